# attention A/B: kernel tests, then the attn_bench table with and without a switch ($1 = env assignment for B)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_decode_attn.py -q -x --timeout 300 2>&1 | tail -3
echo "=== A (default)"; python tools/attn_bench.py 2>&1 | tail -10
if [ -n "$1" ]; then echo "=== B ($1)"; env $1 python tools/attn_bench.py 2>&1 | tail -10; fi
