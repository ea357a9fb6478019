mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_decode_attn.py -q -x --timeout 300 -s 2>&1 | tail -15 | tee gpurun_out/t_attn.log
timeout -s KILL 300 python tools/attn_bench.py 2>&1 | tail -12 | tee gpurun_out/attn_bench.log
