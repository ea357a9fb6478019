# attention: kernel tests, then the attn_bench table for each env assignment given ("-" = default)
timeout -s KILL 600 python -m pytest tests/test_gpu_decode_attn.py -q -x --timeout 300 2>&1 | tail -2
for e in "$@"; do echo "=== $e"; if [ "$e" = "-" ]; then python tools/attn_bench.py 2>&1 | tail -10; else env $e python tools/attn_bench.py 2>&1 | tail -10; fi; done
