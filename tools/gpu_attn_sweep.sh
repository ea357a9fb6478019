timeout -s KILL 120 python -m pytest tests/test_gpu_decode_attn.py -q -x --timeout 60 2>&1 | tail -1
timeout -s KILL 120 python tools/attn_bench.py 2>&1 | tail -10
timeout -s KILL 60 python tools/attn_private_only.py 128
timeout -s KILL 60 python tools/attn_private_only.py 512
