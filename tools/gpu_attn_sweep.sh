python -m pytest tests/test_gpu_decode_attn.py -q -x 2>&1 | tail -1
python tools/attn_bench.py 2>&1 | tail -10
python tools/attn_trace.py 128 64 2>&1 | grep -E "P0|O done|shared phase"
