# decode-attention parity + item trace + kernel bench (one gpurun call); args: extra HK_ATTN_SPLITS values
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_decode_attn.py -q -x --timeout 300 2>&1 | tail -3
python tools/attn_items.py 128 2>&1 | tail -6
python tools/attn_items.py 128 private 2>&1 | tail -5
python tools/attn_items.py 1 2>&1 | tail -6
python tools/attn_bench.py 2>&1 | tail -11
for sp in "$@"; do echo "== HK_ATTN_SPLITS=$sp"; HK_ATTN_SPLITS=$sp python tools/attn_bench.py 2>&1 | tail -11 | head -7; done
