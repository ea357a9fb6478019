python -m pytest tests/test_gpu_decode_attn.py -q -x 2>&1 | tail -2
for sp in 4 6 8; do
  echo "splits=$sp"; HK_ATTN_SPLITS=$sp python tools/attn_bench.py 2>&1 | grep -E "c2 llama  k=   1|c2 llama  k= 128|c2 llama  k= 256|qwen   k= 128"
done
