for kp in 64 128 256; do for sp in 4 8; do
  echo "kp=$kp splits=$sp"; HK_ATTN_PRIV_KEYS=$kp HK_ATTN_SPLITS=$sp python tools/attn_bench.py 2>&1 | grep -E "c2 llama  k=   1|c2 llama  k= 128|c2 llama  k= 256"
done; done
