python -m pytest tests/test_gpu_decode_attn.py -q -x 2>&1 | tail -2
python tools/attn_trace.py 128 128 2>&1 | tail -22
for sp in 2 4 8; do for kp in 64 128 256; do
  echo "splits=$sp priv_keys=$kp"; HK_ATTN_SPLITS=$sp HK_ATTN_PRIV_KEYS=$kp python tools/attn_bench.py 2>&1 | grep "c2 llama" | grep -E "k=   1|k= 128|k= 256"
done; done
python tools/attn_bench.py
