for fam in "" qkv rope attn o rms gu down; do
  echo "== $fam"; HK_DEBUG_DOUBLE=$fam timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1))"
done
