for env in "" "HK_NO_L2_PREFETCH=1"; do
  echo "== $env"; env $env timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'])"
done
