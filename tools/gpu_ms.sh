# ms_per_step of bench.py (configs[1], 2 steps) for each env setting given as an argument
for env in "" "$@"; do
  echo "== [$env]"; env $env timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1))"
done
