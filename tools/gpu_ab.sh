# A/B of an env switch on the full bench (ms_per_step), plus executor GPU tests
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_executor.py tests/test_gpu_kernels.py -q -x --timeout 400 2>&1 | tail -3
for env in "" "$@"; do
  echo "== [$env]"; env $env timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), d['value'])"
done
