mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_executor.py tests/test_gpu_dropin.py -q --timeout 900 2>&1 | tail -3
for w in "c2" "c3" "c4_w1"; do
  timeout -s KILL 1200 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), round(d['ms_per_step'],1))"
done
