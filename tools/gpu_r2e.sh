mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -s -k full_depth 2>&1 | tail -4
for env in "" "HK_DEBUG_SKIP=rms" "HK_GEMM_CLUSTER=1" "HK_GEMM_CLUSTER=1 HK_DEBUG_SKIP=rms" "HK_DEBUG_SKIP=rms,rope" "HK_GEMM_CLUSTER=1 HK_DEBUG_SKIP=rms,rope"; do
  v=$(env $env timeout -s KILL 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['value']))")
  echo "[$env] ms/run tok/s: $v"
done | tee gpurun_out/r2e_ablate.txt
