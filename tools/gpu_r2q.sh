# ncu of the T=2048 prefill GEMMs with token-tile-fastest grids (cold, serialised)
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 8 -o gpurun_out/r2q_prefill_gemm python tools/ncu_probes.py prefill_gemm > gpurun_out/r2q_a.log 2>&1; tail -2 gpurun_out/r2q_a.log
