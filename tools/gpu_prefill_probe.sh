# prefill GEMM timing (events) at T=2048/1024 and one ncu --set full capture of the persistent gate/up and the down GEMM
mkdir -p gpurun_out
python tools/ncu_probes.py prefill_gemm_time 2048
python tools/ncu_probes.py prefill_gemm_time 1024
HK_GEMM_SWIGLU_PERSIST=0 python tools/ncu_probes.py prefill_gemm_time 2048 | grep gate_up
ncu --set full --clock-control none --import-source on -k regex:"gemm_swiglu_pk_kernel|gemm_tc_kernel" -c 8 -o gpurun_out/r2r_prefill_gemm python tools/ncu_probes.py prefill_gemm > gpurun_out/r2r_a.log 2>&1; tail -2 gpurun_out/r2r_a.log
