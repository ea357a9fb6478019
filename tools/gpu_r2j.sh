mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 8 -o gpurun_out/r2_prefill_gemm python tools/ncu_probes.py prefill_gemm > gpurun_out/r2j_a.log 2>&1; tail -3 gpurun_out/r2j_a.log
ncu --set full --clock-control none -k regex:page_move -c 4 -o gpurun_out/r2_pool python tools/ncu_probes.py pool > gpurun_out/r2j_b.log 2>&1; tail -3 gpurun_out/r2j_b.log
ncu --set full --clock-control none -k regex:attn_decode -c 1 -o gpurun_out/r2_attn_c5 python tools/ncu_probes.py attn_c5 128 > gpurun_out/r2j_c.log 2>&1; tail -3 gpurun_out/r2j_c.log
ls -la gpurun_out/*.ncu-rep
