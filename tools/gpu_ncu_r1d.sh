mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 1 \
   -o gpurun_out/attn_k128_r1d python tools/attn_probe.py 128 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1200 -c 2 \
   -o gpurun_out/gemm_r1d python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
ls -la gpurun_out/*r1d*
