mkdir -p gpurun_out
# per-launch durations of ~3 decode iterations (skip init + pin prefill + early iterations)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 900 --csv \
   --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
# full capture of the decode attention kernel and a weight-streaming GEMM
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 2000 -c 2 \
   -o gpurun_out/attn_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3000 -c 4 \
   -o gpurun_out/gemm_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/ncu3.log
ls -la gpurun_out
