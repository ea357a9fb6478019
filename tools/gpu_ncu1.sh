mkdir -p gpurun_out
# per-launch durations of 2 decode iterations of configs[1] (c2_short: same shapes, 8 decode tokens)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1400 -c 660 --csv \
   --log-file gpurun_out/launches_r1.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu1.log 2>&1
tail -2 gpurun_out/ncu1.log
# full capture of the decode attention kernels and a weight-streaming GEMM (gate/up)
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 600 -c 2 \
   -o gpurun_out/attn_full python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1200 -c 4 \
   -o gpurun_out/gemm_full python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu3.log
ls -la gpurun_out
