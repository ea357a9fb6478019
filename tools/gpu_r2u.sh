# round-2 ncu launch list of decode iterations of configs[1] (c2_short) with the current kernels
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1400 -c 520 --csv \
   --log-file gpurun_out/launches_r2u.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r2u.csv 14 > gpurun_out/launches_r2u.txt; cat gpurun_out/launches_r2u.txt
