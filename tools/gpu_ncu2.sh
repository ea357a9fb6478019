mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1400 -c 520 --csv \
   --log-file gpurun_out/launches_r1b.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r1b.csv 14
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 200 -c 1 \
   -o gpurun_out/attn_r1b python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1600 -c 4 \
   -o gpurun_out/gemm_r1b python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
ls gpurun_out/*r1b*
