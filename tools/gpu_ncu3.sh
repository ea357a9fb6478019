timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 700 --csv \
   --log-file gpurun_out/launches_prefill.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_prefill.csv 14
