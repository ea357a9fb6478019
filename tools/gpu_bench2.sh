mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -q -x --timeout 300 2>&1 | tail -5 | tee gpurun_out/t2.log
timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -3 | tee gpurun_out/bench2.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 700 --csv \
   --log-file gpurun_out/launches_r1.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu_l.log 2>&1
tail -2 gpurun_out/ncu_l.log
