mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
timeout -s KILL 900 python bench.py --steps 2 --warmup 1 2>&1 | tail -20 | tee gpurun_out/bench1.log
