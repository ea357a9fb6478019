set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 400 2>&1 | tail -30 | tee gpurun_out/t_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke.log
timeout -s KILL 900 python bench.py 2>&1 | tail -5 | tee gpurun_out/bench.log
timeout -s KILL 600 python bench.py --impl reference 2>&1 | tail -3 | tee gpurun_out/bench_ref.log
