set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "gemm" 2>&1 | tail -30 | tee gpurun_out/t_gemm.log
timeout -s KILL 400 python -m pytest tests/test_gpu_kernels.py -q --timeout 200 -k "not gemm" 2>&1 | tail -40 | tee gpurun_out/t_kern.log
timeout -s KILL 600 python -m pytest tests/test_gpu_executor.py -q --timeout 300 2>&1 | tail -40 | tee gpurun_out/t_exec.log
