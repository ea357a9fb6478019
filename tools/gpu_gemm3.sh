timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 2>&1 | tail -1
python tools/gemm_sweep.py 64
