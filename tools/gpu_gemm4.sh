timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 2>&1 | tail -2
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 2 -c 1 -o gpurun_out/sk_gu python tools/gemm_sweep.py 64 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 66 -c 1 -o gpurun_out/sk_lm python tools/gemm_sweep.py 64 > /dev/null 2>&1
ls gpurun_out/sk_*.ncu-rep
