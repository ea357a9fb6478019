timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 -k "argmax" 2>&1 | grep -E "Error|assert|Mismatch|where" | head -20
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 3 -c 1 -o gpurun_out/gemm_sk_qkv python tools/gemm_sweep.py 64 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 130 -c 1 -o gpurun_out/gemm_sk_gu python tools/gemm_sweep.py 64 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
