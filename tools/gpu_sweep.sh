mkdir -p gpurun_out
python tools/gemm_sweep.py 64 2>&1 | tee gpurun_out/sweep_cluster.log
HK_GEMM_NO_CLUSTER=1 python tools/gemm_sweep.py 64 2>&1 | tee gpurun_out/sweep_nocluster.log
