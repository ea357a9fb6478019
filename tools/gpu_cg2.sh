# CTA-pair prefill GEMMs: kernel tests in every routing, event timing, whole-run A/B of $1 (default HK_GEMM_CG2=0)
mkdir -p gpurun_out
AB=${1:-HK_GEMM_CG2=0}
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 -k "gemm" 2>&1 | tail -2
env $AB timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 -k "gemm" 2>&1 | tail -2
for e in HK_NOTHING=1 "$AB"; do echo "== $e"; env $e timeout -s KILL 300 python tools/ncu_probes.py prefill_gemm_time 2048; env $e timeout -s KILL 300 python tools/ncu_probes.py prefill_gemm_time 1024; done
bash tools/gpu_prefill_ab.sh "$AB"
