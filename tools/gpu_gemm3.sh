echo "## stream-K 1 CTA/SM x 8 stages"; python tools/gemm_sweep.py 64
echo "## stream-K 2 CTA/SM x 4 stages"; HK_SK_CTAS_PER_SM=2 python tools/gemm_sweep.py 64
echo "## stream-K 3 CTA/SM x 4 stages"; HK_SK_CTAS_PER_SM=3 python tools/gemm_sweep.py 64
