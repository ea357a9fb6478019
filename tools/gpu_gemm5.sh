for env in "" HK_SK_ALL=1 "HK_SK_ALL=1 HK_SK_HYBRID=1"; do echo "== [$env]"; env $env python tools/gemm_sweep.py 64 2>&1 | grep -v "^#" | tail -6; done
