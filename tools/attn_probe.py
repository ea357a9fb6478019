"""One decode-attention launch at the configs[1] shape and decode step k (for ncu captures).

    ncu --set full -k regex:attn_decode -c 1 python tools/attn_probe.py 128
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from test_gpu_decode_attn import make_case, run  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
case = make_case(32, 8, [(64, 128, [16 + k] * 64)], seed=1)
_, ms, nbytes = run(case)
print(f"k={k}: algorithmic bytes {nbytes:.0f}")
