"""Per-chunk timeline of a shared tile (clock64 cycles; debug stamps of decode_attn.cu cstamp):
softmax thread 0: S(c) ready, exps packed, PV(c-1) waited, P(c) stored; MMA issuer: S(c) issued, PV(c) issued.

    python tools/attn_chunks.py K [n_shared_ctas]
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_16104_b200 import _lib  # noqa: E402
from test_gpu_decode_attn import make_case, run  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n_sh = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if len(sys.argv) > 3 and sys.argv[3] == "qwen":
    case = make_case(40, 8, [(128, 512, [32 + (i % 40) for i in range(128)])], seed=2)
else:
    case = make_case(32, 8, [(64, 128, [16 + k] * 64)], seed=1)
run(case, iters=3)
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.hkx_decode_attention_trace(C.c_void_p(buf.data_ptr()))
run(case)
lib.hkx_decode_attention_trace(None)
t = buf.cpu().numpy().astype(np.float64)
ch = t[16384:16384 + 148 * 64].reshape(148, 8, 8)[:n_sh]
names = ["S ready", "exps", "PV(c-1) waited", "P stored", "S issued", "PV issued", "max done", "bar passed"]
base = ch[:, 0, 4][:, None]
print("median cycles relative to S(0) issue, per chunk (rows) x event (cols):")
print("      " + " ".join(f"{n:>15s}" for n in names))
for c in range(8):
    vals = ch[:, c, :] - base
    if np.all(ch[:, c, 0] == 0):
        break
    print(f"c={c}: " + " ".join(f"{np.median(vals[:, e]):15.0f}" for e in range(8)))
