"""Per-CTA phase timeline of the decode attention kernels (debug: %globaltimer stamps)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_16104_b200 import _lib  # noqa: E402
from test_gpu_decode_attn import make_case, run  # noqa: E402


def warm_gpu(seconds=0.5):
    """Bring SM clocks up before timing short kernels."""
    import time
    import torch
    x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    t = time.time()
    while time.time() - t < seconds:
        for _ in range(20):
            x = (x @ x).clamp_(-1, 1)
        torch.cuda.synchronize()


warm_gpu()

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
case = make_case(32, 8, [(64, 128, [16 + k] * 64)], seed=1)
run(case, iters=3)  # warm
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
_lib.load().hkx_decode_attention_trace(C.c_void_p(buf.data_ptr()))
run(case)
_lib.load().hkx_decode_attention_trace(None)
t = buf[:148 * 24].view(-1, 24).cpu().numpy().astype(np.float64)  # [CTA][24] stamps
n_sh = int(sys.argv[2]) if len(sys.argv) > 2 else 128
sh = t[:n_sh]
rest = t[n_sh:][t[n_sh:, 0] > 0]
t0 = sh[:, 0].min() if len(rest) == 0 else min(sh[:, 0].min(), rest[:, 0].min())
us = lambda x: (x - t0) / 1e3
print(f"k={k}: shared CTAs {n_sh}: start {us(sh[:,0]).min():.1f}..{us(sh[:,0]).max():.1f} us; "
      f"queue-only CTAs {len(rest)} start {us(rest[:,0]).min() if len(rest) else 0:.1f} us")
order = [(0, "start"), (1, "tmem+bars"), (2, "q in smem"), (7, "S0 ready"), (8, "P0 written"), (3, "O done"),
         (4, "partial out"), (5, "merge")]
prev = None
for idx, name in order:
    if prev is not None:
        d = (sh[:, idx] - sh[:, prev[0]]) / 1e3
        print(f"  {prev[1]:>14s} -> {name:<14s} mean {d.mean():7.2f} us  max {d.max():7.2f}")
    prev = (idx, name)
print(f"  queue loop ends: shared CTAs {us(sh[:,12]).min():.1f}..{us(sh[:,12]).max():.1f} us, "
      f"queue-only CTAs {us(rest[:,12]).min() if len(rest) else 0:.1f}..{us(rest[:,12]).max() if len(rest) else 0:.1f} us")
mhz = (sh[:, 23] - sh[:, 22]) / (sh[:, 5] - sh[:, 0]) * 1e3
print(f"  SM clock inside shared CTAs: {mhz.mean():.0f} MHz; shared phase ends {us(sh[:,5]).min():.1f}..{us(sh[:,5]).max():.1f} us")
# chunk 1 of the softmax warps (thread 0): S1 ready (9) -> row max exchanged (10) -> exps packed (11) -> PV(0) done (6)
c1 = [(9, "O done"), (10, "l exchanged"), (11, "staged"), (6, "bulk stored")]
for (i0, n0), (i1, n1) in zip(c1, c1[1:]):
    d = sh[:, i1] - sh[:, i0]
    print(f"  c1 {n0:>14s} -> {n1:<14s} mean {d.mean():8.0f} cycles  max {d.max():8.0f}")
allc = t[t[:, 0] > 0]
print(f"  tail: queue end {us(allc[:,12]).max():.2f}, grid barrier entered {us(allc[:,16]).min():.2f}..{us(allc[:,16]).max():.2f}, "
      f"merge start {us(allc[:,13]).min():.2f}..{us(allc[:,13]).max():.2f}, merge end {us(allc[:,17]).min():.2f}..{us(allc[:,17]).max():.2f} us")
m = allc[(allc[:, 18] > 0) & (allc[:, 20] > 0)]
if len(m):
    print(f"  merge16 (thread 0, cycles): entry -> batch consumed {np.median(m[:,19]-m[:,18]):.0f} (max {np.max(m[:,19]-m[:,18]):.0f}), "
          f"-> stored {np.median(m[:,20]-m[:,19]):.0f}; CTAs with pairs {len(m)}")
