"""Per-item timeline of the private queue of the decode attention kernel
(debug %globaltimer stamps: claim, first page landed, done; SM and warp).

    python tools/attn_items.py K [private]    # configs[1] shape at k=K (or private-only rows)
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


def warm_gpu(seconds=0.5):
    import time
    x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    t = time.time()
    while time.time() - t < seconds:
        for _ in range(20):
            x = (x @ x).clamp_(-1, 1)
        torch.cuda.synchronize()


warm_gpu()

k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
if len(sys.argv) > 2 and sys.argv[2] == "private":
    case = make_case(32, 8, [(1, 0, [16 + k]) for _ in range(64)], seed=3)
else:
    case = make_case(32, 8, [(64, 128, [16 + k] * 64)], seed=1)
run(case, iters=3)
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.hkx_decode_attention_trace(C.c_void_p(buf.data_ptr()))
run(case)
lib.hkx_decode_attention_trace(None)
t = buf.cpu().numpy().astype(np.float64)
cta = t[:148 * 24].reshape(148, 24)
items = t[32768:32768 + 6000 * 4].reshape(-1, 4)
items = items[items[:, 0] > 0]
t0 = cta[:, 0][cta[:, 0] > 0].min()
us = lambda x: (x - t0) / 1e3
lat = (items[:, 1] - items[:, 0]) / 1e3
run_ = (items[:, 2] - items[:, 1]) / 1e3
print(f"{len(items)} items; claim {us(items[:,0]).min():.2f}..{us(items[:,0]).max():.2f} us, "
      f"done {us(items[:,2]).min():.2f}..{us(items[:,2]).max():.2f} us")
for name, v in (("claim->first page", lat), ("first page->done", run_)):
    q = np.percentile(v, [0, 10, 50, 90, 100])
    print(f"  {name:>18s}: " + " ".join(f"{x:6.2f}" for x in q) + "  (min p10 p50 p90 max us)")
sm = (items[:, 3].astype(np.int64) >> 8)
wp = (items[:, 3].astype(np.int64) & 255)
key = sm * 16 + wp
per = {}
for i, kk in enumerate(key):
    per.setdefault(kk, []).append(i)
busy = []
ends = []
for kk, idx in per.items():
    idx = sorted(idx, key=lambda i: items[i, 0])
    busy.append(sum(items[i, 2] - items[i, 0] for i in idx) / 1e3)
    ends.append(us(items[idx[-1], 2]))
print(f"  warps used {len(per)}; items/warp {len(items)/len(per):.2f}; busy/warp p50 {np.median(busy):.2f} us; "
      f"warp end p10 {np.percentile(ends,10):.2f} p50 {np.median(ends):.2f} p90 {np.percentile(ends,90):.2f} max {max(ends):.2f}")
# bandwidth timeline: items' bytes are unknown here; show in-flight item count over time
grid = np.arange(0, us(items[:, 2]).max() + 0.5, 0.5)
act = [(np.sum((us(items[:, 0]) <= g) & (us(items[:, 2]) > g))) for g in grid]
print("  active items every 0.5us: " + " ".join(str(a) for a in act))
sh_end = us(cta[:, 5][cta[:, 5] > 0])
if len(sh_end):
    print(f"  shared CTAs' phase end {sh_end.min():.2f}..{sh_end.max():.2f} us; merge start (stamp 13) "
          f"{us(cta[:,13][cta[:,13]>0]).min():.2f}..{us(cta[:,13][cta[:,13]>0]).max():.2f}")
