"""K3b decode attention throughput at configs[1] / configs[4] shapes (algorithmic bytes / CUDA-event time).

    python tools/attn_bench.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import json  # noqa: E402

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

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(f"# decode attention, algorithmic bytes (shared KV once per group + private KV + q/o) / launch time; "
      f"peak {peak} GB/s (MEASURED_PEAKS.json)")
for name, H, Hkv, members, shared, ks in [("c2 llama", 32, 8, 64, 128, [1, 32, 64, 128, 192, 256]),
                                          ("c5 qwen", 40, 8, 128, 512, [1, 64, 128, 256])]:
    for k in ks:
        case = make_case(H, Hkv, [(members, shared, [16 * (2 if H == 40 else 1) + k] * members)], seed=k)
        _, ms, nbytes = run(case, iters=50)
        gbs = nbytes / ms / 1e6
        print(f"{name:9s} k={k:4d}: {ms * 1e3:8.2f} us  {nbytes / 1e6:8.2f} MB  {gbs:7.0f} GB/s  frac {gbs / peak:.3f}")
