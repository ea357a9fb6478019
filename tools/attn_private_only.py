"""Private-only decode attention (no shared groups): configs[1] rows at k=128, for profiling the private queue."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from test_gpu_decode_attn import make_case, run  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
# 64 calls, each with 2048 + 16 + k private tokens but no sharing -> pure private work
case = make_case(32, 8, [(1, 0, [16 + k]) for _ in range(64)], seed=3)
_, ms, nbytes = run(case, iters=50)
print(f"private-only k={k}: {ms * 1e3:.2f} us, {nbytes / ms / 1e6:.0f} GB/s")
