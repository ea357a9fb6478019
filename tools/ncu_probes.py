"""Launch-once probes for ncu captures (round 2 evidence named by north_star):

    python tools/ncu_probes.py prefill_gemm   # T=2048 QKV / O / gate-up / down tcgen05 GEMMs (tensor-pipe %)
    python tools/ncu_probes.py pool           # K1 page gather / copy of 256 Llama-3-8B pages (2 MiB each)
    python tools/ncu_probes.py attn_c5 K      # decode attention at configs[4] (Qwen2.5-32B, 8K shared, 128 rows)
Each prints the algorithmic bytes / FLOPs of the launch it makes.
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch  # noqa: E402

from paper_2603_16104_b200 import _lib  # noqa: E402

what = sys.argv[1]
lib = _lib.load()
if what == "prefill_gemm":
    T = 2048
    for name, N, K, epi in [("qkv", 6144, 4096, 3), ("o", 4096, 4096, 3), ("gate_up", 28672, 4096, 4),
                            ("down", 4096, 14336, 3)]:
        W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        out = torch.zeros(T, N // 2 if epi == 4 else N, device="cuda", dtype=torch.bfloat16 if epi == 4 else torch.float32)
        for _ in range(2):  # warm + captured
            assert lib.hkx_gemm_bf16(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()),
                                     N, K, T, epi, None, 0, None) == 0, _lib.last_error()
        torch.cuda.synchronize()
        print(f"{name}: N={N} K={K} T={T}: {2 * N * K * T / 1e12:.3f} TFLOP per launch")
elif what == "prefill_gemm_time":
    # CUDA-event timing of the same launches (20 back to back, inputs resident; not under a profiler)
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    peak = 1392.0
    for name, N, K, epi in [("qkv", 6144, 4096, 3), ("o", 4096, 4096, 3), ("gate_up", 28672, 4096, 4),
                            ("down", 4096, 14336, 3)]:
        W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        out = torch.zeros(T, N // 2 if epi == 4 else N, device="cuda", dtype=torch.bfloat16 if epi == 4 else torch.float32)
        call = lambda: lib.hkx_gemm_bf16(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()),
                                         N, K, T, epi, None, 0, None)
        for _ in range(3):
            assert call() == 0, _lib.last_error()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        tf = 2 * N * K * T / us / 1e6
        print(f"{name:8s} T={T}: {us:8.1f} us  {tf:7.1f} TFLOP/s  frac {tf / peak:.3f}")
elif what == "decode_gemm_time":
    # decode GEMM weight streaming (T = 64, inputs resident, L2 flushed between launches) vs weight-tile count
    T = 64
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, N, K, epi in [("gate_up 224 tiles", 28672, 4096, 4), ("swiglu 296 tiles", 37888, 4096, 4),
                            ("swiglu 148 tiles", 18944, 4096, 4), ("qkv", 6144, 4096, 3), ("o", 4096, 4096, 3),
                            ("down", 4096, 14336, 3)]:
        W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        out = torch.zeros(16 * T * N, device="cuda", dtype=torch.float32)
        call = lambda: lib.hkx_gemm_bf16(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()),
                                         N, K, T, epi, None, 0, None)
        for _ in range(3):
            assert call() == 0, _lib.last_error()
        ts = []
        for _ in range(10):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        print(f"{name:18s} N={N:6d} K={K:6d}: {us:7.1f} us  {N * K * 2 / us / 1e3:7.0f} GB/s")
elif what == "pool":
    from paper_2603_16104_b200.engine import LLAMA3_8B, Engine, EngineConfig
    eng = Engine(LLAMA3_8B, EngineConfig(pages_per_worker=1024, max_calls=8, max_step_tokens=256, max_ctx_tokens=2048))
    pb = eng.page_bytes()
    n = 256
    dst = torch.empty(n * pb, dtype=torch.uint8, device="cuda")
    pages = list(range(0, 2 * n, 2))
    for _ in range(2):
        eng.pool_gather(0, pages, dst.data_ptr())
        eng.pool_copy(0, pages, list(range(2 * n, 3 * n)))
    torch.cuda.synchronize()
    print(f"pool: {n} pages x {pb} B; gather / copy move {2 * n * pb / 1e6:.1f} MB each (read + write)")
    eng.close()
elif what == "attn_c5":
    from test_gpu_decode_attn import make_case, run
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    case = make_case(40, 8, [(128, 512, [32 + k] * 128)], seed=1)
    _, ms, nbytes = run(case)
    # shared part: 128 rows x 5 heads = 640 rows per kv head over 8192 keys; QK^T + PV = 4 * rows * keys * 128 flops
    flops = 4.0 * 640 * 8192 * 128 * 8
    print(f"c5 k={k}: algorithmic bytes {nbytes:.0f}, shared-tile tensor FLOPs {flops:.3e}")
