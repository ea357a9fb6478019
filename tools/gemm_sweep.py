"""Decode-GEMM split-K sweep on the B200 (weights cycled through > L2 of copies).

    python tools/gemm_sweep.py
Prints achieved weight-streaming GB/s per (shape, splits) with CUDA events.
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_16104_b200 import _lib  # noqa: E402

lib = _lib.load()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
shapes = [("qkv", 6144, 4096, 3), ("o", 4096, 4096, 3), ("gate_up", 28672, 4096, 4), ("gate_up_f32", 28672, 4096, 2),
          ("down", 4096, 14336, 3), ("lm_head", 128256, 4096, 5)]
st = torch.cuda.current_stream()
for name, N, K, epi in shapes:
    copies = max(2, int(400e6 // (N * K * 2)))
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
    X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    if epi in (2, 3):
        out = torch.zeros(8 if T <= 256 else 1, T, N, device="cuda")
    elif epi == 4:
        out = torch.zeros(T, N // 2, device="cuda", dtype=torch.bfloat16)
    else:
        out = torch.zeros(N // 128 + 1, T, 2, device="cuda")
    for splits in [0]:
        for i in range(3):
            lib.hkx_gemm_bf16(C.c_void_p(Ws[i % copies].data_ptr()), C.c_void_p(X.data_ptr()),
                              C.c_void_p(out.data_ptr()), N, K, T, epi, None, splits, C.c_void_p(st.cuda_stream))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 60
        a.record()
        for i in range(iters):
            rc = lib.hkx_gemm_bf16(C.c_void_p(Ws[i % copies].data_ptr()), C.c_void_p(X.data_ptr()),
                                   C.c_void_p(out.data_ptr()), N, K, T, epi, None, splits, C.c_void_p(st.cuda_stream))
            assert rc == 0, _lib.last_error()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / iters * 1e3
        print(f"{name:8s} N={N:6d} K={K:6d} T={T} splits={splits}: {us:7.2f} us  {N * K * 2 / us / 1e3:7.1f} GB/s  "
              f"{2 * N * K * T / us / 1e6:7.1f} TFLOP/s")
    del Ws
