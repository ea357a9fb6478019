"""TEST INFRASTRUCTURE ONLY — bounded CPU sample of the LLM-operator hot path
for bench.py's cpu_baseline leg.

The oracle port (oracle/transformer.py math) runs one batched greedy decode
step of configs[1] — 64 branches, context 2,064 + k tokens, Llama-3-8B width —
through `layers` of the 32 layers plus the LM head on the host cores (numpy /
BLAS, all threads). Full-depth step time is extrapolated as
32 * t_layer + t_head; tokens/s = branches / step time. Weight VALUES do not
affect the timing, so the sample uses constant-filled fp32 tensors instead of
the (slow to generate) counter-based init.
"""
from __future__ import annotations

import os
import time

import numpy as np


def decode_step_sample(d=4096, H=32, Hkv=8, hd=128, F=14336, V=128256, L=32, branches=64, ctx=2064,
                       layers=1, reps=2):
    qkv = (H + 2 * Hkv) * hd
    G = H // Hkv
    w_qkv = np.full((qkv, d), 1e-3, np.float32)
    w_o = np.full((d, H * hd), 1e-3, np.float32)
    w_gu = np.full((2 * F, d), 1e-3, np.float32)
    w_d = np.full((d, F), 1e-3, np.float32)
    lm = np.full((V, d), 1e-3, np.float32)
    K = np.full((branches, ctx, Hkv, hd), 1e-2, np.float32)  # per-branch caches (no prefix sharing)
    Vc = np.full((branches, ctx, Hkv, hd), 1e-2, np.float32)
    x = np.full((branches, d), 0.5, np.float32)

    def layer(x):
        h = x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-5)
        t = h @ w_qkv.T
        q = t[:, :H * hd].reshape(branches, Hkv, G, hd)
        s = np.einsum("bkgd,bskd->bkgs", q, K) / np.sqrt(hd)
        s = np.exp(s - s.max(-1, keepdims=True))
        s /= s.sum(-1, keepdims=True)
        o = np.einsum("bkgs,bskd->bkgd", s, Vc).reshape(branches, H * hd)
        x = x + o @ w_o.T
        h = x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-5)
        gu = h @ w_gu.T
        g, u = gu[:, :F], gu[:, F:]
        a = g / (1 + np.exp(-g)) * u
        return x + a @ w_d.T

    def head(x):
        h = x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-5)
        return np.argmax(h @ lm.T, axis=-1)

    layer(x)  # warm
    t_layer = 1e30
    t_head = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        y = x
        for _ in range(layers):
            y = layer(y)
        t1 = time.perf_counter()
        head(y)
        t2 = time.perf_counter()
        t_layer = min(t_layer, (t1 - t0) / layers)
        t_head = min(t_head, t2 - t1)
    step = L * t_layer + t_head
    return {
        "tokens_per_s": branches / step,
        "step_s": step,
        "t_layer_s": t_layer,
        "t_head_s": t_head,
        "cores": os.cpu_count(),
        "sample": f"{branches}-branch greedy decode step of configs[1] at Llama-3-8B width, ctx {ctx}, "
                  f"{layers} of {L} layers + LM head timed (best of {reps}), step = {L}*t_layer + t_head; "
                  "numpy fp32 oracle port, all host threads",
    }
