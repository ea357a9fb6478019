"""TEST INFRASTRUCTURE ONLY — CPU fp32 restatement of the random-init decoder.

The reference (/root/reference/proj) has no model — its LLM operator is a
hash (evaluator.cpp:37-58) — so the math of this decoder is pinned to an
independent implementation instead: HuggingFace transformers' LlamaForCausalLM
/ Qwen2ForCausalLM in fp32 with the same weights (tests/test_oracle_hf_cpu.py).
This numpy decoder is the oracle for the transformer math of the B200 engine
(csrc/cuda/engine.cu):
standard Llama-3 / Qwen2.5 decoder layers (RMSNorm, RoPE rotate-half, GQA
causal attention, SwiGLU MLP, untied LM head, optional QKV bias) with the
engine's counter-based weight init reproduced bit-for-bit (init_uniform_kernel,
ops.cu) and — in bf16 mode — rounding to bf16 at the points where the device
stores bf16 (GEMM inputs/outputs, q/k/v, attention output). Accumulations are
fp32 here; the device's accumulation order differs, hence the tolerances
(1e-2 relative logits in bf16, 1e-5 in fp32 mode) used by the tests.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def round_bf16(v: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 -> fp32, round to nearest even (finite inputs)."""
    b = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def _init_range(out: np.ndarray, lo: int, hi: int, base: np.uint64, scale: float, bf16: bool, chunk: int) -> None:
    """splitmix64 counter init of out[lo:hi] in cache-sized chunks, in-place uint64 arithmetic."""
    with np.errstate(over="ignore"):
        ar = np.arange(chunk, dtype=np.uint64)
        x = np.empty(chunk, dtype=np.uint64)
        t = np.empty(chunk, dtype=np.uint64)
        c1, c2, c3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)
        s30, s27, s31, s40 = np.uint64(30), np.uint64(27), np.uint64(31), np.uint64(40)
        sc = np.float32(scale)
        for s in range(lo, hi, chunk):
            e = min(hi, s + chunk)
            m = e - s
            xv, tv = x[:m], t[:m]
            np.add(ar[:m], base + np.uint64(s) + c1, out=xv)          # splitmix64(base + i)
            np.right_shift(xv, s30, out=tv); np.bitwise_xor(xv, tv, out=xv); np.multiply(xv, c2, out=xv)
            np.right_shift(xv, s27, out=tv); np.bitwise_xor(xv, tv, out=xv); np.multiply(xv, c3, out=xv)
            np.right_shift(xv, s31, out=tv); np.bitwise_xor(xv, tv, out=xv)
            np.right_shift(xv, s40, out=xv)
            u = xv.astype(np.float32) * np.float32(1.0 / 8388608.0) - np.float32(1.0)
            v = u * sc
            out[s:e] = round_bf16(v) if bf16 else v


def init_uniform(n: int, seed: int, tid: int, scale: float, bf16: bool, chunk: int = 1 << 16) -> np.ndarray:
    """Mirror of init_uniform_kernel (ops.cu): w[i] = scale * ((splitmix64(base + i) >> 40) * 2^-23 - 1),
    base = seed * C1 + tid * C2. Large tensors are filled by all host threads
    (numpy releases the GIL inside these ufuncs)."""
    base = np.uint64((seed * 0xD1B54A32D192ED03 + tid * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
    out = np.empty(n, dtype=np.float32)
    workers = min(os.cpu_count() or 1, 32)
    if n < (1 << 22) or workers == 1:
        _init_range(out, 0, n, base, scale, bf16, chunk)
        return out
    from concurrent.futures import ThreadPoolExecutor
    step = -(-n // workers)
    step = -(-step // chunk) * chunk
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(lambda lo: _init_range(out, lo, min(n, lo + step), base, scale, bf16, chunk), range(0, n, step)))
    return out


@dataclass
class Weights:
    embed: np.ndarray
    layers: list
    lm_head: np.ndarray


def build_weights(m) -> Weights:
    """Same tensor ids / scales as hk_engine::init_weights (engine.cu)."""
    bf = not m.fp32
    d, H, Hkv, hd, F, V = m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.ffn_dim, m.vocab
    qkv = (H + 2 * Hkv) * hd
    s_d = np.float32(math.sqrt(3.0 / d))
    s_o = np.float32(math.sqrt(3.0 / (H * hd)))
    s_f = np.float32(math.sqrt(3.0 / F))
    embed = init_uniform(V * d, m.seed, 1, 1.0, bf).reshape(V, d)
    layers = []
    for l in range(m.n_layers):
        t0 = 16 + 16 * l
        lw = {
            "wqkv": init_uniform(qkv * d, m.seed, t0 + 1, float(s_d), bf).reshape(qkv, d),
            "bqkv": init_uniform(qkv, m.seed, t0 + 2, 0.1, bf) if m.qkv_bias else None,
            "wo": init_uniform(d * H * hd, m.seed, t0 + 3, float(np.float32(0.5) * s_o), bf).reshape(d, H * hd),
            "wgu": init_uniform(2 * F * d, m.seed, t0 + 4, float(s_d), bf).reshape(2 * F, d),
            "wd": init_uniform(d * F, m.seed, t0 + 5, float(np.float32(0.5) * s_f), bf).reshape(d, F),
        }
        layers.append(lw)
    lm_head = init_uniform(V * d, m.seed, 2, float(s_d), bf).reshape(V, d)
    return Weights(embed, layers, lm_head)


def rope_table(m, max_pos: int) -> np.ndarray:
    """(cos, sin) per position, computed in float64 then stored fp32, as engine.cu does."""
    half = m.head_dim // 2
    i = np.arange(half, dtype=np.float64)
    inv = np.power(np.float64(m.rope_theta), -2.0 * i / m.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


class Decoder:
    """Incremental greedy decoder with a contiguous KV cache."""

    def __init__(self, m, weights: Optional[Weights] = None, max_pos: int = 16384):
        self.m = m
        self.w = weights or build_weights(m)
        self.bf = not m.fp32
        self.cos, self.sin = rope_table(m, max_pos)

    def _r(self, v):
        return round_bf16(v) if self.bf else v.astype(np.float32)

    def _rms(self, x):
        ms = np.mean(x.astype(np.float64) ** 2, axis=-1, keepdims=True)
        return (x / np.sqrt(ms + self.m.rms_eps)).astype(np.float32)

    def _rope(self, x, pos):
        half = self.m.head_dim // 2
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(np.float32)

    def forward(self, ids: Sequence[int], cache: Optional[list] = None, start: int = 0, all_logits: bool = False):
        """Run tokens ids at positions start.. ; returns (logits of the last token
        — of every token with all_logits — and the cache)."""
        m = self.m
        H, Hkv, hd, d, F = m.n_heads, m.n_kv_heads, m.head_dim, m.d_model, m.ffn_dim
        G = H // Hkv
        T = len(ids)
        pos = np.arange(start, start + T)
        x = self.w.embed[np.asarray(ids)].astype(np.float32)
        if cache is None:
            cache = [(np.zeros((0, Hkv, hd), np.float32), np.zeros((0, Hkv, hd), np.float32)) for _ in range(m.n_layers)]
        new_cache = []
        scale = np.float32(1.0 / math.sqrt(hd))
        for l, lw in enumerate(self.w.layers):
            h = self._r(self._rms(x))
            qkv = h @ lw["wqkv"].T
            if lw["bqkv"] is not None:
                qkv = qkv + lw["bqkv"]
            qkv = self._r(qkv)
            q = qkv[:, :H * hd].reshape(T, H, hd)
            k = qkv[:, H * hd:(H + Hkv) * hd].reshape(T, Hkv, hd)
            v = qkv[:, (H + Hkv) * hd:].reshape(T, Hkv, hd)
            q = self._r(self._rope(q, pos))
            k = self._r(self._rope(k, pos))
            K = np.concatenate([cache[l][0], k], axis=0)
            Vv = np.concatenate([cache[l][1], v], axis=0)
            new_cache.append((K, Vv))
            S = K.shape[0]
            o = np.empty((T, H, hd), np.float32)
            kpos = np.arange(S)
            mask = kpos[None, None, :] > pos[:, None, None]
            for g in range(Hkv):
                qg = q[:, g * G:(g + 1) * G, :].reshape(T * G, hd)          # (T G), hd
                sc = (qg @ K[:, g, :].T).reshape(T, G, S) * scale           # T,G,S (BLAS)
                sc = np.where(mask, -np.inf, sc)
                sc = sc - sc.max(axis=-1, keepdims=True)
                p = np.exp(sc)
                p = p / p.sum(axis=-1, keepdims=True)
                o[:, g * G:(g + 1) * G, :] = (p.astype(np.float32).reshape(T * G, S) @ Vv[:, g, :]).reshape(T, G, hd)
            o = self._r(o.reshape(T, H * hd))
            x = x + (o @ lw["wo"].T)
            h = self._r(self._rms(x))
            gu = self._r(h @ lw["wgu"].T)
            g_, u_ = gu[:, :F], gu[:, F:]
            a = self._r((g_ / (np.float32(1.0) + np.exp(-g_))) * u_)
            x = x + (a @ lw["wd"].T)
        hl = self._r(self._rms(x if all_logits else x[-1:]))
        logits = (hl @ self.w.lm_head.T).astype(np.float32)
        return (logits if all_logits else logits[0]), new_cache

    def generate(self, ids: Sequence[int], n_new: int, forced: Optional[Sequence[int]] = None, prefilled=None):
        """Greedy decode n_new tokens. With `forced` (teacher forcing) the given
        tokens are fed instead of the argmax, so logits can be compared step by
        step against another implementation's sequence. `prefilled` = (logits
        of the last prompt token, cache over the whole prompt) skips the prefill."""
        out, all_logits = [], []
        if n_new == 0:
            return out, all_logits
        logits, cache = prefilled if prefilled is not None else self.forward(list(ids), None, 0)
        p = len(ids)
        for k in range(n_new):
            all_logits.append(logits)
            nxt = int(np.argmax(logits))
            out.append(nxt)
            if k + 1 == n_new:
                break
            feed = nxt if forced is None else int(forced[k])
            logits, cache = self.forward([feed], cache, p)
            p += 1
        return out, all_logits


def top2_margin(logits: np.ndarray) -> float:
    part = np.partition(logits, -2)[-2:]
    return float(part[1] - part[0])


class PrefixReuse:
    """Greedy decoding of many prompts that reuses the KV of the longest prompt
    prefix seen before. Exact, not an approximation: K/V at position p depend
    only on tokens 0..p (causal), which is the same fact the reference's block
    cache relies on (simulator.cpp:69-121). A fully seen prompt re-runs its last
    position for the logits (as the engine does)."""

    def __init__(self, dec: Decoder):
        self.dec = dec
        self.store: list = []  # (prompt ids, cache over the prompt)

    def prefill(self, ids: Sequence[int]):
        a = np.asarray(ids, dtype=np.int64)
        best, bj = None, 0
        for p, cache in self.store:
            n = min(len(p), len(a))
            ne = np.flatnonzero(p[:n] != a[:n])
            j = int(ne[0]) if len(ne) else n
            if j > bj:
                best, bj = cache, j
        bj = min(bj, len(a) - 1)
        c0 = [(K[:bj], V[:bj]) for K, V in best] if bj > 0 else None
        logits, cache = self.dec.forward(a[bj:].tolist(), c0, bj)
        self.store.append((a, cache))
        return logits, cache

    def generate(self, ids: Sequence[int], n_new: int, forced: Optional[Sequence[int]] = None):
        if n_new == 0:
            return [], []
        if forced is not None and n_new > 1:
            # teacher forcing: all positions in one causal pass over prompt || forced[:-1]
            first, cache = self.prefill(ids)
            rest, _ = self.dec.forward([int(t) for t in forced[:n_new - 1]], cache, len(ids), all_logits=True)
            logits = [first] + list(rest)
            return [int(np.argmax(lg)) for lg in logits], logits
        return self.dec.generate(ids, n_new, forced=forced, prefilled=self.prefill(ids))
