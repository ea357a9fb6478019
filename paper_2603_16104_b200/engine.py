"""Device engine handle (hk_engine_* of include/helium_b200.h) and model presets.

Model shapes are the public model cards named by BASELINE.json (weights are
random, initialised on device from a counter-based seed shared with
oracle/transformer.py):
  * tiny        configs[0]: 2 layers, d 256, 2 q / 1 kv heads x 128, FFN 768, vocab 32768
  * llama3_8b   32 L, d 4096, 32 q / 8 kv x 128, FFN 14336, vocab 128256, rope 5e5
  * qwen25_32b  64 L, d 5120, 40 q / 8 kv x 128, FFN 27648, vocab 152064, rope 1e6, qkv bias
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence

import numpy as np

from . import _lib


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    qkv_bias: bool = False
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    seed: int = 0
    fp32: bool = False

    def to_c(self) -> _lib.ModelConfigC:
        return _lib.ModelConfigC(self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.head_dim,
                                 self.ffn_dim, self.vocab, int(self.qkv_bias), self.rope_theta, self.rms_eps,
                                 self.seed, int(self.fp32), 0)

    def params(self) -> int:
        qkv = (self.n_heads + 2 * self.n_kv_heads) * self.head_dim
        per = qkv * self.d_model + self.d_model * self.n_heads * self.head_dim + 3 * self.ffn_dim * self.d_model
        return self.n_layers * per + 2 * self.vocab * self.d_model

    def kv_bytes_per_token(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * (4 if self.fp32 else 2)


TINY = ModelConfig("tiny", 2, 256, 2, 1, 128, 768, 32768, rope_theta=10000.0)
LLAMA3_8B = ModelConfig("llama3_8b", 32, 4096, 32, 8, 128, 14336, 128256, rope_theta=500000.0)
QWEN25_32B = ModelConfig("qwen25_32b", 64, 5120, 40, 8, 128, 27648, 152064, qkv_bias=True, rope_theta=1000000.0,
                         rms_eps=1e-6)
PRESETS = {m.name: m for m in (TINY, LLAMA3_8B, QWEN25_32B)}


def reduced(m: ModelConfig, n_layers: int, vocab: Optional[int] = None) -> ModelConfig:
    """Same widths, fewer layers (and optionally a smaller vocab) for CPU-oracle parity runs."""
    return replace(m, name=f"{m.name}_L{n_layers}", n_layers=n_layers, vocab=vocab or m.vocab)


@dataclass
class EngineConfig:
    device: int = 0
    n_workers: int = 1
    pages_per_worker: int = 4096
    block_tokens: int = 16
    max_calls: int = 256
    max_step_tokens: int = 8192 + 256
    max_ctx_tokens: int = 16384
    use_device_trie: bool = True

    def to_c(self) -> _lib.EngineConfigC:
        return _lib.EngineConfigC(self.device, self.n_workers, self.pages_per_worker, self.block_tokens,
                                  self.max_calls, self.max_step_tokens, self.max_ctx_tokens,
                                  int(self.use_device_trie))


def pages_for(sim_cfg, max_calls: int, max_private_tokens: int, block: int = 16) -> int:
    """Pool size: the reference cache capacity in pages + private pages of live calls."""
    cap = max(w.capacity for w in sim_cfg.workers)
    return cap // block + max_calls * (max_private_tokens // block + 2) + 64


class Engine:
    """A device engine: weights + one KV block pool / device trie per worker."""

    def __init__(self, model: ModelConfig, cfg: EngineConfig):
        lib = _lib.load()
        self.model, self.cfg = model, cfg
        mc, ec = model.to_c(), cfg.to_c()
        self.handle = lib.hk_engine_create(C.byref(mc), C.byref(ec))
        if not self.handle:
            raise RuntimeError(f"hk_engine_create: {_lib.last_error()}")

    def close(self):
        if getattr(self, "handle", None):
            try:
                _lib.load().hk_engine_destroy(self.handle)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.handle = None

    def __del__(self):
        self.close()

    def page_bytes(self) -> int:
        return _lib.load().hk_engine_page_bytes(self.handle)

    def reset(self):
        _lib.check_status(_lib.load().hk_engine_reset(self.handle), "hk_engine_reset")

    def generate(self, ids: Sequence[int], n_new: int, want_logits: bool = False):
        lib = _lib.load()
        a = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        out = np.zeros(max(n_new, 1), dtype=np.uint32)
        logits = np.zeros((n_new, self.model.vocab), dtype=np.float32) if want_logits else None
        rc = lib.hk_generate(self.handle, a.ctypes.data_as(_lib.u32p), len(a), n_new,
                             out.ctypes.data_as(_lib.u32p),
                             logits.ctypes.data_as(_lib.f32p) if want_logits else None)
        _lib.check_status(rc, "hk_generate")
        return (out[:n_new], logits) if want_logits else out[:n_new]

    def stats(self) -> dict:
        s = _lib.EngineStatsC()
        _lib.check_status(_lib.load().hk_engine_stats_get(self.handle, C.byref(s)), "hk_engine_stats_get")
        return {k: getattr(s, k) for k, _ in s._fields_}

    def profile(self, enable: bool = True):
        _lib.check_status(_lib.load().hk_engine_profile(self.handle, int(enable)), "hk_engine_profile")

    def kernel_ms(self, family: str):
        n = C.c_uint64()
        b = C.c_double()
        ms = _lib.load().hk_engine_kernel_ms(self.handle, family.encode(), C.byref(n), C.byref(b))
        return ms, n.value, b.value

    # K1 / K2 entry points (device pointers / host arrays)
    def trie_apply(self, worker: int, ops: List[dict]):
        arr = (_lib.TrieOpC * max(len(ops), 1))()
        keep = []
        for i, op in enumerate(ops):
            k = None
            if not op.get("erase"):
                k = np.ascontiguousarray(np.asarray(op["key"], dtype=np.uint64))
                keep.append(k)
            arr[i] = _lib.TrieOpC(op["node"], op["parent"], op.get("page", -1), int(op.get("erase", 0)), op["phash"],
                                  k.ctypes.data_as(_lib.u64p) if k is not None else None)
        _lib.check_status(_lib.load().hk_trie_apply(self.handle, worker, arr, len(ops)), "hk_trie_apply")

    def trie_match(self, worker: int, prompts: List[Sequence[int]]):
        flat = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.uint64) for p in prompts])
                                    if prompts else np.zeros(0, np.uint64))
        offs = np.zeros(len(prompts) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(p) for p in prompts])
        stride = max(1, max((len(p) // self.cfg.block_tokens for p in prompts), default=1))
        matched = np.zeros(len(prompts), np.int32)
        path = np.full((len(prompts), stride), -1, np.int32)
        pt = np.full((len(prompts), stride), -1, np.int32)
        rc = _lib.load().hk_trie_match(self.handle, worker, flat.ctypes.data_as(_lib.u64p),
                                       offs.ctypes.data_as(_lib.u64p), len(prompts),
                                       matched.ctypes.data_as(_lib.i32p), path.ctypes.data_as(_lib.i32p),
                                       pt.ctypes.data_as(_lib.i32p), stride)
        _lib.check_status(rc, "hk_trie_match")
        return matched, path, pt

    def set_pin_exchange(self, role: int, fn=None):
        """K6 pinned-prefix replication (hk_engine_set_pin_exchange): role 0
        computes pins locally; role 1 computes them and calls fn(worker,
        device_ptr, nbytes) with the newly pinned pages; role 2 skips the
        compute and expects fn to fill the buffer. An exception raised by fn
        fails the run (hk_simulate raises "simulate: pin exchange ...")."""
        self._pin_fn, self._pin_exc = fn, None

        def _cb(_user, worker, buf, nbytes):
            try:
                fn(int(worker), int(buf or 0), int(nbytes))
                return 0
            except Exception as e:  # surfaced by take_pin_exchange_error()
                self._pin_exc = e
                return 1

        self._pin_cb = _lib.PinExchangeFn(_cb) if fn is not None else _lib.PinExchangeFn()  # NULL
        _lib.check_status(_lib.load().hk_engine_set_pin_exchange(self.handle, role, self._pin_cb, None),
                          "hk_engine_set_pin_exchange")

    def take_pin_exchange_error(self):
        e, self._pin_exc = getattr(self, "_pin_exc", None), None
        return e

    # step-level entry points (include/helium_b200.h: hk_slot_*, hk_step, hk_pin_prefill, hk_kv_broadcast)
    def slot_alloc(self, worker: int = 0) -> int:
        s = _lib.load().hk_slot_alloc(self.handle, worker)
        if s < 0:
            raise RuntimeError(f"hk_slot_alloc: {_lib.last_error()}")
        return s

    def slot_free(self, worker: int, slot: int):
        _lib.check_status(_lib.load().hk_slot_free(self.handle, worker, slot), "hk_slot_free")

    def step(self, worker: int, segs: List[dict], want_logits: bool = False):
        """One ragged forward. Each seg: slot, start, count, sample, ids (list of
        vocab ids, or None for a decode step of the slot's last sampled token),
        pages (the call's block table), write_kv (default True). Returns the
        sampled token per seg (-1 where it does not sample) [and the logits
        [n][vocab] of the sampling segs' last positions]."""
        arr = (_lib.StepSegC * max(len(segs), 1))()
        keep = []
        for i, g in enumerate(segs):
            ids = None
            if g.get("ids") is not None:
                ids = np.ascontiguousarray(np.asarray(g["ids"], dtype=np.uint32))
                keep.append(ids)
            pages = np.ascontiguousarray(np.asarray(g["pages"], dtype=np.int32))
            keep.append(pages)
            count = len(ids) if ids is not None else int(g.get("count", 1))
            arr[i] = _lib.StepSegC(int(g.get("slot", -1)), int(g["start"]), count, int(bool(g.get("sample", False))),
                                   ids.ctypes.data_as(_lib.u32p) if ids is not None else None,
                                   pages.ctypes.data_as(_lib.i32p), len(pages), int(bool(g.get("write_kv", True))))
        sampled = np.full(max(len(segs), 1), -1, dtype=np.int32)
        logits = np.zeros((len(segs), self.model.vocab), dtype=np.float32) if want_logits else None
        rc = _lib.load().hk_step(self.handle, worker, arr, len(segs), sampled.ctypes.data_as(_lib.i32p),
                                 logits.ctypes.data_as(_lib.f32p) if want_logits else None)
        _lib.check_status(rc, "hk_step")
        return (sampled[:len(segs)], logits) if want_logits else sampled[:len(segs)]

    def pin_prefill(self, worker: int, ids: Sequence[int], pages: Sequence[int]):
        a = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
        _lib.check_status(_lib.load().hk_pin_prefill(self.handle, worker, a.ctypes.data_as(_lib.u32p), len(a),
                                                     p.ctypes.data_as(_lib.i32p), len(p)), "hk_pin_prefill")

    def kv_broadcast(self, worker: int, role: int, pages: Sequence[int], fn):
        """K6 page broadcast (hk_kv_broadcast): role 1 gathers `pages` and calls
        fn(device_ptr, nbytes); role 2 calls fn to fill the buffer, then
        scatters it into `pages`."""
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
        err = []

        def _cb(_user, _worker, buf, nbytes):
            try:
                fn(int(buf or 0), int(nbytes))
                return 0
            except Exception as e:  # re-raised below
                err.append(e)
                return 1

        cb = _lib.PinExchangeFn(_cb)
        rc = _lib.load().hk_kv_broadcast(self.handle, worker, role, p.ctypes.data_as(_lib.i32p), len(p), cb, None)
        if err:
            raise err[0]
        _lib.check_status(rc, "hk_kv_broadcast")

    def pool_gather(self, worker: int, pages: Sequence[int], dst_ptr: int):
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
        _lib.check_status(_lib.load().hk_pool_gather(self.handle, worker, p.ctypes.data_as(_lib.i32p), len(p),
                                                     C.c_void_p(dst_ptr)), "hk_pool_gather")

    def pool_scatter(self, worker: int, src_ptr: int, pages: Sequence[int]):
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
        _lib.check_status(_lib.load().hk_pool_scatter(self.handle, worker, C.c_void_p(src_ptr),
                                                      p.ctypes.data_as(_lib.i32p), len(p)), "hk_pool_scatter")

    def pool_copy(self, worker: int, src: Sequence[int], dst: Sequence[int]):
        s = np.ascontiguousarray(np.asarray(src, dtype=np.int32))
        d = np.ascontiguousarray(np.asarray(dst, dtype=np.int32))
        _lib.check_status(_lib.load().hk_pool_copy(self.handle, worker, s.ctypes.data_as(_lib.i32p),
                                                   d.ctypes.data_as(_lib.i32p), len(s)), "hk_pool_copy")
