"""ctypes binding of libhelium_b200.so (include/helium_b200.h).

The library is built in-tree (python -m paper_2603_16104_b200.build). Loading
fails loudly if it is missing: there is no Python or CPU fallback for any entry
point of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libhelium_b200.so"

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)


class SimConfigC(C.Structure):
    _fields_ = [("n_workers", C.c_uint32), ("capacity", u64p), ("block", u64p), ("prefill_budget", u64p),
                ("proactive_pin", C.c_int32), ("pin_threshold", C.c_uint64), ("pin_capacity_frac", C.c_double),
                ("seed", C.c_uint64), ("stochastic", C.c_int32), ("collect_trace", C.c_int32),
                ("max_iterations", C.c_uint64)]


class MetricsC(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("prompt_tokens", C.c_uint64), ("cache_served_tokens", C.c_uint64),
                ("prefill_computed_tokens", C.c_uint64), ("decode_tokens", C.c_uint64),
                ("hit_rate_pct", C.c_double), ("calls", C.c_uint64), ("recompute_tokens", C.c_uint64),
                ("pin_compute_tokens", C.c_uint64)]


class ModelConfigC(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("d_model", C.c_uint32), ("n_heads", C.c_uint32),
                ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32), ("ffn_dim", C.c_uint32),
                ("vocab", C.c_uint32), ("qkv_bias", C.c_uint32), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("seed", C.c_uint64), ("fp32", C.c_uint32), ("reserved", C.c_uint32)]


class EngineConfigC(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_workers", C.c_uint32), ("pages_per_worker", C.c_uint32),
                ("block_tokens", C.c_uint32), ("max_calls", C.c_uint32), ("max_step_tokens", C.c_uint32),
                ("max_ctx_tokens", C.c_uint32), ("use_device_trie", C.c_uint32)]


class TrieOpC(C.Structure):
    _fields_ = [("node", C.c_int32), ("parent", C.c_int32), ("page", C.c_int32), ("erase", C.c_int32),
                ("phash", C.c_uint64), ("key", u64p)]


class StepSegC(C.Structure):
    _fields_ = [("slot", C.c_int32), ("start", C.c_int32), ("count", C.c_int32), ("sample", C.c_int32),
                ("ids", u32p), ("pages", i32p), ("n_pages", C.c_int32), ("write_kv", C.c_int32)]


class WorkflowSpecC(C.Structure):
    _fields_ = [("workers", C.c_int32), ("capacities", u64p), ("n_capacities", C.c_size_t), ("scheduler", C.c_char_p),
                ("seed", C.c_uint64), ("stochastic", C.c_int32), ("prune", C.c_int32), ("merge_duplicates", C.c_int32),
                ("cache_substitute", C.c_int32), ("proactive_pin", C.c_int32), ("pin_threshold", C.c_uint64),
                ("pin_capacity_frac", C.c_double), ("block", C.c_uint64), ("prefill_budget", C.c_uint64),
                ("alpha", C.c_double), ("run_sim", C.c_int32), ("collect_trace", C.c_int32),
                ("max_iterations", C.c_uint64)]


class EngineStatsC(C.Structure):
    _fields_ = [("pin_ms", C.c_double), ("iter_ms", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("launches", C.c_uint64), ("steps", C.c_uint64),
                ("step_tokens", C.c_uint64), ("attn_bytes", C.c_double)]


# cross-worker output exchange: int fn(void* user, int worker, int op, int query, uint64_t* tokens, uint64_t n)
OutputExchangeFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_uint64)
# K6 pin exchange callback: int fn(void* user, int worker, void* device_buf, uint64_t bytes)
PinExchangeFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_uint64)

_SIGS = {
    "hk_engine_stats_get": (C.c_int, [C.c_void_p, C.POINTER(EngineStatsC)]),
    "hk_last_error": (C.c_char_p, []),
    "hk_abi_version": (C.c_int, []),
    "hk_simulate": (C.c_void_p, [u8p, C.c_size_t, C.POINTER(SimConfigC), C.c_void_p, C.c_uint32]),
    "hk_simulate_ex": (C.c_void_p, [u8p, C.c_size_t, C.POINTER(SimConfigC), C.c_void_p, C.c_uint32,
                                    OutputExchangeFn, C.c_void_p]),
    "hk_run_metrics": (C.c_int, [C.c_void_p, C.POINTER(MetricsC)]),
    "hk_run_worker_stat": (C.c_size_t, [C.c_void_p, C.c_int, u64p, C.c_size_t]),
    "hk_run_report": (C.c_size_t, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t]),
    "hk_run_outputs": (C.c_size_t, [C.c_void_p, u64p, C.c_size_t]),
    "hk_run_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "hk_run_call_outputs": (C.c_size_t, [C.c_void_p, u64p, C.c_size_t]),
    "hk_run_call_logits": (C.c_size_t, [C.c_void_p, f32p, C.c_size_t]),
    "hk_run_free": (None, [C.c_void_p]),
    "hk_kv_create": (C.c_void_p, [C.c_size_t, C.c_size_t]),
    "hk_kv_lookup": (C.c_size_t, [C.c_void_p, u64p, C.c_size_t, C.c_uint64]),
    "hk_kv_insert": (C.c_size_t, [C.c_void_p, u64p, C.c_size_t, C.c_size_t, C.c_int, C.c_uint64]),
    "hk_kv_release": (None, [C.c_void_p, C.c_uint64]),
    "hk_kv_counters": (None, [C.c_void_p, u64p]),
    "hk_kv_destroy": (None, [C.c_void_p]),
    "hk_plan_partition_calls": (C.c_int64, [u8p, C.c_size_t, C.c_int, u8p, C.c_size_t]),
    "hk_plan_schedule": (C.c_int64, [u8p, C.c_size_t, C.c_int, u64p, C.c_size_t, C.c_double, u8p, C.c_size_t]),
    "hk_plan_call_groups": (C.c_int64, [u8p, C.c_size_t, C.POINTER(C.c_int64), i32p, i32p, u64p, C.c_size_t]),
    "hk_static_pin_prefixes": (C.c_int64, [u8p, C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                           u64p, C.c_size_t, u64p, C.c_size_t]),
    "hk_run_workflow": (C.c_void_p, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(WorkflowSpecC), C.c_void_p,
                                     C.c_void_p]),
    "hk_run_document": (C.c_size_t, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t]),
    "hk_run_plan": (C.c_size_t, [C.c_void_p, u8p, C.c_size_t]),
    "hk_pcache_create": (C.c_void_p, [C.c_size_t]),
    "hk_pcache_load": (C.c_void_p, [C.c_char_p, C.c_size_t]),
    "hk_pcache_save": (C.c_size_t, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "hk_pcache_size": (C.c_size_t, [C.c_void_p]),
    "hk_pcache_capacity": (C.c_size_t, [C.c_void_p]),
    "hk_pcache_contains": (C.c_int, [C.c_void_p, C.c_uint64]),
    "hk_pcache_lookup": (C.c_int64, [C.c_void_p, C.c_uint64, u64p, C.c_size_t]),
    "hk_pcache_insert": (C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_size_t]),
    "hk_pcache_keys": (C.c_size_t, [C.c_void_p, u64p, C.c_size_t]),
    "hk_pcache_harvest": (C.c_int64, [C.c_void_p, u8p, C.c_size_t, C.c_void_p]),
    "hk_pcache_harvest_calls": (C.c_int64, [C.c_void_p, u8p, C.c_size_t, u64p, C.c_size_t]),
    "hk_pcache_destroy": (None, [C.c_void_p]),
    "hk_synth_llm_len": (C.c_size_t, [u64p, C.c_size_t, C.c_double, C.c_int, C.c_uint64, C.c_int]),
    "hk_synth_llm_output": (C.c_size_t, [u64p, C.c_size_t, C.c_double, C.c_int, C.c_uint64, C.c_int, u64p,
                                         C.c_size_t]),
    "hk_fnv1a64": (C.c_uint64, [C.c_void_p, C.c_size_t, C.c_uint64]),
    "hk_hash_combine": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "hk_vocab_of": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "hk_gen_token": (C.c_uint64, [C.c_uint32, C.c_uint32]),
    "hk_engine_create": (C.c_void_p, [C.POINTER(ModelConfigC), C.POINTER(EngineConfigC)]),
    "hk_engine_destroy": (None, [C.c_void_p]),
    "hk_engine_page_bytes": (C.c_size_t, [C.c_void_p]),
    "hk_engine_reset": (C.c_int, [C.c_void_p]),
    "hk_engine_set_pin_exchange": (C.c_int, [C.c_void_p, C.c_int, PinExchangeFn, C.c_void_p]),
    "hk_engine_set_graphs": (C.c_int, [C.c_void_p, C.c_int]),
    "hk_pool_gather": (C.c_int, [C.c_void_p, C.c_int, i32p, C.c_size_t, C.c_void_p]),
    "hk_pool_scatter": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, i32p, C.c_size_t]),
    "hk_pool_copy": (C.c_int, [C.c_void_p, C.c_int, i32p, i32p, C.c_size_t]),
    "hk_trie_apply": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(TrieOpC), C.c_size_t]),
    "hk_trie_match": (C.c_int, [C.c_void_p, C.c_int, u64p, u64p, C.c_size_t, i32p, i32p, i32p, C.c_size_t]),
    "hk_generate": (C.c_int, [C.c_void_p, u32p, C.c_size_t, C.c_size_t, u32p, f32p]),
    "hk_slot_alloc": (C.c_int, [C.c_void_p, C.c_int]),
    "hk_slot_free": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "hk_step": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(StepSegC), C.c_size_t, i32p, f32p]),
    "hk_pin_prefill": (C.c_int, [C.c_void_p, C.c_int, u32p, C.c_size_t, i32p, C.c_size_t]),
    "hk_kv_broadcast": (C.c_int, [C.c_void_p, C.c_int, C.c_int, i32p, C.c_size_t, PinExchangeFn, C.c_void_p]),
    "hk_engine_kernel_ms": (C.c_double, [C.c_void_p, C.c_char_p, u64p, C.POINTER(C.c_double)]),
    "hk_engine_profile": (C.c_int, [C.c_void_p, C.c_int]),
    # include/helium_b200_kernels.h
    "hkx_gemm_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                C.c_int, C.c_void_p]),
    "hkx_gemm_bench": (C.c_double, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int]),
    "hkx_decode_attention": (C.c_double, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, i32p,
                                          i32p, i32p, C.c_int, C.c_void_p, C.c_int]),
    "hkx_decode_attention_trace": (C.c_int, [C.c_void_p]),
    "hkx_gemm_trace_dump": (C.c_int, [C.c_char_p]),
    "hkx_span_trace": (C.c_int, [C.c_int]),
    "hkx_prefill_attention": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i32p,
                                        C.c_int, C.c_void_p]),
    "hkx_prefill_attention_segs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                             C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_void_p]),
    "hkx_decode_attention_bytes": (C.c_double, [C.c_int, C.c_int, C.c_int, i32p, i32p, i32p, i32p, C.c_int]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2603_16104_b200.build` "
                           "(there is no fallback implementation)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().hk_last_error().decode(errors="replace")


def check(ok, what: str):
    if not ok:
        raise RuntimeError(f"{what}: {last_error()}")
    return ok


def check_status(rc: int, what: str):
    if rc < 0:
        raise RuntimeError(f"{what}: {last_error()}")
    return rc


def u64_array(seq):
    import numpy as np
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.uint64))
    return a, a.ctypes.data_as(u64p)
