"""TEST INFRASTRUCTURE ONLY — ctypes access to the compiled reference.

Loads oracle/_ref/libhelios_ref.so (built by oracle/Makefile from the
unmodified reference sources) and exposes the reference pipeline, KvCache,
static_pin_prefixes, synth_* and token hashes. Only tests/, __graft_entry__
.smoke() and bench.py's reference/cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libhelios_ref.so"
u64p = C.POINTER(C.c_uint64)
u8pp = C.POINTER(C.POINTER(C.c_uint8))

_lib = None


def available() -> bool:
    return LIB.exists() or Path("/root/reference/proj/src").exists()


def build() -> Path:
    if not LIB.exists():
        subprocess.run(["make", "-C", str(HERE), "-j8"], check=True, capture_output=True)
    return LIB


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_free.argtypes = [C.c_void_p]
    lib.ref_run.argtypes = [C.c_char_p] * 4 + [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
    lib.ref_time_run_workflow.argtypes = [C.c_char_p] * 4 + [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_void_p)]
    lib.ref_generate_workload.argtypes = [C.c_char_p, C.c_int] + [C.POINTER(C.c_void_p)] * 3
    lib.ref_kv_new.restype = C.c_void_p
    lib.ref_kv_new.argtypes = [C.c_size_t, C.c_size_t]
    lib.ref_kv_free.argtypes = [C.c_void_p]
    lib.ref_kv_lookup.restype = C.c_size_t
    lib.ref_kv_lookup.argtypes = [C.c_void_p, u64p, C.c_size_t, C.c_uint64]
    lib.ref_kv_insert.restype = C.c_size_t
    lib.ref_kv_insert.argtypes = [C.c_void_p, u64p, C.c_size_t, C.c_size_t, C.c_int, C.c_uint64]
    lib.ref_kv_release.argtypes = [C.c_void_p, C.c_uint64]
    lib.ref_kv_counters.argtypes = [C.c_void_p, u64p]
    lib.ref_static_pins.argtypes = [C.c_char_p] * 4 + [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                                       C.POINTER(C.c_void_p)]
    lib.ref_synth_llm_len.restype = C.c_size_t
    lib.ref_synth_llm_len.argtypes = [u64p, C.c_size_t, C.c_double, C.c_int, C.c_uint64, C.c_int]
    lib.ref_synth_llm_output.restype = C.c_size_t
    lib.ref_synth_llm_output.argtypes = [u64p, C.c_size_t, C.c_double, C.c_int, C.c_uint64, C.c_int, u64p,
                                         C.c_size_t]
    lib.ref_fnv1a64.restype = C.c_uint64
    lib.ref_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
    lib.ref_hash_combine.restype = C.c_uint64
    lib.ref_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
    lib.ref_tokenize.restype = C.c_size_t
    lib.ref_tokenize.argtypes = [C.c_char_p, u64p, C.c_size_t]
    lib.ref_role_marker.restype = C.c_uint64
    lib.ref_role_marker.argtypes = [C.c_int]
    lib.ref_cli_run.argtypes = [C.c_char_p] * 4 + [C.POINTER(C.c_void_p)]
    lib.ref_pcache_new.restype = C.c_void_p
    lib.ref_pcache_new.argtypes = [C.c_size_t]
    lib.ref_pcache_load.restype = C.c_void_p
    lib.ref_pcache_load.argtypes = [C.c_char_p]
    lib.ref_pcache_free.argtypes = [C.c_void_p]
    lib.ref_pcache_insert.argtypes = [C.c_void_p, C.c_uint64, u64p, C.c_size_t]
    lib.ref_pcache_lookup.restype = C.c_longlong
    lib.ref_pcache_lookup.argtypes = [C.c_void_p, C.c_uint64]
    lib.ref_pcache_save.restype = C.c_void_p
    lib.ref_pcache_save.argtypes = [C.c_void_p]
    _lib = lib
    return lib


def _err():
    return load().ref_last_error().decode()


def _take_str(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    load().ref_free(p)
    return s


def _j(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def run(workflow, inputs, profile, spec, want_plan: bool = True) -> Tuple[dict, Optional[bytes]]:
    """Reference pipeline + simulate(); returns (result dict, HKPLAN01 blob)."""
    lib = load()
    out = C.c_void_p()
    plan = C.c_void_p()
    n = C.c_size_t()
    rc = lib.ref_run(_j(workflow), _j(inputs), _j(profile), _j(spec), C.byref(out),
                     C.byref(plan) if want_plan else None, C.byref(n) if want_plan else None)
    if rc != 0:
        raise RuntimeError(_err())
    res = json.loads(_take_str(out))
    blob = None
    if want_plan:
        blob = C.string_at(plan, n.value)
        lib.ref_free(plan)
    return res, blob


def cli_run(workflow, inputs, profile, flags: dict) -> dict:
    """`helios run` (tools/helios_main.cpp:83-115) with the reference simulate():
    report / csv / outputs / schedule documents and the saved prompt cache."""
    out = C.c_void_p()
    if load().ref_cli_run(_j(workflow), _j(inputs), _j(profile), _j(flags), C.byref(out)) != 0:
        raise RuntimeError(_err())
    return json.loads(_take_str(out))


class PromptCache:
    """The reference's PromptCache (prompt_cache.cpp), for differential tests."""

    def __init__(self, capacity: int = 4096, _h=None):
        self.h = _h if _h is not None else load().ref_pcache_new(capacity)
        if not self.h:
            raise RuntimeError(_err())

    def __del__(self):
        if getattr(self, "h", None):
            load().ref_pcache_free(self.h)
            self.h = None

    @staticmethod
    def deserialize(text: str) -> "PromptCache":
        h = load().ref_pcache_load(text.encode())
        if not h:
            raise RuntimeError(_err())
        return PromptCache(_h=h)

    def insert(self, sig: int, value: Sequence[int]) -> None:
        a = np.ascontiguousarray(np.asarray(list(value) or [0], dtype=np.uint64))
        load().ref_pcache_insert(self.h, sig, a.ctypes.data_as(u64p), len(value))

    def lookup_len(self, sig: int) -> int:
        return int(load().ref_pcache_lookup(self.h, sig))

    def serialize(self) -> str:
        return _take_str(C.c_void_p(load().ref_pcache_save(self.h)))


def time_run_workflow(workflow, inputs, profile, spec, reps: int = 3) -> Tuple[float, str]:
    lib = load()
    best = C.c_double()
    mj = C.c_void_p()
    rc = lib.ref_time_run_workflow(_j(workflow), _j(inputs), _j(profile), _j(spec), reps, C.byref(best), C.byref(mj))
    if rc != 0:
        raise RuntimeError(_err())
    return best.value, _take_str(mj)


def generate_workload(spec: dict, random: bool = False) -> Tuple[str, str, str]:
    lib = load()
    a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
    if lib.ref_generate_workload(_j(spec), int(random), C.byref(a), C.byref(b), C.byref(c)) != 0:
        raise RuntimeError(_err())
    return _take_str(a), _take_str(b), _take_str(c)


def static_pins(workflow, inputs, profile, spec, worker, block, threshold, budget) -> List[List[int]]:
    lib = load()
    out = C.c_void_p()
    if lib.ref_static_pins(_j(workflow), _j(inputs), _j(profile), _j(spec), worker, block, threshold, budget,
                           C.byref(out)) != 0:
        raise RuntimeError(_err())
    return json.loads(_take_str(out))


def _arr(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.uint64))
    return a, a.ctypes.data_as(u64p)


class RefKvCache:
    """The reference KvCache itself (simulator.cpp:14-128)."""

    def __init__(self, cap: int, block: int):
        self._h = load().ref_kv_new(cap, block)
        if not self._h:
            raise RuntimeError(_err())

    def __del__(self):
        if getattr(self, "_h", None):
            load().ref_kv_free(self._h)

    def lookup(self, seq: Sequence[int], hold: int = 0) -> int:
        a, p = _arr(seq)
        return load().ref_kv_lookup(self._h, p, len(a), hold)

    def insert(self, seq: Sequence[int], length: int, pinned: bool, hold: int = 0) -> int:
        a, p = _arr(seq)
        return load().ref_kv_insert(self._h, p, len(a), length, int(pinned), hold)

    def release(self, hold: int):
        load().ref_kv_release(self._h, hold)

    def counters(self):
        out = (C.c_uint64 * 3)()
        load().ref_kv_counters(self._h, out)
        return list(out)


def synth_llm_len(prompt, len_out, det, seed=0, stochastic=False) -> int:
    a, p = _arr(prompt)
    return load().ref_synth_llm_len(p, len(a), len_out, int(det), seed, int(stochastic))


def synth_llm_output(prompt, len_out, det, seed=0, stochastic=False) -> List[int]:
    a, p = _arr(prompt)
    n = synth_llm_len(prompt, len_out, det, seed, stochastic)
    out = np.zeros(max(n, 1), dtype=np.uint64)
    load().ref_synth_llm_output(p, len(a), len_out, int(det), seed, int(stochastic), out.ctypes.data_as(u64p), n)
    return out[:n].tolist()


def fnv1a64(data: bytes, seed: int = 0xcbf29ce484222325) -> int:
    return load().ref_fnv1a64(data, len(data), seed)


def hash_combine(h: int, v: int) -> int:
    return load().ref_hash_combine(h, v)


def tokenize(text: str) -> List[int]:
    buf = np.zeros(max(1, len(text)), dtype=np.uint64)
    n = load().ref_tokenize(text.encode(), buf.ctypes.data_as(u64p), len(buf))
    return buf[:n].tolist()


def role_marker(role: int) -> int:
    return load().ref_role_marker(role)


def sim_config_dict(spec: dict, n_workers: int) -> dict:
    """The SimConfig ref_capi.cpp builds from `spec` (same defaults as RunSpec)."""
    caps = spec.get("capacities", [4096])
    cap = [caps[0] if len(caps) == 1 else caps[w] for w in range(n_workers)]
    return {
        "capacity": cap,
        "block": [spec.get("block", 16)] * n_workers,
        "prefill_budget": [spec.get("prefill_budget", 0)] * n_workers,
        "proactive_pin": spec.get("proactive_pin", True),
        "pin_threshold": spec.get("pin_threshold", 200),
        "pin_capacity_frac": spec.get("pin_capacity_frac", 0.5),
        "seed": spec.get("seed", 0),
        "stochastic": spec.get("stochastic", False),
        "collect_trace": spec.get("collect_trace", False),
        "max_iterations": spec.get("max_iterations", 0),
    }
