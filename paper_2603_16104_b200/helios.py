"""Python mirror of the reference's L4 execution API over the C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/helios/simulator.hpp and evaluator.hpp so parity
tests read like the reference's own tests (test_simulator.cpp). All work is
done by libhelium_b200.so; this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib


# ------------------------------------------------------------------ KvCache
class KvCache:
    """class KvCache (simulator.hpp:18-62)."""

    def __init__(self, capacity_tokens: int, block_tokens: int):
        lib = _lib.load()
        self._h = lib.hk_kv_create(capacity_tokens, block_tokens)
        if not self._h:
            raise RuntimeError(_lib.last_error())
        self._cap, self._block = capacity_tokens, block_tokens

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().hk_kv_destroy(h)
            self._h = None

    def capacity(self) -> int:
        return self._cap

    def block(self) -> int:
        return self._block

    def _counters(self):
        out = (C.c_uint64 * 3)()
        _lib.load().hk_kv_counters(self._h, out)
        return list(out)

    def used_tokens(self) -> int:
        return self._counters()[0]

    def pinned_tokens(self) -> int:
        return self._counters()[1]

    def evicted_tokens(self) -> int:
        return self._counters()[2]

    def lookup(self, seq: Sequence[int], hold: int = 0) -> int:
        a, p = _lib.u64_array(seq)
        return _lib.load().hk_kv_lookup(self._h, p, len(a), hold)

    def insert(self, seq: Sequence[int], length: int, pinned: bool, hold: int = 0) -> int:
        a, p = _lib.u64_array(seq)
        return _lib.load().hk_kv_insert(self._h, p, len(a), length, int(pinned), hold)

    def release(self, hold: int) -> None:
        _lib.load().hk_kv_release(self._h, hold)


# ------------------------------------------------------------------- config
@dataclass
class SimWorkerConfig:
    capacity: int = 4096
    block: int = 16
    prefill_budget: int = 0


@dataclass
class SimConfig:
    workers: List[SimWorkerConfig] = field(default_factory=list)
    proactive_pin: bool = True
    pin_threshold: int = 200
    pin_capacity_frac: float = 0.5
    seed: int = 0
    stochastic: bool = False
    collect_trace: bool = False
    max_iterations: int = 0

    def to_c(self):
        n = len(self.workers)
        cap = (C.c_uint64 * n)(*[w.capacity for w in self.workers])
        blk = (C.c_uint64 * n)(*[w.block for w in self.workers])
        bud = (C.c_uint64 * n)(*[w.prefill_budget for w in self.workers])
        c = _lib.SimConfigC(n, cap, blk, bud, int(self.proactive_pin), self.pin_threshold,
                            self.pin_capacity_frac, self.seed, int(self.stochastic), int(self.collect_trace),
                            self.max_iterations)
        c._keep = (cap, blk, bud)
        return c


@dataclass
class SimMetrics:
    """SimMetrics (simulator.hpp:108-120) + the reports of simulator.cpp:393-425."""
    iterations: int
    prompt_tokens: int
    cache_served_tokens: int
    prefill_computed_tokens: int
    decode_tokens: int
    hit_rate_pct: float
    calls: int
    pinned_tokens: List[int]
    evicted_tokens: List[int]
    outputs: Dict[int, List[List[int]]]
    metrics_json: str
    calls_csv: str
    trace_csv: str
    recompute_tokens: int = 0
    pin_compute_tokens: List[int] = field(default_factory=list)
    pin_seconds: float = 0.0
    iter_seconds: float = 0.0
    call_outputs: Dict[tuple, List[int]] = field(default_factory=dict)
    call_logits: Dict[tuple, List[float]] = field(default_factory=dict)  # device logit of each generated token


def _report(h, which: int) -> str:
    lib = _lib.load()
    n = lib.hk_run_report(h, which, None, 0)
    buf = C.create_string_buffer(n)
    lib.hk_run_report(h, which, buf, n)
    return buf.value.decode()


def _worker_stat(h, which: int) -> List[int]:
    lib = _lib.load()
    n = lib.hk_run_worker_stat(h, which, None, 0)
    out = (C.c_uint64 * max(n, 1))()
    lib.hk_run_worker_stat(h, which, out, n)
    return list(out)[:n]


def _outputs(h) -> Dict[int, List[List[int]]]:
    lib = _lib.load()
    n = lib.hk_run_outputs(h, None, 0)
    buf = np.zeros(max(n, 1), dtype=np.uint64)
    lib.hk_run_outputs(h, buf.ctypes.data_as(_lib.u64p), n)
    words = buf[:n].tolist()
    out, i = {}, 1
    for _ in range(words[0]):
        nid = int(np.int64(np.uint64(words[i])))
        b = words[i + 1]
        i += 2
        vals = []
        for _ in range(b):
            ln = words[i]
            vals.append(words[i + 1:i + 1 + ln])
            i += 1 + ln
        out[nid] = vals
    return out


def _call_outputs(h) -> Dict[tuple, List[int]]:
    lib = _lib.load()
    n = lib.hk_run_call_outputs(h, None, 0)
    buf = np.zeros(max(n, 1), dtype=np.uint64)
    lib.hk_run_call_outputs(h, buf.ctypes.data_as(_lib.u64p), n)
    w = buf[:n].tolist()
    out, i = {}, 1
    for _ in range(w[0]):
        op, q, ln = int(np.int64(np.uint64(w[i]))), int(w[i + 1]), w[i + 2]
        out[(op, q)] = w[i + 3:i + 3 + ln]
        i += 3 + ln
    return out


def _call_logits(h, outs: Dict[tuple, List[int]]) -> Dict[tuple, List[float]]:
    lib = _lib.load()
    n = lib.hk_run_call_logits(h, None, 0)
    buf = np.zeros(max(n, 1), dtype=np.float32)
    lib.hk_run_call_logits(h, buf.ctypes.data_as(_lib.f32p), n)
    res, i = {}, 0
    for k in sorted(outs):  # same (op, query) order as hk_run_call_outputs
        ln = len(outs[k])
        if not np.isnan(buf[i:i + ln]).all():
            res[k] = buf[i:i + ln].tolist()
        i += ln
    return res


def simulate(plan: bytes, cfg: SimConfig, engine=None, verify_lookup: bool = False,
             only_worker: int = -1, exchange=None) -> SimMetrics:
    """simulate() (simulator.hpp:128-130) on a flattened HKPLAN01 plan.

    engine=None runs the synthetic LLM body (reference mode S); an Engine runs
    the device transformer (mode T). only_worker >= 0 runs one worker of the
    schedule (one process per GPU; exact when that worker has no cross-worker
    dependency). Raises RuntimeError with the reference's messages
    ("simulate: ...") on invalid schedules/configs.

    exchange (with only_worker >= 0): fn(worker, op, query, tokens: np.ndarray
    uint64 view) called at every completion of every worker in the same order
    in all processes — the owner's array holds the generated ids, the others
    must fill theirs (exchange.make_output_exchange broadcasts over
    torch.distributed). Cross-worker dependencies are then served and the
    metrics cover the whole workflow (SURVEY.md §8(e) exchange 2).
    """
    lib = _lib.load()
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    c = cfg.to_c()
    flags = (1 if verify_lookup else 0) | ((only_worker + 1) << 8)
    err = []
    if exchange is not None:
        def _cb(_user, worker, op, query, toks, n):
            try:
                exchange(int(worker), int(op), int(query), np.ctypeslib.as_array(toks, shape=(int(n),)))
                return 0
            except Exception as e:  # re-raised below as the cause
                err.append(e)
                return 1
        cb = _lib.OutputExchangeFn(_cb)
        h = lib.hk_simulate_ex(buf, len(plan), C.byref(c), engine.handle if engine is not None else None, flags,
                               cb, None)
    else:
        h = lib.hk_simulate(buf, len(plan), C.byref(c), engine.handle if engine is not None else None, flags)
    if not h:
        cause = err[0] if err else (engine.take_pin_exchange_error() if engine is not None else None)
        raise RuntimeError(_lib.last_error()) from cause
    try:
        mc = _lib.MetricsC()
        lib.hk_run_metrics(h, C.byref(mc))
        t = (C.c_double * 2)()
        lib.hk_run_timing(h, t)
        return SimMetrics(
            iterations=mc.iterations, prompt_tokens=mc.prompt_tokens, cache_served_tokens=mc.cache_served_tokens,
            prefill_computed_tokens=mc.prefill_computed_tokens, decode_tokens=mc.decode_tokens,
            hit_rate_pct=mc.hit_rate_pct, calls=mc.calls, pinned_tokens=_worker_stat(h, 0),
            evicted_tokens=_worker_stat(h, 1), outputs=_outputs(h), metrics_json=_report(h, 0),
            calls_csv=_report(h, 1), trace_csv=_report(h, 2), recompute_tokens=mc.recompute_tokens,
            pin_compute_tokens=_worker_stat(h, 2), pin_seconds=t[0], iter_seconds=t[1],
            call_outputs=(co := _call_outputs(h)), call_logits=_call_logits(h, co))
    finally:
        lib.hk_run_free(h)


class PromptCache:
    """class PromptCache (prompt_cache.hpp:15-40) over the C ABI: an LRU map
    from operator signature to the tokens that operator produced, saved and
    loaded in the reference's JSON document byte for byte (prompt_cache.cpp),
    so the reference's optimizer (substitute_cached, optimizer.cpp:71-95) can
    serve a warm resubmission from values this executor generated."""

    def __init__(self, capacity: int = 4096, _handle=None):
        self._lib = _lib.load()
        self.handle = _handle if _handle is not None else self._lib.hk_pcache_create(capacity)
        if not self.handle:
            raise RuntimeError(_lib.last_error())

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            self._lib.hk_pcache_destroy(h)

    def contains(self, sig: int) -> bool:
        return bool(self._lib.hk_pcache_contains(self.handle, sig))

    def lookup(self, sig: int) -> Optional[List[int]]:
        """None on miss; a hit refreshes recency."""
        n = self._lib.hk_pcache_lookup(self.handle, sig, None, 0)
        if n < 0:
            return None
        out = (C.c_uint64 * max(1, n))()
        self._lib.hk_pcache_lookup(self.handle, sig, out, n)
        return list(out[:n])

    def insert(self, sig: int, value: Sequence[int]) -> None:
        arr, ptr = _lib.u64_array(list(value) or [0])
        _lib.check_status(self._lib.hk_pcache_insert(self.handle, sig, ptr, len(value)), "PromptCache.insert")

    def size(self) -> int:
        return int(self._lib.hk_pcache_size(self.handle))

    def capacity(self) -> int:
        return int(self._lib.hk_pcache_capacity(self.handle))

    def keys_lru_first(self) -> List[int]:
        n = self._lib.hk_pcache_keys(self.handle, None, 0)
        out = (C.c_uint64 * max(1, n))()
        self._lib.hk_pcache_keys(self.handle, out, n)
        return list(out[:n])

    def serialize(self) -> str:
        n = self._lib.hk_pcache_save(self.handle, None, 0)
        buf = C.create_string_buffer(n)
        self._lib.hk_pcache_save(self.handle, buf, n)
        return buf.value.decode()

    @staticmethod
    def deserialize(json_text: str) -> "PromptCache":
        b = json_text.encode()
        h = _lib.load().hk_pcache_load(b, len(b))
        if not h:
            raise RuntimeError(_lib.last_error())
        return PromptCache(_handle=h)

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.serialize())

    @staticmethod
    def load(path: str) -> "PromptCache":
        with open(path) as f:
            return PromptCache.deserialize(f.read())


def harvest_into_cache(plan: bytes, m: SimMetrics, cache: PromptCache) -> int:
    """harvest_into_cache (optimizer.cpp:113-125) with THIS run's values: every
    untainted format / lambda / llm node of `plan` (exported with its
    signature section), every query; llm values are the tokens the run's LLM
    body generated (the device transformer's under an Engine). Returns the
    number of entries inserted."""
    words = [len(m.call_outputs)]
    for (op, q), toks in sorted(m.call_outputs.items()):
        words += [op & (2**64 - 1), q, len(toks), *toks]
    arr, ptr = _lib.u64_array(words)
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    n = _lib.load().hk_pcache_harvest_calls(cache.handle, buf, len(plan), ptr, len(words))
    if n < 0:
        raise RuntimeError(_lib.last_error())
    return int(n)


def run_workflow(workflow: str, inputs: str, profile: str, workers: int = 1, capacities=(4096,),
                 cache: Optional["PromptCache"] = None, engine=None, **spec) -> dict:
    """run_workflow (run_pipeline.cpp:47-81) natively: the reference's JSON
    documents in, `helios run`'s documents out ({"report", "calls_csv",
    "trace_csv", "outputs_json", "schedule_json", "plan"}). spec keys mirror
    RunSpec: seed, stochastic, prune, merge_duplicates, cache_substitute,
    proactive_pin, pin_threshold, pin_capacity_frac, block, prefill_budget,
    alpha, run_sim, collect_trace, max_iterations."""
    lib = _lib.load()
    caps, cptr = _lib.u64_array(list(capacities))
    c = _lib.WorkflowSpecC(workers, cptr, len(capacities), spec.get("scheduler", "cache_aware").encode(),
                           spec.get("seed", 0), int(spec.get("stochastic", False)), int(spec.get("prune", True)),
                           int(spec.get("merge_duplicates", True)), int(spec.get("cache_substitute", True)),
                           int(spec.get("proactive_pin", True)), spec.get("pin_threshold", 200),
                           spec.get("pin_capacity_frac", 0.5), spec.get("block", 16), spec.get("prefill_budget", 0),
                           spec.get("alpha", 0.0), int(spec.get("run_sim", True)), int(spec.get("collect_trace", False)),
                           spec.get("max_iterations", 0))
    h = lib.hk_run_workflow(workflow.encode(), inputs.encode(), profile.encode(), C.byref(c),
                            cache.handle if cache is not None else None, engine.handle if engine is not None else None)
    if not h:
        raise RuntimeError(_lib.last_error())
    try:
        def doc(which):
            n = lib.hk_run_document(h, which, None, 0)
            buf = C.create_string_buffer(n)
            lib.hk_run_document(h, which, buf, n)
            return buf.value.decode()
        n = lib.hk_run_plan(h, None, 0)
        plan = (C.c_uint8 * n)()
        lib.hk_run_plan(h, plan, n)
        return {"report": doc(0), "outputs_json": doc(1), "schedule_json": doc(2), "calls_csv": _report(h, 1),
                "trace_csv": _report(h, 2), "plan": bytes(plan)}
    finally:
        lib.hk_run_free(h)


def sim_metrics_json(m: SimMetrics) -> str:
    return m.metrics_json


def sim_calls_csv(m: SimMetrics) -> str:
    return m.calls_csv


def sim_trace_csv(m: SimMetrics) -> str:
    return m.trace_csv


def needs_output_exchange(plan: bytes, cfg: SimConfig) -> bool:
    """True when some call of the schedule waits on a call of another worker,
    i.e. one-process-per-worker runs need simulate(..., exchange=...)."""
    for w in range(len(cfg.workers)):
        try:
            simulate(plan, cfg, only_worker=w)  # synthetic body: host control plane only
        except RuntimeError as e:
            if "cross-worker dependency" in str(e):
                return True
            raise
    return False


def worker_pins(plan: bytes, cfg: SimConfig, worker: int) -> List[List[int]]:
    """The prefixes simulate() pins on `worker` (simulator.cpp:257-263): budget
    = pin_capacity_frac x capacity; none when proactive pinning is off."""
    if not cfg.proactive_pin:
        return []
    w = cfg.workers[worker]
    return static_pin_prefixes(plan, worker, w.block, cfg.pin_threshold, int(cfg.pin_capacity_frac * w.capacity))


def static_pin_prefixes(plan: bytes, worker: int, block: int, threshold: int, budget_tokens: int) -> List[List[int]]:
    """static_pin_prefixes (simulator.hpp:67-69)."""
    lib = _lib.load()
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    cap = 1 << 22
    toks = np.zeros(cap, dtype=np.uint64)
    lens = np.zeros(4096, dtype=np.uint64)
    n = lib.hk_static_pin_prefixes(buf, len(plan), worker, block, threshold, budget_tokens,
                                   toks.ctypes.data_as(_lib.u64p), cap, lens.ctypes.data_as(_lib.u64p), 4096)
    if n < 0:
        raise RuntimeError(_lib.last_error())
    out, off = [], 0
    for i in range(n):
        ln = int(lens[i])
        out.append(toks[off:off + ln].tolist())
        off += ln
    return out


def synth_llm_len(prompt: Sequence[int], len_out: float, deterministic: bool, seed: int = 0,
                  stochastic: bool = False) -> int:
    a, p = _lib.u64_array(prompt)
    if len_out < 0:
        raise RuntimeError("negative len_out")
    return _lib.load().hk_synth_llm_len(p, len(a), len_out, int(deterministic), seed, int(stochastic))


def synth_llm_output(prompt: Sequence[int], len_out: float, deterministic: bool, seed: int = 0,
                     stochastic: bool = False) -> List[int]:
    a, p = _lib.u64_array(prompt)
    n = synth_llm_len(prompt, len_out, deterministic, seed, stochastic)
    out = np.zeros(max(n, 1), dtype=np.uint64)
    _lib.load().hk_synth_llm_output(p, len(a), len_out, int(deterministic), seed, int(stochastic),
                                    out.ctypes.data_as(_lib.u64p), n)
    return out[:n].tolist()


def fnv1a64(data: bytes, seed: int = 0xcbf29ce484222325) -> int:
    return _lib.load().hk_fnv1a64(data, len(data), seed)


def hash_combine(h: int, v: int) -> int:
    return _lib.load().hk_hash_combine(h, v)


def vocab_of(token: int, vocab: int) -> int:
    return _lib.load().hk_vocab_of(token, vocab)


def gen_token(vid: int, vocab: int) -> int:
    return _lib.load().hk_gen_token(vid, vocab)


def plan_call_groups(plan: bytes) -> Dict[tuple, tuple]:
    """{(op, query): (trt group node, static prefix tokens)} (hk_plan_call_groups)."""
    lib = _lib.load()
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    n = lib.hk_plan_call_groups(buf, len(plan), None, None, None, None, 0)
    if n < 0:
        raise RuntimeError(_lib.last_error())
    op = (C.c_int64 * max(n, 1))()
    q = (C.c_int32 * max(n, 1))()
    g = (C.c_int32 * max(n, 1))()
    t = (C.c_uint64 * max(n, 1))()
    lib.hk_plan_call_groups(buf, len(plan), op, q, g, t, n)
    return {(op[i], q[i]): (g[i], t[i]) for i in range(n)}


def plan_schedule(plan: bytes, workers: int, capacities: Sequence[int], alpha: float = 0.0) -> bytes:
    """Native cache-aware planner (partition_workflow + build_call_tree +
    plan_operators, scheduler.cpp / trt.cpp): the plan's value graph re-planned
    for `workers` workers; returns the new HKPLAN01 blob."""
    lib = _lib.load()
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    caps, cptr = _lib.u64_array(list(capacities))
    n = lib.hk_plan_schedule(buf, len(plan), workers, cptr, len(capacities), alpha, None, 0)
    if n < 0:
        raise RuntimeError(_lib.last_error())
    out = (C.c_uint8 * n)()
    lib.hk_plan_schedule(buf, len(plan), workers, cptr, len(capacities), alpha, out, n)
    return bytes(out)


def partition_calls(plan: bytes, workers: int) -> bytes:
    """Opt-in call-level partition (hk_plan_partition_calls): every operator's
    calls dealt round-robin over `workers`. DIVERGES from the reference, which
    places whole operators (scheduler.cpp:59-115)."""
    lib = _lib.load()
    buf = (C.c_uint8 * len(plan)).from_buffer_copy(plan)
    n = lib.hk_plan_partition_calls(buf, len(plan), workers, None, 0)
    if n < 0:
        raise RuntimeError(_lib.last_error())
    out = (C.c_uint8 * n)()
    lib.hk_plan_partition_calls(buf, len(plan), workers, out, n)
    return bytes(out)


def replicate_workers(cfg: "SimConfig", workers: int) -> "SimConfig":
    """SimConfig with the first worker's (capacity, block, budget) for every worker."""
    from dataclasses import replace
    return replace(cfg, workers=[cfg.workers[0]] * workers)
