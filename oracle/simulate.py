"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference's
executor for small cases, with a pluggable LLM body.

Restates, line by line in behaviour:
  * KvCache                 simulator.cpp:14-128   (O(N) LRU scan, as the reference)
  * static_pin_prefixes     simulator.cpp:132-199
  * simulate                simulator.cpp:222-389
  * Evaluator::prompt/value evaluator.cpp:79-157, apply_lambda workflow.cpp:258-273
  * synth_* / hashes        evaluator.cpp:13-58, tokens.cpp:7-65
over the HKPLAN01 blob (include/helium_b200.h). In synthetic mode it is pinned
against the reference's committed golden reports (tests/test_oracle_cpu.py);
in model mode the LLM body is oracle.transformer.Decoder greedy decoding and
the generated vocab id v becomes Token gen_token(v) — the same definitions the
B200 executor uses.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

MASK = (1 << 64) - 1
FNV_OFF = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


# ------------------------------------------------------------------ hashes
def fnv1a64(data: bytes, h: int = FNV_OFF) -> int:
    for b in data:
        h = ((h ^ b) * FNV_PRIME) & MASK
    return h


def hash_combine(h: int, v: int) -> int:
    h = ((h ^ 0x9E3779B97F4A7C15) * FNV_PRIME) & MASK
    return fnv1a64(struct.pack("<Q", v), h)


def hash_tokens(toks: List[int], seed: int = FNV_OFF) -> int:
    return fnv1a64(struct.pack(f"<{len(toks)}Q", *toks), seed)


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def _digest(prompt: List[int], seed: int) -> int:
    h = hash_combine(hash_tokens(prompt), seed)
    return fnv1a64(b"\x02", h)


def synth_output_len(prompt, len_out: float, seed: int, stochastic: bool) -> int:
    if len_out < 0:
        raise RuntimeError("negative len_out")
    base = int(math.floor(len_out + 0.5)) if len_out >= 0 else 0  # llround for non-negative
    if not stochastic:
        return base
    h = splitmix64(hash_combine(_digest(prompt, seed), 0x6C656E))
    return h % (2 * base + 1)


def synth_llm_len(prompt, len_out, det, seed, stochastic) -> int:
    return synth_output_len(prompt, len_out, 0 if det else seed, stochastic)


def synth_llm_output(prompt, len_out, det, seed, stochastic) -> List[int]:
    s = 0 if det else seed
    n = synth_output_len(prompt, len_out, s, stochastic)
    d = _digest(prompt, s)
    return [splitmix64(hash_combine(d, i)) for i in range(n)]


def gen_token(vid: int, vocab: int) -> int:
    h = fnv1a64(bytes([0x03]) + struct.pack("<I", vid))
    return (h - h % vocab + vid) & MASK


# ---------------------------------------------------------------- HKPLAN01
@dataclass
class Plan:
    batch: int
    pool: List[int]
    spans: List[Tuple[int, int]]
    nodes: Dict[int, dict]
    outputs: List[int]
    tree: List[dict]
    sigma: List[List[Tuple[int, int]]]

    def span(self, s: int) -> List[int]:
        o, n = self.spans[s]
        return self.pool[o:o + n]


def parse_plan(blob: bytes) -> Plan:
    w = struct.unpack(f"<{len(blob) // 8}Q", blob)
    i = 0

    def u():
        nonlocal i
        i += 1
        return w[i - 1]

    def s64():
        v = u()
        return v - (1 << 64) if v >> 63 else v

    assert u() == 0x31304E414C504B48, "bad magic"
    batch = u()
    nt = u()
    pool = list(w[i:i + nt])
    i += nt
    ns = u()
    spans = [(u(), u()) for _ in range(ns)]
    nodes = {}
    for _ in range(u()):
        nid, kind, flags = s64(), u(), u()
        lo = struct.unpack("<d", struct.pack("<Q", u()))[0]
        na = u()
        a = [s64() for _ in range(na)]
        nodes[nid] = {"kind": kind, "det": bool(flags & 1), "has_profile": bool(flags & 2), "len_out": lo, "a": a}
    outputs = [s64() for _ in range(u())]
    tree = []
    for _ in range(u()):
        parent, is_leaf, op, q = s64(), u(), s64(), s64()
        parts = [(u(), s64(), s64()) for _ in range(u())]
        preds = [s64() for _ in range(u())]
        tree.append({"parent": parent, "leaf": bool(is_leaf), "op": op, "query": q, "parts": parts, "preds": preds})
    sigma = []
    for _ in range(u()):
        sigma.append([(s64(), s64()) for _ in range(u())])
    if i < len(w):  # optional HKSIG001 signature section (prompt cache keys): not used by simulate()
        assert w[i] == 0x3130304749534b48, "plan: trailing bytes"
        i = len(w)
    assert i == len(w)
    return Plan(batch, pool, spans, nodes, outputs, tree, sigma)


class Evaluator:
    def __init__(self, plan: Plan, seed: int, stochastic: bool, strict: bool):
        self.p, self.seed, self.stochastic, self.strict = plan, seed, stochastic, strict
        self.memo: Dict[Tuple[int, int], List[int]] = {}

    def prompt(self, llm: int, q: int) -> List[int]:
        n = self.p.nodes[llm]
        out: List[int] = []
        a = n["a"]
        for k in range(0, len(a), 2):
            out += self.p.span(a[k + 1]) if a[k] == 0 else self.value(a[k + 1], q)
        return out

    def value(self, nid: int, q: int) -> List[int]:
        key = (nid, q)
        if key in self.memo:
            return self.memo[key]
        n = self.p.nodes[nid]
        k, a = n["kind"], n["a"]
        if k == 0:
            v = list(self.p.span(a[q]))
        elif k == 1:
            v = list(self.value(a[0], q))
        elif k == 2:
            ins = [self.value(x, q) for x in a[2:]]
            if a[0] == 0:
                v = list(ins[0])
            elif a[0] == 1:
                v = [t for s in ins for t in s]
            else:
                v = list(ins[0])[:a[1]]
        elif k == 3:
            v = []
            for j in range(0, len(a), 2):
                v += self.p.span(a[j + 1]) if a[j] == 0 else self.value(a[j + 1], q)
        else:
            if self.strict:
                raise RuntimeError(f"llm node {nid} query {q} evaluated before its call completed")
            pr = self.prompt(nid, q)
            v = synth_llm_output(pr, n["len_out"], n["det"], self.seed, self.stochastic)
        self.memo[key] = v
        return v


# ------------------------------------------------------------------ KvCache
class KvCache:
    """simulator.cpp:14-128, including the O(N) eviction scan."""

    def __init__(self, cap: int, block: int):
        if block == 0:
            raise RuntimeError("kv block size must be positive")
        if cap < block:
            raise RuntimeError("kv capacity below one block")
        self.cap, self.block = cap, block
        self.used = self.pinned = self.evicted = self.clock = 0
        self.nodes = [{"parent": -1, "kids": {}, "pinned": False, "holds": 0, "last": 0, "free": False}]
        self.free: List[int] = []
        self.holds: Dict[int, List[int]] = {}

    def _touch(self, i):
        self.clock += 1
        self.nodes[i]["last"] = self.clock

    def _create(self, parent, key):
        if self.free:
            idx = self.free.pop()
            self.nodes[idx] = {"parent": -1, "kids": {}, "pinned": False, "holds": 0, "last": 0, "free": False}
        else:
            idx = len(self.nodes)
            self.nodes.append({"parent": -1, "kids": {}, "pinned": False, "holds": 0, "last": 0, "free": False})
        self.nodes[idx]["parent"] = parent
        self.nodes[parent]["kids"][key] = idx
        return idx

    def _evict_one(self) -> bool:
        victim, best = -1, 0
        for i in range(1, len(self.nodes)):
            n = self.nodes[i]
            if n["free"] or n["pinned"] or n["holds"] > 0 or n["kids"]:
                continue
            if victim < 0 or n["last"] < best:
                victim, best = i, n["last"]
        if victim < 0:
            return False
        v = self.nodes[victim]
        p = self.nodes[v["parent"]]
        for k, c in list(p["kids"].items()):
            if c == victim:
                del p["kids"][k]
                break
        v["free"] = True
        self.free.append(victim)
        self.used -= self.block
        self.evicted += self.block
        return True

    def lookup(self, seq, hold=0) -> int:
        matched, cur, b = 0, 0, self.block
        for off in range(0, len(seq) - b + 1, b):
            nxt = self.nodes[cur]["kids"].get(tuple(seq[off:off + b]))
            if nxt is None:
                break
            self._touch(nxt)
            if hold:
                self.nodes[nxt]["holds"] += 1
                self.holds.setdefault(hold, []).append(nxt)
            matched += b
            cur = nxt
        return matched

    def insert(self, seq, length, pinned, hold=0) -> int:
        length = min(length, len(seq))
        stored, cur, b = 0, 0, self.block
        for off in range(0, length - b + 1, b):
            key = tuple(seq[off:off + b])
            nxt = self.nodes[cur]["kids"].get(key)
            if nxt is None:
                while self.used + b > self.cap:
                    if not self._evict_one():
                        return stored
                nxt = self._create(cur, key)
                self.used += b
                stored += b
            n = self.nodes[nxt]
            if pinned and not n["pinned"]:
                n["pinned"] = True
                self.pinned += b
            self._touch(nxt)
            if hold:
                n["holds"] += 1
                self.holds.setdefault(hold, []).append(nxt)
            cur = nxt
        return stored

    def release(self, hold):
        for i in self.holds.pop(hold, []):
            self.nodes[i]["holds"] -= 1


def static_pin_prefixes(p: Plan, worker: int, block: int, threshold: int, budget: int) -> List[List[int]]:
    place = {}
    for w, wq in enumerate(p.sigma):
        for c in wq:
            place[c] = w
    cnt = [0] * len(p.tree)
    for i, t in enumerate(p.tree):
        if not t["leaf"] or place.get((t["op"], t["query"])) != worker:
            continue
        v = i
        while v >= 0:
            cnt[v] += 1
            v = p.tree[v]["parent"]

    def path(n):
        out = []
        while n >= 0:
            out.append(n)
            n = p.tree[n]["parent"]
        return out[::-1]

    cands = []
    for i in range(1, len(p.tree)):
        if cnt[i] < 2:
            continue
        n = p.tree[i]
        prefix, concrete = [], True
        for anc in path(n["parent"]):
            parts = p.tree[anc]["parts"]
            if not all(pt[0] for pt in parts):
                concrete = False
                break
            for pt in parts:
                prefix += p.span(pt[1])
        if not concrete:
            continue
        for pt in n["parts"]:
            if not pt[0]:
                break
            prefix += p.span(pt[1])
        prefix = prefix[:len(prefix) - len(prefix) % block]
        if len(prefix) < threshold or not prefix:
            continue
        cands.append(prefix)
    cands.sort(key=lambda c: (-len(c), c))
    uniq = []
    for c in cands:
        if not uniq or uniq[-1] != c:
            uniq.append(c)
    chosen, out, total = set(), [], 0
    for c in uniq:
        marginal = sum(block for off in range(0, len(c) - block + 1, block) if tuple(c[:off + block]) not in chosen)
        if total + marginal > budget:
            continue
        for off in range(0, len(c) - block + 1, block):
            chosen.add(tuple(c[:off + block]))
        total += marginal
        out.append(c)
    return out


# ----------------------------------------------------------------- simulate
@dataclass
class SimCfg:
    capacity: List[int]
    block: List[int]
    prefill_budget: List[int]
    proactive_pin: bool = True
    pin_threshold: int = 200
    pin_capacity_frac: float = 0.5
    seed: int = 0
    stochastic: bool = False
    collect_trace: bool = False
    max_iterations: int = 0

    @staticmethod
    def from_meta(sc: dict) -> "SimCfg":
        return SimCfg(list(sc["capacity"]), list(sc["block"]), list(sc["prefill_budget"]), sc["proactive_pin"],
                      sc["pin_threshold"], sc["pin_capacity_frac"], sc["seed"], sc["stochastic"],
                      sc.get("collect_trace", False), sc.get("max_iterations", 0))


def simulate(p: Plan, cfg: SimCfg, body: Optional[Callable[[List[int], int, float, bool], List[int]]] = None):
    """Returns (metrics dict, calls rows, trace rows, outputs, prompts{(op,q): prompt}).
    body(prompt, out_len, len_out, det, call) -> output tokens; None = synth_llm_output."""
    W = len(p.sigma)
    if W == 0:
        raise RuntimeError("simulate: no workers")
    if len(cfg.capacity) != W:
        raise RuntimeError("simulate: worker config count does not match schedule")
    leaf_of = {(t["op"], t["query"]): i for i, t in enumerate(p.tree) if t["leaf"]}
    seen, total = set(), 0
    for wq in p.sigma:
        for c in wq:
            if c not in leaf_of:
                raise RuntimeError("simulate: scheduled call is not a tree leaf")
            if c in seen:
                raise RuntimeError("simulate: call scheduled twice")
            seen.add(c)
            total += 1
    if total != len(leaf_of):
        raise RuntimeError("simulate: schedule does not cover all calls")
    ev = Evaluator(p, cfg.seed, cfg.stochastic, True)
    caches, budgets, pinned = [], [], []
    for w in range(W):
        c = KvCache(cfg.capacity[w], cfg.block[w])
        caches.append(c)
        budgets.append(cfg.prefill_budget[w] if cfg.prefill_budget[w] > 0 else max(cfg.capacity[w] // 8, cfg.block[w]))
        if cfg.proactive_pin:
            bud = int(cfg.pin_capacity_frac * cfg.capacity[w])
            for pin in static_pin_prefixes(p, w, cfg.block[w], cfg.pin_threshold, bud):
                c.insert(pin, len(pin), True)
        pinned.append(c.pinned)
    leaf_done = [False] * len(p.tree)
    admitted = [[False] * len(wq) for wq in p.sigma]
    live: List[List[dict]] = [[] for _ in range(W)]
    backlog = [0] * W
    m = {"iterations": 0, "prompt_tokens": 0, "cache_served_tokens": 0, "prefill_computed_tokens": 0,
         "decode_tokens": 0}
    calls, trace, prompts = [], [], {}
    guard = cfg.max_iterations or 10_000_000
    holdc = completed = it = 0
    while completed < total:
        it += 1
        if it > guard:
            raise RuntimeError("simulate: iteration guard tripped")
        for w in range(W):
            cache = caches[w]
            row = {"iter": it, "worker": w, "active": 0, "admitted": 0, "prefill": 0, "decode": 0}
            for qi, call in enumerate(p.sigma[w]):
                if admitted[w][qi]:
                    continue
                if backlog[w] >= budgets[w]:
                    break
                leaf = leaf_of[call]
                if not all(leaf_done[x] for x in p.tree[leaf]["preds"]):
                    continue
                admitted[w][qi] = True
                op, q = call
                pr = ev.prompt(op, q)
                nd = p.nodes[op]
                if not nd["has_profile"]:
                    raise RuntimeError(f"no profile entry for llm node {op}")
                holdc += 1
                lc = {"id": call, "leaf": leaf, "prompt": pr,
                      "out_len": synth_llm_len(pr, nd["len_out"], nd["det"], cfg.seed, cfg.stochastic),
                      "hold": holdc, "decoded": 0, "pd": 0, "row": len(calls), "fin": False}
                lc["done"] = cache.lookup(pr, holdc)
                if lc["done"] == len(pr):
                    lc["pd"] = it
                backlog[w] += len(pr) - lc["done"]
                calls.append([op, q, w, it, 0, 0, len(pr), lc["done"], 0])
                m["prompt_tokens"] += len(pr)
                m["cache_served_tokens"] += lc["done"]
                prompts[call] = pr
                live[w].append(lc)
                row["admitted"] += 1
            row["active"] = len(live[w])
            left = budgets[w]
            for lc in live[w]:
                if left == 0:
                    break
                rem = len(lc["prompt"]) - lc["done"]
                if rem == 0:
                    continue
                chunk = min(left, rem)
                lc["done"] += chunk
                left -= chunk
                backlog[w] -= chunk
                m["prefill_computed_tokens"] += chunk
                row["prefill"] += chunk
                cache.insert(lc["prompt"], lc["done"], False, lc["hold"])
                if lc["done"] == len(lc["prompt"]):
                    lc["pd"] = it
            for lc in live[w]:
                if lc["fin"] or lc["done"] < len(lc["prompt"]):
                    continue
                if lc["out_len"] > 0:
                    if lc["pd"] >= it:
                        continue
                    lc["decoded"] += 1
                    row["decode"] += 1
                    m["decode_tokens"] += 1
                    if lc["decoded"] < lc["out_len"]:
                        continue
                op, q = lc["id"]
                nd = p.nodes[op]
                if body is None:
                    out = synth_llm_output(lc["prompt"], nd["len_out"], nd["det"], cfg.seed, cfg.stochastic)
                else:
                    out = body(lc["prompt"], lc["out_len"], nd["len_out"], nd["det"], lc["id"]) if lc["out_len"] else []
                if len(out) != lc["out_len"]:
                    raise RuntimeError("simulate: output length drifted from plan")
                ev.memo[(op, q)] = out
                cache.insert(lc["prompt"] + out, len(lc["prompt"]) + len(out), False, 0)
                cache.release(lc["hold"])
                leaf_done[lc["leaf"]] = True
                r = calls[lc["row"]]
                r[4], r[5], r[8] = lc["pd"], it, len(out)
                lc["fin"] = True
                completed += 1
            live[w] = [lc for lc in live[w] if not lc["fin"]]
            if cfg.collect_trace:
                trace.append(row)
    m["iterations"] = it
    m["hit_rate_pct"] = 100.0 * m["cache_served_tokens"] / m["prompt_tokens"] if m["prompt_tokens"] else 0.0
    m["pinned_tokens"] = pinned
    m["evicted_tokens"] = [c.evicted for c in caches]
    m["calls"] = len(calls)
    ev.strict = False
    outputs = {o: [ev.value(o, b) for b in range(p.batch)] for o in p.outputs}
    return m, calls, trace, outputs, prompts


def calls_csv(calls) -> str:
    s = "op,query,worker,admitted_iter,prefill_done_iter,completed_iter,prompt_tokens,cached_tokens,output_tokens\n"
    return s + "".join(",".join(str(x) for x in r) + "\n" for r in calls)


def trace_csv(trace) -> str:
    s = "iter,worker,active,admitted,prefill_tokens,decode_tokens\n"
    return s + "".join(f"{r['iter']},{r['worker']},{r['active']},{r['admitted']},{r['prefill']},{r['decode']}\n"
                       for r in trace)
