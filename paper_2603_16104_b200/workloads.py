"""Synthetic workflows of BASELINE.json's configs, in the reference's wire format.

Each builder returns (workflow, inputs, profile, spec) as JSON-able dicts in the
format of workflow_io.cpp (parse_workflow / parse_inputs / parse_profile) plus
a RunSpec-like dict. They restate the survey probes that produced the golden
SimMetrics of SURVEY.md §8(d) / BASELINE.md.

The executor input (an HKPLAN01 blob) is produced from these by the reference
planner (partition -> plan_operators -> call tree; out of scope for the B200
port) through integration/plan_export.hpp, and
committed under paper_2603_16104_b200/plans/ by tests/golden/make_golden.py so
the GPU box (which has no /root/reference) can run them.
"""
from __future__ import annotations

import gzip
import json
from pathlib import Path
from typing import Dict, List, Tuple

PLANS = Path(__file__).resolve().parent / "plans"


def words(tag: str, n: int) -> str:
    """n distinct words tag0..tag{n-1} (tests/support/builders.hpp:117-124)."""
    return " ".join(f"{tag}{i}" for i in range(n))


class WB:
    """Tiny workflow builder; node ids 0,1,2,... in creation order."""

    def __init__(self):
        self.nodes: List[dict] = []
        self.outputs: List[int] = []
        self.profile: Dict[str, dict] = {}

    def _add(self, kind: str, args: dict) -> int:
        nid = len(self.nodes)
        self.nodes.append({"id": nid, "kind": kind, "args": args})
        return nid

    def input(self, name: str) -> int:
        return self._add("input", {"name": name})

    def data(self, text: str) -> int:
        return self._add("data", {"values": [text]})

    def fmt(self, template: str, ins: List[int]) -> int:
        nid = self._add("format", {"template": template})
        self.nodes[nid]["_ins"] = ins
        return nid

    def llm(self, messages: List[Tuple[str, list]], len_out: float, deterministic: bool = True) -> int:
        msgs = []
        for role, parts in messages:
            jp = []
            for p in parts:
                jp.append({"ref": p} if isinstance(p, int) else {"text": p})
            msgs.append({"role": role, "parts": jp})
        nid = self._add("llm", {"messages": msgs, "deterministic": deterministic})
        self.profile[str(nid)] = {"len_out": float(len_out)}
        return nid

    def output(self, src: int) -> int:
        nid = self._add("output", {})
        self.nodes[nid]["_ins"] = [src]
        self.outputs.append(nid)
        return nid

    def workflow(self) -> dict:
        nodes, edges = [], []
        for n in self.nodes:
            ins = n.get("_ins")
            nodes.append({k: v for k, v in n.items() if k != "_ins"})
            if ins is not None:
                for s, src in enumerate(ins):
                    edges.append({"from": src, "to": n["id"], "slot": s})
        wf = {"nodes": nodes, "outputs": self.outputs}
        if edges:
            wf["edges"] = edges  # llm edges are derived from message refs by parse_workflow
        return wf


def sys_msg(text: str):
    return ("system", [text])


def user_msg(parts: list):
    return ("user", parts)


# --------------------------------------------------------------------- configs
def c1_tiny_mapred():
    """configs[0]: 4-branch map-reduce, 512-token shared static prefix, B=1."""
    b = WB()
    q = b.input("q")
    pre = words("pre", 510)
    maps = [b.llm([sys_msg(pre), user_msg([f"branch{k}:", q])], 32) for k in range(4)]
    parts: list = ["Question:", q]
    for m in maps:
        parts += ["Answer:", m]
    red = b.llm([sys_msg(words("reducer", 64)), user_msg(parts)], 48)
    b.output(red)
    inputs = {"q": [words("ask", 16)]}
    spec = {"workers": 1, "capacities": [8192], "prefill_budget": 256}
    return b.workflow(), inputs, b.profile, spec


def c2_branches(n_branches: int = 64, prefix_words: int = 2046, decode: int = 256, capacity: int = 262144,
                budget: int = 8192, pin: bool = True):
    """configs[1]: one op, B branches x (2K shared system prefix + 16-word query), greedy decode."""
    b = WB()
    q = b.input("q")
    op = b.llm([sys_msg(words("pre", prefix_words)), user_msg([q])], decode)
    b.output(op)
    inputs = {"q": [words(f"b{i}_", 16) for i in range(n_branches)]}
    spec = {"workers": 1, "capacities": [capacity], "prefill_budget": budget, "proactive_pin": pin}
    return b.workflow(), inputs, b.profile, spec


def c2_ops(n_ops: int = 64, workers: int = 1, prefix_words: int = 2046, decode: int = 256,
           capacity: int = 262144, budget: int = 8192, shared_prefix: bool = True, branches_per_op: int = 1):
    """C2': n_ops operators sharing the 2K system prompt, each
    with its own 15-word branch text; partitioned by operator over `workers`."""
    b = WB()
    q = b.input("q")
    for k in range(n_ops):
        pre = words("pre", prefix_words) if shared_prefix else words(f"pre{k}_", prefix_words)
        op = b.llm([sys_msg(pre), user_msg([words(f"br{k}_", 15), q])], decode)
        b.output(op)
    inputs = {"q": ["go"] if branches_per_op == 1 else [f"go{i}" for i in range(branches_per_op)]}
    spec = {"workers": workers, "capacities": [capacity], "prefill_budget": budget}
    return b.workflow(), inputs, b.profile, spec


def c3_reflect_spec():
    """configs[2]: generate -> critique -> refine via the reference's workload
    generator (workload_gen.cpp gen_reflect); materialised by make_golden.py."""
    gen = {"pattern": "reflect", "agents": 2, "batch": 8, "system_tokens": 512, "context_tokens": 1024,
           "question_tokens": 32, "len_out": 128, "len_jitter": False, "seed": 7}
    spec = {"workers": 1, "capacities": [262144], "prefill_budget": 8192}
    return gen, spec


def c4_overlap(workers: int = 1, batch: int = 64, decode: int = 128):
    """configs[3] (C4'): 8 operators, prefix overlap 0-90 % of a 1024-token
    prompt, B=64 synthetic-token queries each (512 calls)."""
    b = WB()
    T = 1024
    ratios = [0, 15, 30, 45, 60, 75, 90, 90]
    inputs = {}
    for f, r in enumerate(ratios):
        S = T * r // 100
        qn = f"u{f}"
        q = b.input(qn)
        msgs = []
        if S >= 2:
            msgs.append(sys_msg(words(f"fam{f}_", S - 2)))
        msgs.append(user_msg([q]))
        op = b.llm(msgs, decode)
        b.output(op)
        inputs[qn] = [{"token_count": T - S} for _ in range(batch)]
    spec = {"workers": workers, "capacities": [262144], "prefill_budget": 8192}
    return b.workflow(), inputs, b.profile, spec


def c5_pressure(n_branches: int = 128, ctx_words: int = 8190, decode: int = 256, capacity: int = 16384):
    """configs[4]: 128 branches x 8K shared context under a 16K-token cache."""
    b = WB()
    q = b.input("q")
    op = b.llm([sys_msg(words("ctx", ctx_words)), user_msg([q])], decode)
    b.output(op)
    inputs = {"q": [words(f"c{i}_", 32) for i in range(n_branches)]}
    spec = {"workers": 1, "capacities": [capacity], "prefill_budget": 8192}
    return b.workflow(), inputs, b.profile, spec


def c2_per_gpu(n_gpus: int, n_branches: int = 64, prefix_words: int = 2046, decode: int = 256):
    """Weak-scaling form of configs[1] for N GPUs: N operators of n_branches
    branches each, one per worker, all sharing the 2K system prompt so the
    pinned prefix is identical on every worker (K6 replication)."""
    b = WB()
    q = b.input("q")
    for k in range(n_gpus):
        op = b.llm([sys_msg(words("pre", prefix_words)), user_msg([f"op{k}", q])], decode)
        b.output(op)
    inputs = {"q": [words(f"b{i}_", 16) for i in range(n_branches)]}
    worker_of = {str(b.nodes[i]["id"]): k for k, i in enumerate(
        [n["id"] for n in b.nodes if n["kind"] == "llm"])}
    spec = {"workers": n_gpus, "capacities": [262144], "prefill_budget": 8192, "worker_of": worker_of}
    return b.workflow(), inputs, b.profile, spec


# ------------------------------------------------------------------ plan I/O
def load_plan(name: str) -> Tuple[bytes, dict]:
    """Committed plan blob + its sim config (from make_golden.py)."""
    with gzip.open(PLANS / f"{name}.plan.gz", "rb") as f:
        blob = f.read()
    meta = json.loads((PLANS / f"{name}.json").read_text())
    return blob, meta


def sim_config_from_meta(meta: dict):
    from .helios import SimConfig, SimWorkerConfig
    sc = meta["sim"]
    return SimConfig(
        workers=[SimWorkerConfig(c, b, p) for c, b, p in zip(sc["capacity"], sc["block"], sc["prefill_budget"])],
        proactive_pin=sc["proactive_pin"], pin_threshold=sc["pin_threshold"],
        pin_capacity_frac=sc["pin_capacity_frac"], seed=sc["seed"], stochastic=sc["stochastic"],
        collect_trace=sc.get("collect_trace", False), max_iterations=sc.get("max_iterations", 0))


def engine_sizing(blob: bytes, sc) -> dict:
    """Engine limits for a plan, from the executor's own synthetic-mode run
    (mode S: the reference's control plane with synth_llm_output, no device):
    the most calls live in one iteration on one worker, the longest call
    context (prompt + output), and the most private (uncached prompt + output)
    tokens of a call."""
    from .helios import simulate
    m = simulate(blob, sc)
    rows = [list(map(int, r.split(","))) for r in m.calls_csv.strip().split("\n")[1:]]
    # op,query,worker,admitted_iter,prefill_done_iter,completed_iter,prompt_tokens,cached_tokens,output_tokens
    events = {}
    for r in rows:
        events.setdefault(r[2], []).append((r[3], 1))
        events[r[2]].append((r[5] + 1, -1))
    max_live = 0
    for ev in events.values():
        live = 0
        for _, dlt in sorted(ev):
            live += dlt
            max_live = max(max_live, live)
    return {"max_live": max_live,
            "max_ctx": max((r[6] + r[8] for r in rows), default=0),
            "max_private": max((r[6] - r[7] + r[8] for r in rows), default=0),
            "decode_tokens": m.decode_tokens}
