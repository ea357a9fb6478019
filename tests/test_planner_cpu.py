"""Native cache-aware planner (csrc/host/planner.cpp) against
the reference planner compiled from its sources (oracle/_ref).

For a plan exported by the reference pipeline (bind -> rewrite -> partition ->
plan_operators -> build_call_tree), hk_plan_schedule re-plans the same value
graph natively: the call tree (parents, leaves, segment contents,
dependencies), the per-worker schedule and the simulate() reports of the
re-planned blob must equal the reference's — on every committed plan (1-8
workers, C1-C5) and on random workflow DAGs of every operator kind, 1-4
workers, mixed capacities.
"""
import random

import pytest

from conftest import needs_ref
from oracle import simulate as osim
from paper_2603_16104_b200 import helios
from paper_2603_16104_b200 import workloads as wl

PLANS = ["t_small", "t_press", "c1", "c1_w2", "c2", "c2_nopin", "c3", "c3_w2", "c4_w1", "c4_w2", "c4_w4", "c4_w8",
         "c5", "c2p_w2", "c2p_w4", "c2p_w8", "c2x2", "c2x4"]


def _tree(blob):
    p = osim.parse_plan(blob)
    out = []
    for t in p.tree:
        parts = []
        for is_static, v, q in t["parts"]:
            parts.append(("s", tuple(p.pool[p.spans[v][0]:p.spans[v][0] + p.spans[v][1]])) if is_static else ("p", v, q))
        out.append((t["parent"], t["leaf"], t["op"], t["query"], tuple(parts), tuple(t["preds"])))
    return out, p.sigma


def _check(blob, caps, workers, alpha=0.0):
    mine = helios.plan_schedule(blob, workers, caps, alpha)
    t_ref, s_ref = _tree(blob)
    t_mine, s_mine = _tree(mine)
    assert s_mine == s_ref
    assert t_mine == t_ref
    return mine


@needs_ref
@pytest.mark.parametrize("name", PLANS)
def test_native_planner_matches_committed_plans(name):
    blob, meta = wl.load_plan(name)
    sim = meta["sim"]
    caps = sim["capacity"] if len(set(sim["capacity"])) > 1 else sim["capacity"][:1]
    mine = _check(blob, caps, len(sim["capacity"]))
    sc = wl.sim_config_from_meta(meta)
    a, b = helios.simulate(blob, sc), helios.simulate(mine, sc)
    assert (a.metrics_json, a.calls_csv) == (b.metrics_json, b.calls_csv)


@needs_ref
@pytest.mark.parametrize("seed", range(40))
def test_native_planner_matches_reference_random_workflows(seed):
    from oracle import refpy
    rng = random.Random(1000 + seed)
    wf, inp, prof = refpy.generate_workload(
        {"llm_ops": rng.randint(1, 7), "batch": rng.randint(1, 4), "allow_nondeterminism": True, "seed": seed},
        random=True)
    workers = rng.choice([1, 2, 3, 4])
    caps = [rng.choice([64, 256, 4096])] if rng.random() < 0.5 else [rng.choice([64, 256, 4096]) for _ in range(workers)]
    alpha = rng.choice([0.0, 0.0, 0.25])
    spec = {"workers": workers, "capacities": caps, "alpha": alpha, "seed": seed}
    res, blob = refpy.run(wf, inp, prof, spec)
    mine = _check(blob, caps, workers, alpha)
    meta = {"sim": refpy.sim_config_dict(spec, len(res["sigma"]))}
    m = helios.simulate(mine, wl.sim_config_from_meta(meta))
    assert m.metrics_json == res["metrics_json"]


@needs_ref
def test_native_planner_replans_for_other_worker_counts():
    """configs[3] (C4', 8 operators) planned for 1 worker by the reference,
    re-planned natively for 2/4/8: equal to the reference's own c4_w2/4/8 plans."""
    blob1, _ = wl.load_plan("c4_w1")
    for w in (2, 4, 8):
        ref, meta = wl.load_plan(f"c4_w{w}")
        mine = helios.plan_schedule(blob1, w, meta["sim"]["capacity"][:1])
        assert _tree(mine) == _tree(ref), w


def test_native_planner_errors():
    blob, _ = wl.load_plan("t_small")
    with pytest.raises(RuntimeError, match="workers must be positive"):
        helios.plan_schedule(blob, 0, [4096])
    with pytest.raises(RuntimeError, match="capacity list"):
        helios.plan_schedule(blob, 2, [1, 2, 3])
