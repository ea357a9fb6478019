"""CPU parity of the host executor against the reference (mode S).

Oracle: the unmodified reference library (oracle/_ref) and the committed
fixtures made from it (tests/golden/make_golden.py). Known answers restate
test_tokens.cpp, test_evaluator.cpp and test_simulator.cpp of the reference.
"""
import json
import random
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import needs_ref
from paper_2603_16104_b200 import _lib, helios
from paper_2603_16104_b200 import workloads as wl

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def words_tokens(tag, n):
    return [helios.fnv1a64(f"{tag}{i}".encode()) for i in range(n)]


# ------------------------------------------------------------- tokens.cpp
def test_fnv_golden_vectors():
    # test_tokens.cpp:10-15
    assert helios.fnv1a64(b"") == 0xcbf29ce484222325
    assert helios.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert helios.fnv1a64(b"foobar") == 0x85944171f73967e8


def test_role_marker_tokens():
    # <|system|>, <|assistant|>, <|user|>
    assert helios.fnv1a64(b"<|system|>") == 0xe623f1012d67351a
    assert helios.fnv1a64(b"<|assistant|>") == 0x669ecc550a1d822d
    assert helios.fnv1a64(b"<|user|>") == 0xa6d93b62fd109f5c


@needs_ref
def test_hash_combine_and_synth_match_reference():
    from oracle import refpy
    rng = random.Random(1)
    for _ in range(200):
        h, v = rng.getrandbits(64), rng.getrandbits(64)
        assert helios.hash_combine(h, v) == refpy.hash_combine(h, v)
    for _ in range(60):
        prompt = [rng.getrandbits(64) for _ in range(rng.randint(0, 40))]
        len_out = rng.choice([0.0, 1.0, 7.4, 7.6, 32.0])
        for det in (True, False):
            for stoch in (False, True):
                seed = rng.getrandbits(16)
                assert helios.synth_llm_len(prompt, len_out, det, seed, stoch) == \
                    refpy.synth_llm_len(prompt, len_out, det, seed, stoch)
                assert helios.synth_llm_output(prompt, len_out, det, seed, stoch) == \
                    refpy.synth_llm_output(prompt, len_out, det, seed, stoch)


def test_synth_known_answers():
    # test_evaluator.cpp:79-120: det output ignores seed; rounding 7.4->7, 7.6->8;
    # stochastic length in [0, 2*base]
    p = words_tokens("w", 10)
    assert helios.synth_llm_output(p, 5, True, 1) == helios.synth_llm_output(p, 5, True, 2)
    assert helios.synth_llm_output(p, 5, False, 1) != helios.synth_llm_output(p, 5, False, 2)
    assert helios.synth_llm_len(p, 7.4, True) == 7
    assert helios.synth_llm_len(p, 7.6, True) == 8
    for s in range(50):
        n = helios.synth_llm_len(p, 6, False, s, True)
        assert 0 <= n <= 12
    with pytest.raises(RuntimeError, match="negative len_out"):
        helios.synth_llm_len(p, -1, True)


def test_gen_token_residue():
    for vid in (0, 1, 12345, 128255):
        t = helios.gen_token(vid, 128256)
        assert helios.vocab_of(t, 128256) == vid
        assert t != vid


# ------------------------------------------------------------ KvCache known answers
def numbered(tag, n):
    return words_tokens(tag, n)


def test_kv_block_granularity():
    # test_simulator.cpp:45-56
    c = helios.KvCache(64, 4)
    assert c.insert(numbered("a", 3), 3, False) == 0
    assert c.used_tokens() == 0
    assert c.insert(numbered("a", 11), 11, False) == 8
    assert c.used_tokens() == 8
    assert c.lookup(numbered("a", 11)) == 8
    assert c.lookup(numbered("a", 6)) == 4
    assert c.lookup(numbered("b", 11)) == 0
    assert c.insert(numbered("a", 11), 11, False) == 0


def test_kv_lru_eviction():
    # test_simulator.cpp:58-68
    c = helios.KvCache(16, 4)
    assert c.insert(numbered("a", 8), 8, False) == 8
    assert c.insert(numbered("b", 8), 8, False) == 8
    assert c.used_tokens() == 16
    c.lookup(numbered("a", 8))
    assert c.insert(numbered("c", 4), 4, False) == 4
    assert c.lookup(numbered("a", 8)) == 8
    assert c.lookup(numbered("b", 8)) == 4
    assert c.evicted_tokens() == 4


def test_kv_pins_and_holds():
    # test_simulator.cpp:70-98
    c = helios.KvCache(16, 4)
    assert c.insert(numbered("pin", 8), 8, True) == 8
    assert c.pinned_tokens() == 8
    for r in range(6):
        c.insert(numbered(f"fill{r}", 8), 8, False)
    assert c.lookup(numbered("pin", 8)) == 8
    assert c.used_tokens() <= 16

    c = helios.KvCache(16, 4)
    assert c.insert(numbered("held", 8), 8, False, 7) == 8
    assert c.insert(numbered("x", 8), 8, False) == 8
    assert c.insert(numbered("y", 8), 8, False) == 8
    assert c.lookup(numbered("held", 8)) == 8
    assert c.lookup(numbered("x", 8)) == 0
    c.release(7)
    c.insert(numbered("z", 16), 16, False)
    assert c.lookup(numbered("held", 8)) < 8

    c = helios.KvCache(8, 4)
    assert c.insert(numbered("pin", 8), 8, True) == 8
    assert c.insert(numbered("new", 8), 8, False) == 0
    assert c.lookup(numbered("pin", 8)) == 8


def test_kv_ctor_errors():
    with pytest.raises(RuntimeError, match="kv block size must be positive"):
        helios.KvCache(16, 0)
    with pytest.raises(RuntimeError, match="kv capacity below one block"):
        helios.KvCache(3, 4)


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_kvtree_matches_reference_fuzz(seed):
    """Random lookup/insert/release streams, lockstep with the reference KvCache."""
    from oracle import refpy
    rng = random.Random(seed)
    block = rng.choice([2, 4, 16])
    cap = block * rng.randint(2, 40)
    mine, ref = helios.KvCache(cap, block), refpy.RefKvCache(cap, block)
    alphabet = [rng.getrandbits(64) for _ in range(6)]  # small alphabet -> shared prefixes
    holds = []
    for step in range(1500):
        op = rng.random()
        n = rng.randint(0, block * 8)
        seq = [rng.choice(alphabet) for _ in range(n)]
        if op < 0.35:
            hold = rng.choice([0, 0, step + 1])
            if hold:
                holds.append(hold)
            assert mine.lookup(seq, hold) == ref.lookup(seq, hold)
        elif op < 0.85:
            ln = rng.randint(0, n)
            pinned = rng.random() < 0.05
            hold = rng.choice([0, 0, step + 1])
            if hold:
                holds.append(hold)
            assert mine.insert(seq, ln, pinned, hold) == ref.insert(seq, ln, pinned, hold)
        elif holds:
            h = holds.pop(rng.randrange(len(holds)))
            mine.release(h)
            ref.release(h)
        assert [mine.used_tokens(), mine.pinned_tokens(), mine.evicted_tokens()] == ref.counters()


# ------------------------------------------------------------ simulate, mode S
PLAN_NAMES = ["c1", "c2", "c2_nopin", "c2p_w1", "c2p_w2", "c2p_w4", "c2p_w8", "c3", "c4_w1", "c4_w2",
              "c4_w4", "c4_w8", "c5", "c2x1", "c2x2", "c2x4", "c2x8", "t_small", "t_press"]


def _digest(outputs):
    import hashlib
    h = hashlib.sha256()
    for k in sorted(outputs, key=int):
        h.update(f"{k}:".encode())
        for v in outputs[k]:
            h.update(len(v).to_bytes(8, "little"))
            for t in v:
                h.update(int(t).to_bytes(8, "little"))
    return h.hexdigest()


@pytest.mark.parametrize("name", PLAN_NAMES)
def test_simulate_synthetic_matches_reference_golden(name):
    """Byte-identical sim_metrics_json / calls / trace / outputs on the committed plans."""
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    m = helios.simulate(blob, wl.sim_config_from_meta(meta))
    assert m.metrics_json == gold["metrics_json"]
    assert m.calls_csv == gold["calls_csv"]
    assert m.trace_csv == gold["trace_csv"]
    assert _digest(m.outputs) == gold["outputs_sha256"]
    if "outputs" in gold:
        assert {str(k): v for k, v in m.outputs.items()} == gold["outputs"]


def _ref_and_mine(wf, inputs, profile, spec):
    from oracle import refpy
    res, blob = refpy.run(wf, inputs, profile, spec)
    meta = {"sim": refpy.sim_config_dict(spec, len(res["sigma"]))}
    m = helios.simulate(blob, wl.sim_config_from_meta(meta))
    return res, m


@needs_ref
@pytest.mark.parametrize("seed", range(40))
def test_simulate_random_workflows_match_reference(seed):
    """Random DAGs of every operator kind (workload_gen.cpp:427-489), W in {1,2,3},
    deterministic and stochastic runs, with and without pins / tiny caches."""
    from oracle import refpy
    rng = random.Random(seed)
    wf, inp, prof = refpy.generate_workload(
        {"llm_ops": rng.randint(1, 6), "batch": rng.randint(1, 4), "allow_nondeterminism": True, "seed": seed},
        random=True)
    spec = {"workers": rng.choice([1, 2, 3]), "capacities": [rng.choice([64, 256, 4096])],
            "prefill_budget": rng.choice([0, 16, 64]), "block": rng.choice([4, 16]),
            "proactive_pin": rng.random() < 0.7, "pin_threshold": rng.choice([16, 200]),
            "seed": rng.getrandbits(16), "stochastic": rng.random() < 0.5, "collect_trace": True}
    if spec["capacities"][0] < spec["block"]:
        spec["capacities"] = [spec["block"] * 4]
    res, m = _ref_and_mine(json.loads(wf), json.loads(inp), json.loads(prof), spec)
    assert m.metrics_json == res["metrics_json"]
    assert m.calls_csv == res["calls_csv"]
    assert m.trace_csv == res["trace_csv"]
    assert {str(k): v for k, v in m.outputs.items()} == res["outputs"]


@needs_ref
@pytest.mark.parametrize("pattern", ["mapred", "debate", "reflect", "iterative", "parallel", "trading_mini"])
def test_simulate_generator_patterns_match_reference(pattern):
    from oracle import refpy
    wf, inp, prof = refpy.generate_workload({"pattern": pattern, "agents": 3, "batch": 3, "seed": 5,
                                             "system_tokens": 120, "context_tokens": 60})
    for spec in ({"workers": 2, "capacities": [1024], "prefill_budget": 64, "seed": 3, "collect_trace": True},
                 {"workers": 1, "capacities": [256], "prefill_budget": 32, "stochastic": True, "seed": 9,
                  "collect_trace": True}):
        res, m = _ref_and_mine(json.loads(wf), json.loads(inp), json.loads(prof), spec)
        assert m.metrics_json == res["metrics_json"]
        assert m.calls_csv == res["calls_csv"]
        assert m.trace_csv == res["trace_csv"]
        assert {str(k): v for k, v in m.outputs.items()} == res["outputs"]


# ------------------------------------------------------------ test_simulator.cpp fixtures
def _tiny(wb_fn, spec):
    from oracle import refpy
    b = wl.WB()
    wb_fn(b)
    return _ref_and_mine(b.workflow(), {}, b.profile, spec)


@needs_ref
def test_cold_call_timeline():
    # test_simulator.cpp:134-153
    def mk(b):
        op = b.llm([wl.sys_msg(wl.words("sys", 30)), wl.user_msg([wl.words("ask", 10)])], 5)
        b.output(op)
    res, m = _tiny(mk, {"workers": 1, "capacities": [4096], "prefill_budget": 16, "proactive_pin": False,
                        "plan_capacities": [4096]})
    assert m.prompt_tokens == 42 and m.prefill_computed_tokens == 42 and m.cache_served_tokens == 0
    assert m.decode_tokens == 5 and m.iterations == 8
    row = m.calls_csv.strip().split("\n")[1].split(",")
    assert row[4] == "3" and row[5] == "8"
    assert m.metrics_json == res["metrics_json"]


@needs_ref
def test_dependent_call_hits_shared_system_prompt():
    # test_simulator.cpp:155-173
    def mk(b):
        persona = wl.words("persona", 40)
        first = b.llm([wl.sys_msg(persona), wl.user_msg(["answer: something"])], 4)
        second = b.llm([wl.sys_msg(persona), wl.user_msg(["critique:", first])], 4)
        b.output(second)
    res, m = _tiny(mk, {"workers": 1, "capacities": [4096], "proactive_pin": False})
    rows = [r.split(",") for r in m.calls_csv.strip().split("\n")[1:]]
    assert int(rows[1][3]) > int(rows[0][5])
    assert rows[1][7] == "32" and m.cache_served_tokens == 32
    assert m.metrics_json == res["metrics_json"]


@needs_ref
def test_burst_admission_serves_exactly_pins():
    # test_simulator.cpp:175-194
    from oracle import refpy
    b = wl.WB()
    q = b.input("q")
    op = b.llm([wl.sys_msg(wl.words("bulk", 60)), wl.user_msg(["solve:", q])], 3)
    b.output(op)
    spec = {"workers": 1, "capacities": [8192], "prefill_budget": 8192, "proactive_pin": True,
            "pin_threshold": 32, "plan_capacities": [4096]}
    inputs = {"q": ["same question"] * 4}
    res, m = _ref_and_mine(b.workflow(), inputs, b.profile, spec)
    res2, blob = refpy.run(b.workflow(), inputs, b.profile, spec)
    pins = helios.static_pin_prefixes(blob, 0, 16, 32, 4096)
    assert len(pins) == 1
    assert m.cache_served_tokens == 4 * len(pins[0])
    assert m.pinned_tokens[0] == len(pins[0])
    assert m.metrics_json == res["metrics_json"]


@needs_ref
def test_static_pin_prefixes_match_reference():
    # test_simulator.cpp:100-132
    from oracle import refpy
    b = wl.WB()
    q = b.input("q")
    persona = wl.words("persona", 40)
    a = b.llm([wl.sys_msg(persona), wl.user_msg(["answer:", q])], 3)
    bb = b.llm([wl.sys_msg(persona), wl.user_msg(["check:", q])], 3)
    lone = b.llm([wl.sys_msg(wl.words("other", 40)), wl.user_msg([q])], 3)
    for n in (a, bb, lone):
        b.output(n)
    wf, inputs = b.workflow(), {"q": ["the question"]}
    spec = {"workers": 1, "worker_of": {str(a): 0, str(bb): 0, str(lone): 0},
            "sigma": [[[a, 0], [bb, 0], [lone, 0]]]}
    _, blob = refpy.run(wf, inputs, b.profile, spec)
    pins = helios.static_pin_prefixes(blob, 0, 16, 16, 4096)
    assert len(pins) == 1 and len(pins[0]) == 32
    assert pins == refpy.static_pins(wf, inputs, b.profile, spec, 0, 16, 16, 4096)
    assert helios.static_pin_prefixes(blob, 0, 16, 64, 4096) == []
    assert helios.static_pin_prefixes(blob, 0, 16, 16, 16) == []
    assert helios.static_pin_prefixes(blob, 1, 16, 16, 4096) == []


@needs_ref
def test_simulate_validation_errors():
    from oracle import refpy
    b = wl.WB()
    op = b.llm([wl.sys_msg("tiny"), wl.user_msg(["go"])], 2)
    b.output(op)
    _, blob = refpy.run(b.workflow(), {}, b.profile, {"workers": 1})
    with pytest.raises(RuntimeError, match="simulate: worker config count does not match schedule"):
        helios.simulate(blob, helios.SimConfig(workers=[helios.SimWorkerConfig()] * 2))
    with pytest.raises(RuntimeError, match="simulate: call scheduled twice"):
        refpy.run(b.workflow(), {}, b.profile, {"workers": 1, "sigma": [[[op, 0], [op, 0]]]})
    _, blob2 = refpy.run(b.workflow(), {}, b.profile, {"workers": 1, "sigma": [[[op, 0], [op, 0]]], "skip_sim": True})
    with pytest.raises(RuntimeError, match="simulate: call scheduled twice"):
        helios.simulate(blob2, helios.SimConfig(workers=[helios.SimWorkerConfig()]))
    _, blob3 = refpy.run(b.workflow(), {}, b.profile, {"workers": 1, "sigma": [[]], "skip_sim": True})
    with pytest.raises(RuntimeError, match="simulate: schedule does not cover all calls"):
        helios.simulate(blob3, helios.SimConfig(workers=[helios.SimWorkerConfig()]))
    with pytest.raises(RuntimeError, match="simulate: iteration guard tripped"):
        helios.simulate(blob, helios.SimConfig(workers=[helios.SimWorkerConfig(4096, 16, 1)], max_iterations=3))
    with pytest.raises(RuntimeError, match="plan: bad magic"):
        helios.simulate(b"\0" * 64, helios.SimConfig(workers=[helios.SimWorkerConfig()]))


@pytest.mark.parametrize("name,W", [("c2p_w2", 2), ("c4_w4", 4), ("c2x4", 4)])
def test_only_worker_slices_equal_the_full_run(name, W):
    """One-worker mode (one process per GPU) reproduces each worker's call rows
    of the full multi-worker run when workers are independent."""
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    rows = gold["calls_csv"].strip().split("\n")[1:]
    sc = wl.sim_config_from_meta(meta)
    total_decode = 0
    iters = 0
    for w in range(W):
        m = helios.simulate(blob, sc, only_worker=w)
        mine = m.calls_csv.strip().split("\n")[1:]
        assert mine == [r for r in rows if r.split(",")[2] == str(w)]
        total_decode += m.decode_tokens
        iters = max(iters, m.iterations)
    gm = json.loads(gold["metrics_json"])
    assert total_decode == gm["decode_tokens"] and iters == gm["iterations"]


@needs_ref
def test_only_worker_rejects_cross_worker_dependencies():
    from oracle import refpy
    b = wl.WB()
    a = b.llm([wl.sys_msg("writer"), wl.user_msg(["go"])], 3)
    c = b.llm([wl.sys_msg("writer"), wl.user_msg([a])], 3)
    b.output(c)
    _, blob = refpy.run(b.workflow(), {}, b.profile, {"workers": 2, "worker_of": {str(a): 0, str(c): 1},
                                                      "sigma": [[[a, 0]], [[c, 0]]], "skip_sim": True})
    sc = helios.SimConfig(workers=[helios.SimWorkerConfig()] * 2)
    with pytest.raises(RuntimeError, match="cross-worker dependency"):
        helios.simulate(blob, sc, only_worker=1)


# ------------------------------------------------------------ C-ABI surface
def test_cabi_exports_every_declared_symbol():
    header = "".join(h.read_text() for h in sorted((ROOT / "include").glob("*.h")))
    declared = set(re.findall(r"\b(hkx?_[a-z0-9_]+)\s*\(", header))
    lib = _lib.load()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) >= declared
    assert lib.hk_abi_version() == 1


def test_plan_trt_static_groups_match_the_shared_prompt_structure():
    """§8(f)4: the decode-attention planner takes its prefix-shared groups from the
    plan's call-level TRT (trt.cpp:489-530): the deepest branching node whose root
    path is all static text. configs[1]: the 64 branches share the 2,048-token
    pinned system prompt; configs[4]: 128 branches share 8,192 tokens; configs[0]:
    the 4 maps share 512 tokens and the reducer has no group of size > 1."""
    from collections import Counter
    groups = {}
    for n in ("c1", "c2", "c4_w1", "c5"):
        blob, _ = wl.load_plan(n)
        groups[n] = Counter(helios.plan_call_groups(blob).values())
    (g2, n2), = groups["c2"].items()
    assert g2[1] == 2048 and n2 == 64
    (g5, n5), = groups["c5"].items()
    assert g5[1] == 8192 and n5 == 128
    assert sorted(groups["c1"].values()) == [1, 4] and max(groups["c1"], key=groups["c1"].get)[1] == 512
    # C4': one group of 64 calls per operator; static prefixes grow with the overlap ratio
    assert sorted(groups["c4_w1"].values()) == [64] * 8
    assert sorted(t for _, t in groups["c4_w1"])[-1] >= 0.9 * 1024 - 2
