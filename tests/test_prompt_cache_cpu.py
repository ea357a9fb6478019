"""Cross-run prompt cache: PromptCache (prompt_cache.cpp) and
harvest_into_cache (optimizer.cpp:113-125) of the executor, against the
reference library compiled by oracle/Makefile.

* the LRU + JSON document are checked in lock-step with the reference's
  PromptCache (byte-identical serialisation after every operation);
* harvest from a finished executor run (synth LLM body) equals the
  reference's harvest_into_cache document on random DAGs of every operator
  kind, including nondeterministic (tainted) llm nodes;
* a warm resubmission planned by the reference's optimizer with the cache this
  executor harvested substitutes the cached operators (CacheFetch) and the
  executor then reproduces the reference's run of that rewritten graph.
"""
import json
import random

import pytest

from conftest import needs_ref
from paper_2603_16104_b200 import helios
from paper_2603_16104_b200 import workloads as wl


@needs_ref
@pytest.mark.parametrize("cap", [1, 3, 8])
def test_prompt_cache_lockstep_with_reference(cap):
    from oracle import refpy
    ref, mine = refpy.PromptCache(cap), helios.PromptCache(cap)
    rng = random.Random(cap)
    for step in range(400):
        sig = rng.randrange(12) * 0x9E3779B97F4A7C15 % 2**64
        if rng.random() < 0.6:
            v = [rng.randrange(2**64) for _ in range(rng.randrange(5))]
            ref.insert(sig, v)
            mine.insert(sig, v)
        else:
            a, b = ref.lookup_len(sig), mine.lookup(sig)
            assert (a < 0 and b is None) or a == len(b), step
        assert mine.serialize() == ref.serialize(), step
    assert mine.size() == len(mine.keys_lru_first()) <= cap
    assert mine.capacity() == cap


@needs_ref
def test_prompt_cache_json_round_trip_and_errors():
    from oracle import refpy
    ref = refpy.PromptCache(4)
    for s, v in [(1, [5, 6]), (2, []), (3, [2**64 - 1]), (1, [7])]:
        ref.insert(s, v)
    doc = ref.serialize()
    mine = helios.PromptCache.deserialize(doc)
    assert mine.serialize() == doc
    assert mine.keys_lru_first() == [2, 3, 1]  # the overwrite of 1 made it most recent
    assert refpy.PromptCache.deserialize(mine.serialize()).serialize() == doc
    assert mine.lookup(2) == [] and mine.lookup(9) is None
    assert mine.keys_lru_first() == [3, 1, 2]  # a hit refreshes recency
    with pytest.raises(RuntimeError, match="prompt cache capacity must be positive"):
        helios.PromptCache(0)
    for bad in ("{", '{"capacity": 2, "entries": [{"sig": "zz", "tokens": []}]}', '{"entries": []}'):
        with pytest.raises(RuntimeError, match="prompt cache json"):
            helios.PromptCache.deserialize(bad)
    with pytest.raises(RuntimeError, match="prompt cache capacity must be positive"):
        helios.PromptCache.deserialize('{"capacity": 0, "entries": []}')


def _run(wf, inputs, prof, spec):
    from oracle import refpy
    res, blob = refpy.run(wf, inputs, prof, spec)
    meta = {"sim": refpy.sim_config_dict(spec, len(res["sigma"]))}
    return res, blob, helios.simulate(blob, wl.sim_config_from_meta(meta))


@needs_ref
@pytest.mark.parametrize("seed", range(24))
def test_harvest_matches_reference_random_workflows(seed):
    """Random DAGs (workload_gen.cpp:427-489: data / input / format / lambda /
    llm, some nondeterministic) — the executor's harvest of its own run equals
    the reference's Evaluator-driven harvest, byte for byte."""
    from oracle import refpy
    rng = random.Random(seed)
    wf, inp, prof = refpy.generate_workload(
        {"llm_ops": rng.randint(1, 6), "batch": rng.randint(1, 4), "allow_nondeterminism": True, "seed": seed},
        random=True)
    cap = rng.choice([2, 8, 4096])
    spec = {"workers": rng.choice([1, 2]), "capacities": [4096], "seed": seed,
            "stochastic": rng.random() < 0.3, "harvest": True, "cache_capacity": cap}
    res, blob, m = _run(wf, inp, prof, spec)
    assert m.metrics_json == res["metrics_json"]
    cache = helios.PromptCache(cap)
    n = helios.harvest_into_cache(blob, m, cache)
    assert n == res["harvested"]
    assert cache.serialize() == res["prompt_cache_out"]


def _mapred(reducer_words: str):
    """configs[0]'s map-reduce with a choice of reducer prompt (the maps are shared)."""
    wf, inputs, prof, spec = wl.c1_tiny_mapred()
    for n in wf["nodes"]:
        if n["kind"] == "llm" and n["args"]["messages"][0]["parts"][0]["text"].startswith("reducer0"):
            n["args"]["messages"][0]["parts"][0]["text"] = wl.words(reducer_words, 64)
    return wf, inputs, prof, spec


@needs_ref
def test_warm_resubmission_served_from_harvested_cache():
    """Submission 1 cold; the executor harvests its values; submission 2 (a
    different reducer over the same maps) is planned by the reference's
    optimizer with that cache: the 4 maps become CacheFetch nodes, only the
    reducer runs, and the executor's run of the rewritten plan equals the
    reference's (metrics, calls, outputs) and the cold run of submission 2."""
    wf1, inputs, prof1, spec = _mapred("reducer")
    _, blob1, m1 = _run(wf1, inputs, prof1, spec)
    cache = helios.PromptCache(4096)
    assert helios.harvest_into_cache(blob1, m1, cache) == 5  # 4 maps + reducer, B = 1
    wf2, _, prof2, _ = _mapred("summarizer")
    cold, _, m_cold = _run(wf2, inputs, prof2, spec)
    warm, blob2, m_warm = _run(wf2, inputs, prof2, dict(spec, prompt_cache=cache.serialize()))
    assert warm["rewrite"]["substituted"] == 4 and cold["rewrite"]["substituted"] == 0
    assert m_warm.metrics_json == warm["metrics_json"] and m_warm.calls_csv == warm["calls_csv"]
    assert len(m_warm.call_outputs) == 1 and len(m_cold.call_outputs) == 5
    assert m_warm.decode_tokens < m_cold.decode_tokens
    assert m_warm.outputs == m_cold.outputs  # same reducer output, maps fetched instead of regenerated
    # an identical resubmission is served entirely from the cache
    warm1, _, m_w1 = _run(wf1, inputs, prof1, dict(spec, prompt_cache=cache.serialize()))
    assert warm1["rewrite"]["substituted"] >= 5 and m_w1.calls == 0 and m_w1.outputs == m1.outputs


@needs_ref
def test_harvest_needs_signatures():
    blob, meta = wl.load_plan("t_small")  # committed plans predate the signature section
    m = helios.simulate(blob, wl.sim_config_from_meta(meta))
    with pytest.raises(RuntimeError, match="carries no signatures"):
        helios.harvest_into_cache(blob, m, helios.PromptCache(16))
