"""Cross-run prompt cache on the device: a warm resubmission
served from values the B200 transformer generated.

Submission 1 (configs[0]'s map-reduce) runs on the device; the executor
harvests the transformer's outputs into a PromptCache (harvest_into_cache,
optimizer.cpp:113-125). Submission 2 (the same maps, another reducer) is
planned by the reference's optimizer with that cache (substitute_cached,
optimizer.cpp:71-95): the maps become CacheFetch nodes holding the DEVICE
tokens, only the reducer runs. Its generated ids must equal the reducer's in a
cold device run of submission 2 — which only holds if the fetched values are
the tokens the device generated for the maps in submission 1.
(The reference library of oracle/_ref plans the submissions: test
infrastructure, as in the CPU tests.)"""
import pytest

pytestmark = pytest.mark.gpu

from conftest import needs_ref  # noqa: E402
from paper_2603_16104_b200 import helios  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for  # noqa: E402


def _mapred(reducer_words: str):
    wf, inputs, prof, spec = wl.c1_tiny_mapred()
    for n in wf["nodes"]:
        if n["kind"] == "llm" and n["args"]["messages"][0]["parts"][0]["text"].startswith("reducer0"):
            n["args"]["messages"][0]["parts"][0]["text"] = wl.words(reducer_words, 64)
    return wf, inputs, prof, spec


def _device_run(wf, inputs, prof, spec):
    from oracle import refpy
    res, blob = refpy.run(wf, inputs, prof, spec)
    sc = wl.sim_config_from_meta({"sim": refpy.sim_config_dict(spec, len(res["sigma"]))})
    eng = Engine(TINY, EngineConfig(pages_per_worker=pages_for(sc, 16, 512), max_calls=16, max_step_tokens=1024,
                                    max_ctx_tokens=4096))
    try:
        m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    finally:
        eng.close()
    return res, blob, m


@needs_ref
def test_warm_resubmission_fetches_device_outputs():
    wf1, inputs, prof1, spec = _mapred("reducer")
    _, blob1, m1 = _device_run(wf1, inputs, prof1, spec)
    cache = helios.PromptCache(4096)
    assert helios.harvest_into_cache(blob1, m1, cache) == 5
    # the cached llm values are the device's generated tokens
    from oracle import refpy
    synth = helios.simulate(blob1, wl.sim_config_from_meta({"sim": refpy.sim_config_dict(spec, 1)}))
    assert m1.call_outputs != synth.call_outputs
    wf2, _, prof2, _ = _mapred("summarizer")
    cold_res, _, m_cold = _device_run(wf2, inputs, prof2, spec)
    warm_res, _, m_warm = _device_run(wf2, inputs, prof2, dict(spec, prompt_cache=cache.serialize()))
    assert warm_res["rewrite"]["substituted"] == 4 and cold_res["rewrite"]["substituted"] == 0
    assert len(m_warm.call_outputs) == 1 and len(m_cold.call_outputs) == 5
    (red,) = m_warm.call_outputs
    assert m_warm.call_outputs[red] == m_cold.call_outputs[red]
    assert m_warm.outputs == m_cold.outputs
    assert m_warm.decode_tokens < m_cold.decode_tokens and m_warm.iterations < m_cold.iterations
