"""GPU parity of the executor (hk_simulate with the device body).

* Control plane: for workflows whose prompts do not depend on generated text
  (single operator, or independent operators) the reference's SimMetrics, call
  rows and trace are independent of the LLM body, so the device run must match
  the reference golden reports byte for byte — including evictions (c5, c4).
* Device trie (K2): every admission burst is matched on device AND checked
  against the host tree (verify flag): any divergence raises.
* LLM body: each call's generated token ids must equal the CPU decoder oracle's
  greedy output for that call's prompt (teacher-forced, near-ties excepted);
  with dependencies (c1) the whole run is compared against the Python
  restatement of simulate() driven by the oracle decoder.
"""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import simulate as osim  # noqa: E402
from oracle.transformer import Decoder, top2_margin  # noqa: E402
from paper_2603_16104_b200 import helios  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"
_DEC = {}


def decoder(model):
    if model.name not in _DEC:
        _DEC[model.name] = Decoder(model, max_pos=16384)
    return _DEC[model.name]


def make_engine(sc, model=TINY, max_calls=160, max_private=512, trie=True):
    return Engine(model, EngineConfig(n_workers=len(sc.workers), pages_per_worker=pages_for(sc, max_calls, max_private),
                                      max_calls=max_calls, max_step_tokens=8192 + 512, max_ctx_tokens=12288,
                                      use_device_trie=trie))


def check_calls_against_decoder(model, plan_blob, meta, m, max_calls_checked=8):
    """Teacher-forced comparison of generated ids vs the oracle decoder."""
    p = osim.parse_plan(plan_blob)
    _, _, _, _, prompts = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]))
    dec = decoder(model)
    V = model.vocab
    llm_of_output = {o: p.nodes[o]["a"][0] for o in p.outputs}
    checked = 0
    for out_node, vals in m.outputs.items():
        op = llm_of_output[out_node]
        for q, toks in enumerate(vals):
            if checked >= max_calls_checked:
                return
            ids = [t % V for t in prompts[(op, q)]]
            gpu = [t % V for t in toks]
            ref, logits = dec.generate(ids, len(gpu), forced=gpu)
            for k in range(len(gpu)):
                if ref[k] != gpu[k]:
                    assert top2_margin(logits[k]) < 0.04 * np.abs(logits[k]).max(), (op, q, k)
            checked += 1


@pytest.mark.parametrize("name", ["t_small", "t_press"])
def test_executor_device_matches_reference_control_plane_and_oracle_tokens(name):
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    sc = wl.sim_config_from_meta(meta)
    eng = make_engine(sc)
    m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    assert m.metrics_json == gold["metrics_json"]
    assert m.calls_csv == gold["calls_csv"]
    check_calls_against_decoder(TINY, blob, meta, m)
    eng.close()


def test_executor_c1_dependencies_match_python_oracle_in_model_mode():
    """c1: 4 map calls feed a reducer whose prompt contains generated tokens.
    The Python restatement of simulate() replays the run with the GPU's call
    outputs as its LLM body; every call's output is checked token by token
    against the oracle decoder on exactly the prompt the executor built
    (teacher-forced; only near-ties of the oracle's top two may differ), and
    the control plane and workflow outputs must then agree exactly."""
    blob, meta = wl.load_plan("c1")
    sc = wl.sim_config_from_meta(meta)
    eng = make_engine(sc)
    m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    eng.close()
    dec = decoder(TINY)
    V = TINY.vocab
    exact = total = 0

    def body(prompt, out_len, len_out, det, call):
        nonlocal exact, total
        gpu = m.call_outputs[call]
        assert len(gpu) == out_len
        gids = [t % V for t in gpu]
        ref, logits = dec.generate([t % V for t in prompt], out_len, forced=gids)
        for k in range(out_len):
            total += 1
            if ref[k] == gids[k]:
                exact += 1
            else:
                assert top2_margin(logits[k]) < 0.04 * np.abs(logits[k]).max(), (call, k)
        return gpu

    p = osim.parse_plan(blob)
    om, calls, trace, outs, _ = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]), body=body)
    assert m.calls_csv == osim.calls_csv(calls)
    assert json.loads(m.metrics_json)["cache_served_tokens"] == om["cache_served_tokens"]
    assert {k: v for k, v in m.outputs.items()} == {k: v for k, v in outs.items()}
    assert exact >= total - 2, (exact, total)


@pytest.mark.parametrize("name", ["c5", "c4_w1", "c2_nopin"])
def test_executor_device_trie_and_evictions_at_config_scale(name):
    """Full-size control plane (C5: 28,672 evicted tokens; C4': 69,504) with the
    tiny model as LLM body; device trie verified on every admission burst."""
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    sc = wl.sim_config_from_meta(meta)
    eng = make_engine(sc, max_calls=600, max_private=1200)
    m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    eng.close()
    assert m.metrics_json == gold["metrics_json"]
    assert m.calls_csv == gold["calls_csv"]


def test_graphs_and_pdl_do_not_change_results():
    """CUDA-graph replay + programmatic dependent launch vs plain eager launches:
    identical control plane and identical generated tokens (same kernels)."""
    import subprocess
    import sys
    code = ("import json,sys; sys.path.insert(0,'.');"
            "from paper_2603_16104_b200 import helios, workloads as wl;"
            "from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for;"
            "blob, meta = wl.load_plan('c5'); sc = wl.sim_config_from_meta(meta);"
            "e = Engine(TINY, EngineConfig(pages_per_worker=pages_for(sc, 600, 1200), max_calls=600,"
            " max_step_tokens=8704, max_ctx_tokens=12288));"
            "m = helios.simulate(blob, sc, engine=e);"
            "print(json.dumps({'m': m.metrics_json, 'o': {str(k): v for k, v in m.call_outputs.items()}}))")
    outs = []
    for env in ({}, {"HK_NO_GRAPHS": "1", "HK_NO_PDL": "1"}):
        import os
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env={**os.environ, **env}, cwd=str(Path(__file__).resolve().parents[1]), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().split("\n")[-1]))
    assert outs[0]["m"] == outs[1]["m"]
    assert outs[0]["o"] == outs[1]["o"]


def test_executor_without_device_trie_matches_too():
    blob, meta = wl.load_plan("t_press")
    gold = json.loads((GOLD / "t_press.ref.json").read_text())
    sc = wl.sim_config_from_meta(meta)
    eng = make_engine(sc, trie=False)
    m = helios.simulate(blob, sc, engine=eng)
    eng.close()
    assert m.metrics_json == gold["metrics_json"]
