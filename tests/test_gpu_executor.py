"""GPU parity of the executor (hk_simulate with the device body).

* Control plane: for workflows whose prompts do not depend on generated text
  (single operator, or independent operators) the reference's SimMetrics, call
  rows and trace are independent of the LLM body, so the device run must match
  the reference golden reports byte for byte — including evictions (c5, c4).
* Device trie (K2): every admission burst is matched on device AND checked
  against the host tree (verify flag): any divergence raises.
* LLM body (token ids, logits, model-mode control plane): tests/test_gpu_parity.py.
"""
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

from paper_2603_16104_b200 import helios  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"


def make_engine(sc, model=TINY, max_calls=160, max_private=512, trie=True):
    return Engine(model, EngineConfig(n_workers=len(sc.workers), pages_per_worker=pages_for(sc, max_calls, max_private),
                                      max_calls=max_calls, max_step_tokens=8192 + 512, max_ctx_tokens=12288,
                                      use_device_trie=trie))


@pytest.mark.parametrize("name", ["t_small", "t_press"])
def test_executor_device_matches_reference_control_plane(name):
    """Single-operator workflows: the control plane does not depend on the
    generated text, so the device run equals the reference's mode-S report.
    (Token parity of the same runs: tests/test_gpu_parity.py.)"""
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    sc = wl.sim_config_from_meta(meta)
    eng = make_engine(sc)
    m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    assert m.metrics_json == gold["metrics_json"]
    assert m.calls_csv == gold["calls_csv"]
    eng.close()


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


@pytest.mark.parametrize("name", ["c5", "c4_w1", "c3"])
def test_graphs_and_pdl_do_not_change_results(name):
    """CUDA-graph replay + programmatic dependent launch vs plain eager launches:
    identical control plane and identical generated tokens (same kernels).
    c4_w1 / c3 have ragged decode batches (calls admitted and completing every
    few iterations), where a stale graph scalar would drop attention partials."""
    import subprocess
    import sys
    code = ("import json,sys; sys.path.insert(0,'.');"
            "from paper_2603_16104_b200 import helios, workloads as wl;"
            "from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for;"
            f"blob, meta = wl.load_plan('{name}'); sc = wl.sim_config_from_meta(meta);"
            "e = Engine(TINY, EngineConfig(pages_per_worker=pages_for(sc, 600, 1200), max_calls=600,"
            " max_step_tokens=8704, max_ctx_tokens=12288));"
            "m = helios.simulate(blob, sc, engine=e);"
            "print(json.dumps({'m': m.metrics_json, 'o': {str(k): v for k, v in m.call_outputs.items()}}))")
    outs = []
    for env in ({}, {"HK_NO_GRAPHS": "1", "HK_NO_PDL": "1"}):  # noqa: B007
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
