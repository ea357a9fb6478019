"""The drop-in at run_pipeline.cpp:72 with the DEVICE body: the reference's
run_workflow pipeline calls integration/simulate_b200.hpp with a B200 engine
(tiny random-init model). For workflows whose prompts do not depend on
generated text the control plane must still equal the reference's simulate()
field by field (counters, pinned/evicted per worker, call rows); outputs are
the transformer's tokens (their parity: tests/test_gpu_parity.py)."""
import pytest

pytestmark = pytest.mark.gpu

from test_dropin_cpu import BIN, cases, needs_bin, run_dropin  # noqa: E402


@needs_bin
@pytest.mark.parametrize("name", ["t_press", "c4_w2", "c5"])
@pytest.mark.parametrize("engine", ["tiny", "tiny_f32"])
def test_simulate_b200_device_body_at_run_workflow_call_site(tmp_path, name, engine):
    wf, inputs, profile, spec = cases()[name]
    rc, res = run_dropin(tmp_path, f"{name}_{engine}", wf, inputs, profile, spec, engine=engine, timeout=900)
    assert rc == 0 and res["ok"], res
    eq = res["equal"]
    assert eq["counters"] and eq["pinned_evicted"] and eq["calls_csv"] and eq["metrics_json"], res
    assert not eq["outputs"], "transformer outputs cannot equal synth_llm_output's hash tokens"
