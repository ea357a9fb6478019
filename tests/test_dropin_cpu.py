"""The drop-in at the reference's own call site.

tests/dropin/dropin_main.cpp (built by oracle/Makefile into
oracle/_ref/dropin_test) runs the UNMODIFIED reference pipeline run_workflow
(run_pipeline.cpp:47-81) once with its own simulate() and once with
simulate() at :72 replaced by integration/simulate_b200.hpp — the C++
binding a maintainer adds, compiled against the reference headers and linked
with libhelium_b200.so. In mode S (no engine) every SimMetrics field must be
identical: counters, per-worker pinned/evicted tokens, call rows, trace and
workflow outputs. The GPU variant (tests/test_gpu_dropin.py) serves the same
call with the device transformer.
"""
import json
import subprocess
from pathlib import Path

import pytest

from paper_2603_16104_b200 import workloads as wl

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_test"
needs_bin = pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/dropin_test not built (needs /root/reference)")


def cases():
    c1 = wl.c1_tiny_mapred()
    out = {
        "c1": (c1[0], c1[1], c1[2], dict(c1[3], collect_trace=True)),
        "c1_w2": (c1[0], c1[1], c1[2], dict(c1[3], workers=2, collect_trace=True)),
        "t_press": wl.c2_branches(n_branches=8, prefix_words=254, decode=16, capacity=1024, budget=128),
        "c2": wl.c2_branches(),
        "c4_w2": wl.c4_overlap(workers=2),
        "c5": wl.c5_pressure(),
    }
    out["t_press"] = (*out["t_press"][:3], dict(out["t_press"][3], pin_threshold=64))
    return out


def run_dropin(tmp_path, name, wf, inputs, profile, spec, engine=None, timeout=600):
    d = tmp_path / name
    d.mkdir()
    paths = []
    for k, obj in (("wf", wf), ("in", inputs), ("prof", profile), ("spec", spec)):
        p = d / f"{k}.json"
        p.write_text(json.dumps(obj))
        paths.append(str(p))
    cmd = [str(BIN), *paths] + (["--engine", engine] if engine else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    return r.returncode, res


@needs_bin
@pytest.mark.parametrize("name", ["c1", "c1_w2", "t_press", "c2", "c4_w2", "c5"])
def test_simulate_b200_at_run_workflow_call_site_equals_reference(tmp_path, name):
    wf, inputs, profile, spec = cases()[name]
    rc, res = run_dropin(tmp_path, name, wf, inputs, profile, spec)
    assert rc == 0 and res["ok"], res
    assert all(res["equal"].values()), res
