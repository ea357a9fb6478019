"""Command-line drop-in: `helios_b200 run` (integration/
helios_b200_main.cpp, built by oracle/Makefile against the reference library
like tools/helios_main.cpp) takes the reference CLI's flags and files and
writes its byte-stable reports; simulate() runs in libhelium_b200.so. With the
synthetic LLM body (--engine none) every document must equal the reference's
`helios run` output (tools/helios_main.cpp:83-115, restated with the reference
simulate() in oracle/ref_capi.cpp ref_cli_run), including the workflow /
inputs / profile JSON parsing, every scheduler, the rewrite flags and the
--cache-file prompt cache across two submissions."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_2603_16104_b200 import workloads as wl

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "helios_b200"          # linked against the reference library
NATIVE = ROOT / "paper_2603_16104_b200" / "helios_b200"  # self-contained (build.py)
needs_bin = pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/helios_b200 not built (needs /root/reference)")
needs_ref = pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libhelios_ref.so").exists(),
                               reason="reference library not built")


def _cli(tmp, wf, inputs, prof, flags: dict, cache_path=None, extra=(), binary=None):
    for name, doc in (("wf", wf), ("in", inputs), ("prof", prof)):
        (tmp / f"{name}.json").write_text(doc if isinstance(doc, str) else json.dumps(doc))
    argv = [str(binary or BIN), "run", "--workflow", str(tmp / "wf.json"), "--inputs", str(tmp / "in.json"),
            "--profile", str(tmp / "prof.json"), "--out", str(tmp / "report.json"),
            "--calls-out", str(tmp / "calls.csv"), "--trace-out", str(tmp / "trace.csv"),
            "--outputs-out", str(tmp / "outputs.json"), "--schedule-out", str(tmp / "schedule.json")]
    for k, v in flags.items():
        opt = "--" + {"no_cse": "no-cse", "no_prune": "no-prune", "no_prompt_cache": "no-prompt-cache",
                      "no_proactive_kv": "no-proactive-kv", "prefill_budget": "prefill-budget",
                      "pin_threshold": "pin-threshold", "no_sim": "no-sim"}.get(k, k)
        if v is False:
            continue
        if v is True:
            argv.append(opt)
        elif k == "capacity":
            argv += [opt, ",".join(map(str, v))]
        elif k != "trace":
            argv += [opt, str(v)]
    if cache_path is not None:
        argv += ["--cache-file", str(cache_path)]
    argv += list(extra)
    p = subprocess.run(argv, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    return {k: (tmp / f).read_text() for k, f in (("report", "report.json"), ("calls_csv", "calls.csv"),
                                                   ("trace_csv", "trace.csv"), ("outputs_json", "outputs.json"),
                                                   ("schedule_json", "schedule.json"))}


def _ref(wf, inputs, prof, flags, cache=False, cache_doc=None):
    from oracle import refpy
    f = dict(flags, trace=True)  # --trace-out turns trace collection on (helios_main.cpp:95)
    if cache:
        f["cache"] = cache_doc
    return refpy.cli_run(wf, inputs, prof, f)


CASES = {
    "c1": lambda: (*wl.c1_tiny_mapred()[:3], {"capacity": [8192], "prefill_budget": 256}),
    "c1_w2_lspf": lambda: (*wl.c1_tiny_mapred()[:3], {"workers": 2, "capacity": [8192, 4096], "scheduler": "lspf"}),
    "t_press_random": lambda: (*wl.c2_branches(n_branches=8, prefix_words=254, decode=16, capacity=1024,
                                               budget=128)[:3],
                               {"capacity": [1024], "scheduler": "random", "seed": 3, "pin_threshold": 64}),
    "c1_flags": lambda: (*wl.c1_tiny_mapred()[:3], {"no_cse": True, "no_prune": True, "no_proactive_kv": True,
                                                    "block": 8, "alpha": 0.5, "scheduler": "op_wise"}),
    "c1_stochastic": lambda: (*wl.c1_tiny_mapred()[:3], {"stochastic": True, "seed": 11, "scheduler": "query_wise"}),
}


CASES.update({
    "c1_w2_native": lambda: (*wl.c1_tiny_mapred()[:3], {"workers": 2, "capacity": [8192, 4096]}),
    "c1_flags_native": lambda: (*wl.c1_tiny_mapred()[:3], {"no_cse": True, "no_prune": True, "no_proactive_kv": True,
                                                           "block": 8, "alpha": 0.5}),
    "c1_stochastic_native": lambda: (*wl.c1_tiny_mapred()[:3], {"stochastic": True, "seed": 11}),
    "t_press_native": lambda: (*wl.c2_branches(n_branches=8, prefix_words=254, decode=16, capacity=1024,
                                               budget=128)[:3], {"capacity": [1024], "pin_threshold": 64}),
    "c4_w2_native": lambda: (*wl.c4_overlap(workers=2)[:3], {"workers": 2, "capacity": [262144],
                                                             "prefill_budget": 8192}),
    "c1_nosim_native": lambda: (*wl.c1_tiny_mapred()[:3], {"no_sim": True}),
})


@needs_bin
@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_reports_equal_reference(tmp_path, name):
    wf, inputs, prof, flags = CASES[name]()
    mine = _cli(tmp_path, wf, inputs, prof, flags)
    ref = _ref(wf, inputs, prof, flags)
    for k in mine:
        assert mine[k] == ref[k], k


@needs_ref
@pytest.mark.parametrize("name", sorted(k for k, c in CASES.items() if "scheduler" not in c()[3]))
def test_native_cli_reports_equal_reference(tmp_path, name):
    """The self-contained helios_b200 (JSON IO, bind, rewrites, planner,
    simulate and reports all in libhelium_b200.so) against the reference CLI
    path, byte for byte."""
    wf, inputs, prof, flags = CASES[name]()
    mine = _cli(tmp_path, wf, inputs, prof, flags, binary=NATIVE)
    ref = _ref(wf, inputs, prof, flags)
    for k in mine:
        assert mine[k] == ref[k], k


@needs_ref
@pytest.mark.parametrize("seed", range(30))
def test_native_cli_random_workflows(tmp_path, seed):
    """Random DAGs of every operator kind (workload_gen.cpp:427-489), with
    duplicate subgraphs (CSE), dead nodes (prune), nondeterministic llms,
    1-3 workers, two --cache-file submissions."""
    import random
    from oracle import refpy
    rng = random.Random(seed)
    wf, inp, prof = refpy.generate_workload(
        {"llm_ops": rng.randint(1, 6), "batch": rng.randint(1, 4), "allow_nondeterminism": True, "seed": seed},
        random=True)
    flags = {"workers": rng.choice([1, 2, 3]), "capacity": [rng.choice([64, 256, 4096])], "seed": seed,
             "stochastic": rng.random() < 0.3}
    cache = tmp_path / "cache.json"
    ref_doc = None
    for sub in range(2):
        mine = _cli(tmp_path, wf, inp, prof, flags, cache_path=cache, binary=NATIVE)
        ref = _ref(wf, inp, prof, flags, cache=True, cache_doc=ref_doc)
        ref_doc = ref["cache_out"]
        for k in mine:
            assert mine[k] == ref[k], (sub, k)
        assert cache.read_text() == ref_doc, sub


@needs_bin
@pytest.mark.parametrize("native", [False, True])
def test_cli_prompt_cache_file_two_submissions(tmp_path, native):
    """--cache-file: the first submission writes the cache, the second reads
    it (every operator substituted) — reports and saved cache equal the
    reference CLI's at both submissions."""
    wf, inputs, prof, flags = CASES["c1"]()
    cache = tmp_path / "cache.json"
    ref_doc = None
    for sub in range(2):
        mine = _cli(tmp_path, wf, inputs, prof, flags, cache_path=cache, binary=NATIVE if native else BIN)
        ref = _ref(wf, inputs, prof, flags, cache=True, cache_doc=ref_doc)
        ref_doc = ref["cache_out"]
        assert mine["report"] == ref["report"], sub
        assert cache.read_text() == ref_doc, sub
    assert json.loads(mine["report"])["rewrite"]["substituted"] >= 5


@needs_bin
@pytest.mark.parametrize("native", [False, True])
def test_cli_usage_errors(tmp_path, native):
    BIN_ = NATIVE if native else BIN
    p = subprocess.run([str(BIN_), "run", "--workflow", "x"], capture_output=True, text=True)
    assert p.returncode == 2 and "required" in p.stderr
    p = subprocess.run([str(BIN_), "run", "--bogus", "1"], capture_output=True, text=True)
    assert p.returncode == 2 and "not expected" in p.stderr
    p = subprocess.run([str(BIN_), "run", "--workflow", "a", "--inputs", "b", "--profile", "c", "--format", "xml"],
                       capture_output=True, text=True)
    assert p.returncode == 2
    p = subprocess.run([str(BIN_), "run", "--workflow", str(tmp_path / "missing.json"), "--inputs", "b",
                        "--profile", "c"], capture_output=True, text=True)
    assert p.returncode == 1 and "error" in p.stderr


BAD = {
    "bad_slot": (lambda wf: wf["nodes"].append({"id": 99, "kind": "format", "args": {"template": "x {a}"}})),
    "dup_id": (lambda wf: wf["nodes"].append(dict(wf["nodes"][0]))),
    "missing_edge_src": (lambda wf: wf.setdefault("edges", []).append({"from": 1234, "to": 0, "slot": 0})),
    "bad_kind": (lambda wf: wf["nodes"].append({"id": 98, "kind": "tensor", "args": {}})),
    "bad_role": (lambda wf: wf["nodes"].append({"id": 97, "kind": "llm", "args": {
        "messages": [{"role": "robot", "parts": [{"text": "hi"}]}]}})),
    "output_not_output": (lambda wf: wf["outputs"].append(0)),
}


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_native_cli_rejects_bad_workflows_like_reference(tmp_path, name):
    """Malformed workflows: the native reader fails with the reference's message."""
    from oracle import refpy
    wf, inputs, prof, flags = CASES["c1"]()
    wf = json.loads(json.dumps(wf))
    BAD[name](wf)
    with pytest.raises(RuntimeError) as ref_err:
        refpy.cli_run(wf, inputs, prof, dict(flags, trace=True))
    for f, doc in (("wf", wf), ("in", inputs), ("prof", prof)):
        (tmp_path / f"{f}.json").write_text(json.dumps(doc))
    p = subprocess.run([str(NATIVE), "run", "--workflow", str(tmp_path / "wf.json"), "--inputs",
                        str(tmp_path / "in.json"), "--profile", str(tmp_path / "prof.json")],
                       capture_output=True, text=True)
    assert p.returncode == 1
    assert p.stderr.strip() == "error: " + str(ref_err.value), (p.stderr, str(ref_err.value))
