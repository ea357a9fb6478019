"""Generates the committed fixtures from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden.py

For every named workload it runs the reference pipeline (bind -> optimize ->
partition -> cache-aware plan -> call tree -> simulate, run_pipeline.cpp:47-81)
and writes
  * paper_2603_16104_b200/plans/<name>.plan.gz  the HKPLAN01 executor input
    (integration/plan_export.hpp) + <name>.json (SimConfig, description)
  * tests/golden/<name>.ref.json                reference SimMetrics report,
    call rows, trace, and outputs (full, or an FNV digest for large runs)
The GPU box has no /root/reference; these files are how its tests and the
bench get reference-planned inputs and reference answers.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refpy  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402

GOLD = ROOT / "tests" / "golden"
PLANS = wl.PLANS


def outputs_digest(outputs: dict) -> str:
    h = hashlib.sha256()
    for k in sorted(outputs, key=int):
        h.update(f"{k}:".encode())
        for v in outputs[k]:
            h.update(len(v).to_bytes(8, "little"))
            for t in v:
                h.update(int(t).to_bytes(8, "little"))
    return h.hexdigest()


def emit(name: str, wf, inputs, profile, spec, desc: str, full_outputs: bool = True):
    res, blob = refpy.run(wf, inputs, profile, spec)
    n_workers = len(res["sigma"])
    meta = {"name": name, "description": desc, "sim": refpy.sim_config_dict(spec, n_workers),
            "workers": n_workers, "spec": spec}
    PLANS.mkdir(parents=True, exist_ok=True)
    with open(PLANS / f"{name}.plan.gz", "wb") as raw, \
            gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as f:
        f.write(blob)
    (PLANS / f"{name}.json").write_text(json.dumps(meta, indent=1) + "\n")
    gold = {"name": name, "metrics_json": res["metrics_json"], "calls_csv": res["calls_csv"],
            "trace_csv": res["trace_csv"], "outputs_sha256": outputs_digest(res["outputs"]),
            "sim_seconds": res["sim_seconds"]}
    if full_outputs:
        gold["outputs"] = res["outputs"]
    (GOLD / f"{name}.ref.json").write_text(json.dumps(gold) + "\n")
    m = json.loads(res["metrics_json"])
    print(f"{name:14s} W={n_workers} iters={m['iterations']} prompt={m['prompt_tokens']} "
          f"served={m['cache_served_tokens']} prefilled={m['prefill_computed_tokens']} "
          f"decoded={m['decode_tokens']} hit={m['hit_rate_pct']:.4f} pinned={m['pinned_tokens']} "
          f"evicted={m['evicted_tokens']} plan={len(blob)}B")


def main():
    wf, i, p, s = wl.c1_tiny_mapred()
    emit("c1", wf, i, p, dict(s, collect_trace=True), "configs[0] tiny 4-branch mapred, 512-token prefix")
    wf, i, p, s = wl.c2_branches()
    emit("c2", wf, i, p, s, "configs[1] 64 branches x 2K shared prefix, 256 decode", full_outputs=False)
    wf, i, p, s = wl.c2_branches(pin=False)
    emit("c2_nopin", wf, i, p, s, "configs[1] without proactive pinning", full_outputs=False)
    for w in (1, 2, 4, 8):
        wf, i, p, s = wl.c2_ops(workers=w)
        emit(f"c2p_w{w}", wf, i, p, s, f"C2' 64 ops x B=1 on {w} workers", full_outputs=False)
    gen, s = wl.c3_reflect_spec()
    wft, it, pt = refpy.generate_workload(gen)
    emit("c3", json.loads(wft), json.loads(it), json.loads(pt), s, "configs[2] reflect generate/critique/refine B=8",
         full_outputs=False)
    for w in (1, 2, 4, 8):
        wf, i, p, s = wl.c4_overlap(workers=w)
        emit(f"c4_w{w}", wf, i, p, s, f"configs[3] C4' 512 calls, 0-90% overlap, {w} workers", full_outputs=False)
    wf, i, p, s = wl.c5_pressure()
    emit("c5", wf, i, p, s, "configs[4] 128 branches x 8K context, 16K-token cache (eviction)", full_outputs=False)
    for n in (1, 2, 4, 8):
        wf, i, p, s = wl.c2_per_gpu(n)
        emit(f"c2x{n}", wf, i, p, s, f"configs[1] weak-scaled: {n} ops x 64 branches, one per GPU",
             full_outputs=False)
    wf, i, p, s = wl.c2_branches(decode=8)
    emit("c2_short", wf, i, p, s, "configs[1] with 8 decode tokens (profiling / launch lists)", full_outputs=False)
    # reduced-size model-mode cases (fit the CPU transformer oracle)
    wf, i, p, s = wl.c2_branches(n_branches=4, prefix_words=94, decode=8, capacity=4096, budget=64)
    emit("t_small", wf, i, p, dict(s, pin_threshold=32), "4 branches x 96-token prefix, 8 decode")
    wf, i, p, s = wl.c2_branches(n_branches=8, prefix_words=254, decode=16, capacity=1024, budget=128)
    emit("t_press", wf, i, p, dict(s, pin_threshold=64), "8 branches, 256-token prefix, 1K cache (eviction)")


def main_model_parity():
    """configs[1] with 16 decode tokens: the Llama-width bf16 token-parity run
    (tests/test_gpu_parity.py), short enough for the CPU oracle."""
    wf, i, p, s = wl.c2_branches(decode=16)
    emit("c2_d16", wf, i, p, s, "configs[1] with 16 decode tokens (model parity at Llama width)", full_outputs=False)


def main_cross_worker():
    """Multi-worker plans whose calls wait on calls of another worker (SURVEY
    §8(e) exchange 2): the tiny map-reduce and the reflect workload on 2 workers."""
    wf, i, p, s = wl.c1_tiny_mapred()
    emit("c1_w2", wf, i, p, dict(s, workers=2, collect_trace=True), "configs[0] map-reduce on 2 workers (cross-worker deps)")
    gen, s = wl.c3_reflect_spec()
    wft, it, pt = refpy.generate_workload(gen)
    emit("c3_w2", json.loads(wft), json.loads(it), json.loads(pt), dict(s, workers=2),
         "configs[2] reflect on 2 workers (cross-worker deps)", full_outputs=False)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cross_worker":
        main_cross_worker()
    elif len(sys.argv) > 1 and sys.argv[1] == "model_parity":
        main_model_parity()
    else:
        main()
