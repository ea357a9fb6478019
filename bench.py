"""Benchmark of the B200 LLM-as-operator executor (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A "step" is one complete run of the workflow through the executor
(hk_simulate): pin precompute + every iteration of the reference's simulate()
loop, with the Llama-3-8B-shaped random-init model as the LLM body. At N=1 the
workload is configs[1] (64 branches x 2K shared prefix, 256 greedy tokens);
at N>1 it is the weak-scaled form c2xN (N operators of configs[1], one per
worker/GPU, one process per GPU). Metric: workflow tokens/s = generated
(decode) tokens of all ranks / max-over-ranks device time of the K runs.

  value  : device time from CUDA events on the engine stream, inputs resident
  e2e    : wall time of the C-ABI call hk_simulate(host plan -> host metrics +
           outputs), including every host<->device copy the executor makes
  roofline / attention_roofline : per-kernel-family device time of one extra
           profiled run (CUDA events around every launch) vs MEASURED_PEAKS.json
  cpu_baseline : the numpy oracle port on the host cores, bounded sample
  --impl reference : the reference's own CPU path (oracle/_ref run_workflow,
           whose LLM operator is a hash — no model math) on the same workflow
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "workflow tokens/sec @ Llama-3-8B shape"
UNIT = "tokens/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j["hbm_gbs"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().split("\n") if r.strip()]
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 7 for i in range(4) if r[3 + i].strip() == "Active"})
        load = [s for s in sm if s > 600] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, ws, rank):
    """Reference arm: the reference's own CPU implementation of the path."""
    if rank != 0:
        return
    from oracle import refpy
    from paper_2603_16104_b200 import workloads as wl
    wf, inp, prof, spec = wl.c2_branches() if args.gpus == 1 else wl.c2_per_gpu(args.gpus)
    if not refpy.LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhelios_ref.so not built"}))
        return
    times = []
    mj = None
    for i in range(args.warmup + args.steps):
        t, mj = refpy.time_run_workflow(wf, inp, prof, spec, reps=1)
        if i >= args.warmup:
            times.append(t)
    m = json.loads(mj)
    total = sum(times)
    value = m["decode_tokens"] * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 hash tokens",
        "data": "synthetic", "config": {"workload": "configs[1]" if args.gpus == 1 else f"c2x{args.gpus}",
                                        "decode_tokens_per_step": m["decode_tokens"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": "whole workflow: unmodified reference run_workflow (bind->plan->simulate), "
                                   "single-threaded; its LLM operator is a hash (evaluator.cpp:37-58), no model math"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def inpipeline_spans(eng, one_run):
    """Bytes-weighted GB/s of the decode GEMMs and of the decode attention over
    one whole run, from per-launch spans (wait exit -> last CTA end)."""
    import csv
    import tempfile
    from paper_2603_16104_b200 import _lib
    lib = _lib.load()
    lib.hk_engine_set_graphs(eng.handle, 0)
    lib.hkx_span_trace(1)
    try:
        one_run()
        with tempfile.NamedTemporaryFile(suffix=".csv", delete=False) as f:
            path = f.name
        lib.hkx_gemm_trace_dump(path.encode())
    finally:
        lib.hkx_span_trace(0)
        lib.hk_engine_set_graphs(eng.handle, 1)
    acc = {"gemm": [0.0, 0.0, 0], "attn": [0.0, 0.0, 0]}
    with open(path) as fh:
        for r in csv.DictReader(fh):
            n, k, t = int(r["N"]), int(r["K"]), int(r["T"])
            wd, en = int(r["wait_done"]), int(r["end"])
            if wd >= (1 << 63) or en <= wd:
                continue
            if n == -1 and t > 0:
                fam, b = "attn", k * 1024.0
            elif n > 0 and t <= 64:
                fam, b = "gemm", float(n) * k * 2
            else:
                continue
            acc[fam][0] += b
            acc[fam][1] += (en - wd) * 1e-9
            acc[fam][2] += 1
    os.unlink(path)
    return {f: {"achieved": v[0] / v[1] / 1e9 if v[1] > 0 else None, "launches": v[2]} for f, v in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-pin-broadcast", action="store_true", help="N>1: every rank prefills its pinned prefix itself")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if ws > 1 and args.gpus != ws:
        args.gpus = ws

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    from paper_2603_16104_b200 import helios
    from paper_2603_16104_b200 import workloads as wl
    from paper_2603_16104_b200.engine import PRESETS, Engine, EngineConfig, pages_for

    model = PRESETS[args.model]
    workload = args.workload or ("c2" if args.gpus == 1 else f"c2x{args.gpus}")
    blob, meta = wl.load_plan(workload)
    sc = wl.sim_config_from_meta(meta)
    W = len(sc.workers)
    only = rank if W > 1 else -1
    if W > 1 and W != ws:
        raise SystemExit(f"workload {workload} has {W} workers but {ws} ranks")
    device = local if ws > 1 else 0
    max_calls = 160
    eng = Engine(model, EngineConfig(device=device, n_workers=1, pages_per_worker=pages_for(sc, max_calls, 512),
                                     max_calls=max_calls, max_step_tokens=8192 + 256, max_ctx_tokens=8192,
                                     use_device_trie=True))

    pin_role = 0
    if ws > 1 and not args.no_pin_broadcast:
        # K6: rank 0 prefills the shared pinned prefix, the others receive its
        # KV pages over NCCL instead of recomputing them (when the pins match)
        from paper_2603_16104_b200 import exchange
        pin_role = exchange.enable_pin_broadcast(eng, helios.worker_pins(blob, sc, only if only >= 0 else 0))

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)

    # exchange 2: plans whose calls wait on other workers' calls replay the
    # whole control plane on every rank and broadcast generated ids (NCCL)
    out_ex = None
    if ws > 1 and helios.needs_output_exchange(blob, sc):
        from paper_2603_16104_b200 import exchange
        out_ex = exchange.make_output_exchange("cuda")

    def one_run():
        m = helios.simulate(blob, sc, engine=eng, only_worker=only, exchange=out_ex)
        return m, eng.stats()

    for _ in range(args.warmup):
        one_run()
    dev_ms, wall_s, decode, h2d, d2h, launches, pin_ms = 0.0, 0.0, 0, 0, 0, 0, 0.0
    last_m = None
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            m, st = one_run()
            wall_s += time.perf_counter() - t0
            barrier()
            dev_ms += st["pin_ms"] + st["iter_ms"]
            pin_ms += st["pin_ms"]
            decode += m.decode_tokens
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
            launches += st["launches"]
            last_m = m
    clocks = clk.summary()

    # max over ranks of device time; sum of tokens
    if ws > 1:
        t = torch.tensor([dev_ms, wall_s, float(decode)], dtype=torch.float64, device=f"cuda:{device}")
        mx = t.clone()
        torch.distributed.all_reduce(mx[:2], op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(t[2:], op=torch.distributed.ReduceOp.SUM)
        dev_ms, wall_s, decode = mx[0].item(), mx[1].item(), int(t[2].item())

    # profiled run (not timed): per kernel-family device time
    prof = {}
    if not args.no_profile:
        eng.profile(True)
        one_run()
        for fam in ("gemm", "attn_shared", "attn_private", "attn_prefill", "attn_merge", "small", "trie"):
            ms, n, b = eng.kernel_ms(fam)
            prof[fam] = {"ms": ms, "launches": n, "bytes": b}
        prof_stats = eng.stats()
        eng.profile(False)

    # in-pipeline spans (not timed): one run with PDL but without CUDA graphs and
    # without event brackets; every decode GEMM / attention launch records its
    # first griddepcontrol.wait exit and last CTA end (%globaltimer)
    spans = None
    if not args.no_profile:  # every rank runs it: the runs' exchanges are collectives
        spans = inpipeline_spans(eng, one_run)

    if rank != 0:
        eng.close()
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    hbm, tflops, peak_src = peaks()
    value = decode / (dev_ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, reference workflow)",
        "config": {"workload": f"{workload}: {meta['description']}", "model": model.name,
                   "decode_tokens_per_step": decode // args.steps, "iterations": last_m.iterations,
                   "hit_rate_pct": last_m.hit_rate_pct, "parallelism": f"{args.gpus} worker(s), one per GPU",
                   "l2": "inputs > L2: 15 GB of weights streamed every decode iteration",
                   "pin_precompute_ms_per_step": pin_ms / args.steps,
                   "pin_exchange": {0: "local prefill", 1: "prefill + NCCL broadcast source",
                                    2: "NCCL broadcast receiver"}[pin_role],
                   "output_exchange": out_ex is not None},
        "e2e": {"value": decode / wall_s, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    traffic = {}
    tp = ROOT / "profiles" / "r1_ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text())
    if prof:
        g = prof["gemm"]
        gemm_ach = g["bytes"] / (g["ms"] / 1e3) / 1e9 if g["ms"] > 0 else None
        gu = traffic.get("gemm_tc_kernel<64,4> gate/up (224 CTAs, T=64, N=28672, K=4096)")
        line["roofline"] = {"bound": "hbm", "kernel": "gemm_tc_kernel / gemm_sk_kernel (tcgen05 weight streaming, all GEMMs)",
                            "achieved": gemm_ach, "peak": hbm, "unit": "GB/s",
                            "frac": gemm_ach / hbm if gemm_ach else None,
                            "traffic": (gu["dram_read_bytes"] + gu["dram_write_bytes"]) if gu else None,
                            "traffic_kernel": "gate/up launch, ncu --set full (algorithmic %d B)" % gu["algorithmic_bytes"]
                            if gu else None,
                            "peak_source": peak_src,
                            "share_of_step": g["ms"] / (prof_stats["pin_ms"] + prof_stats["iter_ms"])}
        if spans and spans["gemm"]["achieved"]:
            line["roofline"]["inpipeline"] = {
                "achieved": spans["gemm"]["achieved"], "frac": spans["gemm"]["achieved"] / hbm,
                "launches": spans["gemm"]["launches"],
                "method": "decode split-K GEMMs (T <= 64): weight bytes / (last CTA end - first griddepcontrol.wait "
                          "exit), %globaltimer, one run with PDL and no CUDA graphs / events"}
        # prefix-shared decode attention = shared-prefix items + private-suffix items + merge
        a_ms = prof["attn_shared"]["ms"] + prof["attn_private"]["ms"] + prof["attn_merge"]["ms"]
        a_b = prof["attn_shared"]["bytes"] + prof["attn_private"]["bytes"]
        if a_ms > 0:
            ach = a_b / (a_ms / 1e3) / 1e9
            at = traffic.get("attn_decode_kernel<4> (configs[1] decode, k=128, 148 CTAs)")
            line["attention_roofline"] = {
                "bound": "hbm",
                "kernel": "attn_decode_kernel (tcgen05 prefix-shared tiles, multicast CTA pairs + mma.sync private "
                          "queue + in-kernel merge), one launch per layer",
                "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": (at["dram_read_bytes"] + at["dram_write_bytes"]) if at else None,
                "traffic_kernel": "one decode launch at k=128 (algorithmic %.0f B), ncu --set full" % at["algorithmic_bytes"]
                if at else None,
                "peak_source": peak_src, "algorithmic_bytes_run": a_b,
                "note": "bytes = shared-prefix KV once per group + private KV + Q/O, per layer, summed over the run; "
                        "time = CUDA events around each launch in one profiled run (no PDL overlap)"}
            if spans and spans["attn"]["achieved"]:
                line["attention_roofline"]["inpipeline"] = {
                    "achieved": spans["attn"]["achieved"], "frac": spans["attn"]["achieved"] / hbm,
                    "launches": spans["attn"]["launches"],
                    "method": "same algorithmic bytes / (last CTA end - first griddepcontrol.wait exit) per launch, "
                              "%globaltimer, one run with PDL and no CUDA graphs / events"}
        line["kernel_ms_per_step"] = {k: v["ms"] for k, v in prof.items()}
    if not args.no_cpu_baseline:
        from oracle.cpu_sample import decode_step_sample
        s = decode_step_sample()
        line["cpu_baseline"] = {"value": s["tokens_per_s"], "unit": UNIT, "cores": s["cores"], "kind": "port",
                                "sample": s["sample"]}
    if os.environ.get("HK_GEMM_TRACE"):  # debug: in-pipeline GEMM spans (tools/gemm_trace.py)
        from paper_2603_16104_b200 import _lib
        _lib.load().hkx_gemm_trace_dump(os.environ.get("HK_GEMM_TRACE_OUT", "gpurun_out/gemm_trace.csv").encode())
    eng.close()
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
