"""Phase timeline of ONE decode-attention launch inside the real configs[1]
pipeline (PDL on, eager launches): HK_ATTN_TRACE="step,layer,path" makes the
engine stamp that launch (%globaltimer / clock64, decode_attn.cu) and dump it.

    python tools/attn_pipeline_trace.py STEP [LAYER] [--model llama3_8b] [--workload c2]
"""
import argparse
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("step", type=int)
ap.add_argument("layer", type=int, nargs="?", default=10)
ap.add_argument("--model", default="llama3_8b")
ap.add_argument("--workload", default="c2")
ap.add_argument("--child", action="store_true")
args = ap.parse_args()
path = f"/tmp/attn_trace_{args.step}_{args.layer}.bin"

if not args.child:
    env = dict(os.environ, HK_NO_GRAPHS="1", HK_ATTN_TRACE=f"{args.step},{args.layer},{path}")
    subprocess.run([sys.executable, __file__, str(args.step), str(args.layer), "--model", args.model,
                    "--workload", args.workload, "--child"], env=env, check=True)
    import numpy as np
    t = np.fromfile(path, dtype=np.uint64).astype(np.float64)
    cta = t[:148 * 24].reshape(148, 24)
    sh = cta[cta[:, 1] > 0]  # shared CTAs stamp "tmem+bars"
    starts = cta[:, 0][cta[:, 0] > 0]
    t0 = starts.min()
    us = lambda x: (x - t0) / 1e3
    print(f"step {args.step} layer {args.layer}: {len(sh)} shared CTAs, CTA starts {us(starts).min():.2f}.."
          f"{us(starts).max():.2f} us")
    for (a, na), (b, nb) in zip([(0, "start"), (1, "tmem+bars"), (2, "q in smem"), (7, "S0 ready"), (8, "P0 written"),
                                 (3, "O done")],
                                [(1, "tmem+bars"), (2, "q in smem"), (7, "S0 ready"), (8, "P0 written"), (3, "O done"),
                                 (5, "rows out")]):
        d = (sh[:, b] - sh[:, a]) / 1e3
        print(f"  {na:>12s} -> {nb:<12s} mean {d.mean():6.2f} max {d.max():6.2f} us   (end {us(sh[:, b]).max():.2f})")
    # per-chunk clock64 stamps (chunks 0-7) of tile 0's softmax thread 0 and the MMA issuer, median over shared
    # CTAs, cycles relative to chunk 0's "S ready": 0 S ready, 6 max done, 1 exps done, 3 P written, 4/5 PV_0/PV_1 issue
    cs = t[16384:16384 + 148 * 64].reshape(148, 8, 8)
    cs = cs[cta[:, 1] > 0]
    if len(cs) and (cs[:, 0, 0] > 0).all():
        rel = cs - cs[:, :1, :1]
        print("  chunk  S_ready  max_done  exp_done  P_written  PV0_issue  PV1_issue (cycles, median over shared CTAs)")
        for c in range(8):
            if (cs[:, c, 0] > 0).all():
                med = np.median(rel[:, c, :], axis=0)
                print("  %5d %8.0f %9.0f %9.0f %10.0f %10.0f %10.0f" % (c, med[0], med[6], med[1], med[3], med[4], med[5]))
    items = t[32768:32768 + 6000 * 4].reshape(-1, 4)
    items = items[items[:, 0] > 0]
    if len(items):
        print(f"  private items {len(items)}: claim {us(items[:,0]).min():.2f}..{us(items[:,0]).max():.2f}, first page "
              f"p50 {np.median(us(items[:,1])):.2f}, done {us(items[:,2]).min():.2f}..{us(items[:,2]).max():.2f} us")
    q_end = us(cta[:, 12][cta[:, 12] > 0])
    bar = us(cta[:, 16][cta[:, 16] > 0])
    m0 = us(cta[:, 13][cta[:, 13] > 0])
    m1 = us(cta[:, 17][cta[:, 17] > 0])
    if len(m0):
        print(f"  queue end {q_end.max():.2f}, grid barrier entered ..{bar.max():.2f}, merge start {m0.min():.2f}.."
              f"{m0.max():.2f}, merge end ..{m1.max():.2f} us")
        has = (cta[:, 13] > 0) & (cta[:, 17] > 0)
        dm = (cta[has, 17] - cta[has, 13]) / 1e3
        print("  merge per CTA (us) min/p50/p90/max: " + " ".join(f"{x:.2f}" for x in np.percentile(dm, [0, 50, 90, 100])))
        w = cta[:, 18] > 0
        if w.any():
            c1 = cta[w, 19] - cta[w, 18]
            c2 = cta[w, 20] - cta[w, 19]
            print("  merge16 thread 0 cycles: loads+math p50 %.0f max %.0f; store p50 %.0f max %.0f" % (
                np.median(c1), c1.max(), np.median(c2[c2 > 0]) if (c2 > 0).any() else 0, c2.max()))
    sys.exit(0)

import torch  # noqa: E402

from paper_2603_16104_b200 import helios  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import PRESETS, Engine, EngineConfig, pages_for  # noqa: E402

blob, meta = wl.load_plan(args.workload)
sc = wl.sim_config_from_meta(meta)
size = wl.engine_sizing(blob, sc)
mc = size["max_live"] + 8
eng = Engine(PRESETS[args.model], EngineConfig(pages_per_worker=pages_for(sc, mc, size["max_private"] + 32),
                                               max_calls=mc, max_step_tokens=8192 + mc + 64,
                                               max_ctx_tokens=max(8192, size["max_ctx"] + 64), use_device_trie=True))
helios.simulate(blob, sc, engine=eng)  # the traced step index counts the steps of this run
torch.cuda.synchronize()
eng.close()
