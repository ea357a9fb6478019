"""TEST INFRASTRUCTURE ONLY — bounded CPU sample of the LLM-operator hot path
for bench.py's cpu_baseline leg.

Runs the oracle itself (oracle/transformer.py: Decoder + PrefixReuse, bf16
rounding points, numpy / BLAS on all host threads) on configs[1]'s workflow:
the prompts oracle/simulate.py assembles for plan c2 (64 branches under the
2,048-token pinned system prompt), through a Llama-3-8B-WIDTH model reduced to
`layers` of its 32 layers (full vocab 128,256), with the same counter-based
weights as the engine. Measured: the prefill of every branch (the shared
prefix once, reused through PrefixReuse, then each 16-token suffix) and one
greedy decode step of all 64 branches. The run estimate is prefill + 256 x
that step (the workflow's 256 decode iterations); tokens/s = 16,384 decode
tokens / that estimate. Reported as what it is: a reduced-depth model.
"""
from __future__ import annotations

import os
import time


def workflow_sample(layers: int = 2, plan: str = "c2"):
    import numpy as np

    from oracle import simulate as osim
    from oracle.transformer import Decoder, PrefixReuse
    from paper_2603_16104_b200 import workloads as wl
    from paper_2603_16104_b200.engine import LLAMA3_8B, reduced

    blob, meta = wl.load_plan(plan)
    p = osim.parse_plan(blob)
    _, _, _, _, prompts = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]))  # prompts do not depend on outputs
    m = reduced(LLAMA3_8B, layers)
    n_new = p.nodes[p.nodes[p.outputs[0]]["a"][0]]["len_out"]
    t_init = time.perf_counter()
    dec = PrefixReuse(Decoder(m, max_pos=2400))
    t_init = time.perf_counter() - t_init
    ids = [[t % m.vocab for t in prompts[c]] for c in sorted(prompts)]
    t0 = time.perf_counter()
    states = [dec.prefill(x) for x in ids]
    t1 = time.perf_counter()
    for x, (logits, cache) in zip(ids, states):
        dec.dec.forward([int(np.argmax(logits))], cache, len(x))
    t2 = time.perf_counter()
    steps = int(round(n_new))
    run_s = (t1 - t0) + steps * (t2 - t1)
    tokens = len(ids) * steps
    return {
        "tokens_per_s": tokens / run_s,
        "run_s_estimate": run_s,
        "prefill_s": t1 - t0,
        "decode_step_s": t2 - t1,
        "weight_init_s": t_init,
        "cores": os.cpu_count(),
        "sample": f"configs[1] (plan {plan}: {len(ids)} branches x 2,064-token prompts, shared 2K prefix) through "
                  f"oracle/transformer.py at Llama-3-8B width reduced to {layers} of 32 layers (vocab {m.vocab}); "
                  f"measured: all prefills ({t1 - t0:.1f} s) + one {len(ids)}-branch greedy decode step "
                  f"({t2 - t1:.2f} s); run = prefill + {steps} x step; numpy/BLAS on all host threads",
    }


if __name__ == "__main__":
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    print(json.dumps(workflow_sample()))
