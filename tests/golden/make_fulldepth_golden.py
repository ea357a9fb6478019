"""Full-depth Llama-3-8B-shaped fixture (32 layers, vocab 128,256, bf16
rounding points): the CPU oracle's free-running greedy continuation of two
configs[1] branches (2,048-token shared prefix + 16-word query, 8 tokens).

    python tests/golden/make_fulldepth_golden.py      # ~10 min, ~35 GB RAM

The prompts are the ones oracle/simulate.py assembles for plan c2_short
(Evaluator::prompt, evaluator.cpp:79-99); a single-operator workflow's prompts
do not depend on generated text, so the synthetic-mode replay gives them. The
fixture keeps, per position, the oracle's top-8 (id, logit) and max |logit|, so
the GPU test (tests/test_gpu_parity.py) can judge a device choice that is not
the oracle's argmax against the oracle's gap, and the device logit error.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import simulate as osim  # noqa: E402
from oracle.transformer import Decoder, PrefixReuse  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import LLAMA3_8B  # noqa: E402

GOLD = ROOT / "tests" / "golden"
BRANCHES = (0, 37)
N_NEW = 8
TOPK = 8


def main():
    t0 = time.time()
    blob, meta = wl.load_plan("c2_short")
    p = osim.parse_plan(blob)
    _, _, _, _, prompts = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]))
    op = p.nodes[p.outputs[0]]["a"][0]
    m = LLAMA3_8B
    dec = PrefixReuse(Decoder(m, max_pos=4096))
    print(f"weights {time.time() - t0:.0f}s", flush=True)
    rec = {}
    for q in BRANCHES:
        ids = [t % m.vocab for t in prompts[(op, q)]]
        toks, logits = dec.generate(ids, N_NEW)
        lg = np.stack(logits)
        top = np.argsort(-lg, axis=1, kind="stable")[:, :TOPK]
        rec[q] = {"prompt_len": len(ids), "ids": toks, "top_ids": top.tolist(),
                  "top_logits": np.take_along_axis(lg, top, axis=1).tolist(),
                  "maxabs": np.abs(lg).max(axis=1).tolist()}
        print(f"branch {q}: {toks} {time.time() - t0:.0f}s", flush=True)
    out = {"plan": "c2_short", "model": m.name, "op": op, "n_new": N_NEW, "branches": rec,
           "generator": "tests/golden/make_fulldepth_golden.py", "oracle_seconds": round(time.time() - t0)}
    (GOLD / "model_llama3_8b_c2_short.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
