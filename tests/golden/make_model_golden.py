"""Generates the model-mode fixtures: the CPU oracle's FREE-RUNNING greedy run
of a workflow, i.e. oracle/simulate.py's restatement of simulate()
(simulator.cpp:222-389, pinned to the reference's golden reports by
tests/test_oracle_cpu.py) with oracle/transformer.py's decoder (pinned to
HuggingFace transformers by tests/test_oracle_hf_cpu.py) as the LLM body.

    python tests/golden/make_model_golden.py [name ...]

Writes tests/golden/model_<model>_<name>.npz + .json:
  * per call (op, query): the generated vocab ids, the oracle's logit of each
    chosen id, its top-1 minus top-2 margin and max |logit| at that position;
  * the model-mode SimMetrics (dict), calls CSV and workflow outputs digest —
    in model mode prompts that contain generated text (c1, c3) change the
    control plane, so the device run must match these, not the mode-S goldens.

The GPU test (tests/test_gpu_parity_fp32.py) runs hk_simulate with the same
fp32 engine and requires identical ids for every call, no exemption.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

GOLD = ROOT / "tests" / "golden"
NAMES = ["t_small", "t_press", "c1", "c3", "c4_w1", "c5"]


def model_for(name: str):
    from paper_2603_16104_b200.engine import TINY
    return replace(TINY, fp32=True)


def outputs_digest(outputs: dict) -> str:
    h = hashlib.sha256()
    for k in sorted(outputs, key=int):
        h.update(f"{k}:".encode())
        for v in outputs[k]:
            h.update(len(v).to_bytes(8, "little"))
            for t in v:
                h.update(int(t).to_bytes(8, "little"))
    return h.hexdigest()


def run(name: str) -> str:
    import numpy as np

    from oracle import simulate as osim
    from oracle.transformer import Decoder, PrefixReuse
    from paper_2603_16104_b200 import workloads as wl

    m = model_for(name)
    blob, meta = wl.load_plan(name)
    p = osim.parse_plan(blob)
    V = m.vocab
    dec = PrefixReuse(Decoder(m, max_pos=16384))
    rec = {}
    t0 = time.time()

    def body(prompt, out_len, len_out, det, call):
        ids, logits = dec.generate([t % V for t in prompt], out_len)
        lg = np.stack(logits)
        part = np.partition(lg, -2, axis=1)
        rec[call] = (ids, lg[np.arange(len(ids)), ids], part[:, -1] - part[:, -2], np.abs(lg).max(axis=1))
        return [osim.gen_token(v, V) for v in ids]

    om, calls, _, outs, _ = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]), body=body)
    keys = sorted(rec)
    np.savez_compressed(
        GOLD / f"model_{m.name}{'_f32' if m.fp32 else ''}_{name}.npz",
        calls=np.array([[op, q, len(rec[(op, q)][0])] for op, q in keys], dtype=np.int64).reshape(-1, 3),
        ids=np.concatenate([np.asarray(rec[k][0], np.int32) for k in keys]),
        logit=np.concatenate([rec[k][1] for k in keys]).astype(np.float32),
        margin=np.concatenate([rec[k][2] for k in keys]).astype(np.float32),
        maxabs=np.concatenate([rec[k][3] for k in keys]).astype(np.float32))
    side = {"name": name, "model": m.name, "fp32": m.fp32, "metrics": om, "calls_csv": osim.calls_csv(calls),
            "outputs_sha256": outputs_digest(outs), "oracle_seconds": round(time.time() - t0, 1),
            "generator": "tests/golden/make_model_golden.py"}
    (GOLD / f"model_{m.name}{'_f32' if m.fp32 else ''}_{name}.json").write_text(json.dumps(side, indent=1) + "\n")
    return f"{name}: {len(keys)} calls, {om['decode_tokens']} tokens, {time.time() - t0:.0f}s"


if __name__ == "__main__":
    names = sys.argv[1:] or NAMES
    os.environ.setdefault("OMP_NUM_THREADS", "2")
    with ProcessPoolExecutor(max_workers=min(len(names), 4)) as ex:
        for line in ex.map(run, names):
            print(line, flush=True)
