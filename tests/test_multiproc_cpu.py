"""N>1 path of bench.py on CPU: one process per worker (world_size 2, gloo).

Each rank runs its own schedule worker of a multi-worker plan
(hk_simulate only_worker = rank, synthetic LLM body — no GPU needed), exactly
as `bench.py --gpus N` does on B200s, then the ranks exchange results the way
the benchmark does (max-over-ranks time, sum of tokens). The union of the
ranks' call rows and outputs must equal the reference's golden multi-worker
run, byte for byte.
"""
import json
import os
import socket
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, name, q):
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_16104_b200 import helios
        from paper_2603_16104_b200 import workloads as wl
        blob, meta = wl.load_plan(name)
        sc = wl.sim_config_from_meta(meta)
        m = helios.simulate(blob, sc, only_worker=rank)
        # the benchmark's reductions: max over ranks of time-like values, sum of tokens
        t = torch.tensor([float(m.iterations), float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tok = torch.tensor([float(m.decode_tokens)], dtype=torch.float64)
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
        rows = [None] * world
        dist.all_gather_object(rows, (m.calls_csv, {str(k): v for k, v in m.outputs.items()}))
        if rank == 0:
            q.put({"iters": int(t[0].item()), "max_rank": int(t[1].item()), "decode": int(tok[0].item()),
                   "rows": rows})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2x2", "c4_w2"])
def test_two_rank_gloo_run_equals_reference_multiworker_run(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    gm = json.loads(gold["metrics_json"])
    assert res["max_rank"] == 2
    assert res["iters"] == gm["iterations"]
    assert res["decode"] == gm["decode_tokens"]
    ref_rows = gold["calls_csv"].strip().split("\n")[1:]
    for w, (csv, outs) in enumerate(res["rows"]):
        mine = csv.strip().split("\n")[1:]
        assert mine == [r for r in ref_rows if r.split(",")[2] == str(w)]
    # workflow outputs: the union over ranks, digested like the golden report
    import hashlib
    merged = {}
    for _, outs in res["rows"]:
        for k, v in outs.items():
            assert k not in merged or merged[k] == v
            merged[k] = v
    h = hashlib.sha256()
    for k in sorted(merged, key=int):
        h.update(f"{k}:".encode())
        for v in merged[k]:
            h.update(len(v).to_bytes(8, "little"))
            for t in v:
                h.update(int(t).to_bytes(8, "little"))
    assert h.hexdigest() == gold["outputs_sha256"]
