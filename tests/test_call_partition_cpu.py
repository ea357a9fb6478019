"""§8(f)1: opt-in call-level partition (hk_plan_partition_calls).

The reference places whole operators on workers (partition_workflow,
scheduler.cpp:59-115), so configs[1] — ONE operator with 64 branches — can
only use one worker there. The opt-in transform deals every operator's calls
round-robin over W workers; it DIVERGES from the reference's schedule (no
golden report exists for it), so the checks are the executor's own
invariants: every call runs exactly once, every worker pins the shared
2,048-token prefix (so K6 replicates it from one GPU), decode tokens add up,
and one process per worker (gloo, world size 2, bench.py's N>1 path with the
synthetic body) reproduces the single-process W-worker run's call rows.
"""
import os
import socket
from pathlib import Path

import pytest

from paper_2603_16104_b200 import helios
from paper_2603_16104_b200 import workloads as wl

ROOT = Path(__file__).resolve().parents[1]


def rows(csv):
    return [r.split(",") for r in csv.strip().split("\n")[1:]]


@pytest.mark.parametrize("W", [2, 4, 8])
def test_call_partition_of_configs1(W):
    blob, meta = wl.load_plan("c2")
    sc = wl.sim_config_from_meta(meta)
    blob_w = helios.partition_calls(blob, W)
    sc_w = helios.replicate_workers(sc, W)
    m = helios.simulate(blob_w, sc_w)
    r = rows(m.calls_csv)
    calls = sorted((int(x[0]), int(x[1])) for x in r)
    assert calls == sorted(helios.plan_call_groups(blob))          # every call once
    per_worker = [sum(1 for x in r if int(x[2]) == w) for w in range(W)]
    assert per_worker == [64 // W] * W
    assert m.decode_tokens == 64 * 256
    assert m.pinned_tokens == [2048] * W                           # every worker pins the prefix
    # each worker's pins are the same token sequence -> K6 broadcasts them from one rank
    assert all(helios.worker_pins(blob_w, sc_w, w) == helios.worker_pins(blob_w, sc_w, 0) for w in range(W))
    # one worker at a time (the one-process-per-GPU mode) gives that worker's rows
    for w in range(W):
        mw = helios.simulate(blob_w, sc_w, only_worker=w)
        assert [x for x in rows(mw.calls_csv)] == [x for x in r if int(x[2]) == w]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_16104_b200 import helios as h
        from paper_2603_16104_b200 import workloads as w
        blob, meta = w.load_plan("c2")
        blob_w = h.partition_calls(blob, world)
        sc_w = h.replicate_workers(w.sim_config_from_meta(meta), world)
        m = h.simulate(blob_w, sc_w, only_worker=rank)
        t = torch.tensor([float(m.decode_tokens)])
        dist.all_reduce(t)
        q.put((rank, m.calls_csv, int(t.item())))
    finally:
        dist.destroy_process_group()


def test_call_partition_one_process_per_worker_gloo():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    blob, meta = wl.load_plan("c2")
    m = helios.simulate(helios.partition_calls(blob, 2), helios.replicate_workers(wl.sim_config_from_meta(meta), 2))
    full = rows(m.calls_csv)
    for rank, csv, total in out:
        assert rows(csv) == [x for x in full if int(x[2]) == rank]
        assert total == 64 * 256
