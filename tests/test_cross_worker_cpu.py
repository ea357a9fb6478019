"""Cross-worker dependencies with one process per worker (SURVEY.md §8(e)
exchange 2), host side: two gloo ranks each own one worker of a plan whose
calls wait on calls of the other worker (the map-reduce and reflect workloads
partitioned over 2 workers by the reference planner). Every rank replays the
whole control plane and receives the other worker's outputs through the
exchange callback; both ranks must reproduce the reference's 2-worker run
byte for byte (metrics, call rows, trace, outputs). The synthetic LLM body
stands in for the device (the exchange path is the same)."""
import hashlib
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


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _digest(outputs):
    h = hashlib.sha256()
    for k in sorted(outputs, key=int):
        h.update(f"{k}:".encode())
        for v in outputs[k]:
            h.update(len(v).to_bytes(8, "little"))
            for t in v:
                h.update(int(t).to_bytes(8, "little"))
    return h.hexdigest()


def _main(rank, port, name, q):
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2603_16104_b200 import exchange, helios
        from paper_2603_16104_b200 import workloads as wl
        blob, meta = wl.load_plan(name)
        sc = wl.sim_config_from_meta(meta)
        calls = []
        fn = exchange.make_output_exchange("cpu")

        def counting(worker, op, query, tokens):
            calls.append((worker, op, query, len(tokens)))
            fn(worker, op, query, tokens)

        m = helios.simulate(blob, sc, only_worker=rank, exchange=counting)
        q.put((rank, {"metrics": m.metrics_json, "calls": m.calls_csv, "trace": m.trace_csv,
                      "digest": _digest({str(k): v for k, v in m.outputs.items()}), "n_ex": len(calls),
                      "ex": calls[:8]}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1_w2", "c3_w2"])
def test_two_ranks_with_cross_worker_dependencies_reproduce_reference(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_main, args=(r, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    for r in range(2):
        assert res[r]["metrics"] == gold["metrics_json"]
        assert res[r]["calls"] == gold["calls_csv"]
        assert res[r]["trace"] == gold["trace_csv"]
        assert res[r]["digest"] == gold["outputs_sha256"]
    # both ranks took part in the same exchanges, in the same order
    assert res[0]["n_ex"] == res[1]["n_ex"] > 0 and res[0]["ex"] == res[1]["ex"]


def test_only_worker_without_exchange_still_rejects_cross_worker_plans():
    from paper_2603_16104_b200 import helios
    from paper_2603_16104_b200 import workloads as wl
    blob, meta = wl.load_plan("c1_w2")
    sc = wl.sim_config_from_meta(meta)
    with pytest.raises(RuntimeError, match="cross-worker dependency"):
        helios.simulate(blob, sc, only_worker=0)


def test_needs_output_exchange_detects_cross_worker_plans():
    from paper_2603_16104_b200 import helios
    from paper_2603_16104_b200 import workloads as wl
    for name, want in (("c1_w2", True), ("c3_w2", True), ("c2x2", False), ("c4_w2", False), ("c1", False)):
        blob, meta = wl.load_plan(name)
        assert helios.needs_output_exchange(blob, wl.sim_config_from_meta(meta)) is want, name
