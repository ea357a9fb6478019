"""Cross-worker dependencies with the device body (SURVEY.md §8(e) exchange 2):
two processes share the one B200 of the test box, each owning one worker of
the map-reduce plan partitioned over 2 workers (the reducer waits on maps of
the other worker). The generated ids cross over the gloo exchange. Both ranks
must produce exactly the metrics, call rows and generated tokens of a
single-process run of both workers on the device."""
import json
import os
import socket
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _engine(sc, workers):
    from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for
    return Engine(TINY, EngineConfig(n_workers=workers, pages_per_worker=pages_for(sc, 160, 512), max_calls=160,
                                     max_step_tokens=8192 + 512, max_ctx_tokens=12288, use_device_trie=True))


def _outputs(m):
    return {str(k): [list(map(int, v)) for v in vals] for k, vals in m.outputs.items()}


def _main(rank, port, q):
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2603_16104_b200 import exchange, helios
        from paper_2603_16104_b200 import workloads as wl
        blob, meta = wl.load_plan("c1_w2")
        sc = wl.sim_config_from_meta(meta)
        eng = _engine(sc, 1)
        m = helios.simulate(blob, sc, engine=eng, only_worker=rank, exchange=exchange.make_output_exchange("cpu"))
        q.put((rank, {"metrics": m.metrics_json, "calls": m.calls_csv, "outputs": _outputs(m)}))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_serve_cross_worker_dependencies_on_device():
    from paper_2603_16104_b200 import helios
    from paper_2603_16104_b200 import workloads as wl
    blob, meta = wl.load_plan("c1_w2")
    sc = wl.sim_config_from_meta(meta)
    eng = _engine(sc, 2)
    ref = helios.simulate(blob, sc, engine=eng)
    ref_out = _outputs(ref)
    eng.close()
    gold = json.loads((ROOT / "tests" / "golden" / "c1_w2.ref.json").read_text())
    assert ref.calls_csv == gold["calls_csv"]  # control plane independent of the body here

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_main, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["metrics"] == ref.metrics_json
        assert res[r]["calls"] == ref.calls_csv
        assert res[r]["outputs"] == ref_out
