"""K6 pinned-prefix replication, host side (world_size 2, gloo): the ranks agree
on enabling the exchange only when their workers pin identical prefixes, rank
0 becomes the source and rank 1 the receiver, and the callback moves the page
buffer byte for byte (a host buffer stands in for the device one; on B200 the
same callback runs over NCCL, tests/test_gpu_pin_exchange.py)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


class FakeEngine:
    def __init__(self):
        self.role, self.fn = None, None

    def set_pin_exchange(self, role, fn=None):
        self.role, self.fn = role, fn


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _main(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2603_16104_b200 import exchange
        out = {}
        same = [[1, 2, 3, 4] * 8, [9] * 16]
        eng = FakeEngine()
        out["role_same"] = exchange.enable_pin_broadcast(eng, same, device="cpu")
        nbytes = 4096 + 16
        buf = (C.c_uint8 * nbytes)()
        if rank == 0:
            np.ctypeslib.as_array(buf)[:] = np.arange(nbytes, dtype=np.uint64).astype(np.uint8) ^ 0x5A
        eng.fn(0, C.addressof(buf), nbytes)
        out["buf"] = bytes(buf)
        eng2 = FakeEngine()
        diff = [[1, 2, 3, 4] * 8] if rank == 0 else [[1, 2, 3, 5] * 8]
        out["role_diff"] = exchange.enable_pin_broadcast(eng2, diff, device="cpu")
        eng3 = FakeEngine()
        out["role_empty"] = exchange.enable_pin_broadcast(eng3, [], device="cpu")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_pin_broadcast_roles_and_payload_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_main, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["role_same"] == 1 and res[1]["role_same"] == 2
    expect = bytes(np.arange(4096 + 16, dtype=np.uint64).astype(np.uint8) ^ 0x5A)
    assert res[0]["buf"] == expect and res[1]["buf"] == expect
    assert res[0]["role_diff"] == 0 and res[1]["role_diff"] == 0
    assert res[0]["role_empty"] == 0 and res[1]["role_empty"] == 0


def test_pins_digest_distinguishes_sequences():
    from paper_2603_16104_b200 import exchange
    assert exchange.pins_digest([[1, 2]]) == exchange.pins_digest([[1, 2]])
    assert exchange.pins_digest([[1, 2]]) != exchange.pins_digest([[1], [2]])
    assert exchange.pins_digest([[1, 2]]) != exchange.pins_digest([[2, 1]])
