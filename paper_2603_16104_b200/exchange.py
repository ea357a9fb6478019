"""Exchanges between the ranks of a multi-GPU run.

K6, exchange 1 — pinned-prefix replication across ranks.

The reference pins the same static prefix on every worker that runs >= 2
calls under it (static_pin_prefixes + pin insert, simulator.cpp:132-199,
:257-263; C2' pins 2,048 tokens on each of 8 workers). With one process per
GPU, the source rank computes the pin's KV (the prefill) and the others
receive the pages with one broadcast instead of recomputing them
(hk_engine_set_pin_exchange, role 1 = source, 2 = receiver). Over NCCL the
transfer runs NVLink peer to peer; 256 MiB for C2's prefix at Llama shape.

The exchange is only enabled when every rank's worker pins exactly the same
token sequences (checked with an all-gather of a digest): a worker with a
different prefix (e.g. C4's per-operator overlap) keeps computing its own.

Exchange 2 — generated ids of calls other workers depend on
(make_output_exchange, used with helios.simulate(..., exchange=...)).
"""
from __future__ import annotations

import ctypes as C
import hashlib
from typing import List, Sequence

import numpy as np


class _CudaBytes:
    """uint8 view of a raw device allocation (no copy) for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def buffer_tensor(ptr: int, nbytes: int, device: str):
    """A torch uint8 tensor aliasing `nbytes` at `ptr` (device memory for
    "cuda", host memory for "cpu", the gloo tests)."""
    import torch
    if device == "cpu":
        arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr))
        return torch.from_numpy(arr)
    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=device)


def pins_digest(pins: Sequence[Sequence[int]]) -> bytes:
    h = hashlib.sha256()
    for p in pins:
        h.update(len(p).to_bytes(8, "little"))
        h.update(np.asarray(p, dtype=np.uint64).tobytes())
    return h.digest()


def same_pins_everywhere(pins: List[List[int]], group=None) -> bool:
    """True when every rank pins the same (non-empty) token sequences."""
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    digests = [None] * ws
    dist.all_gather_object(digests, (pins_digest(pins), sum(len(p) for p in pins)), group=group)
    return all(d == digests[0] for d in digests) and digests[0][1] > 0


def global_rank(group_rank: int, group=None) -> int:
    """torch.distributed's `src` is a global rank: map a rank of `group` to it."""
    import torch.distributed as dist
    return group_rank if group is None else dist.get_global_rank(group, group_rank)


def make_broadcast_fn(src: int, device: str, group=None):
    """The callback: broadcast the pin pages from group rank `src` into every rank's buffer."""
    import torch
    import torch.distributed as dist
    g_src = global_rank(src, group)

    def fn(worker: int, ptr: int, nbytes: int):
        t = buffer_tensor(ptr, nbytes, device)
        dist.broadcast(t, src=g_src, group=group)
        if device != "cpu":
            torch.cuda.synchronize()

    return fn


def enable_pin_broadcast(engine, pins: List[List[int]], src: int = 0, device: str = "cuda", group=None) -> int:
    """Enable K6 on `engine` for this rank; returns the role set (0 = the
    ranks' pins differ: every rank computes its own)."""
    import torch.distributed as dist
    if dist.get_world_size(group) < 2 or not same_pins_everywhere(pins, group):
        engine.set_pin_exchange(0)
        return 0
    role = 1 if dist.get_rank(group) == src else 2
    engine.set_pin_exchange(role, make_broadcast_fn(src, device, group))
    return role


# --------------------------------------------------------------- exchange 2
def make_output_exchange(device: str = "cpu", group=None):
    """Cross-worker dependencies with one process per GPU (exchange 2): the
    callback for helios.simulate(..., only_worker=rank, exchange=fn). Rank r
    owns schedule worker r; at each completion of worker w the owner's output
    ids are broadcast from rank w (host ids only, a few KB). Every rank calls
    it in the same order because every rank replays the same control plane."""
    import torch
    import torch.distributed as dist

    def fn(worker: int, op: int, query: int, tokens):
        t = torch.from_numpy(tokens.view(np.int64))  # shares memory with the executor's buffer
        src = global_rank(worker, group)  # worker w is owned by rank w of the group
        if device == "cpu":
            dist.broadcast(t, src=src, group=group)
        else:
            d = t.to(device)
            dist.broadcast(d, src=src, group=group)
            t.copy_(d.cpu())

    return fn
