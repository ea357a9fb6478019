"""GPU parity of K6 pinned-prefix replication (hk_engine_set_pin_exchange).

Two ranks of the C2' plan (c2x2: two operators under the same 2,048-token
system prompt, each pinned on its own worker) are emulated in one process:
worker 0 runs as the broadcast source (computes its pin and hands the pages
to the callback), worker 1 as the receiver (skips the pin prefill; its pool
is poisoned first, so every pinned page must come from the callback). Worker
1's generated tokens and call rows must equal those of a run that prefills
the pin locally; a receiver fed zeros must not (the pages really are used).
"""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_16104_b200 import exchange, helios  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402
from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for  # noqa: E402


def _poison(eng, P):
    # finite junk (random bf16 values): unwritten slots of a page are masked in
    # the softmax but still multiply V, so the pool never holds NaN bit patterns
    g = torch.Generator(device="cuda").manual_seed(7)
    junk = torch.randn(P * eng.page_bytes() // 2, device="cuda", generator=g).to(torch.bfloat16)
    eng.pool_scatter(0, junk.data_ptr(), list(range(P)))
    torch.cuda.synchronize()


def test_pin_broadcast_receiver_matches_local_prefill():
    blob, meta = wl.load_plan("c2x2")
    sc = wl.sim_config_from_meta(meta)
    assert helios.worker_pins(blob, sc, 0) == helios.worker_pins(blob, sc, 1)
    P = pages_for(sc, 160, 512)
    eng = Engine(TINY, EngineConfig(n_workers=1, pages_per_worker=P, max_calls=160, max_step_tokens=8192 + 512,
                                    max_ctx_tokens=12288, use_device_trie=True))
    stash = {}

    def source(worker, ptr, nbytes):
        stash["buf"] = exchange.buffer_tensor(ptr, nbytes, "cuda").clone()
        stash["worker"] = worker

    def receiver(worker, ptr, nbytes):
        assert nbytes == stash["buf"].numel()
        exchange.buffer_tensor(ptr, nbytes, "cuda").copy_(stash["buf"])
        torch.cuda.synchronize()

    def zeros(worker, ptr, nbytes):
        exchange.buffer_tensor(ptr, nbytes, "cuda").zero_()
        torch.cuda.synchronize()

    eng.set_pin_exchange(1, source)
    m0 = helios.simulate(blob, sc, engine=eng, only_worker=0)
    pinned_pages = sum(len(p) for p in helios.worker_pins(blob, sc, 0)) // 16
    assert stash["worker"] == 0 and stash["buf"].numel() == pinned_pages * eng.page_bytes()

    eng.set_pin_exchange(0)
    ref = helios.simulate(blob, sc, engine=eng, only_worker=1)

    _poison(eng, P)
    eng.set_pin_exchange(2, receiver)
    got = helios.simulate(blob, sc, engine=eng, only_worker=1)
    assert got.outputs == ref.outputs
    assert got.calls_csv == ref.calls_csv
    assert got.metrics_json == ref.metrics_json
    assert m0.decode_tokens == got.decode_tokens

    _poison(eng, P)
    eng.set_pin_exchange(2, zeros)
    bad = helios.simulate(blob, sc, engine=eng, only_worker=1)
    assert bad.outputs != ref.outputs  # the receiver really reads the pages it was given


def test_pin_exchange_callback_error_fails_the_run():
    blob, meta = wl.load_plan("c2x2")
    sc = wl.sim_config_from_meta(meta)
    eng = Engine(TINY, EngineConfig(n_workers=1, pages_per_worker=pages_for(sc, 160, 512), max_calls=160,
                                    max_step_tokens=8192 + 512, max_ctx_tokens=12288, use_device_trie=True))

    def boom(worker, ptr, nbytes):
        raise ValueError("peer gone")

    eng.set_pin_exchange(2, boom)
    with pytest.raises(RuntimeError, match="simulate: pin exchange") as ei:
        helios.simulate(blob, sc, engine=eng, only_worker=1)
    assert isinstance(ei.value.__cause__, ValueError)
