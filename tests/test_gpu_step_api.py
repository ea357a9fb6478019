"""Step-level C ABI: hk_slot_alloc / hk_step / hk_pin_prefill /
hk_kv_broadcast for a host that runs its own iteration loop (the reference's
simulate() body: chunked prefill simulator.cpp:331-343, decode :347-374, pins
:257-263) and owns the block tables.

* One call driven step by step equals hk_generate (same engine path).
* A pinned prefix prefilled once and shared by two calls' block tables, their
  suffix prefills and decode rows in ragged steps: each call's tokens equal a
  stand-alone generation of its full prompt (fp32 engine: exact), and the
  step's logits equal the stand-alone logits.
* K6 outside hk_simulate: pages broadcast from worker 0 to worker 1 arrive byte
  for byte and decode to the same tokens.
"""
from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_16104_b200.engine import TINY, LLAMA3_8B, QWEN25_32B, Engine, EngineConfig, reduced  # noqa: E402
from paper_2603_16104_b200.exchange import buffer_tensor  # noqa: E402


def _engine(model, workers=1):
    return Engine(model, EngineConfig(n_workers=workers, pages_per_worker=96, max_calls=8, max_step_tokens=512,
                                      max_ctx_tokens=1024))


def _ids(n, seed, vocab):
    return np.random.default_rng(seed).integers(0, vocab, n).astype(np.uint32)


@pytest.mark.parametrize("model", [replace(TINY, fp32=True), TINY, reduced(LLAMA3_8B, 2, vocab=32768),
                                   reduced(QWEN25_32B, 2, vocab=32768)],
                         ids=["tiny_fp32", "tiny_bf16", "llama_width_bf16", "qwen_width_bf16"])
def test_step_by_step_equals_generate(model):
    prompt, n_new = _ids(70, 1, model.vocab), 8
    ref = _engine(model)
    want = ref.generate(prompt, n_new)
    ref.close()
    eng = _engine(model)
    pages = list(range((len(prompt) + n_new + 15) // 16))
    slot = eng.slot_alloc(0)
    got = [eng.step(0, [dict(slot=slot, start=0, ids=prompt, sample=True, pages=pages)])[0]]
    for k in range(1, n_new):
        got.append(eng.step(0, [dict(slot=slot, start=len(prompt) + k - 1, ids=None, sample=True, pages=pages)])[0])
    eng.slot_free(0, slot)
    eng.close()
    assert [int(t) for t in got] == [int(t) for t in want]


def test_pinned_prefix_shared_by_a_ragged_batch():
    model = replace(TINY, fp32=True)
    pin = _ids(80, 2, model.vocab)          # 5 full pages, shared by both calls' tables
    sfx = [_ids(20, 3, model.vocab), _ids(27, 4, model.vocab)]
    n_new = 8
    ref = _engine(model)
    want = []
    for s in sfx:
        ids, lg = ref.generate(np.concatenate([pin, s]), n_new, want_logits=True)
        want.append((ids, lg))
        ref.reset()
    ref.close()

    eng = _engine(model)
    eng.pin_prefill(0, pin, list(range(5)))
    tables, slots = [], []
    for c, s in enumerate(sfx):
        own = (len(pin) + len(s) + n_new + 15) // 16 - 5
        tables.append(list(range(5)) + list(range(10 + 10 * c, 10 + 10 * c + own)))
        slots.append(eng.slot_alloc(0))
    got = [[], []]
    first, lg0 = eng.step(0, [dict(slot=slots[c], start=len(pin), ids=sfx[c], sample=True, pages=tables[c])
                              for c in range(2)], want_logits=True)
    for c in range(2):
        got[c].append(int(first[c]))
        np.testing.assert_allclose(lg0[c], want[c][1][0], rtol=1e-4, atol=1e-4)
    for k in range(1, n_new):
        # decode rows of both calls in one ragged step (they share the pinned pages)
        segs = [dict(slot=slots[c], start=len(pin) + len(sfx[c]) + k - 1, ids=None, sample=True, pages=tables[c])
                for c in range(2)]
        out, lg = eng.step(0, segs, want_logits=True)
        for c in range(2):
            got[c].append(int(out[c]))
            np.testing.assert_allclose(lg[c], want[c][1][k], rtol=1e-4, atol=1e-4)
    for c in range(2):
        assert got[c] == [int(t) for t in want[c][0]], c
    eng.close()


def test_kv_broadcast_between_workers():
    model = TINY
    pin = _ids(64, 5, model.vocab)
    pages = list(range(4))
    eng = _engine(model, workers=2)
    eng.pin_prefill(0, pin, pages)
    pb = eng.page_bytes()
    wire = torch.zeros(len(pages) * pb, dtype=torch.uint8, device="cuda")

    def send(ptr, nbytes):  # the caller's broadcast (here: into a "wire" tensor)
        assert nbytes == wire.numel()
        wire.copy_(buffer_tensor(ptr, nbytes, "cuda"))
        torch.cuda.synchronize()

    def recv(ptr, nbytes):
        buffer_tensor(ptr, nbytes, "cuda").copy_(wire)
        torch.cuda.synchronize()

    eng.kv_broadcast(0, 1, pages, send)
    eng.kv_broadcast(1, 2, pages, recv)
    a = torch.empty(len(pages) * pb, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    eng.pool_gather(0, pages, a.data_ptr())
    eng.pool_gather(1, pages, b.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(a, b) and a.any()
    # the received pages decode like the source's
    sfx = _ids(9, 6, model.vocab)
    toks = []
    for w in (0, 1):
        slot = eng.slot_alloc(w)
        table = pages + [20, 21]
        seq = [int(eng.step(w, [dict(slot=slot, start=len(pin), ids=sfx, sample=True, pages=table)])[0])]
        for k in range(1, 5):
            seq.append(int(eng.step(w, [dict(slot=slot, start=len(pin) + len(sfx) + k - 1, ids=None, sample=True,
                                              pages=table)])[0]))
        eng.slot_free(w, slot)
        toks.append(seq)
    assert toks[0] == toks[1]
    eng.close()


def test_step_api_errors():
    eng = _engine(TINY)
    with pytest.raises(RuntimeError, match="decode segment"):
        eng.step(0, [dict(slot=0, start=3, ids=None, count=2, pages=[0])])
    with pytest.raises(RuntimeError, match="needs a call slot"):
        eng.step(0, [dict(slot=-1, start=3, ids=None, sample=True, pages=[0])])
    with pytest.raises(RuntimeError, match="page id out of range"):
        eng.step(0, [dict(slot=-1, start=0, ids=[1, 2, 3], pages=[10_000])])
    with pytest.raises(RuntimeError, match="block table shorter"):
        eng.step(0, [dict(slot=-1, start=0, ids=list(range(40)), pages=[0])])
    with pytest.raises(RuntimeError, match="role must be"):
        eng.kv_broadcast(0, 3, [0], lambda p, n: None)
    with pytest.raises(RuntimeError, match="do not cover"):
        eng.pin_prefill(0, list(range(40)), [0])
    eng.close()
