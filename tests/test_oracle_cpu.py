"""Pins the Python restatement oracle (oracle/simulate.py, oracle/transformer.py)
against the reference's committed golden reports and known answers, so it can
serve as the model-mode oracle for the GPU executor."""
import json
import random
from pathlib import Path

import numpy as np
import pytest

from conftest import needs_ref
from oracle import simulate as osim
from oracle import transformer as otr
from paper_2603_16104_b200 import helios
from paper_2603_16104_b200 import workloads as wl

GOLD = Path(__file__).resolve().parent / "golden"


def test_oracle_hashes_match_product_and_goldens():
    assert osim.fnv1a64(b"foobar") == 0x85944171F73967E8
    rng = random.Random(3)
    for _ in range(50):
        h, v = rng.getrandbits(64), rng.getrandbits(64)
        assert osim.hash_combine(h, v) == helios.hash_combine(h, v)
        p = [rng.getrandbits(64) for _ in range(rng.randint(0, 9))]
        lo = rng.choice([0.0, 3.0, 7.6])
        assert osim.synth_llm_output(p, lo, False, 5, True) == helios.synth_llm_output(p, lo, False, 5, True)
    for vid in (0, 7, 32767):
        assert osim.gen_token(vid, 32768) == helios.gen_token(vid, 32768)


@pytest.mark.parametrize("name", ["c1", "t_small", "t_press", "c2", "c3", "c2p_w2", "c4_w4"])
def test_oracle_simulate_matches_reference_golden(name):
    blob, meta = wl.load_plan(name)
    gold = json.loads((GOLD / f"{name}.ref.json").read_text())
    p = osim.parse_plan(blob)
    m, calls, trace, outputs, _ = osim.simulate(p, osim.SimCfg.from_meta(meta["sim"]))
    gm = json.loads(gold["metrics_json"])
    for k in ("iterations", "prompt_tokens", "cache_served_tokens", "prefill_computed_tokens", "decode_tokens",
              "pinned_tokens", "evicted_tokens", "calls"):
        assert m[k] == gm[k], k
    assert abs(m["hit_rate_pct"] - gm["hit_rate_pct"]) < 1e-12
    assert osim.calls_csv(calls) == gold["calls_csv"]
    if meta["sim"].get("collect_trace"):
        assert osim.trace_csv(trace) == gold["trace_csv"]
    if "outputs" in gold:
        assert {str(k): v for k, v in outputs.items()} == gold["outputs"]


@needs_ref
def test_oracle_kvcache_matches_reference_fuzz():
    from oracle import refpy
    rng = random.Random(11)
    for trial in range(3):
        block = rng.choice([2, 4])
        cap = block * rng.randint(2, 20)
        a, b = osim.KvCache(cap, block), refpy.RefKvCache(cap, block)
        alpha = [rng.getrandbits(64) for _ in range(4)]
        holds = []
        for step in range(600):
            seq = [rng.choice(alpha) for _ in range(rng.randint(0, block * 6))]
            r = rng.random()
            if r < 0.35:
                h = rng.choice([0, step + 1])
                holds += [h] if h else []
                assert a.lookup(seq, h) == b.lookup(seq, h)
            elif r < 0.85:
                h = rng.choice([0, step + 1])
                holds += [h] if h else []
                ln = rng.randint(0, len(seq))
                pin = rng.random() < 0.05
                assert a.insert(seq, ln, pin, h) == b.insert(seq, ln, pin, h)
            elif holds:
                h = holds.pop(rng.randrange(len(holds)))
                a.release(h)
                b.release(h)
            assert [a.used, a.pinned, a.evicted] == b.counters()


def test_weight_init_is_reproducible_and_bf16_exact():
    w = otr.init_uniform(1000, 0, 5, 0.1, True)
    assert np.array_equal(w, otr.init_uniform(1000, 0, 5, 0.1, True))
    assert np.all(np.abs(w) <= 0.1006)  # bf16(0.1) = 0.10009765625
    assert np.array_equal(w, otr.round_bf16(w))  # representable in bf16
    # known-answer: first element from the splitmix formula
    h = osim.splitmix64((0 * 0xD1B54A32D192ED03 + 5 * 0x9E3779B97F4A7C15) & osim.MASK)
    u = np.float32(h >> 40) * np.float32(1.0 / 8388608.0) - np.float32(1.0)
    assert w[0] == otr.round_bf16(np.array([u * np.float32(0.1)], np.float32))[0]


def test_decoder_incremental_equals_full_forward():
    from paper_2603_16104_b200.engine import TINY
    dec = otr.Decoder(TINY, max_pos=256)
    ids = list(range(3, 40))
    full, _ = dec.forward(ids)
    _, cache = dec.forward(ids[:-5])
    pos = len(ids) - 5
    for t in ids[-5:]:
        logits, cache = dec.forward([t], cache, pos)
        pos += 1
    # bf16 rounding after differently-blocked BLAS sums flips a few ulps
    assert np.abs(full - logits).max() / np.abs(full).max() < 1e-2
    assert int(np.argmax(full)) == int(np.argmax(logits))
