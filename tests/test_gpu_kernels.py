"""GPU parity of the device kernels (run on a B200 via gpurun).

K4 (tcgen05 GEMM) is checked against a torch fp32 matmul of the same bf16
operands; K1 page moves against torch copies; the transformer path against the
numpy decoder oracle (oracle/transformer.py).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_16104_b200 import _lib  # noqa: E402
from paper_2603_16104_b200.engine import TINY, LLAMA3_8B, Engine, EngineConfig, reduced  # noqa: E402


def _ptr(t):
    return C.c_void_p(t.data_ptr())


GEMM_SHAPES = [
    (128, 64, 1), (256, 128, 16), (512, 256, 33), (384, 192, 64), (256, 512, 100), (1024, 512, 300),
    (6144, 4096, 64), (4096, 4096, 64), (4096, 14336, 64), (28672, 4096, 64), (6144, 4096, 1024),
    (4096, 1024, 2085), (384, 192, 300), (2048, 512, 257),
]


@pytest.mark.parametrize("N,K,T", GEMM_SHAPES)
def test_gemm_tcgen05_matches_torch(N, K, T):
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K * 3 + T)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * (3.0 / K) ** 0.5
    X = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    ref = X.float() @ W.float().t()
    out = torch.zeros(T, N, device="cuda", dtype=torch.float32)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(out), N, K, T, 2, None, 0, None) == 0, _lib.last_error()
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err
    outb = torch.zeros(T, N, device="cuda", dtype=torch.bfloat16)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(outb), N, K, T, 0, None, 0, None) == 0
    torch.cuda.synchronize()
    errb = (outb.float() - ref).abs().max().item() / ref.abs().max().item()
    assert errb < 1e-2, errb
    # the engine's split-K "partials" epilogue (prefill: one split, persistent tiles)
    part = torch.zeros(T, N, device="cuda", dtype=torch.float32)
    sp = lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part), N, K, T, 3, None, 1, None)
    assert sp == 0, _lib.last_error()
    torch.cuda.synchronize()
    errp = (part - ref).abs().max().item() / ref.abs().max().item()
    assert errp < 1e-4, errp


@pytest.mark.parametrize("splits,T,N", [(1, 600, 1024), (3, 600, 1024), (2, 1024, 1024), (2, 1100, 4096),
                                        (1, 2300, 2048)])
def test_gemm_pair_tiles_splitk_partials(splits, T, N):
    """Prefill tiles on CTA pairs (tcgen05 cta_group::2, 256 weight rows x 256
    tokens per cluster): split-K fp32 partials [splits][T][N] sum to the
    product; T = 600 leaves a ragged last token tile whose second half is
    entirely out of bounds (TMA zero fill). (1100, 4096) x 2 splits and
    (2300, 2048): more units than CTA pairs, so the persistent pair kernel walks
    several (split, weight pair, token tile) units per cluster."""
    lib = _lib.load()
    K = 1024
    g = torch.Generator(device="cuda").manual_seed(splits * 1000 + T)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * (3.0 / K) ** 0.5
    X = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    ref = X.float() @ W.float().t()
    part = torch.full((splits, T, N), float("nan"), device="cuda", dtype=torch.float32)
    sp = lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part), N, K, T, 3, None, splits, None)
    assert sp == 0, _lib.last_error()
    torch.cuda.synchronize()
    err = (part.sum(0) - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err


@pytest.mark.parametrize("splits", [1, 2, 3, 7])
def test_gemm_splitk_bias_and_residual(splits):
    lib = _lib.load()
    N, K, T = 512, 1024, 48
    g = torch.Generator(device="cuda").manual_seed(splits)
    W = (torch.rand(N, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    X = (torch.rand(T, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    b = (torch.rand(N, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    ref = X.float() @ W.float().t() + b.float()
    out = torch.zeros(T, N, device="cuda", dtype=torch.float32)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(out), N, K, T, 2, _ptr(b), splits, None) == 0
    resid = torch.ones(T, N, device="cuda", dtype=torch.float32)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(resid), N, K, T, 1, _ptr(b), splits, None) == 0
    torch.cuda.synchronize()
    scale = ref.abs().max().item()
    assert (out - ref).abs().max().item() / scale < 1e-4
    assert (resid - (ref + 1)).abs().max().item() / scale < 1e-4


@pytest.mark.parametrize("T,F,K", [(1, 512, 256), (64, 512, 256), (300, 512, 256), (2085, 2048, 1024)])
def test_gemm_swiglu_epilogue(T, F, K):
    """Decode (T <= 128) and prefill tiles; (2085, 2048, 1024): 32 weight tiles x 9
    token tiles (the last ragged) = 288 tiles over the persistent prefill kernel's
    148 CTAs — two TMEM accumulators in turn, the stage ring wrapping across tiles."""
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(T)
    Wg = (torch.rand(F, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.1
    Wu = (torch.rand(F, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.1
    # physical layout: per 128-row tile, 64 gate rows then the matching 64 up rows
    W = torch.cat([Wg.view(F // 64, 64, K), Wu.view(F // 64, 64, K)], dim=1).reshape(2 * F, K).contiguous()
    X = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    gg, uu = X.float() @ Wg.float().t(), X.float() @ Wu.float().t()
    ref = gg * torch.sigmoid(gg) * uu
    out = torch.zeros(T, F, device="cuda", dtype=torch.bfloat16)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(out), 2 * F, K, T, 4, None, 0, None) == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() / ref.abs().max().item() < 1e-2


@pytest.mark.parametrize("T", [1, 64])
def test_gemm_argmax_epilogue(T):
    lib = _lib.load()
    V, K = 4096, 256
    g = torch.Generator(device="cuda").manual_seed(T + 1)
    W = (torch.rand(V, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    X = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    logits = torch.zeros(T, V, device="cuda")
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(logits), V, K, T, 2, None, 1, None) == 0
    part = torch.zeros(V // 128, T, 2, device="cuda")
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part), V, K, T, 5, None, 0, None) == 0
    torch.cuda.synchronize()
    lv = logits.view(T, V // 128, 128)
    mx, ix = lv.max(dim=-1)
    # the stream-K LM-head path may sum a vocab tile's k-segments in another
    # (fixed, deterministic) order than the single-accumulator reference
    assert torch.allclose(part[..., 0].t(), mx, rtol=1e-5, atol=1e-5)
    idx = part[..., 1].contiguous().view(torch.int32).t()
    top2 = lv.topk(2, dim=-1).values
    clear = (top2[..., 0] - top2[..., 1]) > 1e-3
    ref = ix + torch.arange(V // 128, device="cuda") * 128
    assert torch.equal(idx.long()[clear], ref[clear])
    # and the path is deterministic run to run
    part2 = torch.zeros_like(part)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part2), V, K, T, 5, None, 0, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(part, part2)


def test_gemm_deterministic():
    lib = _lib.load()
    N, K, T = 4096, 4096, 64
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    outs = []
    for _ in range(3):
        o = torch.zeros(T, N, device="cuda")
        assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(o), N, K, T, 2, None, 0, None) == 0
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


# ------------------------------------------------------------------ K1 pool
def test_pool_gather_scatter_copy():
    eng = Engine(TINY, EngineConfig(pages_per_worker=64, max_calls=8, max_step_tokens=256, max_ctx_tokens=1024))
    pb = eng.page_bytes()
    assert pb == TINY.n_layers * 2 * TINY.n_kv_heads * 16 * TINY.head_dim * 2
    # fill pages 0..9 with a known pattern through scatter, read back through gather
    src = torch.arange(10 * pb // 2, device="cuda", dtype=torch.int16).view(torch.uint8)
    eng.pool_scatter(0, src.data_ptr(), list(range(10)))
    dst = torch.zeros_like(src)
    eng.pool_gather(0, list(range(10)), dst.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    eng.pool_copy(0, [0, 1, 2], [20, 21, 22])
    dst2 = torch.zeros(3 * pb, device="cuda", dtype=torch.uint8)
    eng.pool_gather(0, [20, 21, 22], dst2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dst2, src[: 3 * pb])
    # a permuted gather returns pages in list order
    dst3 = torch.zeros(2 * pb, device="cuda", dtype=torch.uint8)
    eng.pool_gather(0, [5, 2], dst3.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dst3[:pb], src[5 * pb:6 * pb]) and torch.equal(dst3[pb:], src[2 * pb:3 * pb])
    eng.close()


# -------------------------------------------------------------- transformer
def _check_generation(model, prompt, n_new, rel_tol, eng_cfg=None):
    """hk_generate with full logits vs the oracle teacher-forced on the device's
    ids: every logit within rel_tol of max |logit|; a device choice that is not
    the oracle's argmax must sit inside the measured error band (oracle gap <=
    2 x the largest logit error of the run). Returns the exact-match count."""
    from oracle.transformer import Decoder
    eng = Engine(model, eng_cfg or EngineConfig(pages_per_worker=256, max_calls=8, max_step_tokens=1024,
                                                max_ctx_tokens=4096))
    toks, logits = eng.generate(prompt, n_new, want_logits=True)
    eng.close()
    dec = Decoder(model, max_pos=4096)
    ref_toks, ref_logits = dec.generate(prompt, n_new, forced=list(toks))
    delta = max(float(np.abs(gl - rl).max()) for gl, rl in zip(logits, ref_logits))
    exact = 0
    for k in range(n_new):
        rl, gl = ref_logits[k], logits[k]
        err = np.abs(gl - rl).max() / np.abs(rl).max()
        assert err < rel_tol, (k, err)
        if ref_toks[k] == toks[k]:
            exact += 1
        else:
            assert rl[ref_toks[k]] - rl[toks[k]] <= 2 * delta, (k, toks[k], ref_toks[k])
    return exact


def test_generate_tiny_bf16_matches_oracle():
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, TINY.vocab, size=77).tolist()
    exact = _check_generation(TINY, prompt, 12, 1e-2)
    assert exact >= 11


def test_generate_tiny_fp32_matches_oracle():
    from dataclasses import replace
    rng = np.random.default_rng(1)
    prompt = rng.integers(0, TINY.vocab, size=50).tolist()
    exact = _check_generation(replace(TINY, fp32=True), prompt, 8, 1e-5)
    assert exact == 8


def test_generate_llama_shape_reduced_depth_matches_oracle():
    m = reduced(LLAMA3_8B, 2, vocab=32768)
    rng = np.random.default_rng(2)
    prompt = rng.integers(0, m.vocab, size=150).tolist()
    exact = _check_generation(m, prompt, 6, 1e-2)
    assert exact >= 5


@pytest.mark.parametrize("T", [1, 17, 64])
def test_lm_head_streamk_argmax_at_llama_vocab(T):
    """The LM head of every decode step: V = 128,256 (1,002 vocab tiles >= one
    wave of 148 SMs, T <= 64) routes to the stream-K kernel (gemm_sk_kernel,
    gemm.cu gemm_bf16) with the fused (max, argmax) epilogue. Checked against a
    torch fp32 matmul of the same bf16 operands: every tile's max within 1e-5
    relative, its index exact where the tile's top two are not a near-tie, and
    the row argmax over the tiles equal to torch's; plus run-to-run determinism."""
    lib = _lib.load()
    V, K = 128256, 4096
    g = torch.Generator(device="cuda").manual_seed(1000 + T)
    W = ((torch.rand(V, K, device="cuda", generator=g) * 2 - 1) * (3.0 / K) ** 0.5).to(torch.bfloat16)
    X = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    ref = X.float() @ W.float().t()
    nt = (V + 127) // 128
    part = torch.zeros(nt, T, 2, device="cuda")
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part), V, K, T, 5, None, 0, None) == 0, _lib.last_error()
    torch.cuda.synchronize()
    pad = torch.full((T, nt * 128 - V), -float("inf"), device="cuda")
    lv = torch.cat([ref, pad], dim=1).view(T, nt, 128)
    mx, ix = lv.max(dim=-1)
    scale = ref.abs().max().item()
    assert (part[..., 0].t() - mx).abs().max().item() <= 1e-5 * scale
    idx = part[..., 1].contiguous().view(torch.int32).t().long()
    top2 = lv.topk(2, dim=-1).values
    clear = (top2[..., 0] - top2[..., 1]) > 1e-4 * scale
    assert torch.equal(idx[clear], (ix + torch.arange(nt, device="cuda") * 128)[clear])
    # row argmax over the tile partials (what argmax_reduce computes) == torch's
    best = part[..., 0].t().argmax(dim=1)
    rows = torch.arange(T, device="cuda")
    dev_ids = idx[rows, best]
    top2r = ref.topk(2, dim=1).values
    clear_r = (top2r[:, 0] - top2r[:, 1]) > 1e-4 * scale
    assert torch.equal(dev_ids[clear_r], ref.argmax(dim=1)[clear_r])
    part2 = torch.zeros_like(part)
    assert lib.hkx_gemm_bf16(_ptr(W), _ptr(X), _ptr(part2), V, K, T, 5, None, 0, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(part, part2)
