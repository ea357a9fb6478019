"""GPU parity of K3b, the prefix-shared paged decode attention (decode_attn.cu),
through the kernel-level C-ABI hkx_decode_attention, against a torch fp32
attention over the same bf16 pages (tolerance: 1e-2 of max |ref|, the bf16
bound BASELINE.json's north_star states for attention).

Cases cover the shapes of the configs (Llama-3-8B G=4 with 64 branches on a
2K shared prefix; Qwen2.5-32B G=5 with 128 branches on 8K; the tiny model G=2),
ragged groups (a lone call, shared ranges that are not a multiple of the
8-page tcgen05 chunk, private ranges split into several items), and repeated
launches (the arrival counters must return to zero).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_16104_b200 import _lib  # noqa: E402

HD = 128
PG = 16


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(_lib.i32p)


def make_case(H, Hkv, groups, seed=0, n_free=64):
    """groups: list of (members, shared_pages, [private tokens per member]).
    Returns tensors + host tables; each member's private tokens include the decode token."""
    rng = np.random.default_rng(seed)
    tables, offs, pos, grow, gsh = [], [0], [], [], []
    next_page = 0
    for members, shared, priv in groups:
        sp = list(range(next_page, next_page + shared))
        next_page += shared
        for m in range(members):
            n_priv = priv[m]
            npg = (n_priv + PG - 1) // PG
            pp = list(range(next_page, next_page + npg))
            next_page += npg
            tables += sp + pp
            offs.append(len(tables))
            pos.append(shared * PG + n_priv - 1)
        grow.append(members)
        gsh.append(shared if members > 1 else 0)
    n_pages = next_page + n_free
    # shuffle physical page ids so tables are not contiguous ranges
    perm = rng.permutation(n_pages)
    tables = [int(perm[p]) for p in tables]
    dev = torch.device("cuda")
    g = torch.Generator(device="cpu").manual_seed(seed)
    kv = (torch.randn(n_pages, 2, Hkv, PG, HD, generator=g) * 0.5).to(torch.bfloat16).to(dev)
    n_rows = len(pos)
    qkv = (torch.randn(n_rows, (H + 2 * Hkv) * HD, generator=g)).to(torch.bfloat16).to(dev)
    return dict(kv=kv, qkv=qkv, tables=tables, offs=offs, pos=pos, grow=grow, gsh=gsh, n_pages=n_pages, H=H, Hkv=Hkv)


def run(case, iters=0):
    lib = _lib.load()
    n_rows = len(case["pos"])
    out = torch.zeros(n_rows, case["H"], HD, dtype=torch.bfloat16, device="cuda")
    t, tp = _i32(case["tables"])
    o, op = _i32(case["offs"])
    p, pp = _i32(case["pos"])
    gr, grp = _i32(case["grow"])
    gs, gsp = _i32(case["gsh"])
    ms = lib.hkx_decode_attention(C.c_void_p(case["qkv"].data_ptr()), C.c_void_p(case["kv"].data_ptr()),
                                  case["n_pages"], n_rows, case["H"], case["Hkv"], tp, op, pp, grp, gsp,
                                  len(case["grow"]), C.c_void_p(out.data_ptr()), iters)
    if ms < 0:
        raise RuntimeError(_lib.last_error())
    torch.cuda.synchronize()
    nbytes = lib.hkx_decode_attention_bytes(n_rows, case["H"], case["Hkv"], op, pp, grp, gsp, len(case["grow"]))
    return out, ms, nbytes


def reference(case):
    H, Hkv = case["H"], case["Hkv"]
    G = H // Hkv
    kv = case["kv"].float()
    qkv = case["qkv"].float()
    outs = []
    for r, pos in enumerate(case["pos"]):
        pages = torch.tensor(case["tables"][case["offs"][r]:case["offs"][r + 1]], device="cuda", dtype=torch.long)
        k = kv[pages, 0].permute(1, 0, 2, 3).reshape(Hkv, -1, HD)[:, :pos + 1]
        v = kv[pages, 1].permute(1, 0, 2, 3).reshape(Hkv, -1, HD)[:, :pos + 1]
        q = qkv[r, :H * HD].view(Hkv, G, HD)
        s = torch.einsum("hgd,hkd->hgk", q, k) / np.sqrt(HD)
        w = torch.softmax(s, dim=-1)
        outs.append(torch.einsum("hgk,hkd->hgd", w, v).reshape(H, HD))
    return torch.stack(outs)


def check(case):
    out, _, _ = run(case)
    ref = reference(case)
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-2 * scale, (err, scale)
    return out


CASES = {
    # configs[1]: 64 branches x 2,048 shared tokens + 16-token suffix + k generated
    "llama_c2": (32, 8, [(64, 128, [16 + k for k in range(1, 65)])]),
    # configs[4]: 128 branches x 8,192 shared, G = 5
    "qwen_c5": (40, 8, [(128, 512, [32 + (k % 40) for k in range(128)])]),
    # tiny model (G = 2, one kv head)
    "tiny": (2, 1, [(4, 6, [20, 21, 40, 3])]),
    # ragged: lone call (no sharing, > 512 keys: split private), a shared range
    # of 13 pages (not a multiple of the 8-page chunk), long private suffixes
    "ragged": (32, 8, [(1, 0, [1500]), (5, 13, [1, 17, 600, 33, 1030]), (2, 4, [5, 6]), (1, 0, [7])]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_decode_attention_matches_fp32_reference(name):
    H, Hkv, groups = CASES[name]
    check(make_case(H, Hkv, groups, seed=hash(name) % 1000))


def test_decode_attention_repeated_launches_are_identical():
    H, Hkv, groups = CASES["ragged"]
    case = make_case(H, Hkv, groups, seed=3)
    a, _, _ = run(case)
    b, _, _ = run(case, iters=5)  # 1 + 5 more launches, counters must reset every time
    ref = reference(case)
    assert torch.equal(a, b)
    assert (b.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


def test_decode_attention_hbm_throughput_reported():
    """Not a pass/fail bar: prints achieved GB/s at the configs[1] mid-decode shape."""
    case = make_case(32, 8, [(64, 128, [16 + 128] * 64)], seed=5)
    _, ms, nbytes = run(case, iters=20)
    print(f"decode attention c2 k=128: {ms * 1e3:.2f} us/launch, {nbytes / ms / 1e6:.0f} GB/s algorithmic")
    assert ms > 0


# ------------------------------------------------ causal prefill (tile path)
PREFILL_CASES = [(2, 1, 10, 0), (2, 1, 33, 0), (2, 1, 60, 0), (2, 1, 77, 5), (2, 1, 130, 0),
                 (32, 8, 10, 0), (32, 8, 33, 17), (32, 8, 64, 0), (32, 8, 100, 300), (40, 8, 50, 0)]


@pytest.mark.parametrize("H,Hkv,n,start", PREFILL_CASES)
def test_prefill_attention_matches_causal_fp32_reference(H, Hkv, n, start):
    g = torch.Generator(device="cpu").manual_seed(n * 131 + start)
    n_pages = (start + n + 15) // 16 + 8
    table = torch.randperm(n_pages, generator=g)[: (start + n + 15) // 16].tolist()
    kv = (torch.randn(n_pages, 2, Hkv, PG, HD, generator=g) * 0.5).to(torch.bfloat16).cuda()
    qkv = torch.randn(n, (H + 2 * Hkv) * HD, generator=g).to(torch.bfloat16).cuda()
    out = torch.zeros(n, H, HD, dtype=torch.bfloat16, device="cuda")
    t, tp = _i32(table)
    rc = _lib.load().hkx_prefill_attention(C.c_void_p(qkv.data_ptr()), C.c_void_p(kv.data_ptr()), n_pages, n, start,
                                           H, Hkv, tp, len(table), C.c_void_p(out.data_ptr()))
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    G = H // Hkv
    pages = torch.tensor(table, device="cuda", dtype=torch.long)
    k = kv[pages, 0].float().permute(1, 0, 2, 3).reshape(Hkv, -1, HD)
    v = kv[pages, 1].float().permute(1, 0, 2, 3).reshape(Hkv, -1, HD)
    q = qkv[:, :H * HD].float().view(n, Hkv, G, HD)
    s = torch.einsum("thgd,hkd->thgk", q, k) / np.sqrt(HD)
    keys = torch.arange(k.shape[1], device="cuda")
    pos = start + torch.arange(n, device="cuda")
    s = s.masked_fill((keys[None, :] > pos[:, None])[:, None, None, :], float("-inf"))
    ref = torch.einsum("thgk,hkd->thgd", torch.softmax(s, dim=-1), v).reshape(n, H, HD)
    err = (out.float() - ref).abs().amax(dim=(1, 2))
    bad = (err > 1e-2 * ref.abs().max()).nonzero().flatten().tolist()
    assert not bad, (bad[:10], err.max().item())


def _causal_ref(q_rows, kv, table, start, H, Hkv):
    n = q_rows.shape[0]
    G = H // Hkv
    pages = torch.tensor(table, device="cuda", dtype=torch.long)
    k = kv[pages, 0].float().permute(1, 0, 2, 3).reshape(Hkv, -1, HD)
    v = kv[pages, 1].float().permute(1, 0, 2, 3).reshape(Hkv, -1, HD)
    q = q_rows[:, :H * HD].float().view(n, Hkv, G, HD)
    s = torch.einsum("thgd,hkd->thgk", q, k) / np.sqrt(HD)
    keys = torch.arange(k.shape[1], device="cuda")
    pos = start + torch.arange(n, device="cuda")
    s = s.masked_fill((keys[None, :] > pos[:, None])[:, None, None, :], float("-inf"))
    return torch.einsum("thgk,hkd->thgd", torch.softmax(s, dim=-1), v).reshape(n, H, HD)


# (H, Hkv, common pages, suffix tokens per segment, segments): the configs[1] shape
# (G=4: 32-row tiles, 2,048-token pinned prefix = 128 pages), configs[4]'s G=5
# (25-row tiles), and common prefixes that are not a multiple of the 8-page chunk
PAIR_CASES = [(32, 8, 128, [16, 16, 16, 16], 4), (32, 8, 37, [20, 27], 2), (40, 8, 77, [25, 11, 25], 3),
              (40, 8, 9, [7, 25], 2), (2, 1, 12, [60, 33, 64], 3)]


@pytest.mark.parametrize("H,Hkv,common,suffix,nseg", PAIR_CASES)
def test_prefill_paired_suffix_segments_match_causal_reference(H, Hkv, common, suffix, nseg):
    """The engine's paired-suffix prefill (plan_prefill_attention with the arena):
    calls of one operator admitted together prefill their suffixes under a
    common cached prefix; two single-tile segments with >= 8 common leading
    pages share one CTA pair (common pages multicast, own pages per CTA).
    Every segment must equal its own causal fp32 attention."""
    g = torch.Generator(device="cpu").manual_seed(H * 1000 + common * 7 + nseg)
    pre = common * PG
    n_pages = common + sum((s + PG) // PG + 1 for s in suffix) + 8
    perm = torch.randperm(n_pages, generator=g).tolist()
    common_pages, nxt = perm[:common], common
    arena, tok0, counts, starts, ptabs = [], [], [], [], []
    t = 0
    for s in suffix[:nseg]:
        own = (pre + s + PG - 1) // PG - common
        ptabs.append(len(arena))
        arena += common_pages + perm[nxt:nxt + own]
        nxt += own
        tok0.append(t)
        counts.append(s)
        starts.append(pre)
        t += s
    kv = (torch.randn(n_pages, 2, Hkv, PG, HD, generator=g) * 0.5).to(torch.bfloat16).cuda()
    qkv = torch.randn(t, (H + 2 * Hkv) * HD, generator=g).to(torch.bfloat16).cuda()
    out = torch.zeros(t, H, HD, dtype=torch.bfloat16, device="cuda")
    a = [_i32(x) for x in (tok0, counts, starts, ptabs, arena)]
    rc = _lib.load().hkx_prefill_attention_segs(C.c_void_p(qkv.data_ptr()), C.c_void_p(kv.data_ptr()), n_pages, nseg,
                                                a[0][1], a[1][1], a[2][1], a[3][1], H, Hkv, a[4][1], len(arena), t,
                                                C.c_void_p(out.data_ptr()))
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    for s in range(nseg):
        rows = slice(tok0[s], tok0[s] + counts[s])
        table = arena[ptabs[s]:ptabs[s] + (starts[s] + counts[s] + PG - 1) // PG]
        ref = _causal_ref(qkv[rows], kv, table, starts[s], H, Hkv)
        err = (out[rows].float() - ref).abs().max().item()
        assert err <= 1e-2 * ref.abs().max().item(), (s, err)
