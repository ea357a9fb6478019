// K3b: prefix-shared paged decode attention (bf16) — the attention of every
// decode token of one (iteration, worker) step of the reference's simulate()
// loop (simulator.cpp:347-374: one token per running call per iteration) —
// and, on the same tile path, the causal prefill of K3a (:331-343).
//
// ONE persistent launch per layer (attn_decode_kernel<G>): one CTA per SM,
// 320 threads, CTAs paired in clusters of 2.
//
//   shared items  decode rows that share a block-table prefix (the branches
//                 of one pinned system prompt, e.g. configs[1]'s 2,048 tokens)
//                 are (token, q-head) pairs of one kv head — 128/G tokens fill
//                 a 128-row tcgen05 tile. One CTA streams TWO tiles of a kv
//                 head over a range of prefix pages (shared2_phase; planner:
//                 ~64 CTAs for a <= 2K prefix, ~2/3 of the SMs for longer
//                 ones). Warp 9 streams K/V straight from the paged pool with
//                 TMA (128B swizzle, 2-stage K and V rings, started before
//                 griddepcontrol.wait: old pages do not depend on this step);
//                 warp 8 alternates the tiles' MMAs (PV_0, S_0', PV_1, S_1')
//                 so one softmax warpgroup's exponentials (one thread per row,
//                 the chunk in registers, P written over S in TMEM) overlap
//                 the other tile's MMAs. Output: the row normalised to bf16 +
//                 (m, l), one partial per item. (shared_phase — one tile per
//                 CTA, CTA pairs multicasting the pages — serves the prefill
//                 tiles, and decode under HK_ATTN_TWO_TILE=0.)
//   private items every decode row's own pages (prompt suffix + generated
//                 tokens) per kv head, as key ranges sized for one round on
//                 the free warps; each warp pulls items from a global queue,
//                 feeds itself a 3-deep TMA page ring and runs mma.sync
//                 m16n8k16 with swapped operands (keys / head dims are the
//                 16-row M side, the G q-heads the 8-wide N side).
//   merge         after a grid-wide arrival (all CTAs co-resident: grid <=
//                 SMs), every SM merges rows (merge16, up to 16 partials per
//                 memory round trip: w_p = l_p 2^(m_p - M));
//                 a row with a single item is written directly. A grid larger
//                 than the SM count falls back to a separate merge launch.
//   prefill tiles causal tiles (rows = prompt tokens x G heads, keys [0, pos])
//                 paired so the later row block's pages serve both CTAs; two
//                 single-tile segments under a common prefix share a pair
//                 (common pages multicast, own pages per CTA).
#include <algorithm>
#include <array>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

constexpr int HD = 128;
constexpr int PG = 16;        // tokens per KV page
constexpr int KC = 128;       // keys per tcgen05 chunk (8 pages)
constexpr int ROWS = 128;     // MMA rows of a shared item

// -------------------------------------------------------------------- merge
// Partials are stored NORMALISED in bf16 (o_p / l_p, half the bytes of fp32
// unnormalised rows; the writes were the slowest step of a shared tile) with
// (m_p, l_p) in fp32 (m in the log2 domain); merge: out = sum_p w_p o_p / sum_p
// w_p with w_p = l_p 2^(m_p - max m).

__device__ __forceinline__ bf16* part_bf16(const DecodeAttnArgs& a) { return reinterpret_cast<bf16*>(a.part_o); }

// per-chunk clock64 stamps of thread 0 (softmax) and the MMA issuer, chunks < 8 (debug trace)
__device__ __forceinline__ void cstamp(const DecodeAttnArgs& a, int c, int k) {
    if (a.trace && c < 8) a.trace[16384 + static_cast<size_t>(blockIdx.x) * 64 + c * 8 + k] = clock64();
}
__device__ __forceinline__ void stamp(const DecodeAttnArgs& a, int cta, int k) {
    if (a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (k == 6 || k == 9 || k == 10 || k == 11) t = clock64();  // fine-grained (cycles) chunk-1 stamps
        a.trace[static_cast<size_t>(cta) * 24 + k] = t;
        if (k == 0 || k == 5) a.trace[static_cast<size_t>(cta) * 24 + 22 + (k == 5)] = clock64();
    }
}

// launch span (debug, HK_GEMM_TRACE): 0 first CTA start, 1 first wait exit, 2 ~last end
__device__ __forceinline__ void span_mark(const DecodeAttnArgs& a, int k) {
    if (a.span && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMin(&a.span[k], k == 2 ? ~t : t);
    }
}

// per private item (debug trace): [claim, first page landed, done, (smid << 8) | warp]
__device__ __forceinline__ void item_stamp(const DecodeAttnArgs& a, int item, int k) {
    if (a.trace && (threadIdx.x & 31) == 0 && item < 6000) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        unsigned long long* q = a.trace + 32768 + static_cast<size_t>(item) * 4;
        q[k] = t;
        if (k == 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            q[3] = (static_cast<unsigned long long>(smid) << 8) | (threadIdx.x >> 5);
        }
    }
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// This CTA's slice of the L2 prefetch of the next kernel's weights (lane 0).
__device__ __forceinline__ void prefetch_next_weights(const DecodeAttnArgs& a) {
    if (!a.l2_prefetch || a.l2_prefetch_bytes == 0) return;
    const size_t per = (a.l2_prefetch_bytes / gridDim.x + 4095) & ~size_t(4095);
    const size_t b0 = per * blockIdx.x;
    if (b0 >= a.l2_prefetch_bytes) return;
    const size_t b1 = b0 + per < a.l2_prefetch_bytes ? b0 + per : a.l2_prefetch_bytes;
    const uint64_t pol = policy_evict_last();
    const char* base = static_cast<const char*>(a.l2_prefetch);
    for (size_t o = b0; o < b1; o += 32768)
        l2_prefetch_bulk(base + o, static_cast<uint32_t>(b1 - o < 32768 ? b1 - o : 32768), pol);
}

// ------------------------------------------------------- shared (tcgen05)
// Warp-specialised, one CTA per SM (320 threads):
//   warp 9  (TMA)     page ids -> smem, then K/V chunks of 8 pages into a
//                     2-stage ring (TMA 2D, 128B swizzle, box 64 x 16);
//   warp 8  (MMA)     one thread issues S(c) = Q K(c)^T into one of two TMEM
//                     S buffers, then O += P(c-1) V(c-1) — QK of the next
//                     chunk overlaps the softmax of the current one;
//   warps 0-7 (softmax) two threads per row (TMEM lane quarter = warp % 4,
//                     column half = warp / 4): scale, row max (exchanged
//                     through smem), lazy O rescale, exp2, P (bf16) into the
//                     A-operand tile, then the epilogue and arrival counters.
// smem (1024-aligned): sQ [2][128][64] | 3 x sK [2][128][64] | 2 x sV | barriers | exchange (P lives in TMEM)
constexpr int SQ_BYTES = ROWS * HD * 2;   // 32 KB
constexpr int SKV_BYTES = KC * HD * 2;    // 32 KB (K or V of one chunk)
constexpr int SH_THREADS = 320;
constexpr int KST = 3;  // K ring depth of a shared tile (V ring: 2)
constexpr int SH_MAX_PAGES = 1024;        // pages of one tile item (16K keys)
constexpr int SH_SMEM = 1024 + SQ_BYTES + (KST + 2) * SKV_BYTES + 256 + 7 * ROWS * 4 + (ROWS + 4) * 4 +
                        SH_MAX_PAGES * 4;

__device__ __forceinline__ uint32_t sw128(int row, int chunk16) {  // byte offset inside a [rows][64] SW128 block
    return static_cast<uint32_t>(row * 128 + ((chunk16 ^ (row & 7)) << 4));
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fmax3(float x, float y, float z) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x), "f"(y), "f"(z));
    return r;
}
template <int G>
__device__ __forceinline__ void shared_phase(const CUtensorMap& tm_kv, const DecodeAttnArgs& a, uint8_t* sm) {
    uint8_t* sQ = sm;
    // K ring of 3 stages, then a V ring of 2 (P lives in tensor memory, so its
    // 32 KB of shared memory became the third K stage: K(c + 3) is requested as
    // soon as S(c) has read K(c), hiding the ~2 us loaded HBM latency)
    uint8_t* sKV = sm + SQ_BYTES;
    auto sK = [&](int c) { return sKV + (c % KST) * SKV_BYTES; };
    auto sV = [&](int c) { return sKV + KST * SKV_BYTES + (c & 1) * SKV_BYTES; };
    uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + (KST + 2) * SKV_BYTES);
    // K and V of a chunk have their own barriers: K(c + 2) streams in as soon as
    // S(c) has read K(c), long before PV(c) frees V(c)
    uint64_t* k_full = bars;        // [KST] K chunk landed (TMA tx)
    uint64_t* k_empty = bars + 3;   // [KST] K chunk consumed (S commit, both CTAs of the pair)
    uint64_t* s_full = bars + 6;    // [2] S buffer written (MMA commit)
    uint64_t* s_free = bars + 8;    // [2] S buffer read (256 softmax threads)
    uint64_t* p_full = bars + 10;   // P written to TMEM (256 softmax threads)
    uint64_t* o_done = bars + 11;   // PV complete (MMA commit)
    uint64_t* q_full = bars + 12;   // Q tile written (256 softmax threads)
    uint64_t* v_full = bars + 13;   // [2] V chunk landed
    uint64_t* v_empty = bars + 15;  // [2] V chunk consumed (PV commit, both CTAs)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 20);

    float* red = reinterpret_cast<float*>(sm + SQ_BYTES + (KST + 2) * SKV_BYTES + 256);  // [2][128] x 2
    int* flags = reinterpret_cast<int*>(red + 7 * ROWS);  // [ROWS] tokens this CTA merges, [ROWS] count
    int* spg = flags + ROWS + 4;                            // page ids of this item

    stamp(a, blockIdx.x, 0);
    const ShItem it = a.sh[blockIdx.x];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = static_cast<int>(cluster_ctarank());  // pair rank: which half of the pages it fetches
    const int nrows = it.ntok * G;
    const int nch = (it.npages + 7) / 8;

    if (tid == 0) {
        tma_prefetch_desc(&tm_kv);
        for (int b = 0; b < KST; ++b) {
            mbar_init(&k_full[b], 1);
            mbar_init(&k_empty[b], 2);  // the MMA issuers of both CTAs of the pair
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&v_full[b], 1);
            mbar_init(&v_empty[b], 2);
            mbar_init(&s_full[b], 1);
            mbar_init(&s_free[b], 256);
        }
        mbar_init(p_full, 256);
        mbar_init(o_done, 1);
        mbar_init(q_full, 256);
        fence_barrier_init();
    }
    if (warp == 8) tmem_alloc(tslot, 512);  // S0 [0,128) | S1 [128,256) | O [256,384) | P [384,448)
    tc_fence_before();
    // the pair's peer multicasts K/V into this CTA's stages and arrives on its
    // barriers: both CTAs' barriers must be initialised first
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    stamp(a, blockIdx.x, 1);

    if (warp == 9) {
        // ---- TMA producer. Decode tiles read shared pages written by earlier
        // steps, so their loads need not wait for this step's producers; a causal
        // prefill tile reads the chunk's own K/V, written by this step's RoPE
        // kernel, and waits for it first.
        for (int i = lane; i < it.npages; i += 32) spg[i] = a.pages[it.ptab + it.page0 + i];
        __syncwarp();
        if (it.flags & 1) pdl_wait();
        if (lane == 0) {
            const int rows_per_head = a.Hkv * PG;  // pool-map rows between K and V of a page
            // the chunk lands in both CTAs of the pair: each fetches every other
            // page once from HBM and multicasts it (the shared prefix is read
            // once for all 2 x 128 rows of this kv head)
            auto load = [&](int c, int v) {
                const int ns = v ? 2 : KST;  // ring depth
                const int b = c % ns;
                uint64_t* full = v ? &v_full[b] : &k_full[b];
                if (c >= ns) mbar_wait(v ? &v_empty[b] : &k_empty[b], ((c / ns) - 1) & 1);
                const int np = min(8, it.npages - c * 8);
                uint8_t* dst = v ? sV(c) : sK(c);
                mbar_expect_tx(full, static_cast<uint32_t>(np) * 2 * 2048);
                if (c * 8 + np <= it.mc_pages) {
                    // pages common to the pair: each CTA fetches every other one and multicasts
                    for (int i = crank; i < np; i += 2) {
                        const int rk = a.layer_row0 + (spg[c * 8 + i] * 2 * a.Hkv + it.kvh) * PG + v * rows_per_head;
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tma_load_2d_mc(dst + h * SKV_BYTES / 2 + i * 2048, &tm_kv, full, h * 64, rk, 3);
                    }
                } else {
                    // this CTA's own pages (e.g. a call's suffix next to its partner's)
                    for (int i = 0; i < np; ++i) {
                        const int rk = a.layer_row0 + (spg[c * 8 + i] * 2 * a.Hkv + it.kvh) * PG + v * rows_per_head;
#pragma unroll
                        for (int h = 0; h < 2; ++h) tma_load_2d(dst + h * SKV_BYTES / 2 + i * 2048, &tm_kv, full, h * 64, rk);
                    }
                }
            };
            // K runs one chunk ahead of V (V(c) is needed a softmax later than K(c))
            for (int c = 0; c <= nch; ++c) {
                if (c < nch) load(c, 0);
                if (c >= 1) load(c - 1, 1);
            }
        }
        pdl_wait();
        pdl_trigger();
    } else if (warp == 8) {
        // ---- MMA issuer
        pdl_wait();
        pdl_trigger();
        if (lane == 0) {
            const uint32_t q0 = smem_u32(sQ);
            auto issue_pv = [&](int j) {
                mbar_wait(p_full, j & 1);
                mbar_wait(&v_full[j & 1], (j >> 1) & 1);
                tc_fence_after();
                cstamp(a, j, 5);
                const int np = min(8, it.npages - j * 8);
                const uint32_t v0 = smem_u32(sV(j));
                const uint32_t idesc = umma_idesc_bf16(ROWS, HD) | (1u << 16);  // B = V, MN-major
                // A = P straight from tensor memory: 16 keys = 8 columns per k-step
                for (int kk = 0; kk < np; ++kk)
                    umma_bf16_ts(tmem + 256, tmem + 384 + kk * 8,
                                 umma_desc_sw128_lbo(v0 + kk * 2048, SKV_BYTES / 2, 1024), idesc,
                                 (j > 0 || kk > 0) ? 1u : 0u);
                umma_commit(o_done);
                umma_commit_mc(&v_empty[j & 1], 3);  // V stage free in both CTAs once both PVs are done
            };
            auto issue_s = [&](int c) {
                const int b = c & 1;
                mbar_wait(&k_full[c % KST], (c / KST) & 1);
                if (c >= 2) mbar_wait(&s_free[b], ((c >> 1) - 1) & 1);
                tc_fence_after();
                cstamp(a, c, 4);
                const int nk = min(8, it.npages - c * 8) * PG;
                const uint32_t idesc = umma_idesc_bf16(ROWS, nk);
                const uint32_t k0 = smem_u32(sK(c));
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * (SKV_BYTES / 2) + (kk & 3) * 32;
                    umma_bf16(tmem + b * 128, umma_desc_sw128(q0 + (kk >> 2) * (SQ_BYTES / 2) + (kk & 3) * 32),
                              umma_desc_sw128(k0 + off), idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(&s_full[b]);
                umma_commit_mc(&k_empty[c % KST], 3);  // K stage free in both CTAs once both S are done
            };
            mbar_wait(q_full, 0);
            issue_s(0);
            if (nch > 1) issue_s(1);
            for (int c = 0; c < nch; ++c) {
                // PV(c) and S(c + 2) are issued only once the softmax warps hold
                // S(c + 1) in registers: a tcgen05.ld queued behind in-flight MMAs
                // waits for them (measured 0.8 us per chunk), so the tensor pipe
                // works while the softmax computes, not while it reads TMEM
                if (c + 1 < nch) mbar_wait(&s_free[(c + 1) & 1], ((c + 1) >> 1) & 1);
                issue_pv(c);
                if (c + 2 < nch) issue_s(c + 2);
            }
        }
        __syncwarp();
    } else {
        // ---- softmax warps: thread = (row, column half)
        const int row = (warp & 3) * 32 + lane;
        const int half = warp >> 2;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const bool causal = (it.flags & 1) != 0;
        const int tok_base = causal ? it.row0 : a.dec_tok0 + it.row0;  // batch token of tile row 0
        pdl_wait();  // q comes from the qkv/RoPE kernel
        pdl_trigger();
        span_mark(a, 1);
        // causal prefill rows attend keys <= their own position
        const int prow = causal && row < nrows ? a.pos[tok_base + row / G] : 0x7fffffff;
        {
            // Q tile rows (token r / G, head kvh*G + r % G); rows >= nrows are zero.
            uint4 qv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int idx = tid + i * 256, r = idx >> 4, ch = idx & 15;
                qv[i] = make_uint4(0u, 0u, 0u, 0u);
                if (r < nrows)
                    qv[i] = __ldg(reinterpret_cast<const uint4*>(
                        a.qkv + static_cast<size_t>(tok_base + r / G) * a.QKV + (it.kvh * G + r % G) * HD +
                        ch * 8));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int idx = tid + i * 256, r = idx >> 4, ch = idx & 15;
                *reinterpret_cast<uint4*>(sQ + (ch >> 3) * (SQ_BYTES / 2) + sw128(r, ch & 7)) = qv[i];
            }
            fence_proxy_async();
            mbar_arrive(q_full);
        }
        stamp(a, blockIdx.x, 2);
        float m_run = -INFINITY, l_half = 0.f;
        float* red_mx = red;             // [2 chunk parity][2][128] row maxima halves
        float* red_l = red + 5 * ROWS;   // [2][128]
        for (int c = 0; c < nch; ++c) {
            const int b = c & 1;
            const int nk = min(8, it.npages - c * 8) * PG;
            mbar_wait(&s_full[b], (c >> 1) & 1);
            tc_fence_after();
            if (c == 0) stamp(a, blockIdx.x, 7);
            if (threadIdx.x == 0) cstamp(a, c, 0);
            // raw scores (the softmax scale is folded into the exp2 argument)
            float s[64];
            {
                // one 64-column load (columns past nk hold stale bits: masked)
                tmem_ld64(t_lane + b * 128 + half * 64, s);
                const int col0 = half * 64;
                const int key0 = (it.page0 + c * 8) * PG + col0;
                if (causal || col0 + 64 > nk) {  // (warp-uniform) full decode chunks need no mask
#pragma unroll
                    for (int e = 0; e < 64; ++e)
                        if (!(col0 + e < nk && key0 + e <= prow)) s[e] = -INFINITY;
                }
            }
            tc_fence_before();
            mbar_arrive(&s_free[b]);  // this thread is done with S buffer b
            float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < 64; ++j) mx4[j & 3] = fmaxf(mx4[j & 3], s[j]);
            float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
            float* xm = red_mx + (c & 1) * 2 * ROWS;  // double-buffered half-row maxima
            xm[half * ROWS + row] = mx;
            if (threadIdx.x == 0) cstamp(a, c, 6);
            named_bar(1, 256);
            if (threadIdx.x == 0) cstamp(a, c, 7);
            mx = fmaxf(xm[row], xm[ROWS + row]) * a.sl2;  // log2 domain
            // lazy rescale (exact: O and l always refer to m_run; p <= 2^8 between
            // rescales). The exponentials only need the new running max, so they
            // are computed (and packed to bf16 in registers) before waiting for
            // PV(c-1); only the O rescale and the P store wait for it.
            const bool need = mx > m_run + 8.f;
            const float al = need ? ex2(m_run - mx) : 1.f;
            if (need) {
                l_half *= al;
                m_run = mx;
            }
            const float nm = -m_run;
            uint32_t pk[32];
            float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float p0 = ex2(fmaf(s[2 * j], a.sl2, nm));
                const float p1 = ex2(fmaf(s[2 * j + 1], a.sl2, nm));
                ls[j & 3] += p0 + p1;
                pk[j] = pack2(p0, p1);
            }
            l_half += (ls[0] + ls[1]) + (ls[2] + ls[3]);
            // PV(c-1) must be done before O is rescaled or P rewritten
            if (threadIdx.x == 0) cstamp(a, c, 1);
            if (c > 0) {
                mbar_wait(o_done, (c - 1) & 1);
                tc_fence_after();
            }
            if (threadIdx.x == 0) cstamp(a, c, 2);
            // tcgen05.ld/st are warp-collective: a warp rescales together
            if (c > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    float v[32];
                    const uint32_t ta = t_lane + 256 + half * 64 + j * 32;
                    tmem_ld32(ta, v);
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] *= al;
                    tmem_st32(ta, v);
                }
                tmem_wait_st();
            }
            // P (bf16 pairs, key-major) into its TMEM columns: the PV MMA reads A from there
            tmem_st32u(t_lane + 384 + half * 32, pk);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_full);
            if (c == 0) stamp(a, blockIdx.x, 8);
            if (threadIdx.x == 0) cstamp(a, c, 3);
        }
        mbar_wait(o_done, (nch - 1) & 1);
        tc_fence_after();
        stamp(a, blockIdx.x, 3);
        stamp(a, blockIdx.x, 9);
        // ---- output rows: normalised bf16 (final rows of a causal tile, else
        // partials), staged row-major in smem (the K/V stages are free) and
        // written by bulk copies, 256 B per (token, head) row
        red_l[half * ROWS + row] = l_half;
        float v[64];
        tmem_ld64(t_lane + 256 + half * 64, v);
        named_bar(1, 256);
        stamp(a, blockIdx.x, 10);
        const float L = red_l[row] + red_l[ROWS + row];
        const float inv = L > 0.f ? __frcp_rn(L) : 0.f;
        constexpr int RS = HD * 2 + 16;  // padded staging row (bytes): conflict-free 16-byte stores
        uint8_t* stage = sKV;
        {
            uint4* dst = reinterpret_cast<uint4*>(stage + row * RS + half * 128);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                dst[e] = make_uint4(pack2(v[8 * e] * inv, v[8 * e + 1] * inv), pack2(v[8 * e + 2] * inv, v[8 * e + 3] * inv),
                                    pack2(v[8 * e + 4] * inv, v[8 * e + 5] * inv), pack2(v[8 * e + 6] * inv, v[8 * e + 7] * inv));
        }
        auto row_pi = [&](int r) {
            return (static_cast<size_t>(it.row0 + r / G) * a.H + it.kvh * G + r % G) * a.max_parts + it.rank;
        };
        if (!causal && half == 0 && row < nrows) a.part_ml[row_pi(row)] = make_float2(m_run, L);
        fence_proxy_async();
        named_bar(1, 256);
        stamp(a, blockIdx.x, 11);
        if (lane < 16) {
            const int r = warp * 16 + lane;
            if (r < nrows) {
                bf16* dst = causal ? a.out + (static_cast<size_t>(tok_base + r / G) * a.H + it.kvh * G + r % G) * HD
                                   : part_bf16(a) + row_pi(r) * HD;
                bulk_s2g(dst, stage + r * RS, HD * 2);
            }
            bulk_commit_wait_read();  // staging reusable; completion is awaited before the grid barrier
        }
        __syncwarp();
        stamp(a, blockIdx.x, 6);
        stamp(a, blockIdx.x, 4);
        stamp(a, blockIdx.x, 5);
    }
    tc_fence_before();
    // neither CTA of the pair may reuse its shared memory while the peer's
    // multicast commits / copies can still target it
    cluster_sync_all();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------- shared, two tiles per CTA (decode)
// The decode tiles of one (kv head, key range): up to 2 x 128 rows in one CTA,
// each tile with its own softmax warpgroup (one thread per row, the whole
// 128-key chunk in registers) and its own TMEM (S | O, P written over S). The
// MMA warp alternates the tiles — PV_0(c), S_0(c+1), PV_1(c), S_1(c+1) — so one
// warpgroup's exponentials overlap the other tile's MMAs: the 128 x 128 chunk
// softmax is bound by the SFU (16 ex2/clk/SM, ~1,024 cycles), the MMAs of a
// chunk by the tensor pipe (~1,024 cycles for S + PV), and the two overlap.
// K/V are read once per CTA (no pairing), K and V rings of 2 stages.
//   smem: sQ [2 tiles][2][128][64] | sK [2][2][128][64] | sV [2][2][128][64] | barriers | page ids
//   TMEM: tile t at columns t * 256: S [0, 128) (P: bf16 pairs in [0, 64)), O [128, 256)
constexpr int S2_Q = 2 * SQ_BYTES;                         // 64 KB
constexpr int S2_BAR = S2_Q + 4 * SKV_BYTES;               // after 2 K + 2 V stages
constexpr int S2_PG = S2_BAR + 256;                        // page ids of the item
static_assert(1024 + S2_PG + SH_MAX_PAGES * 4 <= SH_SMEM - 1024, "shared2 smem overlaps the private barriers");

template <int G>
__device__ __forceinline__ void shared2_phase(const CUtensorMap& tm_kv, const DecodeAttnArgs& a, uint8_t* sm) {
    uint8_t* sK0 = sm + S2_Q;
    auto sQ = [&](int t) { return sm + t * SQ_BYTES; };
    auto sK = [&](int c) { return sK0 + (c & 1) * SKV_BYTES; };
    auto sV = [&](int c) { return sK0 + 2 * SKV_BYTES + (c & 1) * SKV_BYTES; };
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S2_BAR);
    uint64_t* k_full = bars;        // [2] K chunk landed
    uint64_t* k_empty = bars + 2;   // [2] K chunk read by both tiles' S
    uint64_t* v_full = bars + 4;    // [2]
    uint64_t* v_empty = bars + 6;   // [2] V chunk read by both tiles' PV
    uint64_t* s_full = bars + 8;    // [tile] S written (implies the tile's previous PV completed)
    uint64_t* p_full = bars + 10;   // [tile] P written (128 threads)
    uint64_t* q_full = bars + 12;   // [tile] Q tile in smem (128 threads)
    uint64_t* o_fin = bars + 14;    // [tile] last PV of the tile complete
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 16);
    int* spg = reinterpret_cast<int*>(sm + S2_PG);

    stamp(a, blockIdx.x, 0);
    const ShItem it = a.sh[blockIdx.x];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int RB = ROWS / G;  // tokens per tile
    const int ntile = it.ntok > RB ? 2 : 1;
    const int nch = (it.npages + 7) / 8;
    if (it.ntok <= 0 || nch == 0) return;  // padding item (keeps the cluster pairs aligned)

    if (tid == 0) {
        tma_prefetch_desc(&tm_kv);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&k_full[b], 1);
            mbar_init(&k_empty[b], 1);
            mbar_init(&v_full[b], 1);
            mbar_init(&v_empty[b], 1);
            mbar_init(&s_full[b], 1);
            mbar_init(&p_full[b], 128);
            mbar_init(&q_full[b], 128);
            mbar_init(&o_fin[b], 1);
        }
        fence_barrier_init();
    }
    if (warp == 8) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    stamp(a, blockIdx.x, 1);

    if (warp == 9) {
        // ---- TMA producer: decode tiles read shared pages written by earlier
        // steps, so the loads start before griddepcontrol.wait
        for (int i = lane; i < it.npages; i += 32) spg[i] = a.pages[it.ptab + it.page0 + i];
        __syncwarp();
        if (lane == 0) {
            const int rows_per_head = a.Hkv * PG;  // pool-map rows between K and V of a page
            const uint64_t pol = policy_evict_first();
            auto load = [&](int c, int v) {
                const int b = c & 1;
                uint64_t* full = v ? &v_full[b] : &k_full[b];
                if (c >= 2) mbar_wait(v ? &v_empty[b] : &k_empty[b], ((c >> 1) - 1) & 1);
                const int np = min(8, it.npages - c * 8);
                uint8_t* dst = v ? sV(c) : sK(c);
                mbar_expect_tx(full, static_cast<uint32_t>(np) * 2 * 2048);
                for (int i = 0; i < np; ++i) {
                    const int rk = a.layer_row0 + (spg[c * 8 + i] * 2 * a.Hkv + it.kvh) * PG + v * rows_per_head;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (a.kv_evict_first)
                            tma_load_2d_hint(dst + h * SKV_BYTES / 2 + i * 2048, &tm_kv, full, h * 64, rk, pol);
                        else
                            tma_load_2d(dst + h * SKV_BYTES / 2 + i * 2048, &tm_kv, full, h * 64, rk);
                    }
                }
            };
            for (int c = 0; c <= nch; ++c) {
                if (c < nch) load(c, 0);
                if (c >= 1) load(c - 1, 1);
            }
        }
        pdl_wait();
        pdl_trigger();
    } else if (warp == 8) {
        // ---- MMA issuer
        pdl_wait();
        pdl_trigger();
        if (lane == 0) {
            auto issue_s = [&](int t, int c) {
                const int nk = min(8, it.npages - c * 8) * PG;
                const uint32_t idesc = umma_idesc_bf16(ROWS, nk);
                const uint32_t q0 = smem_u32(sQ(t)), k0 = smem_u32(sK(c));
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * (SKV_BYTES / 2) + (kk & 3) * 32;
                    umma_bf16(tmem + t * 256, umma_desc_sw128(q0 + (kk >> 2) * (SQ_BYTES / 2) + (kk & 3) * 32),
                              umma_desc_sw128(k0 + off), idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int c) {
                const int np = min(8, it.npages - c * 8);
                const uint32_t v0 = smem_u32(sV(c));
                const uint32_t idesc = umma_idesc_bf16(ROWS, HD) | (1u << 16);  // B = V, MN-major
                for (int kk = 0; kk < np; ++kk)
                    umma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + kk * 8,
                                 umma_desc_sw128_lbo(v0 + kk * 2048, SKV_BYTES / 2, 1024), idesc,
                                 (c > 0 || kk > 0) ? 1u : 0u);
            };
            for (int t = 0; t < ntile; ++t) mbar_wait(&q_full[t], 0);
            mbar_wait(&k_full[0], 0);
            tc_fence_after();
            for (int t = 0; t < ntile; ++t) issue_s(t, 0);
            umma_commit(&k_empty[0]);
            for (int c = 0; c < nch; ++c) {
                mbar_wait(&v_full[c & 1], (c >> 1) & 1);
                if (c + 1 < nch) mbar_wait(&k_full[(c + 1) & 1], ((c + 1) >> 1) & 1);
                for (int t = 0; t < ntile; ++t) {
                    // P_t(c) is written over S_t(c); S_t(c + 1) is issued after PV_t(c)
                    // (tcgen05 MMAs of one thread execute in order)
                    mbar_wait(&p_full[t], c & 1);
                    tc_fence_after();
                    cstamp(a, c, 4 + t);
                    issue_pv(t, c);
                    if (c + 1 == nch) umma_commit(&o_fin[t]);
                    else issue_s(t, c + 1);
                }
                umma_commit(&v_empty[c & 1]);
                if (c + 1 < nch) umma_commit(&k_empty[(c + 1) & 1]);
            }
        }
        __syncwarp();
    } else {
        // ---- softmax warpgroups: WG t = warps 4t .. 4t + 3, one thread per row of tile t
        const int t = warp >> 2;
        const int row = (warp & 3) * 32 + lane;
        const uint32_t t_lane = tmem + t * 256 + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const int tok0 = it.row0 + t * RB;                       // decode row of this tile's row 0
        const int ntok_t = t < ntile ? min(RB, it.ntok - t * RB) : 0;
        const int nrows = ntok_t * G;
        pdl_wait();  // q comes from the qkv/RoPE kernel
        pdl_trigger();
        span_mark(a, 1);
        if (t < ntile) {
        {
            // Q tile rows (token r / G, head kvh*G + r % G); rows >= nrows are zero
            uint8_t* q = sQ(t);
            const int wt = tid & 127;
            uint4 qv[16];  // every load in flight at once (one round trip)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int idx = wt + i * 128, r = idx >> 4, ch = idx & 15;
                qv[i] = make_uint4(0u, 0u, 0u, 0u);
                if (r < nrows)
                    qv[i] = __ldg(reinterpret_cast<const uint4*>(a.qkv + static_cast<size_t>(a.dec_tok0 + tok0 + r / G) * a.QKV +
                                                                 (it.kvh * G + r % G) * HD + ch * 8));
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int idx = wt + i * 128, r = idx >> 4, ch = idx & 15;
                *reinterpret_cast<uint4*>(q + (ch >> 3) * (SQ_BYTES / 2) + sw128(r, ch & 7)) = qv[i];
            }
            fence_proxy_async();
            mbar_arrive(&q_full[t]);
        }
        stamp(a, blockIdx.x, 2);
        float m_run = -INFINITY, l_run = 0.f;
        for (int c = 0; c < nch; ++c) {
            const int nk = min(8, it.npages - c * 8) * PG;
            mbar_wait(&s_full[t], c & 1);
            tc_fence_after();
            if (c == 0) stamp(a, blockIdx.x, 7);
            if (tid == 0) cstamp(a, c, 0);
            float s[128];
            {
                float* s0 = s;
                float* s1 = s + 64;
                tmem_ld64(t_lane, *reinterpret_cast<float(*)[64]>(s0));
                tmem_ld64(t_lane + 64, *reinterpret_cast<float(*)[64]>(s1));
            }
            if (nk < 128) {
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e >= nk) s[e] = -INFINITY;
            }
            // the chunk loop is issue-bound: three-input max (FMNMX3) and packed
            // fp32x2 FMA / add (FFMA2 / FADD2) halve those instruction counts
            float m4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
            for (int j = 4; j < 124; j += 8) {
#pragma unroll
                for (int q = 0; q < 4; ++q) m4[q] = fmax3(m4[q], s[j + q], s[j + 4 + q]);
            }
            m4[0] = fmax3(m4[0], s[124], s[125]);
            m4[1] = fmax3(m4[1], s[126], s[127]);
            float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
            mx *= a.sl2;  // log2 domain
            if (tid == 0) cstamp(a, c, 6);
            // lazy rescale (exact: O and l always refer to m_run; p <= 2^8 between rescales)
            const bool need = mx > m_run + 8.f;
            const float al = need ? ex2(m_run - mx) : 1.f;
            if (need) {
                l_run *= al;
                m_run = mx;
            }
            const float nm = -m_run;
            uint32_t pk[64];
            const float2 sl2v = make_float2(a.sl2, a.sl2), nmv = make_float2(nm, nm);
            float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const float2 x = __ffma2_rn(make_float2(s[2 * j], s[2 * j + 1]), sl2v, nmv);
                const float p0 = ex2(x.x), p1 = ex2(x.y);
                ls2[j & 1] = __fadd2_rn(ls2[j & 1], make_float2(p0, p1));
                pk[j] = pack2(p0, p1);
            }
            l_run += (ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y);
            if (tid == 0) cstamp(a, c, 1);
            // s_full(c) implies PV(c - 1) completed: O may be rescaled now
            if (c > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float v[32];
                    const uint32_t ta = t_lane + 128 + j * 32;
                    tmem_ld32(ta, v);
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] *= al;
                    tmem_st32(ta, v);
                }
            }
            // P (bf16 pairs, key-major) over S's first 64 columns: the PV MMA reads A there
            tmem_st32u(t_lane, *reinterpret_cast<uint32_t(*)[32]>(pk));
            tmem_st32u(t_lane + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[t]);
            if (c == 0) stamp(a, blockIdx.x, 8);
            if (tid == 0) cstamp(a, c, 3);
        }
        mbar_wait(&o_fin[t], 0);
        tc_fence_after();
        stamp(a, blockIdx.x, 3);
        // ---- output rows: normalised bf16 partials + (m, l), staged row-major in
        // smem (the K/V stages are free) and written by bulk copies, 256 B per row
        float v[128];
        tmem_ld64(t_lane + 128, *reinterpret_cast<float(*)[64]>(v));
        tmem_ld64(t_lane + 192, *reinterpret_cast<float(*)[64]>(v + 64));
        const float inv = l_run > 0.f ? __frcp_rn(l_run) : 0.f;
        constexpr int RS = HD * 2 + 16;  // padded staging row (bytes)
        uint8_t* stage = sK0 + t * ROWS * RS;
        {
            uint4* dst = reinterpret_cast<uint4*>(stage + row * RS);
#pragma unroll
            for (int e = 0; e < 16; ++e)
                dst[e] = make_uint4(pack2(v[8 * e] * inv, v[8 * e + 1] * inv), pack2(v[8 * e + 2] * inv, v[8 * e + 3] * inv),
                                    pack2(v[8 * e + 4] * inv, v[8 * e + 5] * inv), pack2(v[8 * e + 6] * inv, v[8 * e + 7] * inv));
        }
        const size_t pi = (static_cast<size_t>(tok0 + row / G) * a.H + it.kvh * G + row % G) * a.max_parts + it.rank;
        if (row < nrows) a.part_ml[pi] = make_float2(m_run, l_run);
        fence_proxy_async();
        named_bar(3 + t, 128);
        stamp(a, blockIdx.x, 11);
        {
            // each thread of the warpgroup copies one row
            if (row < nrows) bulk_s2g(part_bf16(a) + pi * HD, stage + row * RS, HD * 2);
            bulk_commit_wait_read();  // staging reusable; completion is awaited before the grid barrier
        }
        stamp(a, blockIdx.x, 5);
        }  // t < ntile
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------ private (tensor cores)
// One warp per item (a token's own pages for one kv head). MMA rows are the G
// q-heads of the token (rows >= G are zero padding): per 16-key page,
// S = Q K^T is 8 x 2 mma.sync m16n8k16 and O += P V is 16 more, operands read
// with ldmatrix from TMA-swizzled page tiles (conflict-free). The warp feeds
// itself: lane 0 keeps PV_ST pages (4 TMA boxes each) in flight in the warp's
// own ring and refills a stage as soon as the warp has read it.
constexpr int PV_ST = 3;  // pages in flight per private warp

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of (row, 16-byte chunk c of 16) in a page tile made of two TMA
// boxes [16 rows][64 elems] with 128B swizzle (box = c / 8)
__device__ __forceinline__ uint32_t tile_off(int row, int c) {
    return static_cast<uint32_t>((c >> 3) * 2048 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

// One private item with the calling warp. ring / full: the warp's PV_ST
// stages (8 KB each) and their mbarriers; pc counts the pages this warp has
// already pushed through the ring (mbarrier phase bookkeeping).
// The queue is software-pipelined: `next` holds the next item's index (its
// atomic was issued before this item started); while this item's pages
// stream, the warp loads the next item's record and page ids into `nit` /
// `npage`, so a new item starts without waiting on L2 round trips.
struct PvNext {
    int idx;     // next item index (raw atomic result in lane 0)
    PvItem it;   // its record (valid when idx < n_pv after the prefetch)
    int page;    // its page id for this lane
};
__device__ __forceinline__ void prefetch_next(const DecodeAttnArgs& a, PvNext& nx) {
    nx.idx = __shfl_sync(0xffffffffu, nx.idx, 0);
    if (nx.idx < a.n_pv) {
        nx.it = a.pv[nx.idx];
        const int nnp = (nx.it.kend - nx.it.kbeg + PG - 1) / PG;
        const int lane = threadIdx.x & 31;
        nx.page = lane < nnp ? a.pages[nx.it.ptab + nx.it.kbeg / PG + lane] : 0;
    }
}

// Issue page i of item `it` into the warp's ring (lane 0 only): K and V, two
// TMA boxes each.
__device__ __forceinline__ void pv_issue(const CUtensorMap& tm_kv, const DecodeAttnArgs& a, const PvItem& it,
                                         uint8_t* ring, uint64_t* full, int pc, int i, int page) {
    const int s = (pc + i) % PV_ST;
    uint64_t* bar = &full[s];
    uint8_t* dst = ring + s * 8192;
    const int rk = a.layer_row0 + (page * 2 * a.Hkv + it.kvh) * PG;
    const int rows_per_head = a.Hkv * PG;
    mbar_expect_tx(bar, 8192);
    if (a.kv_evict_first) {
        const uint64_t pol = policy_evict_first();
        tma_load_2d_hint(dst, &tm_kv, bar, 0, rk, pol);
        tma_load_2d_hint(dst + 2048, &tm_kv, bar, 64, rk, pol);
        tma_load_2d_hint(dst + 4096, &tm_kv, bar, 0, rk + rows_per_head, pol);
        tma_load_2d_hint(dst + 6144, &tm_kv, bar, 64, rk + rows_per_head, pol);
        return;
    }
    tma_load_2d(dst, &tm_kv, bar, 0, rk);
    tma_load_2d(dst + 2048, &tm_kv, bar, 64, rk);
    tma_load_2d(dst + 4096, &tm_kv, bar, 0, rk + rows_per_head);
    tma_load_2d(dst + 6144, &tm_kv, bar, 64, rk + rows_per_head);
}

// Pages of `it` that were written by earlier steps: every page before the one
// holding the item's last key (the decode token's own K/V, written by this
// step's RoPE kernel, lives there). They may be loaded before griddepcontrol.wait.
__device__ __forceinline__ int pv_safe_pages(const PvItem& it) {
    return (it.kend - 1) / PG - it.kbeg / PG;
}

template <int G>
__device__ __forceinline__ void private_item(const CUtensorMap& tm_kv, const DecodeAttnArgs& a, const PvItem& it,
                                             int my_page, uint8_t* ring, uint64_t* full, int& pc, PvNext& nx,
                                             int pre = 0, int item = 0) {
    item_stamp(a, item, 0);
    static_assert(G <= 8, "private item: G q-heads must fit rows 0-7 of the MMA tile");
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int np = (it.kend - it.kbeg + PG - 1) / PG;
    const uint32_t ring_s = smem_u32(ring);
    // (my_page: page ids of the item, one per lane; np <= 32 for this kernel's key splits)
    auto issue = [&](int i, int page) { pv_issue(tm_kv, a, it, ring, full, pc, i, page); };
#pragma unroll
    for (int i = 0; i < PV_ST; ++i) {
        const int pg = __shfl_sync(0xffffffffu, my_page, i);
        if (lane == 0 && i >= pre && i < np) issue(i, pg);
    }
    // Q^T as the B operand: column gid = q head kvh*G + gid (heads >= G are zero)
    uint32_t qa[8][2];
    {
        const bf16* qp = a.qkv + static_cast<size_t>(a.dec_tok0 + it.row) * a.QKV + (it.kvh * G + gid) * HD + 2 * tig;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            qa[ks][0] = gid < G ? *reinterpret_cast<const uint32_t*>(qp + ks * 16) : 0u;
            qa[ks][1] = gid < G ? *reinterpret_cast<const uint32_t*>(qp + ks * 16 + 8) : 0u;
        }
    }
    // Swapped operands (the q heads are the 8-wide N dimension, keys / dims the
    // 16-row M dimension): S^T = K Q^T is 8 mma per page and O^T += V^T P^T is
    // 8 more (half the MMAs of a 16-row Q tile padded from G rows). Lane
    // (gid, tig) holds heads h0 = 2 tig, h1 = 2 tig + 1 (heads >= G are zero
    // padding) for keys gid, gid + 8 (S^T) and dims mt*16 + gid (+ 8) (O^T).
    float o[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads h0, h1 (log2 domain)
    // ldmatrix lane roles: matrix mi = lane / 8, row within it rr = lane % 8
    const int mi = lane >> 3, rr = lane & 7;
    for (int i = 0; i < np; ++i) {
        const int s = (pc + i) % PV_ST;
        mbar_wait(&full[s], ((pc + i) / PV_ST) & 1);
        if (i == 0) item_stamp(a, item, 1);
        const uint32_t kt = ring_s + s * 8192, vt = kt + 4096;
        // S^T = K Q^T: A = K [16 keys][16 dims] (ldmatrix), B = Q^T; two
        // accumulators halve the dependent MMA chain
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            uint32_t af[4];
            ldsm_x4(kt + tile_off((mi & 1) * 8 + rr, 2 * ks + (mi >> 1)), af[0], af[1], af[2], af[3]);
            if (ks & 1)
                mma16816(sb, af, qa[ks][0], qa[ks][1]);
            else
                mma16816(sa, af, qa[ks][0], qa[ks][1]);
        }
        const int kb = it.kbeg + i * PG;
        const bool vlo = kb + gid < it.kend, vhi = kb + gid + 8 < it.kend;
        const float s0 = vlo ? (sa[0] + sb[0]) * a.sl2 : -INFINITY;  // key gid, head h0
        const float s1 = vlo ? (sa[1] + sb[1]) * a.sl2 : -INFINITY;  // key gid, head h1
        const float s2 = vhi ? (sa[2] + sb[2]) * a.sl2 : -INFINITY;  // key gid + 8, head h0
        const float s3 = vhi ? (sa[3] + sb[3]) * a.sl2 : -INFINITY;  // key gid + 8, head h1
        float x0 = fmaxf(s0, s2), x1 = fmaxf(s1, s3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
            x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
        }
        if (x0 > m0) {  // (uniform over the 8 lanes of a head pair)
            const float al = ex2(m0 - x0);
            l0 *= al;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                o[j][0] *= al;
                o[j][2] *= al;
            }
            m0 = x0;
        }
        if (x1 > m1) {
            const float al = ex2(m1 - x1);
            l1 *= al;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                o[j][1] *= al;
                o[j][3] *= al;
            }
            m1 = x1;
        }
        const float p0 = ex2(s0 - m0), p1 = ex2(s1 - m1), p2 = ex2(s2 - m0), p3 = ex2(s3 - m1);
        l0 += p0 + p2;
        l1 += p1 + p3;
        // P^T as the B operand [16 keys][8 heads]: transpose the two 8x8 bf16
        // blocks of the S^T accumulator layout in registers
        const uint32_t pb0 = movmatrix_t(pack2(p0, p1)), pb1 = movmatrix_t(pack2(p2, p3));
        // O^T += V^T P^T: A = V^T [16 dims][16 keys] via ldmatrix.trans of the [key][dim] tile
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            uint32_t af[4];
            ldsm_x4_t(vt + tile_off((mi >> 1) * 8 + rr, 2 * mt + (mi & 1)), af[0], af[1], af[2], af[3]);
            mma16816(o[mt], af, pb0, pb1);
        }
        // every lane has read stage s (the shuffle syncs the warp): refill it
        const int pg = __shfl_sync(0xffffffffu, my_page, (i + PV_ST) & 31);
        if (lane == 0 && i + PV_ST < np) issue(i + PV_ST, pg);
        if (i == 0) prefetch_next(a, nx);
    }
    pc += np;
    item_stamp(a, item, 2);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const int h0 = 2 * tig, h1 = h0 + 1;
    // The G normalised rows go through the warp's (now free) ring as bf16
    // [G][128], then out as 16-byte stores: whole 32-byte sectors, instead of
    // 2-byte stores of the accumulator layout that leave every sector of the
    // rows partially written until the last lane's store lands.
    const float i0 = l0 > 0.f ? __frcp_rn(l0) : 0.f, i1 = l1 > 0.f ? __frcp_rn(l1) : 0.f;
    bf16* st = reinterpret_cast<bf16*>(ring);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (h0 < G) {
            st[h0 * HD + j * 16 + gid] = __float2bfloat16_rn(o[j][0] * i0);
            st[h0 * HD + j * 16 + gid + 8] = __float2bfloat16_rn(o[j][2] * i0);
        }
        if (h1 < G) {
            st[h1 * HD + j * 16 + gid] = __float2bfloat16_rn(o[j][1] * i1);
            st[h1 * HD + j * 16 + gid + 8] = __float2bfloat16_rn(o[j][3] * i1);
        }
    }
    __syncwarp();
    const bool direct = it.part < 0;
    for (int c = lane; c < G * 16; c += 32) {
        const int head = c >> 4, d8 = (c & 15) * 8;
        const uint4 v = *reinterpret_cast<const uint4*>(st + head * HD + d8);
        bf16* dst = direct ? a.out + (static_cast<size_t>(a.dec_tok0 + it.row) * a.H + it.kvh * G + head) * HD + d8
                           : part_bf16(a) +
                                 ((static_cast<size_t>(it.row) * a.H + it.kvh * G + head) * a.max_parts + it.part) * HD + d8;
        *reinterpret_cast<uint4*>(dst) = v;
    }
    __syncwarp();
    fence_proxy_async();  // the ring's next TMA writes follow these generic accesses
    if (!direct && gid == 0) {
        const size_t pi0 = (static_cast<size_t>(it.row) * a.H + it.kvh * G + h0) * a.max_parts + it.part;
        if (h0 < G) a.part_ml[pi0] = make_float2(m0, l0);
        if (h1 < G) a.part_ml[pi0 + a.max_parts] = make_float2(m1, l1);
        // the row's last partial also fills the rest of its 32-byte sector of (m, l)
        // slots (masked by the merge): a partly written sector is completed from
        // DRAM when the merge reads it — a full memory round trip on its critical path
        if (it.part + 1 == a.n_parts[it.row])
            for (int q = it.part + 1; q < ((it.part | 3) + 1) && q < a.max_parts; ++q) {
                if (h0 < G) a.part_ml[pi0 - it.part + q] = make_float2(-INFINITY, 0.f);
                if (h1 < G) a.part_ml[pi0 + a.max_parts - it.part + q] = make_float2(-INFINITY, 0.f);
            }
    }
}

// out[row][head] = merge of the row's n_parts partials. A 16-lane group per
// (row, head), lane owns 8 dims; the part count, every (m, l) and every part's
// 8 dims of a batch of up to 16 parts are loaded at once (one memory round
// trip); unused slots are masked, never multiplied (they may hold stale bits).
// All 32 lanes of the warp must call it (two pairs per warp).
__device__ __forceinline__ void merge16(const DecodeAttnArgs& a, int pair, int n_pairs) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, sub = lane & 15;
    const bool active = pair < n_pairs;
    const int row = active ? pair / a.H : 0, head = active ? pair % a.H : 0;
    if (a.trace && threadIdx.x == 0) a.trace[static_cast<size_t>(blockIdx.x) * 24 + 18] = clock64();
    const int np = active ? a.n_parts[row] : 0;
    const size_t base = (static_cast<size_t>(row) * a.H + head) * a.max_parts;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float M = -INFINITY, L = 0.f;
    // the first batch's loads are issued together with the part count (they do
    // not depend on it; unused slots are masked): one L2 round trip per row
    // (a.any_merge = the step's max part count bounds the first batch: no loads of unused slots)
    const int lim = a.any_merge > 1 ? min(16, a.any_merge) : 16;
    float2 ml = sub < lim ? __ldcg(&a.part_ml[base + sub]) : make_float2(-INFINITY, 0.f);
    uint4 v[16];  // 8 bf16 dims of each of the batch's parts
#pragma unroll
    for (int k = 0; k < 16; ++k)
        v[k] = k < lim ? __ldcg(reinterpret_cast<const uint4*>(part_bf16(a) + (base + k) * HD) + sub) : make_uint4(0u, 0u, 0u, 0u);
    for (int k0 = 0; k0 < a.max_parts; k0 += 16) {
        if (!__any_sync(full, k0 < np)) break;
        if (k0 > 0) {
            ml = __ldcg(&a.part_ml[base + k0 + sub]);
#pragma unroll
            for (int k = 0; k < 16; ++k)
                v[k] = __ldcg(reinterpret_cast<const uint4*>(part_bf16(a) + (base + k0 + k) * HD) + sub);
        }
        const bool mine = k0 + sub < np;
        float mx = mine ? ml.x : -INFINITY;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(full, mx, o));
        const float Mn = fmaxf(M, mx);
        const float sc = M == -INFINITY ? 0.f : exp2f(M - Mn);  // rescale the previous batches
        const float w = mine ? exp2f(ml.x - Mn) * ml.y : 0.f;  // l_p 2^(m_p - M)
        float lw = w;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) lw += __shfl_xor_sync(full, lw, o);
        L = L * sc + lw;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] *= sc;
        const int g0 = lane & 16;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const float wk = __shfl_sync(full, w, g0 + k);
            if (k0 + k < np) {
                const uint32_t u[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc[2 * e] += wk * __uint_as_float(u[e] << 16);
                    acc[2 * e + 1] += wk * __uint_as_float(u[e] & 0xffff0000u);
                }
            }
        }
        M = Mn;
    }
    if (a.trace && threadIdx.x == 0) a.trace[static_cast<size_t>(blockIdx.x) * 24 + 19] = clock64();
    if (!active || np <= 1) return;
    const float inv = L > 0.f ? __frcp_rn(L) : 0.f;
    uint4 w4;
    w4.x = pack2(acc[0] * inv, acc[1] * inv);
    w4.y = pack2(acc[2] * inv, acc[3] * inv);
    w4.z = pack2(acc[4] * inv, acc[5] * inv);
    w4.w = pack2(acc[6] * inv, acc[7] * inv);
    *reinterpret_cast<uint4*>(a.out + (static_cast<size_t>(a.dec_tok0 + row) * a.H + head) * HD + sub * 8) = w4;
    if (a.trace && threadIdx.x == 0) a.trace[static_cast<size_t>(blockIdx.x) * 24 + 20] = clock64();
}

// Fallback merge launch (when the attention grid exceeds one CTA per SM).
__global__ void __launch_bounds__(256) attn_merge_rows_kernel(DecodeAttnArgs a, int n_pairs) {
    pdl_trigger();
    pdl_wait();
    merge16(a, (blockIdx.x * blockDim.x + threadIdx.x) >> 4, n_pairs);
}

// ------------------------------------------------------------ the kernel
// One CTA per SM (persistent). CTA b < n_sh first streams shared item b on
// the tensor cores (all 10 warps); then warps 0-7 of every CTA pull private
// items from a global queue until it is empty, each with its own TMA ring in
// the (now free) shared memory. No SM waits for another's phase.
constexpr int DA_PV_WARPS = 8;
constexpr int DA_SMEM = SH_SMEM + 256;

template <int G>
__global__ void __launch_bounds__(SH_THREADS, 1) attn_decode_kernel(const __grid_constant__ CUtensorMap tm_kv,
                                                                    DecodeAttnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // stay in the shared address space (pointer arithmetic on the array) so
    // plain stores compile to STS
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    pdl_trigger();  // the next kernel (O projection) may launch; it waits for us before reading
    span_mark(a, 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* ring = sm + warp * PV_ST * 8192;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + SH_SMEM - 1024) + warp * PV_ST;
    int pc = 0, pre = 0;
    PvNext nx;
    nx.idx = a.n_pv;
    if (blockIdx.x < a.n_sh) {
        if (a.sh[blockIdx.x].flags & 2)
            shared2_phase<G>(tm_kv, a, sm);
        else
            shared_phase<G>(tm_kv, a, sm);
        __syncthreads();
        if (warp >= DA_PV_WARPS) return;
        // the planner sizes private items for one round on the queue-only CTAs;
        // a shared CTA only joins the queue when there are none or too few (the
        // claim of an already empty queue is an L2 round trip on its tail)
        const int q_ctas = static_cast<int>(gridDim.x) - a.n_sh;
        if (q_ctas <= 0 || a.n_pv > q_ctas * DA_PV_WARPS) {
            if (lane == 0) {
                for (int s = 0; s < PV_ST; ++s) mbar_init(&full[s], 1);
                fence_barrier_init();
            }
            __syncwarp();
            nx.idx = lane == 0 ? atomicAdd(a.pv_next, 1) : 0;
            prefetch_next(a, nx);
        }
    } else {
        stamp(a, blockIdx.x, 0);
        // Queue-only CTA: claim the first item and start streaming its pages
        // that earlier steps wrote (metadata and old KV do not depend on the
        // predecessor kernel), then wait for q and this step's K/V.
        if (warp < DA_PV_WARPS) {
            if (lane == 0) {
                for (int s = 0; s < PV_ST; ++s) mbar_init(&full[s], 1);
                fence_barrier_init();
            }
            __syncwarp();
            nx.idx = lane == 0 ? atomicAdd(a.pv_next, 1) : 0;
            prefetch_next(a, nx);
            if (nx.idx < a.n_pv) {
                pre = min(PV_ST, pv_safe_pages(nx.it));
#pragma unroll
                for (int i = 0; i < PV_ST; ++i) {
                    const int pg = __shfl_sync(0xffffffffu, nx.page, i);
                    if (lane == 0 && i < pre) pv_issue(tm_kv, a, nx.it, ring, full, pc, i, pg);
                }
            }
        }
        pdl_wait();  // q and this step's own K/V come from the qkv/RoPE kernel
        span_mark(a, 1);
        if (warp >= DA_PV_WARPS) return;
    }
    while (nx.idx < a.n_pv) {
        const PvItem it = nx.it;
        const int my_page = nx.page;
        const int cur = __shfl_sync(0xffffffffu, nx.idx, 0);
        nx.idx = lane == 0 ? atomicAdd(a.pv_next, 1) : 0;  // claim the next item now; used after page 0
        private_item<G>(tm_kv, a, it, my_page, ring, full, pc, nx, pre, cur);
        pre = 0;
    }
    if (warp == 0) stamp(a, blockIdx.x, 12);
    // this CTA's work is done; HBM idles while stragglers finish and rows merge:
    // pull its slice of the O-projection weights into L2 (opt-in, HK_L2_PREFETCH_O)
    if (threadIdx.x == 0) prefetch_next_weights(a);
    bulk_wait_all();  // a shared tile's bulk-copied output rows are written (before the grid barrier / exit)
    if (!a.merge_in_kernel) {
        // the last warp out rewinds the queue for the next launch
        if (lane == 0 && atomicAdd(a.pv_done, 1) == static_cast<int>(gridDim.x) * DA_PV_WARPS - 1) {
            *a.pv_next = 0;
            *a.pv_done = 0;
        }
        span_mark(a, 2);
        return;
    }
    // Grid-wide arrival: every CTA of this grid is resident (one per SM, and
    // the launch guarantees grid <= SMs), so spinning cannot deadlock. After
    // it, all partials exist: the rows are merged by every SM in parallel.
    named_bar(2, DA_PV_WARPS * 32);
    const int tid = threadIdx.x;
    if (warp == 0) stamp(a, blockIdx.x, 16);
    if (tid == 0) {
        __threadfence();
        atomicAdd(a.grid_arrive, 1);
        int seen;
        do {
            asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.grid_arrive) : "memory");
        } while (seen < static_cast<int>(gridDim.x));
        __threadfence();  // acquire: every CTA's partials are visible from here on
    }
    named_bar(2, DA_PV_WARPS * 32);
    if (warp == 0) stamp(a, blockIdx.x, 13);
    const int n_pairs = a.n_rows * a.H;
    for (int pb = blockIdx.x * (DA_PV_WARPS * 2); pb < n_pairs; pb += gridDim.x * (DA_PV_WARPS * 2))
        merge16(a, pb + (tid >> 4), n_pairs);
    named_bar(2, DA_PV_WARPS * 32);
    if (warp == 0) stamp(a, blockIdx.x, 17);
    // the last CTA out rewinds the queue and the barrier for the next launch
    if (tid == 0 && atomicAdd(a.pv_done, 1) == static_cast<int>(gridDim.x) - 1) {
        *a.pv_next = 0;
        *a.pv_done = 0;
        *a.grid_arrive = 0;
    }
    span_mark(a, 2);
}

template <int G>
void launch_g(const DecodeAttnArgs& a, const CUtensorMap& tm, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        HK_CUDA(cudaFuncSetAttribute(attn_decode_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, DA_SMEM));
        configured = true;
    }
    // every SM: shared items first, the rest of the grid starts on the private queue at once
    int grid = std::max(a.n_sh, a.n_pv > 0 ? g_num_sms : 1);
    grid += grid & 1;  // CTA pairs (clusters of 2)
    if (a.n_sh & 1) throw std::runtime_error("decode_attention: shared items must come in pairs");
    DecodeAttnArgs k = a;
    static const bool merge_separate = std::getenv("HK_ATTN_MERGE_SEPARATE") && std::atoi(std::getenv("HK_ATTN_MERGE_SEPARATE")) != 0;
    k.merge_in_kernel = a.any_merge && grid <= g_num_sms && !merge_separate ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(SH_THREADS);
    cfg.dynamicSmemBytes = DA_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    HK_CUDA(cudaLaunchKernelEx(&cfg, attn_decode_kernel<G>, tm, k));
    HK_LAUNCHED(1);
    static const bool no_merge = std::getenv("HK_ATTN_DEBUG_NO_MERGE") != nullptr;  // timing experiments only
    if (a.n_rows > 0 && a.any_merge && !no_merge && !k.merge_in_kernel) {
        const int pairs = a.n_rows * a.H;  // 16 lanes each
        static const bool merge_plain = std::getenv("HK_ATTN_MERGE_NO_PDL") != nullptr;
        if (merge_plain)
            attn_merge_rows_kernel<<<(pairs * 16 + 255) / 256, 256, 0, st>>>(a, pairs);
        else
            launch_pdl(attn_merge_rows_kernel, dim3((pairs * 16 + 255) / 256), dim3(256), 0, st, a, pairs);
        HK_LAUNCHED(1);
    }
}

}  // namespace

void decode_attention(const DecodeAttnArgs& a, const CUtensorMap& tm_kv, cudaStream_t st) {
    switch (a.H / a.Hkv) {
        case 1: launch_g<1>(a, tm_kv, st); break;
        case 2: launch_g<2>(a, tm_kv, st); break;
        case 4: launch_g<4>(a, tm_kv, st); break;
        case 5: launch_g<5>(a, tm_kv, st); break;
        default: throw std::runtime_error("decode_attention: unsupported GQA group size");
    }
}

// Host planning: every shared group is tiled into (128/G rows) x kv heads;
// each tile is streamed by a cluster of S CTAs (S uniform per launch, about
// one CTA per SM overall, <= 8 portable) that split its 8-page chunks. Every
// row then gets private items over its own pages, split at kPrivKeys keys.
void plan_decode_attention(const std::vector<DecodeRowIn>& rows, const std::vector<DecodeGroupIn>& groups, int H,
                           int Hkv, int max_parts, int num_sms, DecodePlan& plan) {
    const int G = H / Hkv;
    const int rb = ROWS / G;
    const double kv_tok = 2.0 * HD * 2;  // K + V bytes of one key of one kv head
    plan.sh.clear();
    plan.pv.clear();
    plan.n_parts.assign(rows.size(), 0);
    plan.shared_bytes = plan.private_bytes = 0;
    // decode tiles: two row blocks per CTA (shared2_phase), or CTA pairs of one row
    // block each with multicast pages (shared_phase; HK_ATTN_TWO_TILE=0)
    static const bool two_tile = !(std::getenv("HK_ATTN_TWO_TILE") && std::atoi(std::getenv("HK_ATTN_TWO_TILE")) == 0);
    int tiles = 0;  // shared CTAs per split x kv heads
    for (const auto& g : groups)
        if (g.shared_pages > 0 && g.members > 1) {
            const int nrb = (g.members + rb - 1) / rb;
            tiles += (two_tile ? (nrb + 1) / 2 : nrb + (nrb & 1)) * Hkv;
        }
    plan.sh_cluster = 1;
    // private key split: about 8 private warps per SM over the whole step
    double priv_keys = 0;
    for (const auto& g : groups) {
        const int k0 = (g.shared_pages > 0 && g.members > 1) ? g.shared_pages * PG : 0;
        for (int m = 0; m < g.members; ++m) priv_keys += rows[static_cast<size_t>(g.row0 + m)].pos + 1 - k0;
    }
    static const int env_priv_keys = std::getenv("HK_ATTN_PRIV_KEYS") ? std::atoi(std::getenv("HK_ATTN_PRIV_KEYS")) : 0;
    // Shared split count S (measured on B200, tools/attn_bench.py, profiles/
    // r1_attention.txt): shared CTAs should cover ~64 SMs for a <= 2K-token
    // prefix (the private queue keeps the other SMs streaming), every SM for
    // longer prefixes; SMs without a shared item start on the private queue
    // at once.
    int best_s = 1;
    {
        double rows_n = 0;
        for (const auto& g : groups) rows_n += g.members;
        const double priv_pages_per_row = rows_n > 0 ? priv_keys / rows_n / PG : 0;
        int max_nch = 0;
        for (const auto& g : groups)
            if (g.shared_pages > 0 && g.members > 1) max_nch = std::max(max_nch, (g.shared_pages + 7) / 8);
        // long shared prefixes (> 2K tokens, e.g. configs[4]'s 8K) are tensor-bound: one CTA per SM
        // (r1c re-measure: ~64 shared CTAs at every k for a 2K prefix — the
        // private items then run as one round on the other ~84 SMs)
        (void)priv_pages_per_row;
        // two-tile CTAs: ~2/3 of the SMs for long prefixes (configs[4] at k = 1 / 128 / 256: 96 shared
        // CTAs 47.9 / 50.0 / 52.8 us, 144 CTAs 44.4 / 56.5 / 71.2 us — the private rows need the rest)
        const int target = max_nch > 16 ? (two_tile ? num_sms * 2 / 3 : num_sms) : 64;
        if (tiles > 0) best_s = std::max(1, std::min(8, static_cast<int>(std::lround(static_cast<double>(target) / tiles))));
        static const int env_splits = std::getenv("HK_ATTN_SPLITS") ? std::atoi(std::getenv("HK_ATTN_SPLITS")) : 0;
        if (env_splits > 0) best_s = env_splits;
    }
    // Private split: each (row, kv head) is cut into npv items so that all
    // items run as ONE round on the warps that are free while the shared tiles
    // stream (an item pays one HBM latency before its first page; a second
    // round of short items doubles that, measured with tools/attn_items.py).
    double priv_pages = 0;
    for (const auto& g : groups) {
        const int k0 = (g.shared_pages > 0 && g.members > 1) ? g.shared_pages * PG : 0;
        for (int m = 0; m < g.members; ++m) priv_pages += (rows[static_cast<size_t>(g.row0 + m)].pos + 1 - k0 + PG - 1) / PG;
    }
    const int sh_ctas = tiles * best_s;
    const double q_warps = 8.0 * (sh_ctas < num_sms ? num_sms - sh_ctas : num_sms);
    for (const auto& g : groups) {
        const bool shared = g.shared_pages > 0 && g.members > 1;
        const int shared_pages = shared ? g.shared_pages : 0;
        int splits = 0;
        if (shared) {
            const int nch = (shared_pages + 7) / 8;
            splits = std::max(1, std::min({nch, best_s, max_parts / 2}));
            int cpc = (nch + splits - 1) / splits;
            cpc = std::min(cpc, SH_MAX_PAGES / 8);
            splits = (nch + cpc - 1) / cpc;
            // row blocks of the same (kv head, page range) are adjacent CTAs: they
            // stream the same pages at the same time, so L2 serves the second copy
            // row blocks of the same (kv head, page range) are CTA pairs (clusters
            // of 2) that fetch the pages once and multicast them; an odd count is
            // padded with an empty row block that only helps fetch
            const int nrb = (g.members + rb - 1) / rb;
            if (two_tile) {
                for (int h = 0; h < Hkv; ++h)
                    for (int k = 0; k < splits; ++k)
                        for (int j = 0; j < nrb; j += 2) {
                            ShItem it{};
                            it.row0 = g.row0 + j * rb;
                            it.ntok = std::min(2 * rb, g.members - j * rb);
                            it.kvh = h;
                            it.ptab = rows[static_cast<size_t>(g.row0)].ptab;
                            it.page0 = k * cpc * 8;
                            it.npages = std::min(cpc * 8, shared_pages - it.page0);
                            it.rank = k;
                            it.flags = 2;
                            plan.sh.push_back(it);
                        }
            } else
            for (int h = 0; h < Hkv; ++h)
                for (int k = 0; k < splits; ++k)
                    for (int j = 0; j < nrb + (nrb & 1); ++j) {
                        const int r0 = std::min(j * rb, g.members);
                        ShItem it{};
                        it.row0 = g.row0 + r0;
                        it.ntok = std::max(0, std::min(rb, g.members - r0));
                        it.kvh = h;
                        it.ptab = rows[static_cast<size_t>(g.row0)].ptab;
                        it.page0 = k * cpc * 8;
                        it.npages = std::min(cpc * 8, shared_pages - it.page0);
                        it.mc_pages = it.npages;  // both row blocks read the group's shared pages
                        it.rank = k;  // partial index
                        plan.sh.push_back(it);
                    }
            plan.shared_bytes += static_cast<double>(shared_pages) * PG * Hkv * kv_tok;
        }
        for (int m = 0; m < g.members; ++m) {
            const int r = g.row0 + m;
            const DecodeRowIn& in = rows[static_cast<size_t>(r)];
            const int k0 = shared_pages * PG, k1 = in.pos + 1;
            if (k1 <= k0) throw std::runtime_error("decode_attention: shared range covers the decode token");
            const int first = splits;  // the shared items contribute partials 0 .. splits - 1
            // keep a row's partials within one 16-part merge batch when possible
            const int part_cap = first < 16 ? 16 - first : max_parts - first;
            const int row_pages = (k1 - k0 + PG - 1) / PG;
            int npv0 = static_cast<int>(row_pages * q_warps / (Hkv * std::max(1.0, priv_pages)));
            npv0 = std::max(1, std::min(npv0, std::max(1, part_cap)));
            npv0 = std::max(npv0, (row_pages + 31) / 32);  // <= 32 pages (one page id per lane)
            int kp = (row_pages + npv0 - 1) / npv0 * PG;
            if (env_priv_keys > 0)
                kp = std::max((env_priv_keys + PG - 1) / PG * PG, (row_pages + std::max(1, part_cap) - 1) / std::max(1, part_cap) * PG);
            if (kp > 32 * PG) throw std::runtime_error("decode_attention: private range too long for max_parts");
            const int npv = (k1 - k0 + kp - 1) / kp;
            const int parts = first + npv;
            if (parts > max_parts) throw std::runtime_error("decode_attention: too many partials for a row");
            plan.n_parts[static_cast<size_t>(r)] = parts;
            for (int i = 0; i < npv; ++i)
                for (int h = 0; h < Hkv; ++h) {
                    PvItem it{};
                    it.row = r;
                    it.kvh = h;
                    it.ptab = in.ptab;
                    it.kbeg = k0 + i * kp;
                    it.kend = std::min(k1, it.kbeg + kp);
                    it.part = parts == 1 ? -1 : first + i;
                    plan.pv.push_back(it);
                }
            plan.private_bytes += static_cast<double>(k1 - k0) * Hkv * kv_tok;
            plan.private_bytes += 2.0 * H * HD * 2;  // q in, o out
        }
    }
    // the launch pairs CTAs (clusters of 2, for the prefill tiles that follow):
    // an empty two-tile item keeps every pair homogeneous
    if (plan.sh.size() & 1) {
        ShItem pad{};
        pad.flags = 2;
        plan.sh.push_back(pad);
    }
}

double plan_prefill_attention(const std::vector<PrefillSegIn>& segs, int H, int Hkv, DecodePlan& plan,
                              const int32_t* arena) {
    const int G = H / Hkv;
    const int rb = ROWS / G;
    double bytes = 0;
    // tile pairs are emitted longest first: with more pairs than SMs the CTAs
    // run in waves in launch order, so the short early-causal pairs fill the tail
    std::vector<std::array<ShItem, 2>> pairs;
    auto item = [&](const PrefillSegIn& sg, int r0, int h, int npages) {
        ShItem it{};
        it.row0 = sg.tok0 + r0;
        it.ntok = std::max(0, std::min(rb, sg.count - r0));
        it.kvh = h;
        it.ptab = sg.ptab;
        it.page0 = 0;
        it.npages = npages;
        it.mc_pages = npages;
        it.rank = -1;
        it.flags = 1;
        return it;
    };
    auto pages_of = [&](const PrefillSegIn& sg) { return (sg.start + sg.count - 1) / PG + 1; };
    for (size_t si = 0; si < segs.size(); ++si) {
        const PrefillSegIn& sg = segs[si];
        const int nrb = (sg.count + rb - 1) / rb;
        bytes += (static_cast<double>(sg.start) + sg.count) * Hkv * 2.0 * HD * 2 + 2.0 * sg.count * H * HD * 2;
        if (pages_of(sg) > SH_MAX_PAGES) throw std::runtime_error("prefill attention: context too long for a tile");
        // two single-tile segments under a common prefix (the calls of one
        // operator after its pinned system prompt) share a pair: the common
        // pages are multicast, each CTA loads its own suffix pages
        if (arena && nrb == 1 && si + 1 < segs.size()) {
            const PrefillSegIn& sb = segs[si + 1];
            const int na = pages_of(sg), nb = pages_of(sb);
            if ((sb.count + rb - 1) / rb == 1 && na == nb) {
                int common = 0;
                while (common < na && arena[sg.ptab + common] == arena[sb.ptab + common]) ++common;
                if (common >= 8) {
                    for (int h = 0; h < Hkv; ++h) {
                        std::array<ShItem, 2> pr{item(sg, 0, h, na), item(sb, 0, h, na)};
                        pr[0].mc_pages = pr[1].mc_pages = common;
                        pairs.push_back(pr);
                    }
                    bytes += (static_cast<double>(sb.start) + sb.count) * Hkv * 2.0 * HD * 2 + 2.0 * sb.count * H * HD * 2;
                    ++si;
                    continue;
                }
            }
        }
        for (int h = 0; h < Hkv; ++h)
            for (int j = 0; j < nrb + (nrb & 1); j += 2) {
                // a CTA pair shares the pages of its later row block (causal mask
                // trims the earlier one); an odd block count gets an empty partner
                const int last_tok = std::min(sg.count, (j + 2) * rb) - 1;
                const int npages = (sg.start + last_tok) / PG + 1;
                pairs.push_back({item(sg, std::min(j * rb, sg.count), h, npages),
                                 item(sg, std::min((j + 1) * rb, sg.count), h, npages)});
            }
    }
    std::stable_sort(pairs.begin(), pairs.end(),
                     [](const std::array<ShItem, 2>& x, const std::array<ShItem, 2>& y) { return x[0].npages > y[0].npages; });
    for (const auto& pr : pairs) {
        plan.sh.push_back(pr[0]);
        plan.sh.push_back(pr[1]);
    }
    return bytes;
}

}  // namespace hkd
