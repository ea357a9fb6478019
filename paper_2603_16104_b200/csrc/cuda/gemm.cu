// K4: dense contractions on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   out[t][n] = sum_k X[t][k] * W[n][k]      (X: activations [T][K], W: weights [N][K])
//
// The MMA's M side is the weight matrix (128 output features per CTA tile)
// and its N side is the token batch, so a decode step with 64 live calls is a
// 128 x 64 UMMA tile that streams weights once (weight-bandwidth bound, the
// regime of the executor's decode iterations) while a prefill chunk uses
// N = 256 token tiles (tensor bound). Operands are staged by TMA into 128B-
// swizzled shared memory through a multi-stage mbarrier ring; one elected
// thread issues tcgen05.mma into a TMEM accumulator; all four warps drain TMEM
// with tcgen05.ld in the epilogue. Split-K (grid.z) covers skinny decode
// GEMMs; partials are reduced deterministically by splitk_reduce.
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace hkd {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row

struct GemmParams {
    int N, K, T;
    int kb_total, kb_per_split;
    int epi;
    void* out;
    int ldo;
    const bf16* bias;
    float* partial;
    int cluster;  // 1: the grid.z split-K CTAs form a cluster and reduce through DSMEM
    int skip_epi; // timing experiments only (HK_GEMM_DEBUG_SKIP_EPI): no output stores
    int tfirst = 0;  // grid.x = token tiles, grid.y = weight tiles
    unsigned long long* trace;  // debug (HK_GEMM_TRACE): [first CTA start, first wait done, ~last end,
                                //  ~last main-loop end] (atomicMin)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- epilogues shared by the one-CTA and the CTA-pair kernels: this CTA's
// 128 weight rows (TMEM lanes) x BN token columns, after the accumulator is final.

// SwiGLU: W rows interleaved per 128-row tile as [64 gate | 64 up]; bf16 out [T][N/2]
template <int BN>
__device__ __forceinline__ void epi_swiglu(const GemmParams& p, uint32_t tmem, uint8_t* smem, int warp, int lane,
                                           int mtile, int n0) {
    const int row = warp * 32 + lane;
    // TMEM lanes 0-63 hold gate rows, 64-127 the matching up rows (a warp
    // may only read lanes 32w..32w+31): every warp parks its rows in smem,
    // then all 128 threads produce silu(gate) * up with coalesced stores.
    float* xs = reinterpret_cast<float*>(smem);  // [128][BN + 1], pipeline buffers are free now
    if constexpr (BN >= 32) {
        // 32-column TMEM loads: a quarter of the load/wait round trips of x8
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            float v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) xs[row * (BN + 1) + c + j] = v[j];
        }
    } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 8) {
            float v[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) xs[row * (BN + 1) + c + j] = v[j];
        }
    }
    __syncthreads();
    const int nt = min(BN, p.T - n0);
    for (int idx = threadIdx.x; idx < 64 * nt; idx += blockDim.x) {
        const int r = idx & 63, c = idx >> 6;
        const int f = mtile * 64 + r;  // output feature
        if (mtile * BM + r < p.N) {
            const float g = xs[r * (BN + 1) + c], u = xs[(r + 64) * (BN + 1) + c];
            static_cast<bf16*>(p.out)[static_cast<size_t>(n0 + c) * p.ldo + f] =
                f2bf(__fdividef(g, 1.0f + __expf(-g)) * u);
        }
    }
}

// fp32 rows (kEpiPartial / StoreF32 / StoreBf16 / AddF32)
template <int BN>
__device__ __forceinline__ void epi_rows(const GemmParams& p, uint32_t tmem, uint8_t* smem, int warp, int lane, int m0,
                                         int n0, int zsplit) {
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const bool m_ok = m < p.N;
    // Stage the fp32 tile through shared memory as [token][feature] (the
    // pipeline buffers are free now), then every warp writes whole rows of
    // 128 consecutive features: 16-byte stores, 512 contiguous bytes per
    // warp instruction, in the [token][ldo] / [split][token][N] layouts.
    constexpr int SO = BM + 4;  // padded row: conflict-free column writes and float4 row reads
    float* so = reinterpret_cast<float*>(smem);
    const float bias = (p.bias && m_ok && p.epi != kEpiPartial) ? bf2f(p.bias[m]) : 0.f;
#pragma unroll
    for (int c = 0; c < BN; c += 32) {
        if constexpr (BN >= 32) {
            float v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) so[(c + j) * SO + row] = v[j] + bias;
        }
    }
    if constexpr (BN < 32) {
#pragma unroll
        for (int c = 0; c < BN; c += 8) {
            float v[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) so[(c + j) * SO + row] = v[j] + bias;
        }
    }
    __syncthreads();
    const int rows = min(BN, p.T - n0);
    const bool full_m = m0 + BM <= p.N;
    for (int r = warp; r < rows; r += 4) {
        const int n = n0 + r;
        const float4 v = reinterpret_cast<const float4*>(so + r * SO)[lane];
        const int mm = m0 + lane * 4;
        if (p.epi == kEpiPartial) {
            float* dst = p.partial + (static_cast<size_t>(zsplit) * p.T + n) * p.N + mm;
            if (full_m) {
                *reinterpret_cast<float4*>(dst) = v;
            } else {
                const float e[4] = {v.x, v.y, v.z, v.w};
                for (int q = 0; q < 4; ++q)
                    if (mm + q < p.N) dst[q] = e[q];
            }
        } else {
            const float e[4] = {v.x, v.y, v.z, v.w};
            for (int q = 0; q < 4; ++q) {
                if (mm + q >= p.N) break;
                const size_t o = static_cast<size_t>(n) * p.ldo + mm + q;
                if (p.epi == kEpiStoreBf16)
                    static_cast<bf16*>(p.out)[o] = f2bf(e[q]);
                else if (p.epi == kEpiAddF32)
                    static_cast<float*>(p.out)[o] += e[q];
                else
                    static_cast<float*>(p.out)[o] = e[q];
            }
        }
    }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2;
    constexpr int B_BYTES = BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // token-tile-fastest grids (p.tfirst, several token tiles): the CTAs that read
    // one weight tile are launched together, so L2 serves it to all but the first
    const int mtile = p.tfirst ? static_cast<int>(blockIdx.y) : static_cast<int>(blockIdx.x);
    const int ntile = p.tfirst ? static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.y);
    const int m0 = mtile * BM;
    const int n0 = ntile * BN;
    const int kb0 = blockIdx.z * p.kb_per_split;
    const int kb1 = min(kb0 + p.kb_per_split, p.kb_total);
    const int nkb = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    pdl_trigger();  // let the next kernel of the chain get scheduled (it prefetches its own weights)
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[0], gtimer());
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            // Weights do not depend on the previous kernel: start streaming the
            // first stages before waiting for the activations (PDL overlap).
            const int pre = min(STAGES, nkb);
            for (int i = 0; i < pre; ++i) {
                mbar_expect_tx(&full[i], A_BYTES + B_BYTES);
                tma_load_2d_hint(sA + i * A_BYTES, &tmW, &full[i], (kb0 + i) * BK, m0, pol_w);
            }
            pdl_wait();
            if (p.trace) atomicMin(&p.trace[1], gtimer());
            for (int i = 0; i < pre; ++i) tma_load_2d_hint(sB + i * B_BYTES, &tmX, &full[i], (kb0 + i) * BK, n0, pol_x);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
                mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                tma_load_2d_hint(sA + s * A_BYTES, &tmW, &full[s], (kb0 + i) * BK, m0, pol_w);
                tma_load_2d_hint(sB + s * B_BYTES, &tmX, &full[s], (kb0 + i) * BK, n0, pol_x);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
        for (int i = 0; i < nkb; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    umma_bf16(tmem, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                              (i | k) != 0 ? 1u : 0u);
                }
                umma_commit(&empty[s]);
                if (i == nkb - 1) umma_commit(done);
            }
            __syncwarp();
        }
    }

    // ---- epilogue: TMEM -> registers -> global (all 4 warps) ----
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    pdl_wait();  // (already satisfied) predecessor writes are visible to the epilogue
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const bool m_ok = m < p.N;
    if (p.cluster) {
        // Split-K reduction inside the cluster: every CTA parks its fp32 tile
        // (column-major [BN][128]) in its own smem; CTA rank r then sums rows
        // [r*128/s, (r+1)*128/s) over all s peers through DSMEM in rank order
        // (deterministic) and applies the epilogue once. No HBM partials.
        float* tile = reinterpret_cast<float*>(smem);
#pragma unroll 1
        for (int c = 0; c < BN; c += 8) {
            float v[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) tile[(c + j) * BM + row] = v[j];
        }
        cluster_sync_all();
        const int s = static_cast<int>(gridDim.z);
        const int rank = static_cast<int>(cluster_ctarank());
        const int per = ((BM + s - 1) / s + 3) & ~3;  // rows per rank, multiple of 4 (float4)
        const int r0 = min(BM, rank * per), r1 = min(BM, r0 + per);
        const int nq = (r1 - r0) / 4;                  // float4 row groups
        const float4* peer[8];
        cg::cluster_group cl = cg::this_cluster();
#pragma unroll
        for (int q = 0; q < 8; ++q) peer[q] = reinterpret_cast<const float4*>(cl.map_shared_rank(tile, q < s ? q : 0));
        for (int idx = threadIdx.x; idx < nq * BN; idx += blockDim.x) {
            const int rr = r0 + 4 * (idx % nq), c = idx / nq;
            const int off4 = (c * BM + rr) / 4;
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < s) v[q] = peer[q][off4];  // all peers' loads in flight together
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < s) {  // fixed rank order: deterministic sum
                    acc[0] += v[q].x;
                    acc[1] += v[q].y;
                    acc[2] += v[q].z;
                    acc[3] += v[q].w;
                }
            const int n = n0 + c;
            if (n >= p.T) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int mm = m0 + rr + e;
                if (mm >= p.N) continue;
                float r = acc[e];
                if (p.bias && p.epi != kEpiPartial) r += bf2f(p.bias[mm]);
                switch (p.epi) {
                    case kEpiStoreBf16:
                        static_cast<bf16*>(p.out)[static_cast<size_t>(n) * p.ldo + mm] = f2bf(r);
                        break;
                    case kEpiAddF32:
                        static_cast<float*>(p.out)[static_cast<size_t>(n) * p.ldo + mm] += r;
                        break;
                    case kEpiStoreF32:
                        static_cast<float*>(p.out)[static_cast<size_t>(n) * p.ldo + mm] = r;
                        break;
                    default:
                        p.partial[static_cast<size_t>(n) * p.N + mm] = r;
                        break;
                }
            }
        }
        cluster_sync_all();  // peers keep their smem until every rank has read it
    } else if (p.epi == kEpiSwiGLU) {
        epi_swiglu<BN>(p, tmem, smem, warp, lane, mtile, n0);
    } else if (p.epi == kEpiArgmax) {
        float2* red = reinterpret_cast<float2*>(smem);  // [4][BN] (value, index)
#pragma unroll 1
        for (int c = 0; c < BN; c += 8) {
            float v[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float best = m_ok ? v[j] : -INFINITY;
                int bi = m;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ov > best || (ov == best && oi < bi)) {
                        best = ov;
                        bi = oi;
                    }
                }
                if (lane == 0) red[warp * BN + c + j] = make_float2(best, __int_as_float(bi));
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < BN; c += blockDim.x) {
            float2 b = red[c];
            for (int w2 = 1; w2 < 4; ++w2) {
                const float2 o = red[w2 * BN + c];
                if (o.x > b.x) b = o;  // earlier warps hold lower rows: keep them on ties
            }
            const int n = n0 + c;
            if (n < p.T) reinterpret_cast<float2*>(p.out)[static_cast<size_t>(mtile) * p.T + n] = b;
        }
    }
    if (p.epi < kEpiSwiGLU && !p.cluster && !p.skip_epi) {
        epi_rows<BN>(p, tmem, smem, warp, lane, m0, n0, static_cast<int>(blockIdx.z));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[3], ~gtimer());  // last CTA to finish its main loop + stores
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[2], ~gtimer());
}

// ---------------------------------------------------------------------------
// Prefill GEMMs on CTA pairs (tcgen05 cta_group::2): a cluster of two CTAs on
// one TPC computes a 256-weight-row x 256-token tile. Each CTA stages its own
// 128 weight rows and HALF of the token rows (32 KB per k-block instead of
// 48 KB), rank 0 issues M=256 MMAs that read both CTAs' shared memory, and
// each CTA's TMEM holds its 128 rows x 256 tokens for the usual epilogue.
// Halving the operand bytes per MMA keeps shared-memory bandwidth (TMA writes
// + MMA reads) under the per-SM limit that caps the one-CTA M=128 x N=256 tile.
constexpr int C2_BN = 256;  // tokens per pair tile
template <int STAGES>
constexpr size_t smem2_bytes() {
    return 1024 + STAGES * (BM * BK * 2 + (C2_BN / 2) * BK * 2) + (2 * STAGES + 1) * 8 + 16;
}

template <int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2;           // this CTA's 128 weight rows
    constexpr int B_BYTES = (C2_BN / 2) * BK * 2;  // this CTA's 128 of the tile's 256 tokens
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // cluster (2, 1, 1): grid.x = 2 x token tiles (pair member fastest), grid.y = weight-tile
    // pairs — consecutive clusters walk the token tiles of one weight pair (L2 reuse)
    const uint32_t rank = cluster_ctarank();
    const int ntile = static_cast<int>(blockIdx.x) >> 1;
    const int mtile = static_cast<int>(blockIdx.y) * 2 + static_cast<int>(rank);
    const int m0 = mtile * BM;
    const int n0 = ntile * C2_BN;
    const int kb0 = blockIdx.z * p.kb_per_split;
    const int kb1 = min(kb0 + p.kb_per_split, p.kb_total);
    const int nkb = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_cg2(tmem_slot, C2_BN);
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers initialised before any peer TMA completes on them
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    pdl_trigger();
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[0], gtimer());
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            // both CTAs' loads complete on rank 0's full barriers; rank 0 expects the pair's bytes
            const uint32_t full0 = mapa_shared(smem_u32(full), 0);
            const int nb = n0 + static_cast<int>(rank) * (C2_BN / 2);
            const int pre = min(STAGES, nkb);
            for (int i = 0; i < pre; ++i) {
                if (rank == 0) mbar_expect_tx(&full[i], 2 * (A_BYTES + B_BYTES));
                tma_load_2d_cg2(sA + i * A_BYTES, &tmW, full0 + i * 8, (kb0 + i) * BK, m0, pol_w);
            }
            pdl_wait();
            if (p.trace && rank == 0) atomicMin(&p.trace[1], gtimer());
            for (int i = 0; i < pre; ++i)
                tma_load_2d_cg2(sB + i * B_BYTES, &tmX, full0 + i * 8, (kb0 + i) * BK, nb, pol_x);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
                if (rank == 0) mbar_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
                tma_load_2d_cg2(sA + s * A_BYTES, &tmW, full0 + s * 8, (kb0 + i) * BK, m0, pol_w);
                tma_load_2d_cg2(sB + s * B_BYTES, &tmX, full0 + s * 8, (kb0 + i) * BK, nb, pol_x);
            }
        }
    } else if (warp == 1 && rank == 0) {
        constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, C2_BN);
        for (int i = 0; i < nkb; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16_cg2(tmem, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                                  (i | k) != 0 ? 1u : 0u);
                umma_commit_cg2_mc(&empty[s], 3);  // frees stage s in both CTAs
                if (i == nkb - 1) umma_commit_cg2_mc(done, 3);
            }
            __syncwarp();
        }
    }

    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    pdl_wait();
    if (!p.skip_epi) {
        if (p.epi == kEpiSwiGLU)
            epi_swiglu<C2_BN>(p, tmem, smem, warp, lane, mtile, n0);
        else
            epi_rows<C2_BN>(p, tmem, smem, warp, lane, m0, n0, static_cast<int>(blockIdx.z));
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the pair deallocates together
    if (warp == 2) tmem_dealloc_cg2(tmem, C2_BN);
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[3], ~gtimer());
    if (p.trace && threadIdx.x == 0) atomicMin(&p.trace[2], ~gtimer());
}

// Deterministic split-K reduction (fixed summation order) fused with the epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int splits, int T, int N, int epi, void* out,
                                     int ldo, const bf16* __restrict__ bias) {
    const size_t total = static_cast<size_t>(T) * N;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i / N);
        const int m = static_cast<int>(i % N);
        float r = 0.f;
        for (int s = 0; s < splits; ++s) r += partial[static_cast<size_t>(s) * total + i];
        if (bias) r += bf2f(bias[m]);
        switch (epi) {
            case kEpiStoreBf16:
                static_cast<bf16*>(out)[static_cast<size_t>(n) * ldo + m] = f2bf(r);
                break;
            case kEpiAddF32:
                static_cast<float*>(out)[static_cast<size_t>(n) * ldo + m] += r;
                break;
            default:
                static_cast<float*>(out)[static_cast<size_t>(n) * ldo + m] = r;
                break;
        }
    }
}

// fp32 parity-mode GEMM (SIMT, tiled); same contract as the tensor-core path.
__global__ void gemm_f32_kernel(const float* __restrict__ W, const float* __restrict__ X, int N, int K, int T,
                                int epi, void* out, int ldo, const float* __restrict__ bias) {
    __shared__ float sW[32][33];
    __shared__ float sX[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int m0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
    float acc[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            sW[r][tx] = (m0 + r < N && k0 + tx < K) ? W[static_cast<size_t>(m0 + r) * K + k0 + tx] : 0.f;
            sX[r][tx] = (n0 + r < T && k0 + tx < K) ? X[static_cast<size_t>(n0 + r) * K + k0 + tx] : 0.f;
        }
        __syncthreads();
        for (int k = 0; k < 32; ++k) {
            const float w = sW[tx][k];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] += w * sX[ty + 8 * j][k];
        }
        __syncthreads();
    }
    const int m = m0 + tx;
    if (m >= N) return;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int n = n0 + ty + 8 * j;
        if (n >= T) continue;
        float r = acc[j] + (bias ? bias[m] : 0.f);
        float* o = static_cast<float*>(out) + static_cast<size_t>(n) * ldo + m;
        if (epi == kEpiAddF32)
            *o += r;
        else
            *o = r;
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        HK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

CUtensorMap make_map_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    return make_tmap_2d_bf16(base, rows, cols, BK, box_rows);
}

}  // namespace

CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

namespace {

// ---------------------------------------------------------------------------
// Prefill gate/up with the SwiGLU epilogue, persistent: one CTA per SM walks
// its tiles (token tiles fastest) with TWO TMEM accumulators, so the epilogue
// of tile i (TMEM -> registers -> silu(gate) * up -> bf16 stores) runs while
// the MMAs of tile i + 1 stream (the one-tile-per-CTA kernel left the tensor
// pipe idle during every epilogue: 43-50 % tensor-pipe activity at T = 2048).
//   warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (warp w reads TMEM lanes
//   32 (w % 4) .. +31: quarters 0-1 are gate rows, 2-3 the matching up rows).
//   smem: STAGES x (A 128 x 64 | B 256 x 64) | up exchange [64][33] fp32 |
//         output block [32 tokens][64 features] bf16 | barriers
constexpr int PK_BN = 256, PK_STAGES = 3, PK_EC = 32;  // epilogue column chunk (tokens)
constexpr size_t pk_smem_bytes() {
    return 1024 + PK_STAGES * (BM * BK * 2 + PK_BN * BK * 2) + 64 * (PK_EC + 1) * 4 + PK_EC * 64 * 2 +
           (2 * PK_STAGES + 4) * 8 + 16;
}

__global__ void __launch_bounds__(192, 1)
    gemm_swiglu_pk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = PK_BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + PK_STAGES * A_BYTES;
    float* xup = reinterpret_cast<float*>(sB + PK_STAGES * B_BYTES);   // [64][PK_EC + 1]
    bf16* ob = reinterpret_cast<bf16*>(xup + 64 * (PK_EC + 1));          // [PK_EC][64]
    uint64_t* full = reinterpret_cast<uint64_t*>(ob + PK_EC * 64);
    uint64_t* empty = full + PK_STAGES;
    uint64_t* acc_full = empty + PK_STAGES;   // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = (p.N + BM - 1) / BM, nt = (p.T + PK_BN - 1) / PK_BN;
    const int tiles = mt * nt, nkb = p.kb_total;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int st = 0; st < PK_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            pdl_wait();
            int g = 0;  // k-blocks issued so far by this CTA (stage ring position)
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = (t / nt) * BM, n0 = (t % nt) * PK_BN;
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % PK_STAGES;
                    if (g >= PK_STAGES) mbar_wait(&empty[st], ((g / PK_STAGES) - 1) & 1);
                    mbar_expect_tx(&full[st], A_BYTES + B_BYTES);
                    tma_load_2d_hint(sA + st * A_BYTES, &tmW, &full[st], kb * BK, m0, pol_w);
                    tma_load_2d_hint(sB + st * B_BYTES, &tmX, &full[st], kb * BK, n0, pol_x);
                }
            }
        }
    } else if (warp == 1) {
        pdl_wait();
        constexpr uint32_t idesc = umma_idesc_bf16(BM, PK_BN);
        int g = 0, i = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            const int b = i & 1;
            if (i >= 2) mbar_wait(&acc_empty[b], ((i >> 1) - 1) & 1);
            tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int st = g % PK_STAGES;
                mbar_wait(&full[st], (g / PK_STAGES) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_base = smem_u32(sA + st * A_BYTES);
                    const uint32_t b_base = smem_u32(sB + st * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(tmem + b * PK_BN, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                                  (kb | k) != 0 ? 1u : 0u);
                    umma_commit(&empty[st]);
                    if (kb == nkb - 1) umma_commit(&acc_full[b]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---- epilogue warps: 128 threads, thread = TMEM lane (weight row of the tile)
        pdl_wait();
        const int q = warp & 3;  // lane quarter this warp may read
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;  // 0..127
        int i = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            const int b = i & 1;
            const int mtile = t / nt, n0 = (t % nt) * PK_BN;
            mbar_wait(&acc_full[b], (i >> 1) & 1);
            tc_fence_after();
            for (int c0 = 0; c0 < PK_BN; c0 += PK_EC) {
                float v[PK_EC];
                tmem_ld32(tmem + b * PK_BN + c0 + (static_cast<uint32_t>(q * 32) << 16), v);
                if (c0 + PK_EC == PK_BN) {  // the whole accumulator is in registers: free it
                    tc_fence_before();
                    mbar_arrive(&acc_empty[b]);
                }
                if (row >= 64) {
#pragma unroll
                    for (int j = 0; j < PK_EC; ++j) xup[(row - 64) * (PK_EC + 1) + j] = v[j];
                }
                named_bar(1, 128);
                if (row < 64) {
#pragma unroll
                    for (int j = 0; j < PK_EC; ++j) {
                        const float g = v[j], u = xup[row * (PK_EC + 1) + j];
                        ob[j * 64 + row] = f2bf(__fdividef(g, 1.0f + __expf(-g)) * u);
                    }
                }
                named_bar(1, 128);
                // [PK_EC tokens][64 features]: 128-byte rows, 16 bytes per thread x 2
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int idx = et + k * 128, j = idx >> 3, c8 = (idx & 7) * 8;
                    const int n = n0 + c0 + j, f = mtile * 64 + c8;
                    if (n < p.T && f < p.N / 2)
                        *reinterpret_cast<uint4*>(static_cast<bf16*>(p.out) + static_cast<size_t>(n) * p.ldo + f) =
                            *reinterpret_cast<const uint4*>(ob + j * 64 + c8);
                }
                named_bar(1, 128);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// The persistent gate/up kernel on CTA pairs: a cluster of two CTAs walks
// 256-weight-row x 256-token pair tiles (token tiles fastest); per k-block each
// CTA stages its 128 weight rows and half the tokens, rank 0 issues the M=256
// MMAs into the two accumulators, and both CTAs' epilogue warps free an
// accumulator on rank 0's barrier. Same SwiGLU epilogue as above.
constexpr int PK2_STAGES = 6;
constexpr size_t pk2_smem_bytes() {
    return 1024 + PK2_STAGES * (BM * BK * 2 + (PK_BN / 2) * BK * 2) + 64 * (PK_EC + 1) * 4 + PK_EC * 64 * 2 +
           (2 * PK2_STAGES + 4) * 8 + 16;
}

__global__ void __launch_bounds__(192, 1)
    gemm_swiglu_pk2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = (PK_BN / 2) * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + PK2_STAGES * A_BYTES;
    float* xup = reinterpret_cast<float*>(sB + PK2_STAGES * B_BYTES);  // [64][PK_EC + 1]
    bf16* ob = reinterpret_cast<bf16*>(xup + 64 * (PK_EC + 1));         // [PK_EC][64]
    uint64_t* full = reinterpret_cast<uint64_t*>(ob + PK_EC * 64);
    uint64_t* empty = full + PK2_STAGES;
    uint64_t* acc_full = empty + PK2_STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2] (rank 0's: 256 arrivals, both CTAs' epilogues)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = static_cast<int>(blockIdx.x) >> 1, n_pairs = static_cast<int>(gridDim.x) >> 1;
    const int mpt = (p.N + BM - 1) / BM / 2, nt = (p.T + PK_BN - 1) / PK_BN;  // weight-tile pairs, token tiles
    const int tiles = mpt * nt, nkb = p.kb_total;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int st = 0; st < PK2_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 256);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const uint32_t full0 = mapa_shared(smem_u32(full), 0);
            pdl_wait();
            int g = 0;
            for (int t = pair; t < tiles; t += n_pairs) {
                const int m0 = ((t / nt) * 2 + static_cast<int>(rank)) * BM;
                const int nb = (t % nt) * PK_BN + static_cast<int>(rank) * (PK_BN / 2);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % PK2_STAGES;
                    if (g >= PK2_STAGES) mbar_wait(&empty[st], ((g / PK2_STAGES) - 1) & 1);
                    if (rank == 0) mbar_expect_tx(&full[st], 2 * (A_BYTES + B_BYTES));
                    tma_load_2d_cg2(sA + st * A_BYTES, &tmW, full0 + st * 8, kb * BK, m0, pol_w);
                    tma_load_2d_cg2(sB + st * B_BYTES, &tmX, full0 + st * 8, kb * BK, nb, pol_x);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            pdl_wait();
            constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, PK_BN);
            int g = 0, i = 0;
            for (int t = pair; t < tiles; t += n_pairs, ++i) {
                const int b = i & 1;
                if (i >= 2) mbar_wait(&acc_empty[b], ((i >> 1) - 1) & 1);
                tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % PK2_STAGES;
                    mbar_wait(&full[st], (g / PK2_STAGES) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a_base = smem_u32(sA + st * A_BYTES);
                        const uint32_t b_base = smem_u32(sB + st * B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_bf16_cg2(tmem + b * PK_BN, umma_desc_sw128(a_base + k * 32),
                                          umma_desc_sw128(b_base + k * 32), idesc, (kb | k) != 0 ? 1u : 0u);
                        umma_commit_cg2_mc(&empty[st], 3);
                        if (kb == nkb - 1) umma_commit_cg2_mc(&acc_full[b], 3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        pdl_wait();
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;
        const uint32_t acc_empty0 = mapa_shared(smem_u32(acc_empty), 0);
        int i = 0;
        for (int t = pair; t < tiles; t += n_pairs, ++i) {
            const int b = i & 1;
            const int mtile = (t / nt) * 2 + static_cast<int>(rank), n0 = (t % nt) * PK_BN;
            mbar_wait(&acc_full[b], (i >> 1) & 1);
            tc_fence_after();
            for (int c0 = 0; c0 < PK_BN; c0 += PK_EC) {
                float v[PK_EC];
                tmem_ld32(tmem + b * PK_BN + c0 + (static_cast<uint32_t>(q * 32) << 16), v);
                if (c0 + PK_EC == PK_BN) {
                    tc_fence_before();
                    mbar_arrive_cluster(acc_empty0 + b * 8);
                }
                if (row >= 64) {
#pragma unroll
                    for (int j = 0; j < PK_EC; ++j) xup[(row - 64) * (PK_EC + 1) + j] = v[j];
                }
                named_bar(1, 128);
                if (row < 64) {
#pragma unroll
                    for (int j = 0; j < PK_EC; ++j) {
                        const float g = v[j], u = xup[row * (PK_EC + 1) + j];
                        ob[j * 64 + row] = f2bf(__fdividef(g, 1.0f + __expf(-g)) * u);
                    }
                }
                named_bar(1, 128);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int idx = et + k * 128, j = idx >> 3, c8 = (idx & 7) * 8;
                    const int n = n0 + c0 + j, f = mtile * 64 + c8;
                    if (n < p.T && f < p.N / 2)
                        *reinterpret_cast<uint4*>(static_cast<bf16*>(p.out) + static_cast<size_t>(n) * p.ldo + f) =
                            *reinterpret_cast<const uint4*>(ob + j * 64 + c8);
                }
                named_bar(1, 128);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2(tmem, 512);
    }
}

// The fp32-row prefill GEMMs (QKV / O / down partial rows) on persistent CTA
// pairs: the gate/up kernel's pipeline with the row epilogue — per 32-token
// chunk, TMEM -> registers -> smem [32 tokens][128 features] -> 512-byte row
// stores — drained while the next tile's MMAs run. Units are (split, weight
// pair, token tile), token tiles fastest.
constexpr size_t pr2_smem_bytes() {
    return 1024 + PK2_STAGES * (BM * BK * 2 + (PK_BN / 2) * BK * 2) + PK_EC * (BM + 4) * 4 +
           (2 * PK2_STAGES + 4) * 8 + 16;
}

__global__ void __launch_bounds__(192, 1)
    gemm_rows_pk2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = (PK_BN / 2) * BK * 2;
    constexpr int SO = BM + 4;  // padded staging row
    uint8_t* sA = smem;
    uint8_t* sB = smem + PK2_STAGES * A_BYTES;
    float* so = reinterpret_cast<float*>(sB + PK2_STAGES * B_BYTES);  // [PK_EC tokens][SO]
    uint64_t* full = reinterpret_cast<uint64_t*>(so + PK_EC * SO);
    uint64_t* empty = full + PK2_STAGES;
    uint64_t* acc_full = empty + PK2_STAGES;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = static_cast<int>(blockIdx.x) >> 1, n_pairs = static_cast<int>(gridDim.x) >> 1;
    const int mpt = (p.N + BM - 1) / BM / 2, nt = (p.T + PK_BN - 1) / PK_BN;
    const int per_split = mpt * nt;
    const int splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
    const int units = per_split * splits;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int st = 0; st < PK2_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 256);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    auto unit_of = [&](int u, int& m0, int& n0, int& z, int& kb0, int& nkb) {
        z = u / per_split;
        const int r = u % per_split;
        m0 = ((r / nt) * 2 + static_cast<int>(rank)) * BM;
        n0 = (r % nt) * PK_BN;
        kb0 = z * p.kb_per_split;
        nkb = min(p.kb_per_split, p.kb_total - kb0);
    };
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const uint32_t full0 = mapa_shared(smem_u32(full), 0);
            pdl_wait();
            int g = 0;
            for (int u = pair; u < units; u += n_pairs) {
                int m0, n0, z, kb0, nkb;
                unit_of(u, m0, n0, z, kb0, nkb);
                const int nb = n0 + static_cast<int>(rank) * (PK_BN / 2);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % PK2_STAGES;
                    if (g >= PK2_STAGES) mbar_wait(&empty[st], ((g / PK2_STAGES) - 1) & 1);
                    if (rank == 0) mbar_expect_tx(&full[st], 2 * (A_BYTES + B_BYTES));
                    tma_load_2d_cg2(sA + st * A_BYTES, &tmW, full0 + st * 8, (kb0 + kb) * BK, m0, pol_w);
                    tma_load_2d_cg2(sB + st * B_BYTES, &tmX, full0 + st * 8, (kb0 + kb) * BK, nb, pol_x);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            pdl_wait();
            constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, PK_BN);
            int g = 0, i = 0;
            for (int u = pair; u < units; u += n_pairs, ++i) {
                int m0, n0, z, kb0, nkb;
                unit_of(u, m0, n0, z, kb0, nkb);
                const int b = i & 1;
                if (i >= 2) mbar_wait(&acc_empty[b], ((i >> 1) - 1) & 1);
                tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % PK2_STAGES;
                    mbar_wait(&full[st], (g / PK2_STAGES) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a_base = smem_u32(sA + st * A_BYTES);
                        const uint32_t b_base = smem_u32(sB + st * B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_bf16_cg2(tmem + b * PK_BN, umma_desc_sw128(a_base + k * 32),
                                          umma_desc_sw128(b_base + k * 32), idesc, (kb | k) != 0 ? 1u : 0u);
                        umma_commit_cg2_mc(&empty[st], 3);
                        if (kb == nkb - 1) umma_commit_cg2_mc(&acc_full[b], 3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        pdl_wait();
        const int q = warp & 3;  // TMEM lane quarter of this warp
        const int row = q * 32 + lane;
        const int ew = warp - 2;  // 0..3: store warp index
        const uint32_t acc_empty0 = mapa_shared(smem_u32(acc_empty), 0);
        int i = 0;
        for (int u = pair; u < units; u += n_pairs, ++i) {
            int m0, n0, z, kb0, nkb;
            unit_of(u, m0, n0, z, kb0, nkb);
            const int b = i & 1;
            const bool m_ok = m0 + row < p.N;
            const float bias = (p.bias && m_ok && p.epi != kEpiPartial) ? bf2f(p.bias[m0 + row]) : 0.f;
            const bool full_m = m0 + BM <= p.N;
            mbar_wait(&acc_full[b], (i >> 1) & 1);
            tc_fence_after();
            for (int c0 = 0; c0 < PK_BN; c0 += PK_EC) {
                float v[PK_EC];
                tmem_ld32(tmem + b * PK_BN + c0 + (static_cast<uint32_t>(q * 32) << 16), v);
                if (c0 + PK_EC == PK_BN) {
                    tc_fence_before();
                    mbar_arrive_cluster(acc_empty0 + b * 8);
                }
#pragma unroll
                for (int j = 0; j < PK_EC; ++j) so[j * SO + row] = v[j] + bias;
                named_bar(1, 128);
                const int rows = min(PK_EC, p.T - n0 - c0);
                for (int r = ew; r < rows; r += 4) {
                    const int n = n0 + c0 + r;
                    const float4 w = reinterpret_cast<const float4*>(so + r * SO)[lane];
                    const int mm = m0 + lane * 4;
                    if (p.epi == kEpiPartial) {
                        float* dst = p.partial + (static_cast<size_t>(z) * p.T + n) * p.N + mm;
                        if (full_m) {
                            *reinterpret_cast<float4*>(dst) = w;
                        } else {
                            const float e[4] = {w.x, w.y, w.z, w.w};
                            for (int qq = 0; qq < 4; ++qq)
                                if (mm + qq < p.N) dst[qq] = e[qq];
                        }
                    } else {
                        const float e[4] = {w.x, w.y, w.z, w.w};
                        for (int qq = 0; qq < 4; ++qq) {
                            if (mm + qq >= p.N) break;
                            const size_t o = static_cast<size_t>(n) * p.ldo + mm + qq;
                            if (p.epi == kEpiStoreBf16)
                                static_cast<bf16*>(p.out)[o] = f2bf(e[qq]);
                            else if (p.epi == kEpiAddF32)
                                static_cast<float*>(p.out)[o] += e[qq];
                            else
                                static_cast<float*>(p.out)[o] = e[qq];
                        }
                    }
                }
                named_bar(1, 128);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2(tmem, 512);
    }
}

template <int BN, int STAGES>
constexpr size_t smem_bytes() {
    return 1024 + STAGES * (BM * BK * 2 + BN * BK * 2) + (2 * STAGES + 1) * 8 + 16;
}

template <int BN, int STAGES>
void launch_tc(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p, dim3 grid, cudaStream_t st) {
    static bool configured = false;
    constexpr size_t sm = smem_bytes<BN, STAGES>();
    if (!configured) {
        HK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm)));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p.cluster) {
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = 1;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = grid.z;
        cfg.numAttrs = 2;
    }
    HK_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES>, tw, tx, p));
    HK_LAUNCHED(1);
}

template <int STAGES>
void launch_tc2(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p, dim3 grid, cudaStream_t st) {
    static bool configured = false;
    constexpr size_t sm = smem2_bytes<STAGES>();
    if (!configured) {
        HK_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm)));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = sm;
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
    HK_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<STAGES>, tw, tx, p));
    HK_LAUNCHED(1);
}

}  // namespace

int g_num_sms = 148;
unsigned long long g_launches = 0;
bool g_pdl = true;

// HK_GEMM_TRACE=1 (debug; run with HK_NO_GRAPHS=1): every tcgen05 GEMM launch
// gets a slot recording its first CTA start, first griddepcontrol.wait exit
// and last CTA end (%globaltimer); hkx_gemm_trace_dump writes them out.
namespace {
struct GemmTrace {
    unsigned long long* d = nullptr;
    int n = 0, cap = 0;
    std::vector<std::array<int, 6>> meta;  // N, K, T, splits, grid CTAs, prefill rows of the step
};
GemmTrace g_gtrace;
}  // namespace

bool g_span_trace = std::getenv("HK_GEMM_TRACE") != nullptr;  // also hkx_span_trace(1)
int g_trace_prefill_rows = 0;

void span_trace_reset(bool on) {
    g_span_trace = on;
    g_gtrace.n = 0;
    g_gtrace.meta.clear();
    if (g_gtrace.d) HK_CUDA(cudaMemset(g_gtrace.d, 0xff, static_cast<size_t>(g_gtrace.cap) * 4 * 8));
}

unsigned long long* gemm_trace_slot(int N, int K, int T, int splits, int ctas) {
    if (!g_span_trace) return nullptr;
    if (!g_gtrace.d) {
        g_gtrace.cap = 1 << 18;
        HK_CUDA(cudaMalloc(&g_gtrace.d, static_cast<size_t>(g_gtrace.cap) * 4 * 8));
        HK_CUDA(cudaMemset(g_gtrace.d, 0xff, static_cast<size_t>(g_gtrace.cap) * 4 * 8));
    }
    if (g_gtrace.n >= g_gtrace.cap) return nullptr;
    g_gtrace.meta.push_back({N, K, T, splits, ctas, g_trace_prefill_rows});
    return g_gtrace.d + 4 * static_cast<size_t>(g_gtrace.n++);
}

int gemm_trace_dump(const char* path) {
    if (!g_gtrace.d) return 0;
    HK_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(static_cast<size_t>(g_gtrace.n) * 4);
    HK_CUDA(cudaMemcpy(h.data(), g_gtrace.d, h.size() * 8, cudaMemcpyDeviceToHost));
    FILE* f = std::fopen(path, "w");
    if (!f) return -1;
    std::fprintf(f, "slot,N,K,T,splits,ctas,start,wait_done,end,mainloop_end,prefill_rows\n");
    for (int i = 0; i < g_gtrace.n; ++i) {
        const auto& m = g_gtrace.meta[static_cast<size_t>(i)];
        std::fprintf(f, "%d,%d,%d,%d,%d,%d,%llu,%llu,%llu,%llu,%d\n", i, m[0], m[1], m[2], m[3], m[4], h[4 * i],
                     h[4 * i + 1], ~h[4 * i + 2], ~h[4 * i + 3], m[5]);
    }
    std::fclose(f);
    return g_gtrace.n;
}

int gemm_bf16(const bf16* W, const bf16* X, int N, int K, int T, int epi, void* out, int ldo, const bf16* bias,
              float* workspace, size_t workspace_floats, cudaStream_t st, int force_splits, int max_splits) {
    if (T <= 0) return 0;
    if (K % BK != 0) throw std::runtime_error("gemm_bf16: K must be a multiple of 64");
    // The LM head (1,002 vocab tiles, argmax epilogue) runs stream-K, one CTA
    // per SM (97% of HBM peak measured); the per-layer GEMMs keep split-K
    // partials reduced by their consumer row kernels, measured faster
    // (tools/gemm_sweep.py, profiles/r1_gemm_sweep.txt).
    const bool wide = (N + BM - 1) / BM >= g_num_sms;  // at least one whole wave of weight tiles
    static const bool sk_swiglu = std::getenv("HK_SK_SWIGLU") != nullptr;  // opt-in: slower on B200 (sweep)
    static const bool sk_all = std::getenv("HK_SK_ALL") != nullptr;        // experiments: every decode GEMM
    if (T <= 64 && (wide || sk_all) && (epi == kEpiArgmax || (sk_swiglu && epi == kEpiSwiGLU) || sk_all) &&
        force_splits == 0 &&
        bias == nullptr &&
        gemm_streamk_enabled()) {
        gemm_bf16_streamk(W, X, N, K, T, epi, out, ldo, st);
        return 1;  // fully reduced
    }
    int BN;
    if (T <= 16)
        BN = 16;
    else if (T <= 32)
        BN = 32;
    else if (T <= 64)
        BN = 64;
    else if (T <= 128)
        BN = 128;
    else
        BN = 256;
    const int mt = (N + BM - 1) / BM;
    const int nt = (T + BN - 1) / BN;
    const int kb = K / BK;
    int splits = 1;
    if (epi == kEpiSwiGLU || epi == kEpiArgmax) {
        splits = 1;  // epilogue needs the whole K reduction in TMEM
    } else if (force_splits > 0) {
        splits = force_splits;
    } else {
        // skinny (decode) GEMMs: split K across a thread-block cluster so that
        // ~2 CTAs per SM stream weights; reduced through DSMEM (<= 8 per cluster)
        const int slots = BN <= 64 ? 2 * g_num_sms : g_num_sms;
        if (mt * nt * 2 <= slots) splits = std::min(8, slots / (mt * nt));
        splits = std::min(splits, std::max(1, kb / 4));
    }
    splits = std::min(splits, std::max(1, max_splits));
    int kbps = (kb + splits - 1) / splits;
    splits = (kb + kbps - 1) / kbps;  // no empty splits
    // DSMEM cluster reduction is kept behind a switch: measured slower on B200
    // than L2-resident fp32 partials reduced by the consumer row kernel
    // (profiles/r1_gemm_sweep.txt), so partials are the default.
    static const bool use_cluster = std::getenv("HK_GEMM_CLUSTER") != nullptr;
    const bool cluster = splits > 1 && splits <= 8 && use_cluster;
    if (!cluster && epi != kEpiPartial && splits > 1 && static_cast<size_t>(splits) * T * N > workspace_floats) {
        splits = 1;
        kbps = kb;
    }
    const bool via_ws = splits > 1 && !cluster && epi != kEpiPartial;
    static const int skip_epi = std::getenv("HK_GEMM_DEBUG_SKIP_EPI") ? 1 : 0;
    GemmParams p{N, K, T, kb, kbps, via_ws ? kEpiPartial : epi, out, ldo, bias,
                 epi == kEpiPartial ? static_cast<float*>(out) : workspace, cluster ? 1 : 0, skip_epi};
    p.trace = gemm_trace_slot(N, K, T, splits, mt * nt * splits);
    const CUtensorMap tw = make_map_2d(W, static_cast<uint64_t>(N), static_cast<uint64_t>(K), BM);
    const CUtensorMap tx = make_map_2d(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), static_cast<uint32_t>(BN));
    // prefill tiles (256 tokens) on CTA pairs: two weight tiles per cluster
    // (HK_GEMM_CG2=0: one CTA per tile; HK_GEMM_CG2_SWIGLU=1: gate/up too, instead of the persistent kernel)
    static const bool cg2_off = std::getenv("HK_GEMM_CG2") && std::atoi(std::getenv("HK_GEMM_CG2")) == 0;
    static const bool cg2_swiglu = std::getenv("HK_GEMM_CG2_SWIGLU") && std::atoi(std::getenv("HK_GEMM_CG2_SWIGLU")) != 0;
    const bool use_cg2 = BN == 256 && !cg2_off && !cluster && mt % 2 == 0 && epi != kEpiArgmax && !p.skip_epi &&
                         (epi != kEpiSwiGLU || cg2_swiglu);
    static const bool pk_off = std::getenv("HK_GEMM_SWIGLU_PERSIST") && std::atoi(std::getenv("HK_GEMM_SWIGLU_PERSIST")) == 0;
    static const bool pk2_off = std::getenv("HK_GEMM_SWIGLU_PAIRS") && std::atoi(std::getenv("HK_GEMM_SWIGLU_PAIRS")) == 0;
    if (epi == kEpiSwiGLU && BN == 256 && !pk_off && !pk2_off && !cg2_off && !use_cg2 && N % (2 * BM) == 0 &&
        !p.skip_epi && g_num_sms >= 2) {
        // prefill gate/up: persistent CTA pairs
        static bool configured = false;
        constexpr size_t sm = pk2_smem_bytes();
        if (!configured) {
            HK_CUDA(cudaFuncSetAttribute(gemm_swiglu_pk2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm)));
            configured = true;
        }
        const CUtensorMap txh = make_map_2d(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), PK_BN / 2);
        const int pairs = std::min((mt / 2) * nt, g_num_sms / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = sm;
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
        HK_CUDA(cudaLaunchKernelEx(&cfg, gemm_swiglu_pk2_kernel, tw, txh, p));
        HK_LAUNCHED(1);
        return 1;
    }
    if (epi == kEpiSwiGLU && BN == 256 && !pk_off && !use_cg2 && N % BM == 0 && !p.skip_epi) {
        // prefill gate/up: persistent tiles, epilogue under the next tile's MMAs
        static bool configured = false;
        constexpr size_t sm = pk_smem_bytes();
        if (!configured) {
            HK_CUDA(cudaFuncSetAttribute(gemm_swiglu_pk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm)));
            configured = true;
        }
        const CUtensorMap txp = make_map_2d(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), PK_BN);
        launch_pdl(gemm_swiglu_pk_kernel, dim3(std::min(mt * nt, g_num_sms)), dim3(192), sm, st, tw, txp, p);
        HK_LAUNCHED(1);
        return 1;
    }
    static const bool pr2_off = std::getenv("HK_GEMM_ROWS_PERSIST") && std::atoi(std::getenv("HK_GEMM_ROWS_PERSIST")) == 0;
    if (use_cg2 && epi != kEpiSwiGLU && !pr2_off && (mt / 2) * nt * splits > g_num_sms / 2) {  // > one wave of pairs
        // prefill fp32-row GEMMs: persistent CTA pairs, epilogue under the next tile's MMAs
        static bool configured = false;
        constexpr size_t sm = pr2_smem_bytes();
        if (!configured) {
            HK_CUDA(cudaFuncSetAttribute(gemm_rows_pk2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm)));
            configured = true;
        }
        const CUtensorMap txh = make_map_2d(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), PK_BN / 2);
        const int pairs = std::min((mt / 2) * nt * splits, g_num_sms / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = sm;
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
        HK_CUDA(cudaLaunchKernelEx(&cfg, gemm_rows_pk2_kernel, tw, txh, p));
        HK_LAUNCHED(1);
        if (via_ws) {
            const size_t total = static_cast<size_t>(T) * N;
            const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 4096));
            splitk_reduce_kernel<<<blocks, 256, 0, st>>>(workspace, splits, T, N, epi, out, ldo, bias);
            HK_LAUNCHED(1);
        }
        return splits;
    }
    if (use_cg2) {
        const CUtensorMap txh = make_map_2d(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), C2_BN / 2);
        launch_tc2<6>(tw, txh, p, dim3(2 * nt, mt / 2, splits), st);
        if (via_ws) {
            const size_t total = static_cast<size_t>(T) * N;
            const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 4096));
            splitk_reduce_kernel<<<blocks, 256, 0, st>>>(workspace, splits, T, N, epi, out, ldo, bias);
            HK_LAUNCHED(1);
        }
        return splits;
    }
    static const bool wfirst = std::getenv("HK_GEMM_WEIGHT_TILE_FIRST") != nullptr;  // A/B: the old grid order
    p.tfirst = nt > 1 && !wfirst && !cluster ? 1 : 0;
    dim3 grid = p.tfirst ? dim3(nt, mt, splits) : dim3(mt, nt, splits);
    switch (BN) {
        case 16: launch_tc<16, 4>(tw, tx, p, grid, st); break;
        case 32: launch_tc<32, 4>(tw, tx, p, grid, st); break;
        case 64: launch_tc<64, 4>(tw, tx, p, grid, st); break;
        case 128: launch_tc<128, 4>(tw, tx, p, grid, st); break;
        default: launch_tc<256, 4>(tw, tx, p, grid, st); break;
    }
    if (cluster) splits = 1;  // the result is already reduced
    if (via_ws) {
        const size_t total = static_cast<size_t>(T) * N;
        const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 4096));
        splitk_reduce_kernel<<<blocks, 256, 0, st>>>(workspace, splits, T, N, epi, out, ldo, bias);
        HK_LAUNCHED(1);
    }
    return splits;
}

namespace {
__global__ void argmax_reduce_kernel(const float2* __restrict__ part, int n_tiles, int T, int32_t* ids,
                                     float* vals, const int32_t* slots, int32_t* slot_last) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
        const float2 v = part[static_cast<size_t>(i) * T + t];
        const int idx = __float_as_int(v.y);
        if (v.x > best || (v.x == best && idx < bi)) {
            best = v.x;
            bi = idx;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = best;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
                best = sv[w];
                bi = si[w];
            }
        if (bi == 0x7fffffff) bi = 0;  // all-NaN row: an in-range id (the embedding gather indexes with it)
        ids[t] = bi;
        if (vals) vals[t] = best;
        if (slots) slot_last[slots[t]] = bi;
    }
}
}  // namespace

void argmax_reduce(const float2* part, int n_tiles, int T, int32_t* ids, float* vals, const int32_t* slots,
                   int32_t* slot_last, cudaStream_t st) {
    if (T <= 0) return;
    launch_pdl(argmax_reduce_kernel, dim3(T), dim3(256), 0, st, part, n_tiles, T, ids, vals, slots, slot_last);
    HK_LAUNCHED(1);
}

void gemm_f32(const float* W, const float* X, int N, int K, int T, int epi, void* out, int ldo, const float* bias,
              cudaStream_t st) {
    if (T <= 0) return;
    dim3 grid((N + 31) / 32, (T + 31) / 32);
    gemm_f32_kernel<<<grid, 256, 0, st>>>(W, X, N, K, T, epi, out, ldo, bias);
    HK_LAUNCHED(1);
}

}  // namespace hkd
