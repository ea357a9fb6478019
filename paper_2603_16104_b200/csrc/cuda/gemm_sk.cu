// K4, decode shape: stream-K tcgen05 GEMM for skinny (T <= 64 tokens)
// weight-streaming contractions — QKV, O, gate/up (+SwiGLU), down, LM head
// (+argmax) of every decode iteration.
//
//   out[t][n] = sum_k X[t][k] * W[n][k]
//
// Work = (128-row weight tile, 64-wide k-block) units, 16 KB of weights each.
// Exactly one CTA per SM gets an equal contiguous range of units, so every
// SM streams the same number of weight bytes for the whole kernel (no wave
// quantisation, no tail) through an 8-deep TMA ring. A CTA's range crosses
// tile boundaries: each tile segment accumulates in one of two TMEM buffers
// (the epilogue of one segment overlaps the MMAs of the next). A tile split
// across CTAs is finished by its last-arriving CTA, which sums the fp32
// segment partials in k order (deterministic) and applies the epilogue.
//
// Warp roles (192 threads): 0 TMA producer, 1 MMA issuer, 2-5 epilogue
// (one TMEM lane quarter each: row = quarter * 32 + lane).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

constexpr int SK_BM = 128;
constexpr int SK_BK = 64;
constexpr int SK_THREADS = 192;

struct SkParams {
    int N, K, T;
    int kb;      // k-blocks per tile
    int mt;      // weight tiles
    int units;   // units of the stream-K region: (mt - dp_tiles) * kb
    int ctas;    // grid size
    int w;       // whole-tile waves before the stream-K region (tile c + q * ctas, q < w)
    int dp_tiles;
    int epi;
    void* out;
    int ldo;
    float* ws;          // [ctas][2 (head, tail)][BN][128] fp32 segment partials
    int32_t* counters;  // [mt] arrivals of split tiles (zero between launches)
};

__device__ __forceinline__ int sk_u0(int c, const SkParams& p) {
    return static_cast<int>(static_cast<long long>(c) * p.units / p.ctas);
}
// CTA whose unit range holds unit u
__device__ __forceinline__ int sk_cta_of(int u, const SkParams& p) {
    int c = static_cast<int>(static_cast<long long>(u) * p.ctas / p.units);
    while (c + 1 < p.ctas && sk_u0(c + 1, p) <= u) ++c;
    while (c > 0 && sk_u0(c, p) > u) --c;
    return c;
}
__device__ __forceinline__ int sk_arrive(int32_t* ctr) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    return old;
}

// Segment q of CTA c: the first w are whole tiles (data-parallel waves), the
// rest are the CTA's tile pieces of the stream-K region [u0, u1) (region-
// relative units; t_rel indexes region tiles).
struct SkSeg {
    int t;      // global tile
    int ka, kz; // k-block range [ka, kz) within the tile
    int t_rel;  // region tile (stream-K segments), -1 for whole tiles
};
__device__ __forceinline__ SkSeg sk_seg(int c, int q, int u0, int u1, int t_first, const SkParams& p) {
    if (q < p.w) return SkSeg{c + q * p.ctas, 0, p.kb, -1};
    const int tr = t_first + (q - p.w);
    return SkSeg{p.dp_tiles + tr, max(u0, tr * p.kb) - tr * p.kb, min(u1, (tr + 1) * p.kb) - tr * p.kb, tr};
}

template <int BN, int STAGES>
constexpr size_t sk_smem() {
    return 1024 + STAGES * (SK_BM * SK_BK * 2 + BN * SK_BK * 2) + 64 * (BN + 1) * 4 + 4 * BN * 8 + 256;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(SK_THREADS, 1)
    gemm_sk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, SkParams p) {
    constexpr int A_BYTES = SK_BM * SK_BK * 2;
    constexpr int B_BYTES = BN * SK_BK * 2;
    constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : 256));
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = sm;
    uint8_t* sB = sA + STAGES * A_BYTES;
    float* xs = reinterpret_cast<float*>(sB + STAGES * B_BYTES);        // [64][BN + 1] SwiGLU exchange
    float2* red = reinterpret_cast<float2*>(xs + 64 * (BN + 1));        // [4][BN] argmax exchange
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 4 * BN);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    int* flag = reinterpret_cast<int*>(tslot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int u0 = sk_u0(c, p), u1 = sk_u0(c + 1, p);
    const int t_first = u0 / p.kb, t_last = u1 > u0 ? (u1 - 1) / p.kb : t_first - 1;
    const int n_segs = p.w + (t_last - t_first + 1);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tslot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    pdl_trigger();  // the next kernel may launch and prefetch its own weights

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const int n = p.w * p.kb + (u1 - u0);
            auto unit = [&](int i, int& t, int& k) {  // i-th unit of this CTA -> (global tile, k-block)
                if (i < p.w * p.kb) {
                    t = c + (i / p.kb) * p.ctas;
                    k = i % p.kb;
                } else {
                    const int u = u0 + i - p.w * p.kb;
                    t = p.dp_tiles + u / p.kb;
                    k = u % p.kb;
                }
            };
            // Weights do not depend on the previous kernel: start streaming them
            // before waiting for the activations (PDL overlap).
            const int pre = min(STAGES, n);
            for (int i = 0; i < pre; ++i) {
                int t, k;
                unit(i, t, k);
                mbar_expect_tx(&full[i], A_BYTES + B_BYTES);
                tma_load_2d_hint(sA + i * A_BYTES, &tmW, &full[i], k * SK_BK, t * SK_BM, pol_w);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i) {
                int t, k;
                unit(i, t, k);
                tma_load_2d_hint(sB + i * B_BYTES, &tmX, &full[i], k * SK_BK, 0, pol_x);
            }
            for (int i = pre; i < n; ++i) {
                const int s = i % STAGES;
                int t, k;
                unit(i, t, k);
                mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
                mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                tma_load_2d_hint(sA + s * A_BYTES, &tmW, &full[s], k * SK_BK, t * SK_BM, pol_w);
                tma_load_2d_hint(sB + s * B_BYTES, &tmX, &full[s], k * SK_BK, 0, pol_x);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = umma_idesc_bf16(SK_BM, BN);
        int i = 0;
        for (int q = 0; q < n_segs; ++q) {
            const SkSeg sg = sk_seg(c, q, u0, u1, t_first, p);
            const int a = sg.ka, b = sg.kz;
            const int buf = q & 1;
            if (q >= 2) mbar_wait(&acc_empty[buf], ((q >> 1) - 1) & 1);
            tc_fence_after();
            for (int u = a; u < b; ++u, ++i) {
                const int s = i % STAGES;
                mbar_wait(&full[s], (i / STAGES) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                    const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
                    for (int k = 0; k < SK_BK / 16; ++k)
                        umma_bf16(tmem + buf * BN, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32),
                                  idesc, (u > a || k > 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                    if (u == b - 1) umma_commit(&acc_full[buf]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---- epilogue warps
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int etid = threadIdx.x - 64;  // 0..127
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        for (int q = 0; q < n_segs; ++q) {
            const SkSeg sg = sk_seg(c, q, u0, u1, t_first, p);
            const int t = sg.t;
            const int buf = q & 1;
            mbar_wait(&acc_full[buf], (q >> 1) & 1);
            tc_fence_after();
            float v[BN];
#pragma unroll
            for (int j = 0; j < BN; j += 32) {
                if constexpr (BN >= 32) {
                    float w[32];
                    tmem_ld32(t_lane + buf * BN + j, w);
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[j + e] = w[e];
                }
            }
            if constexpr (BN < 32) {
#pragma unroll
                for (int j = 0; j < BN; j += 8) {
                    float w[8];
                    tmem_ld8(t_lane + buf * BN + j, w);
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[j + e] = w[e];
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
            if (sg.ka != 0 || sg.kz != p.kb) {
                // split tile: park this segment, the last arriver sums all segments in k order
                const int tr = sg.t_rel;
                const int slot = tr == t_first ? 0 : 1;
                float* wsp = p.ws + (static_cast<size_t>(c) * 2 + slot) * BN * SK_BM;
#pragma unroll
                for (int j = 0; j < BN; ++j) wsp[j * SK_BM + row] = v[j];
                named_bar(1, 128);
                const int cf = sk_cta_of(tr * p.kb, p), cl = sk_cta_of((tr + 1) * p.kb - 1, p);
                if (etid == 0) *flag = sk_arrive(&p.counters[t]) == cl - cf;
                named_bar(1, 128);
                if (!*flag) continue;
#pragma unroll
                for (int j = 0; j < BN; ++j) v[j] = 0.f;
                for (int cc = cf; cc <= cl; ++cc) {
                    const int sl = (tr == sk_u0(cc, p) / p.kb) ? 0 : 1;
                    const float* src = p.ws + (static_cast<size_t>(cc) * 2 + sl) * BN * SK_BM;
#pragma unroll
                    for (int j = 0; j < BN; ++j) v[j] += __ldcg(src + j * SK_BM + row);
                }
                if (etid == 0) p.counters[t] = 0;
            }
            // ---- final epilogue of tile t
            const int m = t * SK_BM + row;
            const bool m_ok = m < p.N;
            if (p.epi == kEpiSwiGLU) {
                // rows 0-63 gate, 64-127 the matching up rows (interleaved weights)
                if (row >= 64) {
#pragma unroll
                    for (int j = 0; j < BN; ++j) xs[(row - 64) * (BN + 1) + j] = v[j];
                }
                named_bar(1, 128);
                if (row < 64 && m_ok) {
                    const int f = t * 64 + row;
#pragma unroll
                    for (int j = 0; j < BN; ++j)
                        if (j < p.T) {
                            const float g = v[j], u = xs[row * (BN + 1) + j];
                            static_cast<bf16*>(p.out)[static_cast<size_t>(j) * p.ldo + f] = f2bf(g / (1.0f + __expf(-g)) * u);
                        }
                }
                named_bar(1, 128);
            } else if (p.epi == kEpiArgmax) {
#pragma unroll
                for (int j = 0; j < BN; ++j) {
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
                    if (lane == 0) red[quarter * BN + j] = make_float2(best, __int_as_float(bi));
                }
                named_bar(1, 128);
                if (etid < BN && etid < p.T) {
                    float2 bb = red[etid];
                    for (int qq = 1; qq < 4; ++qq) {
                        const float2 o = red[qq * BN + etid];
                        if (o.x > bb.x) bb = o;  // earlier quarters hold lower rows: keep them on ties
                    }
                    reinterpret_cast<float2*>(p.out)[static_cast<size_t>(t) * p.T + etid] = bb;
                }
                named_bar(1, 128);
            } else if (m_ok) {
#pragma unroll
                for (int j = 0; j < BN; ++j) {
                    if (j >= p.T) break;
                    if (p.epi == kEpiStoreBf16)
                        static_cast<bf16*>(p.out)[static_cast<size_t>(j) * p.ldo + m] = f2bf(v[j]);
                    else if (p.epi == kEpiAddF32)
                        static_cast<float*>(p.out)[static_cast<size_t>(j) * p.ldo + m] += v[j];
                    else
                        static_cast<float*>(p.out)[static_cast<size_t>(j) * p.ldo + m] = v[j];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

struct SkBuffers {
    float* ws = nullptr;
    size_t ws_floats = 0;
    int32_t* counters = nullptr;
    int n_counters = 0;
};
SkBuffers g_sk;

template <int BN, int STAGES>
void launch_sk(const CUtensorMap& tw, const CUtensorMap& tx, const SkParams& p, cudaStream_t st) {
    static bool configured = false;
    constexpr size_t smem = sk_smem<BN, STAGES>();
    if (!configured) {
        HK_CUDA(cudaFuncSetAttribute(gemm_sk_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        configured = true;
    }
    launch_pdl(gemm_sk_kernel<BN, STAGES>, dim3(p.ctas), dim3(SK_THREADS), smem, st, tw, tx, p);
    HK_LAUNCHED(1);
}

}  // namespace

bool gemm_streamk_enabled() {
    static const bool off = std::getenv("HK_GEMM_NO_STREAMK") != nullptr;
    return !off;
}

void gemm_streamk_reserve(int max_tiles, int max_bn) {
    const size_t need_ws = static_cast<size_t>(g_num_sms) * 2 * max_bn * SK_BM;
    if (need_ws > g_sk.ws_floats) {
        cudaFree(g_sk.ws);
        HK_CUDA(cudaMalloc(&g_sk.ws, need_ws * sizeof(float)));
        g_sk.ws_floats = need_ws;
    }
    if (max_tiles > g_sk.n_counters) {
        cudaFree(g_sk.counters);
        HK_CUDA(cudaMalloc(&g_sk.counters, static_cast<size_t>(max_tiles) * sizeof(int32_t)));
        HK_CUDA(cudaMemset(g_sk.counters, 0, static_cast<size_t>(max_tiles) * sizeof(int32_t)));
        g_sk.n_counters = max_tiles;
    }
}

void gemm_bf16_streamk(const bf16* W, const bf16* X, int N, int K, int T, int epi, void* out, int ldo,
                       cudaStream_t st) {
    if (T <= 0) return;
    if (T > 64) throw std::runtime_error("gemm_bf16_streamk: T > 64");
    if (K % SK_BK != 0) throw std::runtime_error("gemm_bf16_streamk: K must be a multiple of 64");
    const int BN = T <= 16 ? 16 : (T <= 32 ? 32 : 64);
    SkParams p{};
    p.N = N;
    p.K = K;
    p.T = T;
    p.kb = K / SK_BK;
    p.mt = (N + SK_BM - 1) / SK_BM;
    static const int per_sm = std::getenv("HK_SK_CTAS_PER_SM") ? std::atoi(std::getenv("HK_SK_CTAS_PER_SM")) : 1;
    p.ctas = std::min(g_num_sms * per_sm, p.mt * p.kb);
    // whole-tile waves first (no fixups), stream-K only over the remainder
    // (opt-in: measured slower than pure stream-K on B200, profiles/r1_gemm_sweep.txt)
    static const bool hybrid = std::getenv("HK_SK_HYBRID") != nullptr;
    p.w = hybrid && p.mt >= p.ctas ? p.mt / p.ctas : 0;
    p.dp_tiles = p.w * p.ctas;
    p.units = (p.mt - p.dp_tiles) * p.kb;
    p.epi = epi;
    p.out = out;
    p.ldo = ldo;
    if (g_sk.n_counters < p.mt || g_sk.ws_floats < static_cast<size_t>(p.ctas) * 2 * BN * SK_BM)
        gemm_streamk_reserve(std::max(p.mt, 4096), 64 * per_sm);  // (never inside a graph capture: the first call is eager)
    p.ws = g_sk.ws;
    p.counters = g_sk.counters;
    const CUtensorMap tw = make_tmap_2d_bf16(W, static_cast<uint64_t>(N), static_cast<uint64_t>(K), SK_BK, SK_BM);
    const CUtensorMap tx = make_tmap_2d_bf16(X, static_cast<uint64_t>(T), static_cast<uint64_t>(K), SK_BK,
                                             static_cast<uint32_t>(BN));
    if (per_sm >= 2) {
        switch (BN) {
            case 16: launch_sk<16, 4>(tw, tx, p, st); break;
            case 32: launch_sk<32, 4>(tw, tx, p, st); break;
            default: launch_sk<64, 4>(tw, tx, p, st); break;
        }
    } else {
        switch (BN) {
            case 16: launch_sk<16, 8>(tw, tx, p, st); break;
            case 32: launch_sk<32, 8>(tw, tx, p, st); break;
            default: launch_sk<64, 8>(tw, tx, p, st); break;
        }
    }
}

}  // namespace hkd
