// K3a/K3b: paged attention over the KV block pool, as work items that each
// cover <= 16 query tokens x one GQA group x one page-aligned key range.
//
// The executor's step planner (engine.cu) turns a ragged batch into items:
//   * prefill chunks: 16 consecutive tokens of one call, causal, keys [0, pos]
//     -> written directly (part = -1);
//   * decode, prefix-shared part (K3b): 16 decode tokens of 16 different calls
//     that share a block-table prefix, keys = the shared pages only. The shared
//     KV is streamed once per 16 calls (and from L2 for the other row groups)
//     instead of once per call;
//   * decode, private part: one call's own suffix pages (single-token items);
//   * long ranges are split into key chunks.
// MMA rows are (token, q-head) pairs of one GQA group: row r -> token r / G,
// head r % G, so the G query heads that share a kv head share every K/V tile
// and a single decode token fills G of the 16 rows of one warp (not 1).
// Multi-token items run G warps with 64-key tiles; single-token items run one
// warp with 32-key tiles (7 CTAs/SM keep enough KV bytes in flight).
// Every partial keeps flash-style (m, l, unnormalised o) state in log2 units;
// attention_merge combines the partials of each (token, head). QK^T and PV run
// on tensor cores (mma.sync m16n8k16 bf16 -> f32), K/V tiles are staged with
// 16-byte cp.async into XOR-swizzled shared memory and read with ldmatrix.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

constexpr int HD = 128;
constexpr int BLK = 16;  // tokens per KV page (engine enforces block_tokens == 16)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
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
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// byte offset of 16B chunk `c` of key row `r` in a swizzled [TK][HD] bf16 tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * (HD * 2) + ((c ^ (r & 7)) << 4); }

// Stage keys [k0, k0 + TK) of one kv head (K and V) from their pages: each
// thread issues 16-byte cp.async for whole chunks; rows past kend zero-fill.
template <int TK>
__device__ __forceinline__ void load_tile(uint32_t sK, uint32_t sV, const bf16* __restrict__ kv,
                                          const int32_t* __restrict__ pages, int k0, int kend, size_t head_off,
                                          size_t page_stride, size_t kv_half) {
    const int nthr = blockDim.x;
#pragma unroll 4
    for (int c = threadIdx.x; c < TK * 32; c += nthr) {
        const int r = c >> 5;          // key row in tile
        const int isv = (c >> 4) & 1;  // K or V
        const int ch = c & 15;         // 16B chunk within the 256-byte row
        const int key = k0 + r;
        const bool valid = key < kend;
        const bf16* src = kv;
        if (valid)
            src = kv + static_cast<size_t>(pages[key >> 4]) * page_stride + isv * kv_half + head_off +
                  (key & (BLK - 1)) * HD + ch * 8;
        cp_async16((isv ? sV : sK) + swz(r, ch), src, valid);
    }
}

template <int TK, int STAGES>
__global__ void __launch_bounds__(256) attn_mma_kernel(AttnArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    pdl_trigger();
    pdl_wait();
    const AttnItem it = a.items[blockIdx.x];
    const int G = a.H / a.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int QKV = (a.H + 2 * a.Hkv) * HD;
    const bf16* qkv = static_cast<const bf16*>(a.qkv);
    const bf16* kv = static_cast<const bf16*>(a.kv_layer);
    const int32_t* pages = a.pages + it.ptab;
    const size_t kv_half = static_cast<size_t>(a.Hkv) * BLK * HD;
    const size_t page_stride = 2 * kv_half;
    const size_t head_off = static_cast<size_t>(it.kvh) * BLK * HD;

    constexpr uint32_t TILE = TK * HD * 2;
    const uint32_t sbase = smem_u32(smem);  // [stage][K|V] tiles

    const int n_tiles = it.kend > it.kbeg ? (it.kend - it.kbeg + TK - 1) / TK : 0;
    // STAGES-deep cp.async ring; one commit group per tile slot (possibly empty)
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < n_tiles)
            load_tile<TK>(sbase + s * 2 * TILE, sbase + s * 2 * TILE + TILE, kv, pages, it.kbeg + s * TK, it.kend,
                          head_off, page_stride, kv_half);
        cp_async_commit();
    }

    // rows of this warp: (token, head) pairs
    const int ra = warp * 16 + gid, rb = ra + 8;
    const int ta = ra / G, tb = rb / G;
    const int ha = it.kvh * G + ra % G, hb = it.kvh * G + rb % G;
    const bool va = ta < it.ntok, vb = tb < it.ntok;
    uint32_t qf[HD / 16][4];
    {
        const uint32_t* q0 = reinterpret_cast<const uint32_t*>(qkv + static_cast<size_t>(it.tok0 + ta) * QKV + ha * HD);
        const uint32_t* q1 = reinterpret_cast<const uint32_t*>(qkv + static_cast<size_t>(it.tok0 + tb) * QKV + hb * HD);
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            const int c = ks * 8 + tig;
            qf[ks][0] = va ? q0[c] : 0u;
            qf[ks][1] = vb ? q1[c] : 0u;
            qf[ks][2] = va ? q0[c + 4] : 0u;
            qf[ks][3] = vb ? q1[c + 4] : 0u;
        }
    }
    const int pos0 = va ? a.pos[it.tok0 + ta] : -1;
    const int pos1 = vb ? a.pos[it.tok0 + tb] : -1;
    const float sl2 = a.scale * kLog2e;

    float o[HD / 8][4];
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int ti = 0; ti < n_tiles; ++ti) {
        const uint32_t sK = sbase + (ti % STAGES) * 2 * TILE;
        const uint32_t sV = sK + TILE;
        const int nt = ti + STAGES - 1;
        if (nt < n_tiles) {
            const uint32_t nK = sbase + (nt % STAGES) * 2 * TILE;
            load_tile<TK>(nK, nK + TILE, kv, pages, it.kbeg + nt * TK, it.kend, head_off, page_stride, kv_half);
        }
        cp_async_commit();
        cp_async_wait<STAGES - 1>();
        __syncthreads();
        const int kt0 = it.kbeg + ti * TK;

        float s[TK / 8][4];
#pragma unroll
        for (int j = 0; j < TK / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
            for (int jn = 0; jn < TK / 16; ++jn) {
                const int mi = lane >> 3, rr = lane & 7;
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sK + swz(jn * 16 + (mi >> 1) * 8 + rr, ks * 2 + (mi & 1)), b0, b1, b2, b3);
                mma_bf16(s[2 * jn], qf[ks], b0, b1);
                mma_bf16(s[2 * jn + 1], qf[ks], b2, b3);
            }
        }
        const bool need_mask = it.causal || kt0 + TK > it.kend;
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int j = 0; j < TK / 8; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float x0 = s[j][e] * sl2, x1 = s[j][2 + e] * sl2;
                if (need_mask) {
                    const int key = kt0 + j * 8 + 2 * tig + e;
                    const bool ok = key < it.kend;
                    if (!(ok && (!it.causal || key <= pos0))) x0 = -INFINITY;
                    if (!(ok && (!it.causal || key <= pos1))) x1 = -INFINITY;
                }
                if (!va) x0 = -INFINITY;
                if (!vb) x1 = -INFINITY;
                s[j][e] = x0;
                s[j][2 + e] = x1;
                mx0 = fmaxf(mx0, x0);
                mx1 = fmaxf(mx1, x1);
            }
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float base0 = mn0 == -INFINITY ? 0.f : mn0;
        const float base1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = exp2f(m0 - base0), al1 = exp2f(m1 - base1);
        m0 = mn0;
        m1 = mn1;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int j = 0; j < TK / 8; ++j) {
            s[j][0] = exp2f(s[j][0] - base0);
            s[j][1] = exp2f(s[j][1] - base0);
            s[j][2] = exp2f(s[j][2] - base1);
            s[j][3] = exp2f(s[j][3] - base1);
            rs0 += s[j][0] + s[j][1];
            rs1 += s[j][2] + s[j][3];
        }
        l0 = l0 * al0 + rs0;
        l1 = l1 * al1 + rs1;
#pragma unroll
        for (int j = 0; j < HD / 8; ++j) {
            o[j][0] *= al0;
            o[j][1] *= al0;
            o[j][2] *= al1;
            o[j][3] *= al1;
        }
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks) {
            uint32_t pa[4];
            pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
            pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
            pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
            pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
            for (int jd = 0; jd < HD / 16; ++jd) {
                const int mi = lane >> 3, rr = lane & 7;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sV + swz(ks * 16 + (mi & 1) * 8 + rr, jd * 2 + (mi >> 1)), b0, b1, b2, b3);
                mma_bf16(o[2 * jd], pa, b0, b1);
                mma_bf16(o[2 * jd + 1], pa, b2, b3);
            }
        }
        __syncthreads();
    }

    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

    if (it.part < 0) {
        const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
        bf16* out = static_cast<bf16*>(a.out);
        bf16* oa = out + (static_cast<size_t>(it.tok0 + ta) * a.H + ha) * HD;
        bf16* ob = out + (static_cast<size_t>(it.tok0 + tb) * a.H + hb) * HD;
#pragma unroll
        for (int j = 0; j < HD / 8; ++j) {
            const int d = j * 8 + 2 * tig;
            if (va) *reinterpret_cast<uint32_t*>(oa + d) = pack_bf16(o[j][0] * i0, o[j][1] * i0);
            if (vb) *reinterpret_cast<uint32_t*>(ob + d) = pack_bf16(o[j][2] * i1, o[j][3] * i1);
        }
    } else {
        const size_t pa_ = (static_cast<size_t>(it.tok0 + ta - a.part_tok0) * a.H + ha) * a.max_parts + it.part;
        const size_t pb_ = (static_cast<size_t>(it.tok0 + tb - a.part_tok0) * a.H + hb) * a.max_parts + it.part;
#pragma unroll
        for (int j = 0; j < HD / 8; ++j) {
            const int d = j * 8 + 2 * tig;
            if (va) *reinterpret_cast<float2*>(a.part_o + pa_ * HD + d) = make_float2(o[j][0], o[j][1]);
            if (vb) *reinterpret_cast<float2*>(a.part_o + pb_ * HD + d) = make_float2(o[j][2], o[j][3]);
        }
        if (tig == 0) {
            if (va) a.part_ml[pa_] = make_float2(m0, l0);
            if (vb) a.part_ml[pb_] = make_float2(m1, l1);
        }
    }
}

// fp32 parity-mode attention (SIMT): one warp per (row, head) of an item.
__global__ void attn_simt_f32_kernel(AttnArgs a) {
    const AttnItem it = a.items[blockIdx.x];
    const int G = a.H / a.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int QKV = (a.H + 2 * a.Hkv) * HD;
    const float* qkv = static_cast<const float*>(a.qkv);
    const float* kv = static_cast<const float*>(a.kv_layer);
    const size_t head_stride = static_cast<size_t>(a.block) * HD;
    const float sl2 = a.scale * kLog2e;
    for (int job = warp; job < it.ntok * G; job += nw) {
        const int r = job / G, g = job % G;
        const int h = it.kvh * G + g;
        const int tok = it.tok0 + r;
        const int pos = a.pos[tok];
        float q[HD / 32], acc[HD / 32];
#pragma unroll
        for (int i = 0; i < HD / 32; ++i) {
            q[i] = qkv[static_cast<size_t>(tok) * QKV + h * HD + lane + 32 * i];
            acc[i] = 0.f;
        }
        float m = -INFINITY, l = 0.f;
        for (int key = it.kbeg; key < it.kend; ++key) {
            if (it.causal && key > pos) break;
            const int page = a.pages[it.ptab + key / a.block];
            const float* kp = kv + ((static_cast<size_t>(page) * 2 + 0) * a.Hkv + it.kvh) * head_stride +
                              static_cast<size_t>(key % a.block) * HD;
            const float* vp = kp + static_cast<size_t>(a.Hkv) * head_stride;
            float dot = 0.f;
#pragma unroll
            for (int i = 0; i < HD / 32; ++i) dot += q[i] * kp[lane + 32 * i];
            dot = warp_sum(dot) * sl2;
            const float mn = fmaxf(m, dot);
            const float al = exp2f(m - mn), p = exp2f(dot - mn);
            l = l * al + p;
#pragma unroll
            for (int i = 0; i < HD / 32; ++i) acc[i] = acc[i] * al + p * vp[lane + 32 * i];
            m = mn;
        }
        if (it.part < 0) {
            float* out = static_cast<float*>(a.out);
#pragma unroll
            for (int i = 0; i < HD / 32; ++i)
                out[(static_cast<size_t>(tok) * a.H + h) * HD + lane + 32 * i] = l > 0.f ? acc[i] / l : 0.f;
        } else {
            const size_t pi = (static_cast<size_t>(tok - a.part_tok0) * a.H + h) * a.max_parts + it.part;
#pragma unroll
            for (int i = 0; i < HD / 32; ++i) a.part_o[pi * HD + lane + 32 * i] = acc[i];
            if (lane == 0) a.part_ml[pi] = make_float2(m, l);
        }
    }
}

// out[t][h] = sum_k 2^(m_k - M) o_k / sum_k 2^(m_k - M) l_k ; one warp per (row, head)
__global__ void attn_merge_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                                  const int32_t* __restrict__ n_parts, int n_rows, int tok0, int H, int max_parts,
                                  void* out, bool f32) {
    pdl_trigger();
    pdl_wait();
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= n_rows * H) return;
    const int row = wid / H, h = wid % H;
    const int np = n_parts[row];
    const size_t base = (static_cast<size_t>(row) * H + h) * max_parts;
    float M = -INFINITY;
    for (int k = 0; k < np; ++k) M = fmaxf(M, part_ml[base + k].x);
    const float Mb = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < np; ++k) {
        const float2 ml = part_ml[base + k];
        const float w = exp2f(ml.x - Mb);
        L += w * ml.y;
        const float4 v = reinterpret_cast<const float4*>(part_o + (base + k) * HD)[lane];
        acc.x += w * v.x;
        acc.y += w * v.y;
        acc.z += w * v.z;
        acc.w += w * v.w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const size_t oi = (static_cast<size_t>(tok0 + row) * H + h) * HD + lane * 4;
    if (f32) {
        *reinterpret_cast<float4*>(static_cast<float*>(out) + oi) =
            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    } else {
        bf16* o = static_cast<bf16*>(out) + oi;
        *reinterpret_cast<uint2*>(o) =
            make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
    }
}

template <int TK, int STAGES>
void launch_mma(const AttnArgs& a, int warps, cudaStream_t st) {
    constexpr int smem = STAGES * 2 * TK * HD * 2;  // STAGES x (K + V)
    static bool configured = false;
    if (!configured) {
        HK_CUDA(cudaFuncSetAttribute(attn_mma_kernel<TK, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured = true;
    }
    launch_pdl(attn_mma_kernel<TK, STAGES>, dim3(a.n_items), dim3(warps * 32), smem, st, a);
}

}  // namespace

void attention_partial(const AttnArgs& a, cudaStream_t st) {
    if (a.n_items == 0) return;
    const int G = a.H / a.Hkv;
    if (a.f32) {
        attn_simt_f32_kernel<<<a.n_items, 128, 0, st>>>(a);
    } else {
        if (a.block != BLK) throw std::runtime_error("attention: KV page size must be 16 tokens");
        if (G > 16) throw std::runtime_error("attention: GQA group > 16 unsupported");
        if (a.single)
            launch_mma<32, 3>(a, (G + 15) / 16, st);  // 48 KB: 4 CTAs/SM
        else
            launch_mma<64, 4>(a, G, st);              // 128 KB: deep ring for long shared ranges
    }
    HK_LAUNCHED(1);
}

void attention_merge(const float* part_o, const float2* part_ml, const int32_t* n_parts, int n_rows, int tok0, int H,
                     int hd, int max_parts, void* out, bool f32, cudaStream_t st) {
    if (n_rows == 0) return;
    if (hd != HD) throw std::runtime_error("attention: head_dim must be 128");
    const int warps = n_rows * H;
    launch_pdl(attn_merge_kernel, dim3((warps + 7) / 8), dim3(256), 0, st, part_o, part_ml, n_parts, n_rows, tok0, H,
               max_parts, out, f32);
    HK_LAUNCHED(1);
}

}  // namespace hkd
