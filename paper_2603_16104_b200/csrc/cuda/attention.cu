// fp32 parity-mode paged attention (the bf16 path is the tensor-core
// decode_attention kernel in decode_attn.cu, which also runs causal prefill).
//
// The engine's step planner (engine.cu) turns an fp32 step into work items
// that each cover <= 16 query tokens x one kv head x one page-aligned key
// range: prefill chunks (16 consecutive tokens of one call, causal, written
// directly, part = -1), the prefix-shared part of decode tokens that share a
// block-table prefix, and each decode token's private pages; long ranges are
// split into key chunks. Every partial keeps flash-style (m, l, unnormalised o)
// state in log2 units; attention_merge combines the partials of each
// (token, head). Plain fp32 SIMT arithmetic: this path exists for the 1e-5
// parity mode (tests/test_gpu_parity.py), not for speed.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

constexpr int HD = 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
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

}  // namespace

void attention_partial(const AttnArgs& a, cudaStream_t st) {
    if (a.n_items == 0) return;
    if (!a.f32) throw std::runtime_error("attention_partial: fp32 parity path only (bf16 runs decode_attention)");
    attn_simt_f32_kernel<<<a.n_items, 128, 0, st>>>(a);
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
