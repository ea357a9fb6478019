// K5: row-wise ops of the decoder (embedding gather, RMSNorm, RoPE + paged KV
// write, SwiGLU, greedy argmax) and the counter-based weight init.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// w[i] = scale * u,  u = (splitmix64(seed*C1 + tid*C2 + i) >> 40) * 2^-23 - 1   in [-1, 1)
__global__ void init_uniform_kernel(void* w, bool f32, size_t n, uint64_t seed, uint64_t tid, float scale) {
    const uint64_t base = seed * 0xd1b54a32d192ed03ull + tid * 0x9e3779b97f4a7c15ull;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix64(base + i);
        const float u = static_cast<float>(static_cast<uint32_t>(h >> 40)) * (1.0f / 8388608.0f) - 1.0f;
        const float v = __fmul_rn(u, scale);
        if (f32)
            static_cast<float*>(w)[i] = v;
        else
            static_cast<bf16*>(w)[i] = __float2bfloat16_rn(v);
    }
}

__global__ void fill_kernel(void* w, bool f32, size_t n, float v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (f32)
            static_cast<float*>(w)[i] = v;
        else
            static_cast<bf16*>(w)[i] = __float2bfloat16_rn(v);
    }
}

__global__ void embed_kernel(const void* table, bool f32, int d, const int32_t* ids, const int32_t* slots,
                             const int32_t* slot_last, float* x) {
    const int t = blockIdx.x;
    int id = ids[t];
    if (id < 0) id = slot_last[slots[t]];
    float* xr = x + static_cast<size_t>(t) * d;
    if (f32) {
        const float* row = static_cast<const float*>(table) + static_cast<size_t>(id) * d;
        for (int i = threadIdx.x; i < d; i += blockDim.x) xr[i] = row[i];
    } else {
        const bf16* row = static_cast<const bf16*>(table) + static_cast<size_t>(id) * d;
        for (int i = threadIdx.x; i < d; i += blockDim.x) xr[i] = bf2f(row[i]);
    }
}

__global__ void rmsnorm_kernel(const float* x, const void* w, bool f32, int d, float eps, const int32_t* rows,
                               void* out) {
    const int r = blockIdx.x;
    const int src = rows ? rows[r] : r;
    const float* xr = x + static_cast<size_t>(src) * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
    __shared__ float red[32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / static_cast<float>(d) + eps);
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        if (f32) {
            static_cast<float*>(out)[static_cast<size_t>(r) * d + i] = xr[i] * inv * static_cast<const float*>(w)[i];
        } else {
            const float wv = bf2f(static_cast<const bf16*>(w)[i]);
            static_cast<bf16*>(out)[static_cast<size_t>(r) * d + i] = f2bf(xr[i] * inv * wv);
        }
    }
}

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld<bf16>(const bf16* p) { return bf2f(*p); }
template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ bf16 cvt<bf16>(float v) { return f2bf(v); }

template <typename T>
__global__ void rope_kv_kernel(RopeArgs a) {
    const int t = blockIdx.x;
    const int pos = a.pos[t];
    const int half = a.hd / 2;
    const int nh = a.H + a.Hkv;  // rotated heads (q then k)
    T* row = static_cast<T*>(a.qkv) + static_cast<size_t>(t) * (a.H + 2 * a.Hkv) * a.hd;
    const float2* rp = a.rope + static_cast<size_t>(pos) * half;
    const bool write = a.kvw[t] != 0;
    int page = 0;
    if (write) page = a.pages[a.ptab[t] + pos / a.block];
    const size_t head_stride = static_cast<size_t>(a.block) * a.hd;
    T* kv = static_cast<T*>(a.kv_layer);
    for (int j = threadIdx.x; j < nh * half; j += blockDim.x) {
        const int hh = j / half, i = j % half;
        T* x = row + hh * a.hd;
        const float x1 = ld(x + i), x2 = ld(x + i + half);
        const float2 cs = rp[i];
        const float o1 = x1 * cs.x - x2 * cs.y;
        const float o2 = x2 * cs.x + x1 * cs.y;
        const T q1 = cvt<T>(o1), q2 = cvt<T>(o2);
        x[i] = q1;
        x[i + half] = q2;
        if (write && hh >= a.H) {
            const int kh = hh - a.H;
            T* kd = kv + ((static_cast<size_t>(page) * 2 + 0) * a.Hkv + kh) * head_stride +
                    static_cast<size_t>(pos % a.block) * a.hd;
            kd[i] = q1;
            kd[i + half] = q2;
        }
    }
    if (write) {
        for (int j = threadIdx.x; j < a.Hkv * a.hd; j += blockDim.x) {
            const int kh = j / a.hd, i = j % a.hd;
            T* vd = kv + ((static_cast<size_t>(page) * 2 + 1) * a.Hkv + kh) * head_stride +
                    static_cast<size_t>(pos % a.block) * a.hd;
            vd[i] = row[(a.H + a.Hkv + kh) * a.hd + i];
        }
    }
}

template <typename T>
__global__ void swiglu_kernel(const T* gu, int F, T* out) {
    const int t = blockIdx.x;
    const T* g = gu + static_cast<size_t>(t) * 2 * F;
    const T* u = g + F;
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
        const float gv = ld(g + i);
        const float s = gv / (1.0f + expf(-gv));
        out[static_cast<size_t>(t) * F + i] = cvt<T>(s * ld(u + i));
    }
}

__global__ void argmax_kernel(const float* logits, int V, int32_t* ids, float* vals, const int32_t* slots,
                              int32_t* slot_last) {
    const int r = blockIdx.x;
    const float* row = logits + static_cast<size_t>(r) * V;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const float v = row[i];
        if (v > best || (v == best && i < bi)) {
            best = v;
            bi = i;
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
        ids[r] = bi;
        if (vals) vals[r] = best;
        if (slots) slot_last[slots[r]] = bi;
    }
}

int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

__global__ void init_gu_kernel(void* w, bool f32, int F, int d, uint64_t seed, uint64_t tid, float scale) {
    const uint64_t base = seed * 0xd1b54a32d192ed03ull + tid * 0x9e3779b97f4a7c15ull;
    const size_t n = static_cast<size_t>(2) * F * d;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t p = i / d, col = i % d;
        const size_t tile = p / 128, r = p % 128;
        const size_t lrow = r < 64 ? tile * 64 + r : static_cast<size_t>(F) + tile * 64 + (r - 64);
        const uint64_t h = splitmix64(base + lrow * d + col);
        const float u = static_cast<float>(static_cast<uint32_t>(h >> 40)) * (1.0f / 8388608.0f) - 1.0f;
        const float v = __fmul_rn(u, scale);
        if (f32)
            static_cast<float*>(w)[i] = v;
        else
            static_cast<bf16*>(w)[i] = __float2bfloat16_rn(v);
    }
}

__global__ void swiglu_interleaved_kernel(const float* __restrict__ gu, int F, float* __restrict__ out) {
    const int t = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    const size_t col = static_cast<size_t>(f / 64) * 128 + f % 64;
    const float g = gu[static_cast<size_t>(t) * 2 * F + col];
    const float u = gu[static_cast<size_t>(t) * 2 * F + col + 64];
    out[static_cast<size_t>(t) * F + f] = g / (1.0f + expf(-g)) * u;
}

// One thread per rotated pair (q and k heads) or per value pair (v heads).
template <typename T>
__global__ void qkv_rope_kv_kernel(QkvArgs a) {
    pdl_trigger();
    // everything but the split-K partials (step metadata, page ids, RoPE
    // table, bias) is loaded before griddepcontrol.wait: only the partial
    // loads remain on the critical path after the QKV GEMM
    const RopeArgs& r = a.r;
    const int t = blockIdx.y;
    const int half = r.hd / 2;
    const int n_rot = (r.H + r.Hkv) * half;   // (i, i + half) pairs of q and k heads
    const int n_v = r.Hkv * half;             // v handled as (2j, 2j + 1) pairs
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_rot + n_v) return;
    const int QKV = (r.H + 2 * r.Hkv) * r.hd;
    const size_t tstride = static_cast<size_t>(r.T) * QKV;
    const float* src = a.part + static_cast<size_t>(t) * QKV;
    const int pos = r.pos[t];
    const bool write = r.kvw[t] != 0;
    T* row = static_cast<T*>(r.qkv) + static_cast<size_t>(t) * QKV;
    T* kv = static_cast<T*>(r.kv_layer);
    const size_t head_stride = static_cast<size_t>(r.block) * r.hd;
    int page = 0;
    if (write) page = r.pages[r.ptab[t] + pos / r.block];
    int c0, c1;
    if (j < n_rot) {
        const int hh = j / half, i = j % half;
        c0 = hh * r.hd + i;
        c1 = c0 + half;
    } else {
        const int jj = j - n_rot;
        c0 = (r.H + r.Hkv) * r.hd + 2 * jj;
        c1 = c0 + 1;
    }
    float b0 = 0.f, b1 = 0.f;
    if (a.bias) {
        if (sizeof(T) == 4) {
            b0 = static_cast<const float*>(a.bias)[c0];
            b1 = static_cast<const float*>(a.bias)[c1];
        } else {
            b0 = bf2f(static_cast<const bf16*>(a.bias)[c0]);
            b1 = bf2f(static_cast<const bf16*>(a.bias)[c1]);
        }
    }
    const float2 cs = j < n_rot ? r.rope[static_cast<size_t>(pos) * half + (j % half)] : make_float2(1.f, 0.f);
    pdl_wait();
    float x0 = 0.f, x1 = 0.f;
    for (int s0 = 0; s0 < a.splits; s0 += 8) {
        float p0[8], p1[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const bool ok = s0 + s < a.splits;
            p0[s] = ok ? __ldcg(src + (s0 + s) * tstride + c0) : 0.f;
            p1[s] = ok ? __ldcg(src + (s0 + s) * tstride + c1) : 0.f;
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {  // fixed split order: deterministic
            x0 += p0[s];
            x1 += p1[s];
        }
    }
    if (a.bias) {
        x0 += b0;
        x1 += b1;
    }
    if (j < n_rot) {
        // round to the storage type first: the oracle rotates the stored (bf16) qkv
        const T s0 = cvt<T>(x0), s1 = cvt<T>(x1);
        x0 = ld(&s0);
        x1 = ld(&s1);
        const int i = (j % half);
        const float o1 = x0 * cs.x - x1 * cs.y;
        const float o2 = x1 * cs.x + x0 * cs.y;
        const T q1 = cvt<T>(o1), q2 = cvt<T>(o2);
        row[c0] = q1;
        row[c1] = q2;
        const int hh = j / half;
        if (write && hh >= r.H) {
            T* kd = kv + ((static_cast<size_t>(page) * 2 + 0) * r.Hkv + (hh - r.H)) * head_stride +
                    static_cast<size_t>(pos % r.block) * r.hd;
            kd[i] = q1;
            kd[i + half] = q2;
        }
    } else {
        const T v0 = cvt<T>(x0), v1 = cvt<T>(x1);
        row[c0] = v0;
        row[c1] = v1;
        if (write) {
            const int vc = c0 - (r.H + r.Hkv) * r.hd;
            T* vd = kv + ((static_cast<size_t>(page) * 2 + 1) * r.Hkv + vc / r.hd) * head_stride +
                    static_cast<size_t>(pos % r.block) * r.hd + vc % r.hd;
            vd[0] = v0;
            vd[1] = v1;
        }
    }
}

// bf16 path, vectorised: a thread owns 4 rotated pairs of a q / k head (dims
// i..i+3 and i+64..i+67: one float4 of each half per split) or 8 values of a v
// head, so the split-K partials come in as 16-byte loads and q / K / V go out
// as 8- / 16-byte stores. Per element the arithmetic (split order, bias,
// bf16 rounding before the rotation) is the scalar kernel's.
__device__ __forceinline__ uint2 pack_bf16x4(float a, float b, float c, float d) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&lo);
    u.y = *reinterpret_cast<const uint32_t*>(&hi);
    return u;
}
__global__ void qkv_rope_kv4_kernel(QkvArgs a) {
    pdl_trigger();
    const RopeArgs& r = a.r;
    const int t = blockIdx.y;
    const int half = r.hd / 2;                 // 64
    const int n_rot = (r.H + r.Hkv) * (half / 4);
    const int n_v = r.Hkv * (r.hd / 8);
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_rot + n_v) return;
    const int QKV = (r.H + 2 * r.Hkv) * r.hd;
    const size_t tstride = static_cast<size_t>(r.T) * QKV;
    const float* src = a.part + static_cast<size_t>(t) * QKV;
    const int pos = r.pos[t];
    const bool write = r.kvw[t] != 0;
    bf16* row = static_cast<bf16*>(r.qkv) + static_cast<size_t>(t) * QKV;
    bf16* kv = static_cast<bf16*>(r.kv_layer);
    const size_t head_stride = static_cast<size_t>(r.block) * r.hd;
    const int page = write ? r.pages[r.ptab[t] + pos / r.block] : 0;
    const bf16* bias = static_cast<const bf16*>(a.bias);
    const bool rot = u < n_rot;
    const int hh = rot ? u / (half / 4) : 0;
    const int i = rot ? (u % (half / 4)) * 4 : 0;
    const int c0 = rot ? hh * r.hd + i : (r.H + r.Hkv) * r.hd + (u - n_rot) * 8;
    const int c1 = rot ? c0 + half : c0 + 4;
    float b[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (bias)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            b[e] = bf2f(bias[c0 + e]);
            b[4 + e] = bf2f(bias[c1 + e]);
        }
    float2 cs[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cs[e] = rot ? r.rope[static_cast<size_t>(pos) * half + i + e] : make_float2(1.f, 0.f);
    pdl_wait();
    float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < a.splits; s0 += 4) {
        float4 p0[4], p1[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const bool ok = s0 + s < a.splits;
            const float* base = src + static_cast<size_t>(s0 + s) * tstride;
            p0[s] = ok ? __ldcg(reinterpret_cast<const float4*>(base + c0)) : make_float4(0.f, 0.f, 0.f, 0.f);
            p1[s] = ok ? __ldcg(reinterpret_cast<const float4*>(base + c1)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {  // fixed split order: deterministic
            x[0] += p0[s].x;
            x[1] += p0[s].y;
            x[2] += p0[s].z;
            x[3] += p0[s].w;
            x[4] += p1[s].x;
            x[5] += p1[s].y;
            x[6] += p1[s].z;
            x[7] += p1[s].w;
        }
    }
    if (bias)
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] += b[e];
    float o[8];
    if (rot) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            // round to bf16 first: the oracle rotates the stored qkv
            const float x0 = bf2f(f2bf(x[e])), x1 = bf2f(f2bf(x[4 + e]));
            o[e] = x0 * cs[e].x - x1 * cs[e].y;
            o[4 + e] = x1 * cs[e].x + x0 * cs[e].y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = x[e];
    }
    const uint2 lo = pack_bf16x4(o[0], o[1], o[2], o[3]), hi = pack_bf16x4(o[4], o[5], o[6], o[7]);
    *reinterpret_cast<uint2*>(row + c0) = lo;
    *reinterpret_cast<uint2*>(row + c1) = hi;
    if (!write) return;
    if (rot && hh >= r.H) {
        bf16* kd = kv + ((static_cast<size_t>(page) * 2 + 0) * r.Hkv + (hh - r.H)) * head_stride +
                   static_cast<size_t>(pos % r.block) * r.hd;
        *reinterpret_cast<uint2*>(kd + i) = lo;
        *reinterpret_cast<uint2*>(kd + i + half) = hi;
    } else if (!rot) {
        const int vc = c0 - (r.H + r.Hkv) * r.hd;
        bf16* vd = kv + ((static_cast<size_t>(page) * 2 + 1) * r.Hkv + vc / r.hd) * head_stride +
                   static_cast<size_t>(pos % r.block) * r.hd + vc % r.hd;
        *reinterpret_cast<uint4*>(vd) = make_uint4(lo.x, lo.y, hi.x, hi.y);
    }
}

// Row kernel spread over a thread-block cluster: the RS CTAs of cluster
// (token t) each own d / RS consecutive features (one float4 per thread),
// load the residual and every split-K partial with all loads in flight, and
// exchange their partial sums of squares through distributed shared memory.
constexpr int kRowSplit = 8;
template <typename T>
__global__ void __launch_bounds__(256) add_rmsnorm_kernel(const float* __restrict__ part, int splits, float* x,
                                                          const T* __restrict__ w, int T_, int d, float eps, T* h,
                                                          const int32_t* __restrict__ cmap, T* hc) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x;
    const int n4 = d / 4;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;  // float4 index within the row
    const bool ok = i < n4;
    float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(t) * d);
    const size_t pstride = static_cast<size_t>(T_) * d / 4;
    const float4* pr = reinterpret_cast<const float4*>(part) + static_cast<size_t>(t) * d / 4;
    float4 v = ok ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < splits; s0 += 8) {
        float4 b[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
            b[s] = (ok && s0 + s < splits) ? __ldcg(pr + (s0 + s) * pstride + i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int s = 0; s < 8; ++s) {  // fixed split order: deterministic
            v.x += b[s].x;
            v.y += b[s].y;
            v.z += b[s].z;
            v.w += b[s].w;
        }
    }
    float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    __shared__ float red[8];
    __shared__ float cta_sum;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f;
        for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) a += red[k];
        cta_sum = a;
    }
    cluster_sync_all();
    float tot = 0.f;
    {
        float pv[kRowSplit];
#pragma unroll
        for (int q = 0; q < kRowSplit; ++q) pv[q] = ld_dsmem_f32(mapa_shared(smem_u32(&cta_sum), q));
#pragma unroll
        for (int q = 0; q < kRowSplit; ++q) tot += pv[q];  // rank order: every CTA gets the same total
    }
    const float inv = rsqrtf(tot / static_cast<float>(d) + eps);
    const int cr = cmap ? cmap[t] : -1;
    if (ok) {
        if (splits > 0) xr[i] = v;
        const float o0 = v.x * inv * ld(w + 4 * i), o1 = v.y * inv * ld(w + 4 * i + 1),
                    o2 = v.z * inv * ld(w + 4 * i + 2), o3 = v.w * inv * ld(w + 4 * i + 3);
        T* hr = h + static_cast<size_t>(t) * d + 4 * i;
        if constexpr (sizeof(T) == 2) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(o0, o1), hi = __floats2bfloat162_rn(o2, o3);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(hr) = pk;
            if (cr >= 0) *reinterpret_cast<uint2*>(hc + static_cast<size_t>(cr) * d + 4 * i) = pk;
        } else {
            *reinterpret_cast<float4*>(hr) = make_float4(o0, o1, o2, o3);
            if (cr >= 0) *reinterpret_cast<float4*>(hc + static_cast<size_t>(cr) * d + 4 * i) = make_float4(o0, o1, o2, o3);
        }
    }
    cluster_sync_all();  // peers read cta_sum: keep it alive until everyone has
}

// bf16 path: one CTA per row (no cluster barriers / DSMEM round trips), up
// to 1024 threads x VPT float4; the norm weights are loaded before
// griddepcontrol.wait. Same split order for x as add_rmsnorm_kernel.
template <int VPT>
__global__ void __launch_bounds__(1024) add_rmsnorm_row_kernel(const float* __restrict__ part, int splits, float* x,
                                                               const bf16* __restrict__ w, int T_, int d, float eps,
                                                               bf16* h, const int32_t* __restrict__ cmap, bf16* hc) {
    pdl_trigger();
    const int t = blockIdx.x;
    const int n4 = d / 4;
    uint2 wv[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int i = threadIdx.x + j * blockDim.x;
        wv[j] = i < n4 ? __ldg(reinterpret_cast<const uint2*>(w) + i) : make_uint2(0u, 0u);
    }
    pdl_wait();
    float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(t) * d);
    const size_t pstride = static_cast<size_t>(T_) * d / 4;
    const float4* pr = reinterpret_cast<const float4*>(part) + static_cast<size_t>(t) * d / 4;
    float4 v[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int i = threadIdx.x + j * blockDim.x;
        v[j] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int s0 = 0; s0 < splits; s0 += 8) {
        float4 b[VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int i = threadIdx.x + j * blockDim.x;
#pragma unroll
            for (int s = 0; s < 8; ++s)
                b[j][s] = (i < n4 && s0 + s < splits) ? __ldcg(pr + (s0 + s) * pstride + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < VPT; ++j)
#pragma unroll
            for (int s = 0; s < 8; ++s) {  // fixed split order: deterministic
                v[j].x += b[j][s].x;
                v[j].y += b[j][s].y;
                v[j].z += b[j][s].z;
                v[j].w += b[j][s].w;
            }
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
    __shared__ float red[32];
    __shared__ float tot_s;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        a = warp_sum(a);
        if (threadIdx.x == 0) tot_s = a;
    }
    __syncthreads();
    const float inv = rsqrtf(tot_s / static_cast<float>(d) + eps);
    const int cr = cmap ? cmap[t] : -1;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int i = threadIdx.x + j * blockDim.x;
        if (i >= n4) continue;
        if (splits > 0) xr[i] = v[j];
        const __nv_bfloat162 w01 = *reinterpret_cast<const __nv_bfloat162*>(&wv[j].x);
        const __nv_bfloat162 w23 = *reinterpret_cast<const __nv_bfloat162*>(&wv[j].y);
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v[j].x * inv * __low2float(w01), v[j].y * inv * __high2float(w01));
        const __nv_bfloat162 hi = __floats2bfloat162_rn(v[j].z * inv * __low2float(w23), v[j].w * inv * __high2float(w23));
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(h + static_cast<size_t>(t) * d + 4 * i) = pk;
        if (cr >= 0) *reinterpret_cast<uint2*>(hc + static_cast<size_t>(cr) * d + 4 * i) = pk;
    }
}

}  // namespace

void init_uniform_gu(void* w, bool f32, int F, int d, uint64_t seed, uint64_t tensor_id, float scale, cudaStream_t st) {
    init_gu_kernel<<<grid_for(static_cast<size_t>(2) * F * d), 256, 0, st>>>(w, f32, F, d, seed, tensor_id, scale);
    HK_LAUNCHED(1);
}

void swiglu_interleaved(const float* gu, int T, int F, float* out, cudaStream_t st) {
    if (!T) return;
    swiglu_interleaved_kernel<<<dim3((F + 255) / 256, T), 256, 0, st>>>(gu, F, out);
    HK_LAUNCHED(1);
}

void qkv_rope_kv(const QkvArgs& a, cudaStream_t st) {
    if (!a.r.T) return;
    const int half = a.r.hd / 2;
    const int n = (a.r.H + a.r.Hkv) * half + a.r.Hkv * half;
    dim3 grid((n + 255) / 256, a.r.T);
    static const bool scalar = std::getenv("HK_ROPE_SCALAR") != nullptr;  // A/B: the one-pair-per-thread kernel
    if (a.r.f32)
        launch_pdl(qkv_rope_kv_kernel<float>, grid, dim3(256), 0, st, a);
    else if (!scalar && a.r.hd == 128) {
        const int n4 = (a.r.H + a.r.Hkv) * (half / 4) + a.r.Hkv * (a.r.hd / 8);
        launch_pdl(qkv_rope_kv4_kernel, dim3((n4 + 255) / 256, a.r.T), dim3(256), 0, st, a);
    } else
        launch_pdl(qkv_rope_kv_kernel<bf16>, grid, dim3(256), 0, st, a);
    HK_LAUNCHED(1);
}

void add_rmsnorm(const float* part, int splits, float* x, const void* w, bool f32, int T, int d, float eps, void* h,
                 const int32_t* cmap, void* hc, cudaStream_t st) {
    if (!T) return;
    if (d % 4 || d > 8192 * 4) throw std::runtime_error("add_rmsnorm: d must be a multiple of 4");
    static const bool cluster_rms = std::getenv("HK_RMS_CLUSTER") != nullptr;  // A/B: the 8-CTA cluster kernel
    if (!f32 && !cluster_rms && d / 4 <= 4 * 1024) {
        const int n4 = d / 4;
        const int vpt = n4 <= 1024 ? 1 : (n4 <= 2048 ? 2 : 4);
        const int threads = std::min(1024, ((n4 + vpt - 1) / vpt + 31) / 32 * 32);
        const bf16* wb = static_cast<const bf16*>(w);
        bf16* hb = static_cast<bf16*>(h);
        bf16* hcb = static_cast<bf16*>(hc);
        if (vpt == 1)
            launch_pdl(add_rmsnorm_row_kernel<1>, dim3(T), dim3(threads), 0, st, part, splits, x, wb, T, d, eps, hb, cmap, hcb);
        else if (vpt == 2)
            launch_pdl(add_rmsnorm_row_kernel<2>, dim3(T), dim3(threads), 0, st, part, splits, x, wb, T, d, eps, hb, cmap, hcb);
        else
            launch_pdl(add_rmsnorm_row_kernel<4>, dim3(T), dim3(threads), 0, st, part, splits, x, wb, T, d, eps, hb, cmap, hcb);
        HK_LAUNCHED(1);
        return;
    }
    const int per = (d / 4 + kRowSplit - 1) / kRowSplit;          // float4 per CTA
    const int threads = std::max(32, (per + 31) / 32 * 32);
    if (threads > 256) throw std::runtime_error("add_rmsnorm: d too large");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(T, kRowSplit);
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = kRowSplit;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (f32)
        HK_CUDA(cudaLaunchKernelEx(&cfg, add_rmsnorm_kernel<float>, part, splits, x, static_cast<const float*>(w), T, d,
                                   eps, static_cast<float*>(h), cmap, static_cast<float*>(hc)));
    else
        HK_CUDA(cudaLaunchKernelEx(&cfg, add_rmsnorm_kernel<bf16>, part, splits, x, static_cast<const bf16*>(w), T, d,
                                   eps, static_cast<bf16*>(h), cmap, static_cast<bf16*>(hc)));
    HK_LAUNCHED(1);
}

void init_uniform(void* w, bool f32, size_t n, uint64_t seed, uint64_t tensor_id, float scale, cudaStream_t st) {
    if (!n) return;
    init_uniform_kernel<<<grid_for(n), 256, 0, st>>>(w, f32, n, seed, tensor_id, scale);
    HK_LAUNCHED(1);
}

void fill_const(void* w, bool f32, size_t n, float v, cudaStream_t st) {
    if (!n) return;
    fill_kernel<<<grid_for(n), 256, 0, st>>>(w, f32, n, v);
    HK_LAUNCHED(1);
}

void embed(const void* table, bool f32, int d, const int32_t* ids, const int32_t* slots, const int32_t* slot_last,
           int T, float* x, cudaStream_t st) {
    if (!T) return;
    embed_kernel<<<T, 256, 0, st>>>(table, f32, d, ids, slots, slot_last, x);
    HK_LAUNCHED(1);
}

void rmsnorm(const float* x, const void* w, bool f32, int d, float eps, const int32_t* rows, int R, void* out,
             cudaStream_t st) {
    if (!R) return;
    rmsnorm_kernel<<<R, 256, 0, st>>>(x, w, f32, d, eps, rows, out);
    HK_LAUNCHED(1);
}

void rope_kv_write(const RopeArgs& a, cudaStream_t st) {
    if (!a.T) return;
    if (a.f32)
        rope_kv_kernel<float><<<a.T, 256, 0, st>>>(a);
    else
        rope_kv_kernel<bf16><<<a.T, 256, 0, st>>>(a);
    HK_LAUNCHED(1);
}

void swiglu(const void* gu, bool f32, int T, int F, void* out, cudaStream_t st) {
    if (!T) return;
    if (f32)
        swiglu_kernel<float><<<T, 256, 0, st>>>(static_cast<const float*>(gu), F, static_cast<float*>(out));
    else
        swiglu_kernel<bf16><<<T, 256, 0, st>>>(static_cast<const bf16*>(gu), F, static_cast<bf16*>(out));
    HK_LAUNCHED(1);
}

void argmax_rows(const float* logits, int R, int V, int32_t* ids, float* vals, const int32_t* slots,
                 int32_t* slot_last, cudaStream_t st) {
    if (!R) return;
    argmax_kernel<<<R, 512, 0, st>>>(logits, V, ids, vals, slots, slot_last);
    HK_LAUNCHED(1);
}

}  // namespace hkd
