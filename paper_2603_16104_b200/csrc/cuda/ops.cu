// K5: row-wise ops of the decoder (embedding gather, RMSNorm, RoPE + paged KV
// write, SwiGLU, greedy argmax) and the counter-based weight init.
#include <cfloat>

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

__global__ void argmax_kernel(const float* logits, int V, int32_t* ids, const int32_t* slots, int32_t* slot_last) {
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
        ids[r] = bi;
        if (slots) slot_last[slots[r]] = bi;
    }
}

int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void init_uniform(void* w, bool f32, size_t n, uint64_t seed, uint64_t tensor_id, float scale, cudaStream_t st) {
    if (!n) return;
    init_uniform_kernel<<<grid_for(n), 256, 0, st>>>(w, f32, n, seed, tensor_id, scale);
    HK_CUDA(cudaGetLastError());
}

void fill_const(void* w, bool f32, size_t n, float v, cudaStream_t st) {
    if (!n) return;
    fill_kernel<<<grid_for(n), 256, 0, st>>>(w, f32, n, v);
    HK_CUDA(cudaGetLastError());
}

void embed(const void* table, bool f32, int d, const int32_t* ids, const int32_t* slots, const int32_t* slot_last,
           int T, float* x, cudaStream_t st) {
    if (!T) return;
    embed_kernel<<<T, 256, 0, st>>>(table, f32, d, ids, slots, slot_last, x);
    HK_CUDA(cudaGetLastError());
}

void rmsnorm(const float* x, const void* w, bool f32, int d, float eps, const int32_t* rows, int R, void* out,
             cudaStream_t st) {
    if (!R) return;
    rmsnorm_kernel<<<R, 256, 0, st>>>(x, w, f32, d, eps, rows, out);
    HK_CUDA(cudaGetLastError());
}

void rope_kv_write(const RopeArgs& a, cudaStream_t st) {
    if (!a.T) return;
    if (a.f32)
        rope_kv_kernel<float><<<a.T, 256, 0, st>>>(a);
    else
        rope_kv_kernel<bf16><<<a.T, 256, 0, st>>>(a);
    HK_CUDA(cudaGetLastError());
}

void swiglu(const void* gu, bool f32, int T, int F, void* out, cudaStream_t st) {
    if (!T) return;
    if (f32)
        swiglu_kernel<float><<<T, 256, 0, st>>>(static_cast<const float*>(gu), F, static_cast<float*>(out));
    else
        swiglu_kernel<bf16><<<T, 256, 0, st>>>(static_cast<const bf16*>(gu), F, static_cast<bf16*>(out));
    HK_CUDA(cudaGetLastError());
}

void argmax_rows(const float* logits, int R, int V, int32_t* ids, const int32_t* slots, int32_t* slot_last,
                 cudaStream_t st) {
    if (!R) return;
    argmax_kernel<<<R, 512, 0, st>>>(logits, V, ids, slots, slot_last);
    HK_CUDA(cudaGetLastError());
}

}  // namespace hkd
