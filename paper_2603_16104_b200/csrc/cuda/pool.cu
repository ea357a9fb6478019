// K1: KV block pool page moves. A page is one 16-token block of every layer
// (layout per layer: [page][K|V][kv_head][block][head_dim]). gather packs
// pages into a contiguous staging buffer (e.g. pinned-prefix blocks before an
// NVLink broadcast), scatter unpacks on the receiver, copy moves pages within a
// pool. 16-byte vector copies, one CTA per (page, layer) slice.
#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

__global__ void page_move_kernel(const uint8_t* src_base, uint8_t* dst_base, size_t layer_stride, int L,
                                 size_t page_bytes, const int32_t* src_pages, const int32_t* dst_pages, int mode) {
    const int i = blockIdx.x;   // page index in the list
    const int l = blockIdx.y;   // layer
    const uint8_t* src;
    uint8_t* dst;
    if (mode == 0) {  // gather: pool -> staging
        src = src_base + l * layer_stride + static_cast<size_t>(src_pages[i]) * page_bytes;
        dst = dst_base + (static_cast<size_t>(i) * L + l) * page_bytes;
    } else if (mode == 1) {  // scatter: staging -> pool
        src = src_base + (static_cast<size_t>(i) * L + l) * page_bytes;
        dst = dst_base + l * layer_stride + static_cast<size_t>(dst_pages[i]) * page_bytes;
    } else {  // copy within pool
        src = src_base + l * layer_stride + static_cast<size_t>(src_pages[i]) * page_bytes;
        dst = dst_base + l * layer_stride + static_cast<size_t>(dst_pages[i]) * page_bytes;
    }
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    const size_t n4 = page_bytes / 16;
    for (size_t k = threadIdx.x; k < n4; k += blockDim.x) d4[k] = __ldg(s4 + k);
}

}  // namespace

void pool_gather(const void* kv, size_t layer_stride, int L, size_t page_bytes, const int32_t* pages, int n, void* dst,
                 cudaStream_t st) {
    if (n <= 0) return;
    page_move_kernel<<<dim3(n, L), 256, 0, st>>>(static_cast<const uint8_t*>(kv), static_cast<uint8_t*>(dst),
                                                 layer_stride, L, page_bytes, pages, nullptr, 0);
    HK_LAUNCHED(1);
}

void pool_scatter(void* kv, size_t layer_stride, int L, size_t page_bytes, const int32_t* pages, int n, const void* src,
                  cudaStream_t st) {
    if (n <= 0) return;
    page_move_kernel<<<dim3(n, L), 256, 0, st>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(kv),
                                                 layer_stride, L, page_bytes, nullptr, pages, 1);
    HK_LAUNCHED(1);
}

void pool_copy(void* kv, size_t layer_stride, int L, size_t page_bytes, const int32_t* src, const int32_t* dst, int n,
               cudaStream_t st) {
    if (n <= 0) return;
    page_move_kernel<<<dim3(n, L), 256, 0, st>>>(static_cast<const uint8_t*>(kv), static_cast<uint8_t*>(kv),
                                                 layer_stride, L, page_bytes, src, dst, 2);
    HK_LAUNCHED(1);
}

}  // namespace hkd
