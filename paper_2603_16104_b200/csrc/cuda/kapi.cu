// Kernel-level C-ABI (include/helium_b200_kernels.h).
#include <string>

#include "common.cuh"
#include "helium_b200_kernels.h"
#include "kernels.cuh"

namespace hk {
void set_error(const std::string& s);
}

namespace {
float* g_ws = nullptr;
size_t g_ws_floats = 0;

float* workspace(size_t n) {
    if (n > g_ws_floats) {
        cudaFree(g_ws);
        HK_CUDA(cudaMalloc(&g_ws, n * sizeof(float)));
        g_ws_floats = n;
    }
    return g_ws;
}

void init_sms() {
    static bool done = false;
    if (done) return;
    int dev = 0, sms = 0;
    HK_CUDA(cudaGetDevice(&dev));
    HK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    hkd::g_num_sms = sms;
    done = true;
}
}  // namespace

extern "C" {

int hkx_gemm_bf16(const void* W, const void* X, void* out, int N, int K, int T, int epi, const void* bias, int splits,
                  void* stream) {
    try {
        init_sms();
        const size_t ws = static_cast<size_t>(32) * (T + 256) * N;
        const int ldo = epi == hkd::kEpiSwiGLU ? N / 2 : N;
        hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, ldo,
                       static_cast<const hkd::bf16*>(bias), workspace(ws), ws, static_cast<cudaStream_t>(stream),
                       splits, 64);
        return 0;
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return -1;
    }
}

double hkx_gemm_bench(const void* W, const void* X, void* out, int N, int K, int T, int epi, int splits, int iters) {
    try {
        init_sms();
        const size_t ws = static_cast<size_t>(32) * (T + 256) * N;
        float* w = workspace(ws);
        cudaEvent_t a, b;
        HK_CUDA(cudaEventCreate(&a));
        HK_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 3; ++i)
            hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, N,
                           nullptr, w, ws, nullptr, splits);
        HK_CUDA(cudaEventRecord(a));
        for (int i = 0; i < iters; ++i)
            hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, N,
                           nullptr, w, ws, nullptr, splits);
        HK_CUDA(cudaEventRecord(b));
        HK_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        HK_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms / iters;
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return -1;
    }
}

}  // extern "C"
