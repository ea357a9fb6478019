/*
 * helium_b200_kernels.h — kernel-level entry points (device pointers) used by
 * the parity tests and micro-benchmarks. Not needed by the reference-facing
 * executor API in helium_b200.h.
 */
#ifndef HELIUM_B200_KERNELS_H
#define HELIUM_B200_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* K4 tcgen05 GEMM: out[t][n] (+)= sum_k X[t][k] W[n][k] (+ bias[n]).
 * W bf16 [N][K], X bf16 [T][K]; epi 0 = store bf16, 1 = add into f32,
 * 2 = store f32, 3 = fp32 split-K partials [splits][T][N], 4 = SwiGLU (W rows
 * interleaved [64 gate | 64 up] per 128; out bf16 [T][N/2]), 5 = argmax
 * partials (out float2 [N/128][T] = (max, index as int bits)).
 * splits = 0 picks split-K automatically. stream may be NULL. */
int hkx_gemm_bf16(const void* W, const void* X, void* out, int N, int K, int T, int epi, const void* bias,
                  int splits, void* stream);
/* Times `iters` back-to-back launches of the same GEMM with CUDA events; returns
 * the mean milliseconds per launch (or a negative value on error). */
double hkx_gemm_bench(const void* W, const void* X, void* out, int N, int K, int T, int epi, int splits, int iters);

#ifdef __cplusplus
}
#endif

#endif
