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

/* K3b decode attention of one layer (device pointers; bf16):
 *   qkv [n_rows][(H + 2 Hkv) * 128], kv [n_pages][2][Hkv][16][128], out [n_rows][H][128].
 * Row r attends keys [0, pos[r]] through the page table tables[offs[r] .. offs[r+1])
 * (host arrays). Rows come in n_groups consecutive groups of group_rows[g]
 * rows whose tables share group_shared_pages[g] leading pages (0 = none): the
 * shared pages run on the tcgen05 kernel once per group, the rest per row.
 * Replaces the attention that the reference's decode step implies
 * (simulator.cpp:347-355). iters > 0 also times that many back-to-back calls:
 * returns ms per call (0 when iters == 0) or a negative value on error. */
double hkx_decode_attention(const void* qkv, const void* kv, int n_pages, int n_rows, int H, int Hkv,
                            const int32_t* tables, const int32_t* offs, const int32_t* pos, const int32_t* group_rows,
                            const int32_t* group_shared_pages, int n_groups, void* out, int iters);
/* Causal prefill attention of one chunk on the tensor-core tile path: n_tok
 * tokens at positions start .. start+n_tok-1 (qkv rows 0 .. n_tok-1) attend keys
 * [0, own position] through the page table (host array, table_len pages);
 * out [n_tok][H][128] bf16. Replaces the attention implied by the reference's
 * chunked prefill (simulator.cpp:331-343). Returns 0 or -1. */
int hkx_prefill_attention(const void* qkv, const void* kv, int n_pages, int n_tok, int start, int H, int Hkv,
                          const int32_t* table, int table_len, void* out);
/* Several causal prefill segments in one launch, planned as the engine plans a
 * step: segment s = seg_count[s] tokens at qkv/out rows seg_tok0[s].., positions
 * seg_start[s].., block table arena[seg_ptab[s]..]. Adjacent single-tile
 * segments with >= 8 common leading pages share a multicast CTA pair (the
 * calls of one operator under its pinned prefix). Returns 0 or -1. */
int hkx_prefill_attention_segs(const void* qkv, const void* kv, int n_pages, int n_segs, const int32_t* seg_tok0,
                               const int32_t* seg_count, const int32_t* seg_start, const int32_t* seg_ptab, int H,
                               int Hkv, const int32_t* arena, int arena_len, int n_tok, void* out);
/* Debug: record per-CTA phase timestamps (%globaltimer, ns) of later
 * hkx_decode_attention calls into device_buf ([shared CTAs + private CTAs][8] u64);
 * NULL turns it off. */
int hkx_decode_attention_trace(void* device_buf);
/* debug: dump the HK_GEMM_TRACE per-launch spans (first CTA start, wait exit, last end) as CSV */
int hkx_gemm_trace_dump(const char* path);
/* debug: start (on = 1, clearing earlier spans) or stop span tracing of the
 * GEMM / decode-attention launches (run without CUDA graphs: hk_engine_set_graphs) */
int hkx_span_trace(int on);
/* Algorithmic bytes of that call: shared KV once per group + private KV + q and o. */
double hkx_decode_attention_bytes(int n_rows, int H, int Hkv, const int32_t* offs, const int32_t* pos,
                                  const int32_t* group_rows, const int32_t* group_shared_pages, int n_groups);

#ifdef __cplusplus
}
#endif

#endif
