// Host-callable launchers of the device kernels (one translation unit each).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace hkd {

// GEMM epilogues. kEpiPartial writes fp32 split-K partials [splits][T][N] that
// a consumer row kernel reduces (fused with bias / RoPE / residual / RMSNorm);
// kEpiSwiGLU expects W rows interleaved per 128-row tile as [64 gate | 64 up]
// and writes silu(gate) * up as bf16 [T][N/2]; kEpiArgmax writes per-(tile,
// token) (max, argmax) pairs [N/128][T] for argmax_reduce.
enum : int { kEpiStoreBf16 = 0, kEpiAddF32 = 1, kEpiStoreF32 = 2, kEpiPartial = 3, kEpiSwiGLU = 4, kEpiArgmax = 5 };
extern int g_num_sms;
extern unsigned long long g_launches;  // kernels launched by this library (all launchers count)

// ----------------------------------------------------------------- gemm.cu
// out[t][n] (+)= sum_k X[t][k] W[n][k] (+ bias[n]); tcgen05 path for bf16.
// Returns the split-K factor used (kEpiPartial: `out` must hold splits*T*N floats;
// max_splits bounds it). Other epilogues reduce split partials through `workspace`.
int gemm_bf16(const bf16* W, const bf16* X, int N, int K, int T, int epi, void* out, int ldo, const bf16* bias,
              float* workspace, size_t workspace_floats, cudaStream_t st, int force_splits = 0, int max_splits = 16);
// Stream-K variant for decode shapes (T <= 64): one CTA per SM over equal
// shares of (128-row tile, 64-k) units; the result is fully reduced (no
// split-K partials): kEpiPartial/kEpiStoreF32 write fp32 [T][ldo].
void gemm_bf16_streamk(const bf16* W, const bf16* X, int N, int K, int T, int epi, void* out, int ldo, cudaStream_t st);
bool gemm_streamk_enabled();
// debug: write the HK_GEMM_TRACE launch spans as CSV; returns the launch count
int gemm_trace_dump(const char* path);
// debug (HK_GEMM_TRACE): a span slot [first CTA start, first wait exit, ~last end, ~last main-loop end]
// for one launch; N = -1 marks a decode-attention launch (K = its algorithmic KB)
unsigned long long* gemm_trace_slot(int N, int K, int T, int splits, int ctas);
extern int g_trace_prefill_rows;  // recorded with every trace slot: prefill rows of the step being enqueued
// (re)start span tracing (clears the slots); on = false stops it
void span_trace_reset(bool on);
// allocate the stream-K workspace/counters ahead of any CUDA-graph capture
void gemm_streamk_reserve(int max_tiles, int max_bn);
// ids[t] = argmax over the n_tiles (max, idx) partials of kEpiArgmax (lowest index wins ties);
// vals[t] (optional) = that max logit
void argmax_reduce(const float2* part, int n_tiles, int T, int32_t* ids, float* vals, const int32_t* slots,
                   int32_t* slot_last, cudaStream_t st);
// 2D bf16 tensor map [rows][cols] (row stride cols*2 B), box {box_cols, box_rows}, 128B swizzle
CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows);
void gemm_f32(const float* W, const float* X, int N, int K, int T, int epi, void* out, int ldo, const float* bias,
              cudaStream_t st);

// ------------------------------------------------------------------ ops.cu
// Counter-based weight init shared bit-for-bit with oracle/transformer.py.
void init_uniform(void* w, bool f32, size_t n, uint64_t seed, uint64_t tensor_id, float scale, cudaStream_t st);
void fill_const(void* w, bool f32, size_t n, float v, cudaStream_t st);
// x[t] = embed[id_t] (ids < 0 read the slot's last sampled token)
void embed(const void* table, bool f32, int d, const int32_t* ids, const int32_t* slots, const int32_t* slot_last,
           int T, float* x, cudaStream_t st);
// out[r] = rmsnorm(x[rows ? rows[r] : r]) * w
void rmsnorm(const float* x, const void* w, bool f32, int d, float eps, const int32_t* rows, int R, void* out,
             cudaStream_t st);
// RoPE on q and k of qkv rows; K/V written into their KV pages (tok_kvw != 0).
struct RopeArgs {
    void* qkv;              // [T][(H + 2 Hkv) hd], bf16 or f32
    bool f32;
    int T, H, Hkv, hd;
    const int32_t* pos;     // [T]
    const int32_t* kvw;     // [T] write K/V?
    const int32_t* ptab;    // [T] offset of the token's block table in `pages`
    const int32_t* pages;   // page-table arena
    const float2* rope;     // [max_pos][hd/2] (cos, sin)
    void* kv_layer;         // this layer's pool: [P][2][Hkv][block][hd]
    int block;
};
void rope_kv_write(const RopeArgs& a, cudaStream_t st);
void swiglu(const void* gu, bool f32, int T, int F, void* out, cudaStream_t st);
// gate/up weights are stored with rows interleaved per 128-row tile ([64 gate | 64 up]);
// init maps the physical index back to the logical (gate | up) index of the oracle.
void init_uniform_gu(void* w, bool f32, int F, int d, uint64_t seed, uint64_t tensor_id, float scale, cudaStream_t st);
// fp32 parity path: silu(gate) * up from an interleaved [T][2F] GEMM output
void swiglu_interleaved(const float* gu, int T, int F, float* out, cudaStream_t st);
// Split-K consumer: qkv = sum_s part[s] (+ bias); RoPE on q/k; q -> qkv (bf16 or f32);
// k, v -> this layer's KV pages (tokens with kvw != 0).
struct QkvArgs {
    const float* part;      // [splits][T][QKV]
    int splits;
    const void* bias;       // [QKV] or null
    RopeArgs r;             // r.qkv receives the rotated q (and raw k, v) rows
};
void qkv_rope_kv(const QkvArgs& a, cudaStream_t st);
// Split-K consumer: x[t] += sum_s part[s][t]; h[t] = rmsnorm(x[t]) * w; rows with
// cmap[t] >= 0 are also written to hc[cmap[t]] (compact rows for the LM head).
void add_rmsnorm(const float* part, int splits, float* x, const void* w, bool f32, int T, int d, float eps, void* h,
                 const int32_t* cmap, void* hc, cudaStream_t st);
// ids[r] = argmax_v logits[r][v] (lowest index on ties), vals[r] (optional) its logit;
// also slot_last[slots[r]] = ids[r]
void argmax_rows(const float* logits, int R, int V, int32_t* ids, float* vals, const int32_t* slots,
                 int32_t* slot_last, cudaStream_t st);

// ------------------------------------------------------------ attention.cu
struct AttnItem {
    int tok0;    // first batch token (rows tok0 .. tok0 + ntok - 1)
    int ntok;    // <= 16
    int kvh;     // kv head
    int ptab;    // offset of the rows' block table in the page arena
    int kbeg;    // key range [kbeg, kend), kbeg page aligned
    int kend;
    int causal;  // mask key j > pos(row)
    int part;    // partial index for these rows, -1 = write the final output directly
};
struct AttnArgs {
    const void* qkv;       // [T][(H + 2 Hkv) hd]
    bool f32;
    int H, Hkv, hd, block;
    const int32_t* pos;    // [T]
    const int32_t* pages;  // page arena
    const void* kv_layer;  // [P][2][Hkv][block][hd]
    const AttnItem* items;
    int n_items;
    void* out;             // [T][H][hd] (bf16 or f32)
    float* part_o;         // [rows][H][max_parts][hd], row = token - part_tok0
    float2* part_ml;       // [rows][H][max_parts] (m, l) in log2 units
    int max_parts;
    int part_tok0;         // first batch token that has partials (decode tokens are last)
    float scale;
    int single;            // items hold exactly one token each (private decode suffixes)
};
void attention_partial(const AttnArgs& a, cudaStream_t st);
// out[tok0 + r][h] = merge of the n_parts[r] partials of row r, r < n_rows
void attention_merge(const float* part_o, const float2* part_ml, const int32_t* n_parts, int n_rows, int tok0, int H,
                     int hd, int max_parts, void* out, bool f32, cudaStream_t st);

// --------------------------------------------------------- decode_attn.cu
// K3b (bf16): decode attention of one ragged step, one launch pair per layer.
//   * shared items (tcgen05): 128 MMA rows = (token, q-head) pairs of up to
//     128/G decode tokens sharing a block-table prefix x one kv head x a range
//     of whole shared pages; the shared KV is read once for all those rows;
//   * private items (CUDA cores): one decode token x one kv head x its own
//     pages (suffix + generated tokens).
// Every item leaves a flash partial (m, l, unnormalised o) per row and head
// (a row's only item writes the bf16 output directly); a PDL-chained merge
// kernel combines the partials of rows that have several.
struct ShItem {
    int row0;    // first decode row
    int ntok;    // decode rows covered (<= 128 / G)
    int kvh;
    int ptab;    // block table (arena offset) of the group's first member
    int page0;   // first shared page (index into the table)
    int npages;  // shared pages covered by this item (may be 0)
    int rank;    // partial index (decode items)
    int flags;   // bit0: causal prefill item — row0 is a batch token, keys <= the row's
                 // position, the normalised bf16 output is written directly
    int mc_pages;  // leading pages identical in both CTAs of the pair: those chunks are
                   // fetched once and multicast, later chunks are loaded by each CTA itself
};
struct PvItem {
    int row;     // decode row
    int kvh;
    int ptab;
    int kbeg;    // key range [kbeg, kend), kbeg page aligned
    int kend;
    int part;    // partial index, -1 = sole contributor: write the output directly
    int pad0, pad1;
};
struct DecodeAttnArgs {
    const bf16* qkv;        // [T][QKV]
    const int32_t* pos;     // [T] token positions (causal prefill items)
    int H, Hkv, QKV;
    const bf16* kv_layer;   // this layer's pool [P][2][Hkv][16][128]
    int layer_row0;         // first row of this layer in the pool tensor map
    const int32_t* pages;   // page arena
    const ShItem* sh;
    int n_sh;
    int sh_cluster;         // CTAs per shared cluster (items of one tile are consecutive)
    const PvItem* pv;
    int n_pv;
    float* part_o;          // [rows][H][max_parts][128]
    float2* part_ml;        // [rows][H][max_parts] (m, l), log2 units
    int max_parts;
    const int32_t* n_parts; // [rows] partials per (row, kv head)
    int32_t* counters;      // [rows][Hkv], zero between launches
    int n_rows;             // decode rows of the step
    int any_merge;          // max partials of a row when > 1 (a merge follows), else 0; 1 = unknown
    int32_t* pv_next;       // private work queue head (zero between launches)
    int32_t* pv_done;       // warps / CTAs that left the queue (zero between launches)
    int32_t* grid_arrive;   // grid-wide arrival before the in-kernel merge (zero between launches)
    int merge_in_kernel;    // set by the launcher
    int dec_tok0;           // batch token of decode row 0
    bf16* out;              // [T][H][128]
    float sl2;              // softmax scale * log2(e)
    unsigned long long* trace;  // optional [n_sh + n_pv][8] %globaltimer stamps per CTA phase (null = off)
    const void* l2_prefetch;    // optional: bytes the next kernel streams (O-projection weights), pulled
    size_t l2_prefetch_bytes;   // into L2 by otherwise idle warps while HBM is under-used
    unsigned long long* span = nullptr;  // debug (HK_GEMM_TRACE): launch span slot, see gemm_trace_slot
    int kv_evict_first = 0;  // decode K/V page loads carry an L2 evict_first hint (each page is read once
                             // per step: keeps L2 for what is reused — instructions, metadata, partials)
};
// Host planning of one step's decode rows. Rows of a group are consecutive
// and share `shared_pages` leading pages of their block tables.
struct DecodeRowIn {
    int ptab;  // block table offset in the arena
    int pos;   // position of the decode token (keys [0, pos] are attended)
};
struct DecodeGroupIn {
    int row0, members, shared_pages;
};
struct DecodePlan {
    std::vector<ShItem> sh;
    std::vector<PvItem> pv;
    std::vector<int32_t> n_parts;
    int sh_cluster = 1;
    double shared_bytes = 0, private_bytes = 0;  // algorithmic KV bytes (+ Q/O) per layer
};
void plan_decode_attention(const std::vector<DecodeRowIn>& rows, const std::vector<DecodeGroupIn>& groups, int H,
                           int Hkv, int max_parts, int num_sms, DecodePlan& plan);
// Causal prefill chunks on the same tensor-core tile path: appends paired
// items (prompt tokens x q-heads of one kv head, keys = the call's pages up
// to the chunk's last position) to plan.sh. Returns the algorithmic bytes.
struct PrefillSegIn {
    int tok0;   // batch token of the chunk's first token
    int count;  // tokens in the chunk
    int start;  // position of the first token
    int ptab;   // block table offset in the arena
};
// arena (optional): the host page-id arena the segments' ptab offsets index;
// with it, single-tile segments that share leading pages (calls under one
// pinned prefix) are paired with each other instead of with an empty tile
double plan_prefill_attention(const std::vector<PrefillSegIn>& segs, int H, int Hkv, DecodePlan& plan,
                              const int32_t* arena = nullptr);
// tm_kv: the worker's whole pool as a [L*P*2*Hkv*16][128] bf16 tensor map, box {64, 16}.
void decode_attention(const DecodeAttnArgs& a, const CUtensorMap& tm_kv, cudaStream_t st);

// ------------------------------------------------------------------ pool.cu
// K1: page-granular moves of whole KV pages (all layers) inside one pool.
void pool_gather(const void* kv, size_t layer_stride, int L, size_t page_bytes_layer, const int32_t* pages, int n,
                 void* dst, cudaStream_t st);
void pool_scatter(void* kv, size_t layer_stride, int L, size_t page_bytes_layer, const int32_t* pages, int n,
                  const void* src, cudaStream_t st);
void pool_copy(void* kv, size_t layer_stride, int L, size_t page_bytes_layer, const int32_t* src, const int32_t* dst,
               int n, cudaStream_t st);

// ------------------------------------------------------------------ trie.cu
// K2: device mirror of a worker's KvTree, keyed by prefix hash.
struct DevTrie {
    int max_nodes = 0, block = 16, table_size = 0;
    int32_t* parent = nullptr;   // [max_nodes]
    int32_t* page = nullptr;     // [max_nodes]
    uint64_t* phash = nullptr;   // [max_nodes]
    uint64_t* keys = nullptr;    // [max_nodes][block]
    uint64_t* tab_key = nullptr; // [table_size] prefix hash (0 = empty, 1 = tombstone)
    int32_t* tab_node = nullptr; // [table_size]
};
struct TrieOpDev {
    int32_t node, parent, page, erase;
    uint64_t phash;
};
void trie_apply(DevTrie& t, const TrieOpDev* ops, const uint64_t* keys, int n_ops, cudaStream_t st);
void trie_match(const DevTrie& t, const uint64_t* tokens, const uint64_t* offsets, int n_prompts, int32_t* matched,
                int32_t* node_path, int32_t* page_table, int stride, cudaStream_t st);

}  // namespace hkd
