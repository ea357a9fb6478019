/*
 * helium_b200.h — C-ABI of the B200-native LLM-as-operator executor.
 *
 * Drop-in boundary for the reference's L4 execution layer
 * (/root/reference/proj/include/helios/simulator.hpp, evaluator.hpp). Every
 * entry point below names the reference interface it replaces. Plain
 * pointers and sizes only; no C++ or torch types cross this boundary.
 * Errors: functions return NULL / a negative status and hk_last_error()
 * returns the message (thread-local). Messages thrown by the executor keep the
 * reference's wording ("simulate: ...", simulator.cpp:226-244, :286, :361).
 *
 * ---------------------------------------------------------------------------
 * HKPLAN01 — the executor input (little-endian, 8-byte words)
 * ---------------------------------------------------------------------------
 * It carries exactly what simulate(compiled, profile, call_tree, sigma, cfg)
 * (simulator.hpp:128-130) reads. integration/plan_export.hpp produces it from
 * the reference types.
 *   u64 magic = 0x31304e414c504b48 ("HKPLAN01")
 *   u64 batch                                  CompiledGraph::batch
 *   u64 n_tok,  u64 tok[n_tok]                 interned token pool
 *   u64 n_span, {u64 off, u64 len}[n_span]     spans into the pool
 *   u64 n_node, per node (ascending id):
 *       i64 id, u64 kind, u64 flags, f64 len_out, u64 n_a, i64 a[n_a]
 *       kind 0 BOUND  (data/input/cache_fetch): a[q] = span of query q
 *       kind 1 OUTPUT : a = {input node}
 *       kind 2 LAMBDA : a = {fn (0 identity, 1 concat, 2 truncate), arg, inputs...}
 *       kind 3 FORMAT : a = {(tag, v)...}: tag 0 literal span, tag 1 input node
 *       kind 4 LLM    : a = {(tag, v)...}: prompt template in Evaluator::prompt
 *                       order (role markers included): tag 0 span, tag 1 ref node
 *       flags bit0 deterministic, bit1 has profile (len_out valid)
 *   u64 n_out, i64 out[n_out]                  WorkflowGraph::outputs
 *   u64 n_tnode, per call-tree node:           TemplatedRadixTree pool order
 *       i64 parent, u64 is_leaf, i64 op, i64 query,
 *       u64 n_parts, {u64 is_static, i64 span_or_source, i64 query}[n_parts],
 *       u64 n_preds, i64 preds[n_preds]
 *   u64 n_workers, per worker: u64 n, {i64 op, i64 query}[n]   Schedule sigma
 *   optional, for the prompt cache (integration/plan_export.hpp writes it):
 *   u64 magic2 = 0x3130304749534b48 ("HKSIG001"), u64 n,
 *       per node: i64 id, u64 tainted, u64 sig[batch]    compute_signatures
 *                                                         (signature.cpp:29-104)
 */
#ifndef HELIUM_B200_H
#define HELIUM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HK_ABI_VERSION 1

const char* hk_last_error(void);
int hk_abi_version(void);

/* ------------------------------------------------------------------ config */
/* SimConfig + SimWorkerConfig (simulator.hpp:71-86). Arrays have n_workers entries. */
typedef struct hk_sim_config {
    uint32_t n_workers;
    const uint64_t* capacity;       /* kv tokens per worker */
    const uint64_t* block;          /* kv block size in tokens */
    const uint64_t* prefill_budget; /* 0 = max(capacity/8, block) */
    int32_t proactive_pin;
    uint64_t pin_threshold;
    double pin_capacity_frac;
    uint64_t seed;
    int32_t stochastic;
    int32_t collect_trace;
    uint64_t max_iterations; /* 0 = 10M guard */
} hk_sim_config;

/* SimMetrics counters (simulator.hpp:108-120) + B200 additions. */
typedef struct hk_metrics {
    uint64_t iterations;
    uint64_t prompt_tokens;
    uint64_t cache_served_tokens;
    uint64_t prefill_computed_tokens;
    uint64_t decode_tokens;
    double hit_rate_pct;
    uint64_t calls;
    uint64_t recompute_tokens;  /* last position of fully cached prompts re-run on device */
    uint64_t pin_compute_tokens; /* summed over workers */
} hk_metrics;

typedef struct hk_run hk_run;
typedef struct hk_engine hk_engine;
typedef struct hk_kvcache hk_kvcache;

/* ---------------------------------------------------------------- executor */
/* Replaces simulate() (simulator.cpp:222-389). engine == NULL runs the
 * synthetic LLM body (synth_llm_output, evaluator.cpp:53-58) with the same
 * control plane; otherwise the LLM body is the device transformer of `engine`
 * (one engine worker per schedule worker).
 * flags: bit0 = verify device trie lookups against the host tree. */
hk_run* hk_simulate(const uint8_t* plan, size_t plan_len, const hk_sim_config* cfg, hk_engine* engine,
                    uint32_t flags);
/* Cross-worker dependencies with one process per GPU (SURVEY.md §8(e)
 * exchange 2). With only_worker >= 0 (flags bits 8+) and fn set, every process
 * replays the control plane of ALL workers (the reference's lock-step loop,
 * simulator.cpp:287-380) and runs the LLM body only for its own worker; at
 * every completion of every worker, in the same order in all processes,
 * fn(user, worker, op, query, tokens, n) is called: the owning process passes
 * the n generated ids, the others fill `tokens`. Metrics, call rows and
 * outputs then cover the whole workflow. fn returns 0 on success. */
typedef int (*hk_output_exchange_fn)(void* user, int worker, int op, int query, uint64_t* tokens, uint64_t n);
hk_run* hk_simulate_ex(const uint8_t* plan, size_t plan_len, const hk_sim_config* cfg, hk_engine* engine,
                       uint32_t flags, hk_output_exchange_fn fn, void* user);
int hk_run_metrics(const hk_run* run, hk_metrics* out);
/* per-worker vectors of SimMetrics: which 0 = pinned_tokens, 1 = evicted_tokens,
 * 2 = pin_compute_tokens. Returns the count; copies min(count, cap). */
size_t hk_run_worker_stat(const hk_run* run, int which, uint64_t* out, size_t cap);
/* which: 0 = sim_metrics_json (simulator.cpp:393-405), 1 = sim_calls_csv
 * (:407-415), 2 = sim_trace_csv (:417-425). Returns bytes needed (incl. NUL). */
size_t hk_run_report(const hk_run* run, int which, char* buf, size_t cap);
/* SimMetrics::outputs flattened as u64 words:
 *   n_nodes, {node_id, batch, {len, tokens[len]}[batch]}[n_nodes]
 * Returns the word count; copies min(count, cap) words. */
size_t hk_run_outputs(const hk_run* run, uint64_t* out, size_t cap);
/* Generated tokens of every llm call (not only workflow outputs), as u64 words:
 *   n_calls, {op, query, len, tokens[len]}[n_calls]  in (op, query) order. */
size_t hk_run_call_outputs(const hk_run* run, uint64_t* out, size_t cap);
/* The device's fp32 logit of every token of hk_run_call_outputs, in the same
 * order (NaN where the body has none, e.g. mode S). For parity checks: the
 * greedy choice's logit against the oracle's logit of the same token. */
size_t hk_run_call_logits(const hk_run* run, float* out, size_t cap);
/* executor wall time split (seconds): [0] pin precompute, [1] iterations. */
int hk_run_timing(const hk_run* run, double out[2]);
void hk_run_free(hk_run* run);

/* ------------------------------------------------------------------ KvCache */
/* class KvCache (simulator.hpp:18-62), same node numbering/LRU/holds/pins. */
hk_kvcache* hk_kv_create(size_t capacity_tokens, size_t block_tokens);
size_t hk_kv_lookup(hk_kvcache* c, const uint64_t* seq, size_t n, uint64_t hold);
size_t hk_kv_insert(hk_kvcache* c, const uint64_t* seq, size_t n, size_t len, int pinned, uint64_t hold);
void hk_kv_release(hk_kvcache* c, uint64_t hold);
/* out = {used_tokens, pinned_tokens, evicted_tokens} */
void hk_kv_counters(const hk_kvcache* c, uint64_t out[3]);
void hk_kv_destroy(hk_kvcache* c);

/* static_pin_prefixes (simulator.hpp:67-69) for `worker` of `plan`. Pins are
 * written back to back into tokens (cap words) with their lengths in lens
 * (lens_cap). Returns the number of pins, or -1. */
int64_t hk_static_pin_prefixes(const uint8_t* plan, size_t plan_len, int worker, size_t block, size_t threshold,
                               size_t budget_tokens, uint64_t* tokens, size_t cap, uint64_t* lens, size_t lens_cap);
/* Opt-in call-level partition — DIVERGES from the reference,
 * which places whole operators (partition_workflow, scheduler.cpp:59-115): the
 * plan's calls of every operator are dealt round-robin over `workers` (each
 * worker keeps the plan's schedule order), so one operator's branches can
 * run on several GPUs. Writes the new HKPLAN01 blob; returns its byte size
 * (copies min(size, cap) bytes; out may be NULL) or -1. */
int64_t hk_plan_partition_calls(const uint8_t* plan, size_t plan_len, int workers, uint8_t* out, size_t cap);
/* Native cache-aware planner: re-plans the value graph of
 * `plan` for `workers` workers exactly as the reference's run_workflow does
 * (run_pipeline.cpp:47-69 with the cache-aware scheduler): partition_workflow
 * (scheduler.cpp:59-115), build_call_tree (trt.cpp:527-530) and
 * plan_operators + expand_soft_schedule (scheduler.cpp:474-571), with the
 * CostParams of capacities (one, or one per worker) and alpha (0 = 1/capacity).
 * Writes the new HKPLAN01 blob (call tree + schedule replaced, value graph and
 * signatures kept); returns its byte size (copies min(size, cap); out may be
 * NULL) or -1. */
int64_t hk_plan_schedule(const uint8_t* plan, size_t plan_len, int workers, const uint64_t* capacities, size_t n_caps,
                         double alpha, uint8_t* out, size_t cap);
/* The plan's TRT shared-prefix groups (trt.cpp:489-530), one per llm call in
 * (op, query) order: the deepest call-tree ancestor whose whole root path is
 * static text (-1: none) and that static path's token length. The decode
 * planner groups prefix-shared attention rows by it. Returns the call count
 * (copies min(count, cap)) or -1. */
int64_t hk_plan_call_groups(const uint8_t* plan, size_t plan_len, int64_t* op, int32_t* query, int32_t* group,
                            uint64_t* tokens, size_t cap);

/* ------------------------------------------------------ run_workflow (native) */
/* RunSpec (run_pipeline.hpp:16-38). scheduler: "cache_aware" (the baselines
 * random / lspf / op_wise / query_wise stay in the reference library). */
typedef struct hk_workflow_spec {
    int32_t workers;
    const uint64_t* capacities; /* one, or one per worker (kv tokens) */
    size_t n_capacities;
    const char* scheduler;
    uint64_t seed;
    int32_t stochastic;
    int32_t prune;
    int32_t merge_duplicates;
    int32_t cache_substitute;
    int32_t proactive_pin;
    uint64_t pin_threshold;
    double pin_capacity_frac;
    uint64_t block;
    uint64_t prefill_budget; /* 0 = capacity/8 */
    double alpha;            /* 0 = 1/capacity */
    int32_t run_sim;
    int32_t collect_trace;
    uint64_t max_iterations;
} hk_workflow_spec;
typedef struct hk_pcache hk_pcache;
/* run_workflow (run_pipeline.cpp:47-81) entirely in this library: the
 * reference's workflow / inputs / profile JSON (workflow_io.cpp), validate +
 * bind (workflow.cpp), rewrite (optimizer.cpp: prune, fold duplicates,
 * prompt-cache substitution when `cache` is set), the native planner
 * (hk_plan_schedule), simulate() with the synthetic body (engine NULL) or the
 * device transformer, and the prompt-cache harvest of this run's values.
 * Errors keep the reference's messages ("workflow json: ...", "format node
 * 3: bad slot ...", "simulate: ..."). The run's documents:
 * hk_run_report(0|1|2) = sim metrics json / calls csv / trace csv, and
 * hk_run_document(0|1|2) = run_report_json (run_pipeline.cpp:85-112) / the
 * CLI's outputs json (helios_main.cpp:26-34) / soft_schedule_json
 * (scheduler.cpp:573-581), each exactly the bytes `helios run` writes for
 * --out / --outputs-out / --schedule-out (helios_main.cpp:100-112). */
hk_run* hk_run_workflow(const char* workflow_json, const char* inputs_json, const char* profile_json,
                        const hk_workflow_spec* spec, hk_pcache* cache, hk_engine* engine);
size_t hk_run_document(const hk_run* run, int which, char* buf, size_t cap);
/* the planned HKPLAN01 of hk_run_workflow (copies min(size, cap); returns size) */
size_t hk_run_plan(const hk_run* run, uint8_t* out, size_t cap);

/* ------------------------------------------------------------ prompt cache */
/* class PromptCache (prompt_cache.hpp:15-40): LRU from operator signature to
 * the tokens that operator produced. hk_pcache_save / hk_pcache_load use the
 * reference's JSON document byte for byte (prompt_cache.cpp:47-67), so the
 * reference's optimizer (substitute_cached, optimizer.cpp:71-95) reads a cache
 * harvested here and vice versa. Errors keep the reference wording
 * ("prompt cache capacity must be positive", "prompt cache json: ..."). */
hk_pcache* hk_pcache_create(size_t capacity);
hk_pcache* hk_pcache_load(const char* json, size_t len);
/* writes the JSON document (NUL-terminated, truncated to cap); returns bytes needed incl. NUL */
size_t hk_pcache_save(const hk_pcache* c, char* buf, size_t cap);
size_t hk_pcache_size(const hk_pcache* c);
size_t hk_pcache_capacity(const hk_pcache* c);
int hk_pcache_contains(const hk_pcache* c, uint64_t sig);
/* hit: refreshes recency, copies min(len, cap) tokens, returns len; miss: -1 */
int64_t hk_pcache_lookup(hk_pcache* c, uint64_t sig, uint64_t* out, size_t cap);
int hk_pcache_insert(hk_pcache* c, uint64_t sig, const uint64_t* tokens, size_t n);
/* keys least recently used first; returns the count, copies min(count, cap) */
size_t hk_pcache_keys(const hk_pcache* c, uint64_t* out, size_t cap);
/* harvest_into_cache (optimizer.cpp:113-125) from a finished run of `plan`
 * (which must carry the HKSIG001 section): every untainted format / lambda /
 * llm node, every query; llm values are the tokens this run's LLM body
 * generated (the device transformer's, under an engine). Returns the number
 * of entries inserted, or -1. */
int64_t hk_pcache_harvest(hk_pcache* c, const uint8_t* plan, size_t plan_len, const hk_run* run);
/* The same from call outputs in the hk_run_call_outputs layout (n_calls,
 * {op, query, len, tokens[len]}...), for bindings that keep a run's outputs
 * after freeing it. */
int64_t hk_pcache_harvest_calls(hk_pcache* c, const uint8_t* plan, size_t plan_len, const uint64_t* calls,
                                size_t n_words);
void hk_pcache_destroy(hk_pcache* c);

/* --------------------------------------------------------- LLM body (synth) */
/* synth_llm_len / synth_llm_output (evaluator.hpp:29-32). */
size_t hk_synth_llm_len(const uint64_t* prompt, size_t n, double len_out, int deterministic, uint64_t seed,
                        int stochastic);
size_t hk_synth_llm_output(const uint64_t* prompt, size_t n, double len_out, int deterministic, uint64_t seed,
                           int stochastic, uint64_t* out, size_t cap);
/* tokens.hpp:16-28 */
uint64_t hk_fnv1a64(const void* data, size_t len, uint64_t seed);
uint64_t hk_hash_combine(uint64_t h, uint64_t v);
/* model-mode token maps (new definitions) */
uint32_t hk_vocab_of(uint64_t token, uint32_t vocab);
uint64_t hk_gen_token(uint32_t id, uint32_t vocab);

/* ================================================================ device */
/* Random-init decoder-only transformer (Llama-3 / Qwen2.5 family). */
typedef struct hk_model_config {
    uint32_t n_layers;
    uint32_t d_model;
    uint32_t n_heads;
    uint32_t n_kv_heads;
    uint32_t head_dim;
    uint32_t ffn_dim;
    uint32_t vocab;
    uint32_t qkv_bias;   /* Qwen2.5 has q/k/v biases */
    float rope_theta;
    float rms_eps;
    uint64_t seed;       /* counter-based weight init seed */
    uint32_t fp32;       /* 1 = fp32 storage + fp32 math (parity mode) */
    uint32_t reserved;
} hk_model_config;

typedef struct hk_engine_config {
    int32_t device;             /* CUDA ordinal */
    uint32_t n_workers;         /* KV pools (one per schedule worker on this device) */
    uint32_t pages_per_worker;  /* physical 16-token KV pages per pool */
    uint32_t block_tokens;      /* page size in tokens (must equal SimWorkerConfig::block) */
    uint32_t max_calls;         /* live call slots per worker */
    uint32_t max_step_tokens;   /* max tokens in one ragged forward */
    uint32_t max_ctx_tokens;    /* max context length of one call */
    uint32_t use_device_trie;   /* admission lookups through the device trie (K2) */
} hk_engine_config;

/* K1-K5 live on the engine. Weights are initialised on device from the seed. */
hk_engine* hk_engine_create(const hk_model_config* model, const hk_engine_config* cfg);
void hk_engine_destroy(hk_engine* e);
/* bytes of one KV page (all layers, K and V) */
size_t hk_engine_page_bytes(const hk_engine* e);
/* resets pools, slots and tries of every worker */
int hk_engine_reset(hk_engine* e);

/* K6 pinned-prefix replication (SURVEY.md §8(e) exchange 1; reference
 * static_pin_prefixes + pin insert, simulator.cpp:132-199, :257-263): every
 * worker pins the same prefix, so one rank computes its KV and the others
 * receive the pages instead of recomputing them. The pin precompute of
 * hk_simulate calls fn once per worker that pinned new blocks, with a device
 * buffer of `bytes` = (newly pinned pages, in pin / block order) x
 * hk_engine_page_bytes, each page laid out as hk_pool_gather writes it.
 *   role 0: compute locally, no callback (default)
 *   role 1: compute, then fn(buffer holding the pages)  (broadcast source)
 *   role 2: skip the compute; fn fills the buffer, the engine scatters it
 *           into this worker's pin pages                (receiver)
 * fn returns 0 on success; non-zero fails hk_simulate with "simulate: ...". */
typedef int (*hk_pin_exchange_fn)(void* user, int worker, void* device_buf, uint64_t bytes);
int hk_engine_set_pin_exchange(hk_engine* e, int role, hk_pin_exchange_fn fn, void* user);
/* CUDA-graph replay of repeated step shapes (default on; off for launch-level tracing) */
int hk_engine_set_graphs(hk_engine* e, int on);

/* K1 block pool: page-granular gather / scatter / copy on the device.
 * dst/src are device pointers of n * page_bytes bytes. */
int hk_pool_gather(hk_engine* e, int worker, const int32_t* pages, size_t n, void* dst_device);
int hk_pool_scatter(hk_engine* e, int worker, const void* src_device, const int32_t* pages, size_t n);
int hk_pool_copy(hk_engine* e, int worker, const int32_t* src_pages, const int32_t* dst_pages, size_t n);

/* K2 device trie. Node journal entries mirror KvTree creates/erases. */
typedef struct hk_trie_op {
    int32_t node;
    int32_t parent;
    int32_t page;
    int32_t erase;
    uint64_t phash;
    const uint64_t* key; /* block_tokens tokens (creates only) */
} hk_trie_op;
int hk_trie_apply(hk_engine* e, int worker, const hk_trie_op* ops, size_t n);
/* Batched longest-block-prefix match of n prompts (tokens concatenated,
 * offsets[n+1]). For prompt i writes matched block count, node path and page
 * table rows (stride = max blocks per prompt). Equals KvCache::lookup's
 * matched length and walk (simulator.cpp:69-87) without its side effects. */
int hk_trie_match(hk_engine* e, int worker, const uint64_t* tokens, const uint64_t* offsets, size_t n,
                  int32_t* matched_blocks, int32_t* node_path, int32_t* page_table, size_t stride);

/* ---- step-level entry points: for a host that runs its own
 * iteration loop (the reference's simulate() body, simulator.cpp:331-374) and
 * owns the block tables. Every call is synchronous on the engine stream. */
/* A call slot holds the call's last sampled token on the device (the next
 * decode step's input) and its generated tokens. -1 + hk_last_error on failure. */
int hk_slot_alloc(hk_engine* e, int worker);
int hk_slot_free(hk_engine* e, int worker, int slot);
/* One segment of a ragged step: a prefill chunk of `count` tokens at positions
 * [start, start + count) with their vocab ids, or a decode step (ids == NULL,
 * count == 1) whose input is the slot's last sampled token at position `start`.
 * `pages` is the call's block table covering positions [0, start + count)
 * (page p holds positions [16p, 16p + 16) of the call); the K/V of the
 * segment's positions are written into it when write_kv != 0, earlier
 * positions are read from it (shared prefix pages may appear in several
 * calls' tables). */
typedef struct hk_step_seg {
    int32_t slot;          /* call slot; -1 for a prefill chunk that samples nothing */
    int32_t start;
    int32_t count;
    int32_t sample;        /* greedy-sample the token after the segment's last position */
    const uint32_t* ids;   /* count vocab ids, or NULL (decode) */
    const int32_t* pages;
    int32_t n_pages;
    int32_t write_kv;
} hk_step_seg;
/* One ragged forward (prefill chunks + decode rows, the engine's K3/K4/K5 path;
 * the reference's chunked prefill simulator.cpp:331-343 and decode step
 * :347-374 of one worker and iteration). sampled[i] = the token sampled for
 * segment i (-1 when it does not sample); logits (optional, [n][vocab] fp32)
 * receives the vocab logits of every sampling segment's last position. */
int hk_step(hk_engine* e, int worker, const hk_step_seg* segs, size_t n, int32_t* sampled, float* logits);
/* Prefill a pin (static prefix, simulator.cpp:257-263) into `pages` without
 * sampling: K/V of positions [0, n) land in pages[0 .. ceil(n / 16)). */
int hk_pin_prefill(hk_engine* e, int worker, const uint32_t* ids, size_t n, const int32_t* pages, size_t n_pages);
/* K6 page broadcast outside hk_simulate: role 1 gathers `pages` into a device
 * buffer (n x hk_engine_page_bytes, hk_pool_gather layout) and calls fn with
 * it (the caller broadcasts, e.g. ncclBroadcast); role 2 calls fn to fill the
 * buffer, then scatters it into `pages`. */
int hk_kv_broadcast(hk_engine* e, int worker, int role, const int32_t* pages, size_t n, hk_pin_exchange_fn fn,
                    void* user);

/* Stand-alone greedy generation of one prompt (vocab ids) through the paged
 * engine — prefill then n_new decode steps — used by model parity tests.
 * logits (optional) receives the vocab logits of each sampled position. */
int hk_generate(hk_engine* e, const uint32_t* ids, size_t n, size_t n_new, uint32_t* out_ids, float* logits);

/* Statistics of the last hk_simulate run on this engine: device time measured
 * with CUDA events on the engine stream (pin precompute, iteration loop), the
 * host<->device bytes the executor moved, and kernel launches issued. */
typedef struct hk_engine_stats {
    double pin_ms;
    double iter_ms;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t launches;
    uint64_t steps;
    uint64_t step_tokens;
    double attn_bytes; /* algorithmic attention bytes (KV read once per group + Q/O) */
} hk_engine_stats;
int hk_engine_stats_get(const hk_engine* e, hk_engine_stats* out);

/* Device time (ms) per kernel family accumulated since the last reset, for
 * roofline reporting: names "gemm", "attn_shared", "attn_private", "attn_prefill",
 * "attn_merge", "small", "trie", "kvcopy". Returns -1 for an unknown name. */
double hk_engine_kernel_ms(const hk_engine* e, const char* family, uint64_t* launches, double* bytes);
int hk_engine_profile(hk_engine* e, int enable);

#ifdef __cplusplus
}
#endif

#endif /* HELIUM_B200_H */
