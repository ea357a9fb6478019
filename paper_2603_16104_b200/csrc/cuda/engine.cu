// Device engine: random-init decoder weights, per-worker KV block pools and
// device tries, the ragged step planner and forward pass, and the LlmBody that
// lets the host executor (executor.cpp) run its LLM calls on the B200.
//
// One step = one (iteration, worker) of the reference's simulate() loop
// (simulator.cpp:287-379): every prefill chunk and every decode token of that
// worker's iteration is one ragged forward pass. Tokens are ordered
// [prefill chunks][decode tokens grouped by shared block-table prefix] so that
// the prefix-shared attention items (K3b) cover 16 consecutive rows.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <map>
#include <unordered_map>

#include "common.cuh"
#include "helium_b200.h"
#include "hk_host.hpp"
#include "kernels.cuh"

namespace hk {
void set_error(const std::string& s);
}

namespace {

using hkd::bf16;

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) return nullptr;
    HK_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

struct LayerW {
    void *attn_norm, *wqkv, *bqkv, *wo, *mlp_norm, *wgu, *wd;
};

struct KernelClock {
    // accumulated device time per kernel family, measured with CUDA events
    struct Pair {
        cudaEvent_t a, b;
        int fam;
        double bytes;
    };
    static constexpr int kFamilies = 9;
    // gemm: weight-streaming GEMMs (<= 192 rows, bytes = weights + inputs); gemm_prefill:
    // tensor-bound GEMMs (> 192 rows, "bytes" = FLOPs)
    const char* names[kFamilies] = {"gemm", "attn_shared", "attn_private", "attn_prefill",
                                    "attn_merge", "small", "trie", "kvcopy", "gemm_prefill"};
    double ms[kFamilies] = {0};
    double bytes[kFamilies] = {0};
    uint64_t launches[kFamilies] = {0};
    std::vector<Pair> pending;
    std::vector<cudaEvent_t> free_events;
    bool enabled = false;

    cudaEvent_t ev() {
        if (free_events.empty()) {
            cudaEvent_t e;
            HK_CUDA(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = free_events.back();
        free_events.pop_back();
        return e;
    }
    int begin(int fam, cudaStream_t st) {
        if (!enabled) return -1;
        Pair p{ev(), nullptr, fam, 0};
        HK_CUDA(cudaEventRecord(p.a, st));
        pending.push_back(p);
        return static_cast<int>(pending.size()) - 1;
    }
    void end(int idx, cudaStream_t st, double b = 0, uint64_t n = 1) {
        if (idx < 0) return;
        Pair& p = pending[static_cast<size_t>(idx)];
        p.b = ev();
        p.bytes = b;
        HK_CUDA(cudaEventRecord(p.b, st));
        launches[p.fam] += n;
    }
    void collect() {
        for (Pair& p : pending) {
            HK_CUDA(cudaEventSynchronize(p.b));
            float t = 0;
            HK_CUDA(cudaEventElapsedTime(&t, p.a, p.b));
            ms[p.fam] += t;
            bytes[p.fam] += p.bytes;
            free_events.push_back(p.a);
            free_events.push_back(p.b);
        }
        pending.clear();
    }
    void reset() {
        collect();
        std::fill(ms, ms + kFamilies, 0.0);
        std::fill(bytes, bytes + kFamilies, 0.0);
        std::fill(launches, launches + kFamilies, 0);
    }
};

}  // namespace

struct hk_engine {
    hk_model_config mc{};
    hk_engine_config ec{};
    bool f32 = false;
    size_t esz = 2;
    int L = 0, d = 0, H = 0, Hkv = 0, hd = 0, F = 0, V = 0, QKV = 0;
    cudaStream_t st = nullptr;

    // weights
    void* wbuf = nullptr;
    void *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
    std::vector<LayerW> layers;
    float2* rope = nullptr;

    struct Worker {
        void* kv = nullptr;           // [L][P][2][Hkv][block][hd]
        size_t layer_stride = 0;      // bytes
        int32_t* slot_last = nullptr; // [max_calls]
        int32_t* counters = nullptr;  // [max decode rows][Hkv] decode-attention arrival counters
        CUtensorMap tm_kv{};          // the pool as [L*P*2*Hkv*block][hd] bf16 rows (TMA, box 64 x 16)
        hkd::DevTrie trie;
        int trie_tombs = 0;
        std::vector<int> free_slots;
        std::vector<std::vector<int32_t>> slot_tokens;
        std::vector<std::vector<float>> slot_logits;  // the sampled token's logit, per generated token
    };
    std::vector<Worker> workers;
    size_t page_bytes_layer = 0;

    // step scratch (device)
    int maxT = 0, maxS = 0, max_parts = 32;
    float* x = nullptr;
    void *h = nullptr, *qkv = nullptr, *attn = nullptr, *gu = nullptr, *act = nullptr;
    float* logits = nullptr;
    int32_t* sample_ids = nullptr;  // [maxS] sampled ids, followed by [maxS] their logits (fp32 bits)
    float* ws = nullptr;
    size_t ws_floats = 0;
    float* pbuf = nullptr;  // fp32 split-K partials of QKV / O / down GEMMs
    size_t pbuf_floats = 0;
    void* hs = nullptr;     // normalized rows of sampled tokens (LM head input)
    float2* amax = nullptr; // per (vocab tile, row) argmax partials
    float* part_o = nullptr;
    float2* part_ml = nullptr;
    int max_part_rows = 0;
    // step metadata (device + pinned host mirror), int32 words; a ring so the
    // host can plan step k+1 while step k's upload is still in flight
    struct Meta {
        int32_t* d = nullptr;
        int32_t* h = nullptr;
        size_t cap = 0;
        cudaEvent_t done = nullptr;
    };
    static constexpr int kMetaRing = 4;
    Meta meta[kMetaRing];
    int meta_next = 0;
    int32_t* meta_dev = nullptr;
    size_t meta_dev_cap = 0;

    // CUDA graphs of repeated step shapes (decode iterations): key = step signature
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        unsigned long long launches = 0;
    };
    std::map<std::vector<int64_t>, GraphEntry> graphs;
    std::map<std::vector<int64_t>, int> graph_seen;
    bool use_graphs = true;
    bool l2_prefetch_o = false;  // decode attention pulls the O-projection weights into L2 (opt-in)
    std::vector<int> last_sslots;  // call slot of each sampled row of the last step (logits row order)
    void* pin_xbuf = nullptr;    // K6 pin-exchange buffer (grown on demand, reused across runs)
    uint64_t pin_xbuf_bytes = 0;
    // K6 pinned-prefix replication (hk_engine_set_pin_exchange)
    int pin_role = 0;
    hk_pin_exchange_fn pin_fn = nullptr;
    void* pin_user = nullptr;
    void drop_graphs() {
        for (auto& [k, g] : graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
        graph_seen.clear();
    }
    // trie staging
    uint64_t* tok_d = nullptr;
    size_t tok_cap = 0;
    int32_t* match_d = nullptr;
    size_t match_cap = 0;

    // sampled-id harvest ring
    struct Pending {
        cudaEvent_t ev;
        int worker;
        std::vector<int> slots;
        int32_t* host = nullptr;
    };
    std::vector<Pending> pending;
    std::vector<int32_t*> host_bufs;
    std::vector<cudaEvent_t> free_ev;

    KernelClock clock;
    double attn_alg_bytes_step = 0;

    // run statistics (hk_engine_stats_get)
    hk_engine_stats stats{};
    cudaEvent_t ev_run0 = nullptr, ev_pins = nullptr, ev_end = nullptr;
    unsigned long long launches0 = 0;
    bool pins_marked = false;
    void run_begin() {
        if (!ev_run0) {
            HK_CUDA(cudaEventCreate(&ev_run0));
            HK_CUDA(cudaEventCreate(&ev_pins));
            HK_CUDA(cudaEventCreate(&ev_end));
        }
        stats = hk_engine_stats{};
        launches0 = hkd::g_launches;
        pins_marked = false;
        HK_CUDA(cudaEventRecord(ev_run0, st));
    }
    void mark_pins_done() {
        if (pins_marked) return;
        HK_CUDA(cudaEventRecord(ev_pins, st));
        pins_marked = true;
    }
    void run_end() {
        mark_pins_done();
        HK_CUDA(cudaEventRecord(ev_end, st));
        HK_CUDA(cudaEventSynchronize(ev_end));
        float a = 0, b = 0;
        HK_CUDA(cudaEventElapsedTime(&a, ev_run0, ev_pins));
        HK_CUDA(cudaEventElapsedTime(&b, ev_pins, ev_end));
        stats.pin_ms = a;
        stats.iter_ms = b;
        stats.launches = hkd::g_launches - launches0;
    }

    // ---- construction ----
    hk_engine(const hk_model_config& m, const hk_engine_config& c);
    ~hk_engine();
    void init_weights();
    void reset_workers();

    // ---- execution ----
    struct SegIn {
        int slot = -1;
        int start = 0, count = 0;
        bool from_prompt = true, write_kv = true, sample = false;
        int group = -1;        // TRT static group (decode): Plan::static_group of the call's leaf
        int group_pages = 0;   // full pages of that group's static prefix
        const std::vector<int>* table = nullptr;
        const std::vector<uint64_t>* prompt = nullptr;  // host tokens (Token space)
        const std::vector<uint32_t>* ids = nullptr;     // or raw vocab ids
    };
    void step(int w, std::vector<SegIn>& segs, float* logits_out_host = nullptr);
    void harvest(bool all);
    void sync() {
        HK_CUDA(cudaStreamSynchronize(st));
        harvest(true);
        clock.collect();
    }
    void trie_sync(int w, std::vector<hk::TrieOp>& ops, const std::function<const uint64_t*(int)>& key_of);
    void trie_lookup(int w, const std::vector<const std::vector<uint64_t>*>& prompts, std::vector<std::vector<int>>& paths);
    int alloc_slot(int w) {
        Worker& wk = workers[static_cast<size_t>(w)];
        if (wk.free_slots.empty()) throw std::runtime_error("engine: out of call slots (max_calls)");
        int s = wk.free_slots.back();
        wk.free_slots.pop_back();
        wk.slot_tokens[static_cast<size_t>(s)].clear();
        wk.slot_logits[static_cast<size_t>(s)].clear();
        return s;
    }
    void free_slot(int w, int s) { workers[static_cast<size_t>(w)].free_slots.push_back(s); }
    void* kv_layer(int w, int l) const {
        return static_cast<uint8_t*>(workers[static_cast<size_t>(w)].kv) + l * workers[static_cast<size_t>(w)].layer_stride;
    }
};

hk_engine::hk_engine(const hk_model_config& m, const hk_engine_config& c) : mc(m), ec(c) {
    HK_CUDA(cudaSetDevice(c.device));
    int sms = 0;
    HK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    hkd::g_num_sms = sms;
    f32 = m.fp32 != 0;
    esz = f32 ? 4 : 2;
    L = static_cast<int>(m.n_layers);
    d = static_cast<int>(m.d_model);
    H = static_cast<int>(m.n_heads);
    Hkv = static_cast<int>(m.n_kv_heads);
    hd = static_cast<int>(m.head_dim);
    F = static_cast<int>(m.ffn_dim);
    V = static_cast<int>(m.vocab);
    QKV = (H + 2 * Hkv) * hd;
    if (hd != 128) throw std::runtime_error("engine: head_dim must be 128");
    if (H % Hkv) throw std::runtime_error("engine: n_heads must be a multiple of n_kv_heads");
    if (d % 64 || F % 64 || (H * hd) % 64) throw std::runtime_error("engine: d_model/ffn must be multiples of 64");
    if (c.block_tokens == 0 || c.pages_per_worker == 0 || c.n_workers == 0)
        throw std::runtime_error("engine: bad engine config");
    HK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    use_graphs = std::getenv("HK_NO_GRAPHS") == nullptr;
    // opt-in: measured -2% on configs[1] (the prefetch traffic slows the attention more
    // than the O projection gains; profiles/r1_attention.txt)
    l2_prefetch_o = std::getenv("HK_L2_PREFETCH_O") != nullptr;
    hkd::g_pdl = std::getenv("HK_NO_PDL") == nullptr;
    init_weights();

    // rope table (cos, sin) computed in double, stored fp32 — shared with the oracle
    const int half = hd / 2;
    const int max_pos = static_cast<int>(c.max_ctx_tokens) + 1;
    std::vector<float2> rt(static_cast<size_t>(max_pos) * half);
    for (int p = 0; p < max_pos; ++p)
        for (int i = 0; i < half; ++i) {
            const double inv = std::pow(static_cast<double>(m.rope_theta), -2.0 * i / hd);
            const double ang = p * inv;
            rt[static_cast<size_t>(p) * half + i] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
        }
    rope = dalloc<float2>(rt.size());
    HK_CUDA(cudaMemcpy(rope, rt.data(), rt.size() * sizeof(float2), cudaMemcpyHostToDevice));

    // KV pools
    page_bytes_layer = static_cast<size_t>(2) * Hkv * c.block_tokens * hd * esz;
    workers.resize(c.n_workers);
    for (auto& wk : workers) {
        wk.layer_stride = page_bytes_layer * c.pages_per_worker;
        wk.kv = dalloc<uint8_t>(wk.layer_stride * L);
        HK_CUDA(cudaMemsetAsync(wk.kv, 0, wk.layer_stride * L, st));
        if (!f32)
            wk.tm_kv = hkd::make_tmap_2d_bf16(wk.kv, static_cast<uint64_t>(L) * c.pages_per_worker * 2 * Hkv * c.block_tokens,
                                              static_cast<uint64_t>(hd), 64, c.block_tokens);
        // arrival counters [rows][Hkv] followed by the private work-queue head and exit count
        const size_t ctr_n = static_cast<size_t>(c.max_calls * c.n_workers + 16) * Hkv + 4 * static_cast<size_t>(L);
        wk.counters = dalloc<int32_t>(ctr_n);
        HK_CUDA(cudaMemsetAsync(wk.counters, 0, ctr_n * 4, st));
        wk.slot_last = dalloc<int32_t>(c.max_calls);
        HK_CUDA(cudaMemsetAsync(wk.slot_last, 0, c.max_calls * sizeof(int32_t), st));
        hkd::DevTrie& t = wk.trie;
        t.block = static_cast<int>(c.block_tokens);
        t.max_nodes = static_cast<int>(c.pages_per_worker) + 1;
        t.table_size = 1;
        while (t.table_size < 4 * t.max_nodes) t.table_size <<= 1;
        t.parent = dalloc<int32_t>(t.max_nodes);
        t.page = dalloc<int32_t>(t.max_nodes);
        t.phash = dalloc<uint64_t>(t.max_nodes);
        t.keys = dalloc<uint64_t>(static_cast<size_t>(t.max_nodes) * t.block);
        t.tab_key = dalloc<uint64_t>(t.table_size);
        t.tab_node = dalloc<int32_t>(t.table_size);
        wk.slot_tokens.resize(c.max_calls);
        wk.slot_logits.resize(c.max_calls);
    }
    reset_workers();

    // step scratch
    maxT = static_cast<int>(c.max_step_tokens);
    maxS = static_cast<int>(std::min<uint32_t>(c.max_step_tokens, c.max_calls * c.n_workers + 64));
    x = dalloc<float>(static_cast<size_t>(maxT) * d);
    h = dalloc<uint8_t>(static_cast<size_t>(maxT) * std::max(d, F) * esz);
    qkv = dalloc<uint8_t>(static_cast<size_t>(maxT) * QKV * esz);
    attn = dalloc<uint8_t>(static_cast<size_t>(maxT) * H * hd * esz);
    gu = dalloc<uint8_t>(static_cast<size_t>(maxT) * 2 * F * esz);
    act = dalloc<uint8_t>(static_cast<size_t>(maxT) * F * esz);
    logits = dalloc<float>(static_cast<size_t>(maxS) * V);
    sample_ids = dalloc<int32_t>(2 * static_cast<size_t>(maxS));
    ws_floats = static_cast<size_t>(16) * std::max<size_t>(static_cast<size_t>(c.max_calls) * c.n_workers + 64, 256) *
                std::max({QKV, d, 2 * F});
    ws = dalloc<float>(ws_floats);
    pbuf_floats = std::max(static_cast<size_t>(maxT) * std::max(QKV, d) * 2, static_cast<size_t>(16) * 512 * std::max(QKV, d));
    pbuf = dalloc<float>(pbuf_floats);
    if (!f32) hkd::gemm_streamk_reserve(std::max((V + 127) / 128, 4096), 64);
    hs = dalloc<uint8_t>(static_cast<size_t>(maxS) * d * esz);
    amax = dalloc<float2>(static_cast<size_t>((V + 127) / 128) * maxS);
    max_part_rows = static_cast<int>(c.max_calls * c.n_workers) + 16;
    part_o = dalloc<float>(static_cast<size_t>(max_part_rows) * H * max_parts * hd);
    part_ml = dalloc<float2>(static_cast<size_t>(max_part_rows) * H * max_parts);
    HK_CUDA(cudaStreamSynchronize(st));
}

hk_engine::~hk_engine() {
    cudaStreamSynchronize(st);
    cudaFree(wbuf);
    cudaFree(rope);
    for (auto& wk : workers) {
        cudaFree(wk.kv);
        cudaFree(wk.slot_last);
        cudaFree(wk.counters);
        cudaFree(wk.trie.parent);
        cudaFree(wk.trie.page);
        cudaFree(wk.trie.phash);
        cudaFree(wk.trie.keys);
        cudaFree(wk.trie.tab_key);
        cudaFree(wk.trie.tab_node);
    }
    for (void* p : {static_cast<void*>(x), h, qkv, attn, gu, act, static_cast<void*>(logits),
                    static_cast<void*>(sample_ids), static_cast<void*>(ws), static_cast<void*>(part_o),
                    static_cast<void*>(part_ml), static_cast<void*>(tok_d), static_cast<void*>(match_d),
                    static_cast<void*>(pbuf), hs, static_cast<void*>(amax)})
        cudaFree(p);
    drop_graphs();
    for (Meta& mt : meta) {
        if (mt.h) cudaFreeHost(mt.h);
        if (mt.done) cudaEventDestroy(mt.done);
    }
    cudaFree(meta_dev);
    cudaFree(pin_xbuf);
    for (int32_t* b : host_bufs) cudaFreeHost(b);
    cudaStreamDestroy(st);
}

// Tensor ids and scales of the counter-based init (oracle/transformer.py mirrors this).
void hk_engine::init_weights() {
    const size_t n_embed = static_cast<size_t>(V) * d;
    const size_t per_layer = static_cast<size_t>(d) + static_cast<size_t>(QKV) * d + (mc.qkv_bias ? QKV : 0) +
                             static_cast<size_t>(d) * H * hd + d + static_cast<size_t>(2) * F * d +
                             static_cast<size_t>(d) * F;
    const size_t total = n_embed + per_layer * L + d + n_embed;
    wbuf = dalloc<uint8_t>(total * esz + 256 * (8 * L + 4));
    uint8_t* p = static_cast<uint8_t*>(wbuf);
    auto take = [&](size_t n) {
        void* r = p;
        p += (n * esz + 255) / 256 * 256;
        return r;
    };
    const uint64_t seed = mc.seed;
    const float s_d = std::sqrt(3.0f / static_cast<float>(d));
    const float s_o = std::sqrt(3.0f / static_cast<float>(H * hd));
    const float s_f = std::sqrt(3.0f / static_cast<float>(F));
    embed = take(n_embed);
    hkd::init_uniform(embed, f32, n_embed, seed, 1, 1.0f, st);
    layers.resize(L);
    for (int l = 0; l < L; ++l) {
        LayerW& w = layers[l];
        const uint64_t t0 = 16 + 16 * static_cast<uint64_t>(l);
        w.attn_norm = take(d);
        hkd::fill_const(w.attn_norm, f32, d, 1.0f, st);
        w.wqkv = take(static_cast<size_t>(QKV) * d);
        hkd::init_uniform(w.wqkv, f32, static_cast<size_t>(QKV) * d, seed, t0 + 1, s_d, st);
        w.bqkv = nullptr;
        if (mc.qkv_bias) {
            w.bqkv = take(QKV);
            hkd::init_uniform(w.bqkv, f32, QKV, seed, t0 + 2, 0.1f, st);
        }
        w.wo = take(static_cast<size_t>(d) * H * hd);
        hkd::init_uniform(w.wo, f32, static_cast<size_t>(d) * H * hd, seed, t0 + 3, 0.5f * s_o, st);
        w.mlp_norm = take(d);
        hkd::fill_const(w.mlp_norm, f32, d, 1.0f, st);
        w.wgu = take(static_cast<size_t>(2) * F * d);
        hkd::init_uniform_gu(w.wgu, f32, F, d, seed, t0 + 4, s_d, st);  // rows interleaved [64 gate | 64 up]
        w.wd = take(static_cast<size_t>(d) * F);
        hkd::init_uniform(w.wd, f32, static_cast<size_t>(d) * F, seed, t0 + 5, 0.5f * s_f, st);
    }
    final_norm = take(d);
    hkd::fill_const(final_norm, f32, d, 1.0f, st);
    lm_head = take(n_embed);
    hkd::init_uniform(lm_head, f32, n_embed, seed, 2, s_d, st);
}

void hk_engine::reset_workers() {
    for (auto& wk : workers) {
        wk.free_slots.clear();
        for (int s = static_cast<int>(ec.max_calls) - 1; s >= 0; --s) wk.free_slots.push_back(s);
        hkd::DevTrie& t = wk.trie;
        HK_CUDA(cudaMemsetAsync(t.tab_key, 0, t.table_size * sizeof(uint64_t), st));
        HK_CUDA(cudaMemsetAsync(t.parent, 0xff, t.max_nodes * sizeof(int32_t), st));
        wk.trie_tombs = 0;
    }
}

// --------------------------------------------------------------- harvest
void hk_engine::harvest(bool all) {
    size_t k = 0;
    for (; k < pending.size(); ++k) {
        Pending& p = pending[k];
        if (!all && cudaEventQuery(p.ev) == cudaErrorNotReady) break;
        HK_CUDA(cudaEventSynchronize(p.ev));
        Worker& wk = workers[static_cast<size_t>(p.worker)];
        const size_t S = p.slots.size();
        for (size_t i = 0; i < S; ++i)
            if (p.slots[i] >= 0) {
                wk.slot_tokens[static_cast<size_t>(p.slots[i])].push_back(p.host[i]);
                float v;
                std::memcpy(&v, p.host + S + i, 4);
                wk.slot_logits[static_cast<size_t>(p.slots[i])].push_back(v);
            }
        host_bufs.push_back(p.host);
        free_ev.push_back(p.ev);
    }
    pending.erase(pending.begin(), pending.begin() + static_cast<std::ptrdiff_t>(k));
}

// ------------------------------------------------------------------ step
void hk_engine::step(int w, std::vector<SegIn>& segs, float* logits_out_host) {
    Worker& wk = workers[static_cast<size_t>(w)];
    const int block = static_cast<int>(ec.block_tokens);

    // order: prefill/recompute segs first, then decode segs: rows of a TRT
    // static group (the plan's call-level tree, trt.cpp:489-530) together, in
    // admission order; rows without one are grouped by block-table prefix
    std::vector<int> pre, dec, dec_free;
    for (int i = 0; i < static_cast<int>(segs.size()); ++i) {
        if (segs[i].from_prompt)
            pre.push_back(i);
        else
            (segs[i].group >= 0 ? dec : dec_free).push_back(i);
    }
    auto full_pages = [&](const SegIn& s) { return (s.start) / block; };  // pages strictly before the decode token
    std::stable_sort(dec.begin(), dec.end(), [&](int a, int b) { return segs[a].group < segs[b].group; });
    std::sort(dec_free.begin(), dec_free.end(), [&](int a, int b) {
        const auto& ta = *segs[a].table;
        const auto& tb = *segs[b].table;
        const int na = full_pages(segs[a]), nb = full_pages(segs[b]);
        return std::lexicographical_compare(ta.begin(), ta.begin() + na, tb.begin(), tb.begin() + nb);
    });
    const size_t n_trt_rows = dec.size();
    dec.insert(dec.end(), dec_free.begin(), dec_free.end());
    std::vector<int> order = pre;
    order.insert(order.end(), dec.begin(), dec.end());

    int T = 0;
    const int n_pages = static_cast<int>(ec.pages_per_worker);
    for (int i : order) {
        const SegIn& s = segs[i];
        T += s.count;
        // every page the step touches must exist: a bad table would silently
        // read or overwrite another call's KV
        const size_t need = static_cast<size_t>((s.start + s.count + block - 1) / block);
        if (s.table->size() < need)
            throw std::runtime_error("engine: block table shorter than the segment (" + std::to_string(s.table->size()) +
                                     " pages for " + std::to_string(s.start + s.count) + " tokens)");
        for (size_t k = 0; k < need; ++k)
            if ((*s.table)[k] < 0 || (*s.table)[k] >= n_pages)
                throw std::runtime_error("engine: page id out of range: " + std::to_string((*s.table)[k]));
        if (s.slot >= static_cast<int>(ec.max_calls) || (!s.from_prompt && s.slot < 0))
            throw std::runtime_error("engine: bad call slot");
    }
    if (T == 0) return;
    if (T > maxT) throw std::runtime_error("engine: step exceeds max_step_tokens");
    const int T_pre = T - static_cast<int>(dec.size());

    // metadata layout (int32 words)
    std::vector<int32_t> ids(T), pos(T), slots(T), kvw(T), ptab(T), pages;
    std::vector<hkd::AttnItem> items, items_single;  // multi-token (prefill/shared) | single-token (private)
    std::vector<int32_t> nparts(dec.size(), 0);
    std::vector<int32_t> srows, sslots;
    int t = 0;
    int n_pre_items = 0, n_sh_items = 0, n_pv_items = 0;
    double alg_bytes = 0, alg_single = 0;  // algorithmic attention bytes: multi-token items | private items
    const double kv_tok_bytes = 2.0 * Hkv * hd * esz;
    std::vector<hkd::PrefillSegIn> psegs;
    for (int i : pre) {
        SegIn& s = segs[i];
        const int off = static_cast<int>(pages.size());
        pages.insert(pages.end(), s.table->begin(), s.table->end());
        for (int j = 0; j < s.count; ++j) {
            const int p = s.start + j;
            int id;
            if (s.ids)
                id = static_cast<int>((*s.ids)[static_cast<size_t>(p)]);
            else
                id = s.prompt->empty() ? 0 : static_cast<int>(hk::vocab_of((*s.prompt)[static_cast<size_t>(p)], V));
            ids[t + j] = id;
            pos[t + j] = p;
            slots[t + j] = std::max(s.slot, 0);
            kvw[t + j] = s.write_kv ? 1 : 0;
            ptab[t + j] = off;
        }
        if (f32) {
            for (int c = 0; c < s.count; c += 16) {
                const int n = std::min(16, s.count - c);
                for (int kh = 0; kh < Hkv; ++kh)
                    items.push_back(hkd::AttnItem{t + c, n, kh, off, 0, s.start + c + n, 1, -1});
                n_pre_items += Hkv;
            }
        } else {
            psegs.push_back(hkd::PrefillSegIn{t, s.count, s.start, off});  // tensor-core tiles (decode_attn.cu)
        }
        alg_bytes += (s.start + s.count) * kv_tok_bytes + 2.0 * s.count * H * hd * esz;
        if (s.sample) {
            srows.push_back(t + s.count - 1);
            sslots.push_back(s.slot);
        }
        t += s.count;
    }
    // decode groups: maximal runs (in sorted order) sharing >= 4 full pages
    const int KS = 512;   // key split for shared ranges (fp32 path)
    const int KP = 1024;  // key split for private ranges (fp32 path)
    std::vector<hkd::DecodeRowIn> drows;
    std::vector<hkd::DecodeGroupIn> dgroups;
    size_t gi = 0;
    while (gi < dec.size()) {
        size_t gj = gi + 1;
        int lcp = full_pages(segs[dec[gi]]);
        if (gi < n_trt_rows) {
            // TRT group: the members are known from the plan; the shared pages are the
            // group's static prefix, trimmed to what the members' tables really share
            // (a prefix block evicted and recomputed privately is not shared)
            const int g = segs[dec[gi]].group;
            lcp = std::min(lcp, segs[dec[gi]].group_pages);
            while (gj < n_trt_rows && segs[dec[gj]].group == g) {
                const auto& a = *segs[dec[gi]].table;
                const auto& b = *segs[dec[gj]].table;
                const int n = std::min(lcp, full_pages(segs[dec[gj]]));
                int k = 0;
                while (k < n && a[static_cast<size_t>(k)] == b[static_cast<size_t>(k)]) ++k;
                lcp = k;
                ++gj;
            }
            if (lcp < 4) lcp = 0;  // under one 64-key tile: no shared part
        } else {
            while (gj < dec.size()) {
                const auto& a = *segs[dec[gi]].table;
                const auto& b = *segs[dec[gj]].table;
                int n = std::min(lcp, full_pages(segs[dec[gj]]));
                int k = 0;
                while (k < n && a[static_cast<size_t>(k)] == b[static_cast<size_t>(k)]) ++k;
                if (k < 4) break;  // require at least one shared 64-key tile
                lcp = k;
                ++gj;
            }
        }
        const int members = static_cast<int>(gj - gi);
        const int shared_pages = members > 1 ? lcp : 0;
        const int shared_keys = shared_pages * block;
        const int tg0 = t;
        dgroups.push_back(hkd::DecodeGroupIn{tg0 - T_pre, members, shared_pages});
        // per-member rows (+ private items of the fp32 path)
        for (size_t q = gi; q < gj; ++q) {
            SegIn& s = segs[dec[q]];
            const int off = static_cast<int>(pages.size());
            pages.insert(pages.end(), s.table->begin(), s.table->end());
            ids[t] = -1;
            pos[t] = s.start;
            slots[t] = s.slot;
            kvw[t] = 1;
            ptab[t] = off;
            drows.push_back(hkd::DecodeRowIn{off, s.start});
            const int r = t - T_pre;
            if (f32) {
                int part = shared_keys > 0 ? (shared_keys + KS - 1) / KS : 0;
                for (int k0 = shared_keys; k0 < s.start + 1; k0 += KP) {
                    const int k1 = std::min(k0 + KP, s.start + 1);
                    for (int kh = 0; kh < Hkv; ++kh) items_single.push_back(hkd::AttnItem{t, 1, kh, off, k0, k1, 0, part});
                    n_pv_items += Hkv;
                    ++part;
                }
                if (part > max_parts) throw std::runtime_error("engine: too many attention partials");
                nparts[static_cast<size_t>(r)] = part;
            }
            alg_single += (s.start + 1 - shared_keys) * kv_tok_bytes + 2.0 * H * hd * esz;
            if (s.sample) {
                srows.push_back(t);
                sslots.push_back(s.slot);
            }
            ++t;
        }
        if (shared_keys > 0 && f32) {
            const int off0 = ptab[tg0];
            for (int r0 = tg0; r0 < t; r0 += 16) {
                const int n = std::min(16, t - r0);
                int part = 0;
                for (int k0 = 0; k0 < shared_keys; k0 += KS, ++part)
                    for (int kh = 0; kh < Hkv; ++kh)
                        items.push_back(hkd::AttnItem{r0, n, kh, off0, k0, std::min(k0 + KS, shared_keys), 0, part});
                n_sh_items += Hkv * ((shared_keys + KS - 1) / KS);
            }
        }
        if (shared_keys > 0) alg_bytes += shared_keys * kv_tok_bytes;
        gi = gj;
    }
    hkd::DecodePlan dplan;
    double prefill_bytes = 0;
    if (!f32) {
        if (!dec.empty()) {
            hkd::plan_decode_attention(drows, dgroups, H, Hkv, max_parts, hkd::g_num_sms, dplan);
            nparts = dplan.n_parts;
        }
        prefill_bytes = hkd::plan_prefill_attention(psegs, H, Hkv, dplan, pages.data());  // after the decode tiles
    }
    const int S = static_cast<int>(srows.size());
    if (S > maxS) throw std::runtime_error("engine: too many sampled rows in one step");
    if (static_cast<int>(dec.size()) > max_part_rows) throw std::runtime_error("engine: too many decode rows");
    attn_alg_bytes_step = (alg_bytes + alg_single) * L;

    // pack metadata: ids pos slots kvw ptab | pages | nparts | srows sslots | items
    const int n_multi = static_cast<int>(items.size());
    items.insert(items.end(), items_single.begin(), items_single.end());
    const size_t n_items = items.size();
    std::vector<int32_t> cmap(static_cast<size_t>(T), -1);  // batch row -> LM-head row
    for (int k = 0; k < S; ++k) cmap[static_cast<size_t>(srows[static_cast<size_t>(k)])] = k;
    const size_t words = 6 * static_cast<size_t>(T) + pages.size() + nparts.size() + 2 * static_cast<size_t>(S) +
                         n_items * (sizeof(hkd::AttnItem) / 4) + dplan.sh.size() * (sizeof(hkd::ShItem) / 4) +
                         dplan.pv.size() * (sizeof(hkd::PvItem) / 4) + 64;
    Meta& mt = meta[meta_next];
    meta_next = (meta_next + 1) % kMetaRing;
    if (mt.done) HK_CUDA(cudaEventSynchronize(mt.done));  // this slot's previous step has consumed it
    else HK_CUDA(cudaEventCreateWithFlags(&mt.done, cudaEventDisableTiming));
    if (words > mt.cap) {
        if (mt.h) cudaFreeHost(mt.h);
        mt.cap = words * 2;
        HK_CUDA(cudaMallocHost(&mt.h, mt.cap * sizeof(int32_t)));
    }
    // One device metadata buffer for every step (stream order protects it), so
    // a captured step graph can be replayed with fresh metadata.
    if (words > meta_dev_cap) {
        HK_CUDA(cudaStreamSynchronize(st));
        cudaFree(meta_dev);
        meta_dev_cap = words * 2;
        meta_dev = dalloc<int32_t>(meta_dev_cap);
        drop_graphs();
    }
    int32_t* meta_h = mt.h;
    int32_t* meta_d = meta_dev;
    size_t o = 0;
    auto put = [&](const int32_t* src, size_t n) {
        std::memcpy(meta_h + o, src, n * 4);
        const size_t at = o;
        o += n;
        o = (o + 3) & ~size_t(3);  // 16B alignment for items
        return at;
    };
    // layout: every section before `pages` depends only on the step's shape, so a
    // repeated shape (decode) keeps identical device pointers (CUDA graph replay)
    const size_t o_ids = put(ids.data(), T), o_pos = put(pos.data(), T), o_slots = put(slots.data(), T),
                 o_kvw = put(kvw.data(), T), o_ptab = put(ptab.data(), T),
                 o_np = put(nparts.data(), nparts.size()), o_sr = put(srows.data(), S), o_ss = put(sslots.data(), S),
                 o_items = put(reinterpret_cast<const int32_t*>(items.data()), n_items * sizeof(hkd::AttnItem) / 4),
                 o_cmap = put(cmap.data(), cmap.size()),
                 o_sh = put(reinterpret_cast<const int32_t*>(dplan.sh.data()), dplan.sh.size() * sizeof(hkd::ShItem) / 4),
                 o_pv = put(reinterpret_cast<const int32_t*>(dplan.pv.data()), dplan.pv.size() * sizeof(hkd::PvItem) / 4),
                 o_pages = put(pages.data(), pages.size());
    HK_CUDA(cudaMemcpyAsync(meta_d, meta_h, o * 4, cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += o * 4;
    stats.steps += 1;
    stats.step_tokens += static_cast<uint64_t>(T);
    stats.attn_bytes += attn_alg_bytes_step;
    const int32_t* d_ids = meta_d + o_ids;
    const int32_t* d_pos = meta_d + o_pos;
    const int32_t* d_slots = meta_d + o_slots;
    const int32_t* d_kvw = meta_d + o_kvw;
    const int32_t* d_ptab = meta_d + o_ptab;
    const int32_t* d_pages = meta_d + o_pages;
    const int32_t* d_np = meta_d + o_np;
    const int32_t* d_ss = meta_d + o_ss;
    const int32_t* d_cmap = meta_d + o_cmap;
    (void)o_sr;
    const hkd::AttnItem* d_items = reinterpret_cast<const hkd::AttnItem*>(meta_d + o_items);
    const hkd::ShItem* d_sh = reinterpret_cast<const hkd::ShItem*>(meta_d + o_sh);
    const hkd::PvItem* d_pv = reinterpret_cast<const hkd::PvItem*>(meta_d + o_pv);
    // items are packed pre | (per group: private..., shared...) — launch them as one grid
    (void)n_pre_items;
    (void)n_sh_items;
    (void)n_pv_items;

    // max attention partials of a decode row (> 1: the in-kernel merge runs over that many)
    const int any_merge = [&] {
        const int mx = dplan.n_parts.empty() ? 0 : *std::max_element(dplan.n_parts.begin(), dplan.n_parts.end());
        return mx > 1 ? mx : 0;
    }();
    const float eps = mc.rms_eps;
    const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
    // the step's kernel sequence (eager, or recorded once into a CUDA graph)
    // timing experiments only (HK_DEBUG_DOUBLE=qkv,rope,attn,o,rms,gu,down): launch a kernel
    // family twice per layer to measure its marginal cost inside the real PDL/graph pipeline
    static const std::string dbl_env = std::getenv("HK_DEBUG_DOUBLE") ? std::getenv("HK_DEBUG_DOUBLE") : "";
    auto dbl = [&](const char* fam) { return !dbl_env.empty() && dbl_env.find(fam) != std::string::npos && !dec.empty(); };
    // HK_DEBUG_SKIP=rope,attn: drop a kernel family (wrong tokens; decode lengths are fixed, so the
    // schedule is unchanged) to measure what a perfect fusion of it could save
    static const std::string skip_env = std::getenv("HK_DEBUG_SKIP") ? std::getenv("HK_DEBUG_SKIP") : "";
    auto skip = [&](const char* fam) { return !skip_env.empty() && skip_env.find(fam) != std::string::npos && !dec.empty(); };
    hkd::g_trace_prefill_rows = T_pre;
    unsigned long long* attn_trace_pending = nullptr;  // HK_ATTN_TRACE (debug)
    auto enqueue = [&]() {
    int ck = clock.begin(5, st);
    hkd::embed(embed, f32, d, d_ids, d_slots, wk.slot_last, T, x, st);
    hkd::add_rmsnorm(nullptr, 0, x, layers[0].attn_norm, f32, T, d, eps, h, nullptr, nullptr, st);
    clock.end(ck, st, static_cast<double>(T) * d * (esz + 4));
    // GEMMs into fp32 split-K partials (consumers reduce them), or fused epilogues
    auto gemm = [&](const void* W, const void* X, int N, int K, int rows, int epi, void* out, int ldo) -> int {
        const bool tensor_bound = rows > 192;
        const int c = clock.begin(tensor_bound ? 8 : 0, st);
        int sp = 1;
        if (f32) {
            hkd::gemm_f32(static_cast<const float*>(W), static_cast<const float*>(X), N, K, rows,
                          epi == hkd::kEpiPartial ? hkd::kEpiStoreF32 : epi, out, ldo, nullptr, st);
        } else {
            const int max_sp = static_cast<int>(std::max<size_t>(1, pbuf_floats / (static_cast<size_t>(rows) * N)));
            sp = hkd::gemm_bf16(static_cast<const bf16*>(W), static_cast<const bf16*>(X), N, K, rows, epi, out, ldo,
                                nullptr, ws, ws_floats, st, 0, max_sp);
        }
        clock.end(c, st, tensor_bound ? 2.0 * N * K * rows : static_cast<double>(N) * K * esz + static_cast<double>(rows) * K * esz);
        return sp;
    };
    for (int l = 0; l < L; ++l) {
        const LayerW& lw = layers[static_cast<size_t>(l)];
        const hkd::RopeArgs ra{qkv, f32, T, H, Hkv, hd, d_pos, d_kvw, d_ptab, d_pages, rope, kv_layer(w, l), block};
        {
            if (dbl("qkv")) gemm(lw.wqkv, h, QKV, d, T, hkd::kEpiPartial, pbuf, QKV);
            const int sp = gemm(lw.wqkv, h, QKV, d, T, hkd::kEpiPartial, pbuf, QKV);
            const hkd::QkvArgs qa{pbuf, sp, lw.bqkv, ra};
            ck = clock.begin(5, st);
            if (dbl("rope")) hkd::qkv_rope_kv(qa, st);
            if (!skip("rope")) hkd::qkv_rope_kv(qa, st);
            clock.end(ck, st);
        }
        hkd::AttnArgs aa{qkv, f32, H, Hkv, hd, block, d_pos, d_pages, kv_layer(w, l), d_items,
                         n_multi, attn, part_o, part_ml, max_parts, T_pre, scale, 0};
        if (f32) {
            ck = clock.begin(dec.empty() ? 3 : 1, st);
            hkd::attention_partial(aa, st);
            clock.end(ck, st, alg_bytes);
            aa.items = d_items + n_multi;
            aa.n_items = static_cast<int>(n_items) - n_multi;
            aa.single = 1;
            ck = clock.begin(2, st);
            hkd::attention_partial(aa, st);
            clock.end(ck, st, alg_single);
            ck = clock.begin(4, st);
            hkd::attention_merge(part_o, part_ml, d_np, static_cast<int>(dec.size()), T_pre, H, hd, max_parts, attn,
                                 f32, st);
            clock.end(ck, st);
        } else {
            if (!dplan.pv.empty() || !dplan.sh.empty()) {
                const size_t ctr_words = static_cast<size_t>(ec.max_calls * ec.n_workers + 16) * Hkv;
                hkd::DecodeAttnArgs da{static_cast<const bf16*>(qkv), d_pos, H, Hkv, QKV,
                                       static_cast<const bf16*>(kv_layer(w, l)),
                                       static_cast<int>(static_cast<size_t>(l) * ec.pages_per_worker * 2 * Hkv * block),
                                       d_pages, d_sh, static_cast<int>(dplan.sh.size()), dplan.sh_cluster, d_pv,
                                       static_cast<int>(dplan.pv.size()), part_o, part_ml, max_parts, d_np,
                                       wk.counters, static_cast<int>(dec.size()), any_merge,
                                       // per-layer queue state: the queue head may be claimed before
                                       // griddepcontrol.wait, so layers never share it
                                       wk.counters + ctr_words + 4 * l, wk.counters + ctr_words + 4 * l + 1,
                                       wk.counters + ctr_words + 4 * l + 2, 0, T_pre,
                                       static_cast<bf16*>(attn), scale * 1.4426950408889634f, nullptr,
                                       l2_prefetch_o ? lw.wo : nullptr,
                                       static_cast<size_t>(d) * H * hd * esz};
                static const bool kv_ef = !(std::getenv("HK_ATTN_KV_EVICT_FIRST") &&
                                            std::atoi(std::getenv("HK_ATTN_KV_EVICT_FIRST")) == 0);
                da.kv_evict_first = kv_ef ? 1 : 0;
                // debug (HK_ATTN_TRACE="step,layer,path"): the phase stamps of ONE launch inside the
                // real pipeline (run with HK_NO_GRAPHS=1), dumped to path after the step
                static const char* atr = std::getenv("HK_ATTN_TRACE");
                static unsigned long long* atr_buf = nullptr;
                if (atr) {
                    long st_k = -1, ly = -1;
                    std::sscanf(atr, "%ld,%ld", &st_k, &ly);
                    if (static_cast<long>(stats.steps) == st_k && l == ly) {
                        if (!atr_buf) HK_CUDA(cudaMalloc(&atr_buf, 65536 * 8));
                        HK_CUDA(cudaMemsetAsync(atr_buf, 0, 65536 * 8, st));
                        da.trace = atr_buf;
                        attn_trace_pending = atr_buf;
                    }
                }
                da.span = hkd::gemm_trace_slot(
                    -1, static_cast<int>((dplan.shared_bytes + dplan.private_bytes + prefill_bytes) / 1024),
                    static_cast<int>(dec.size()), static_cast<int>(dplan.sh.size()), 0);
                // one launch: decode tiles + private queue + prefill tiles
                ck = clock.begin(dec.empty() ? 3 : 1, st);
                if (dbl("attn")) hkd::decode_attention(da, wk.tm_kv, st);
                if (!skip("attn")) hkd::decode_attention(da, wk.tm_kv, st);
                clock.end(ck, st, dplan.shared_bytes + dplan.private_bytes + prefill_bytes, 1);
            }
        }
        if (dbl("o")) gemm(lw.wo, attn, d, H * hd, T, hkd::kEpiPartial, pbuf, d);
        int sp = gemm(lw.wo, attn, d, H * hd, T, hkd::kEpiPartial, pbuf, d);
        ck = clock.begin(5, st);
        if (dbl("rms")) hkd::add_rmsnorm(pbuf, 0, x, lw.mlp_norm, f32, T, d, eps, h, nullptr, nullptr, st);
        if (!skip("rms")) hkd::add_rmsnorm(pbuf, sp, x, lw.mlp_norm, f32, T, d, eps, h, nullptr, nullptr, st);
        clock.end(ck, st);
        if (f32) {
            gemm(lw.wgu, h, 2 * F, d, T, hkd::kEpiStoreF32, gu, 2 * F);
            ck = clock.begin(5, st);
            hkd::swiglu_interleaved(static_cast<const float*>(gu), T, F, static_cast<float*>(act), st);
            clock.end(ck, st);
        } else {
            if (dbl("gu")) gemm(lw.wgu, h, 2 * F, d, T, hkd::kEpiSwiGLU, act, F);
            gemm(lw.wgu, h, 2 * F, d, T, hkd::kEpiSwiGLU, act, F);  // SwiGLU fused in the epilogue
        }
        if (dbl("down")) gemm(lw.wd, act, d, F, T, hkd::kEpiPartial, pbuf, d);
        sp = gemm(lw.wd, act, d, F, T, hkd::kEpiPartial, pbuf, d);
        const bool last = l + 1 == L;
        ck = clock.begin(5, st);
        if (last || !skip("rms"))
            hkd::add_rmsnorm(pbuf, sp, x, last ? final_norm : layers[static_cast<size_t>(l) + 1].attn_norm, f32, T, d,
                             eps, h, last && S > 0 ? d_cmap : nullptr, last && S > 0 ? hs : nullptr, st);
        clock.end(ck, st);
    }
    if (S > 0) {
        if (f32 || logits_out_host) {
            gemm(lm_head, hs, V, d, S, hkd::kEpiStoreF32, logits, V);
            ck = clock.begin(5, st);
            hkd::argmax_rows(logits, S, V, sample_ids, reinterpret_cast<float*>(sample_ids + maxS), d_ss, wk.slot_last,
                             st);
            clock.end(ck, st);
        } else {
            gemm(lm_head, hs, V, d, S, hkd::kEpiArgmax, amax, V);  // greedy argmax fused in the epilogue
            ck = clock.begin(5, st);
            hkd::argmax_reduce(amax, (V + 127) / 128, S, sample_ids, reinterpret_cast<float*>(sample_ids + maxS), d_ss,
                               wk.slot_last, st);
            clock.end(ck, st);
        }
    }
    };  // enqueue

    const bool graphable = use_graphs && !clock.enabled && !logits_out_host && !f32;
    if (graphable) {
        // everything the recorded kernels depend on besides metadata contents: the
        // metadata offsets, and every scalar baked into a launch (grid sizes, the
        // decode-attention tile / queue counts, cluster mode and merge bound)
        const std::vector<int64_t> sig{w, T, S, T_pre, n_multi, static_cast<int64_t>(n_items),
                                       static_cast<int64_t>(dec.size()), static_cast<int64_t>(o_pages),
                                       static_cast<int64_t>(dplan.sh.size()), static_cast<int64_t>(dplan.pv.size()),
                                       static_cast<int64_t>(dplan.sh_cluster), any_merge};
        auto it = graphs.find(sig);
        if (it != graphs.end()) {
            HK_CUDA(cudaGraphLaunch(it->second.exec, st));
            hkd::g_launches += it->second.launches;
        } else if (graph_seen[sig]++ >= 1) {
            // second occurrence of this shape: record it once, replay from now on
            const unsigned long long l0 = hkd::g_launches;
            cudaGraph_t g;
            HK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            enqueue();
            HK_CUDA(cudaStreamEndCapture(st, &g));
            GraphEntry ge;
            HK_CUDA(cudaGraphInstantiate(&ge.exec, g, 0));
            HK_CUDA(cudaGraphDestroy(g));
            ge.launches = hkd::g_launches - l0;
            HK_CUDA(cudaGraphLaunch(ge.exec, st));
            graphs[sig] = ge;
        } else {
            enqueue();
        }
    } else {
        enqueue();
    }
    if (attn_trace_pending) {
        const char* atr = std::getenv("HK_ATTN_TRACE");
        const char* path = std::strrchr(atr, ',');
        std::vector<unsigned long long> h(65536);
        HK_CUDA(cudaStreamSynchronize(st));
        HK_CUDA(cudaMemcpy(h.data(), attn_trace_pending, h.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = path ? std::fopen(path + 1, "wb") : nullptr) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    if (S > 0) {
        if (logits_out_host)
            HK_CUDA(cudaMemcpyAsync(logits_out_host, logits, static_cast<size_t>(S) * V * 4, cudaMemcpyDeviceToHost, st));
        // harvest ring: D2H of the sampled ids into pinned memory
        Pending p;
        if (host_bufs.empty()) {
            int32_t* hb;
            HK_CUDA(cudaMallocHost(&hb, static_cast<size_t>(2 * maxS) * 4));
            host_bufs.push_back(hb);
        }
        p.host = host_bufs.back();
        host_bufs.pop_back();
        if (free_ev.empty()) {
            cudaEvent_t e;
            HK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            free_ev.push_back(e);
        }
        p.ev = free_ev.back();
        free_ev.pop_back();
        p.worker = w;
        p.slots = sslots;
        last_sslots = sslots;
        // ids, then their logits (read back for the parity checks; 4 B per token)
        HK_CUDA(cudaMemcpyAsync(p.host, sample_ids, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, st));
        HK_CUDA(cudaMemcpyAsync(p.host + S, sample_ids + maxS, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, st));
        stats.d2h_bytes += static_cast<uint64_t>(S) * 8;
        HK_CUDA(cudaEventRecord(p.ev, st));
        pending.push_back(std::move(p));
        if (pending.size() > 64) harvest(false);
    }
    HK_CUDA(cudaEventRecord(mt.done, st));
}

// -------------------------------------------------------------- device trie
void hk_engine::trie_sync(int w, std::vector<hk::TrieOp>& ops, const std::function<const uint64_t*(int)>& key_of) {
    if (ops.empty()) return;
    Worker& wk = workers[static_cast<size_t>(w)];
    const int block = wk.trie.block;
    // compact per node: first op erase => keep the erase; last op create => keep the final create
    std::unordered_map<int, std::pair<int, int>> first_last;
    for (int i = 0; i < static_cast<int>(ops.size()); ++i) {
        auto it = first_last.find(ops[i].node);
        if (it == first_last.end())
            first_last[ops[i].node] = {i, i};
        else
            it->second.second = i;
    }
    std::vector<hkd::TrieOpDev> dev;
    std::vector<uint64_t> keys;
    for (int i = 0; i < static_cast<int>(ops.size()); ++i) {
        const auto& fl = first_last[ops[i].node];
        const hk::TrieOp& op = ops[i];
        if (op.erase && i == fl.first) {
            dev.push_back({op.node, op.parent, op.page, 1, op.phash});
            keys.insert(keys.end(), block, 0);
            ++wk.trie_tombs;
        } else if (!op.erase && i == fl.second) {
            dev.push_back({op.node, op.parent, op.page, 0, op.phash});
            const uint64_t* k = key_of(op.node);
            keys.insert(keys.end(), k, k + block);
        }
    }
    ops.clear();
    if (dev.empty()) return;
    // stage ops + keys in one device buffer (reuse tok_d)
    const size_t op_words = dev.size() * sizeof(hkd::TrieOpDev) / 8;
    const size_t need = op_words + keys.size();
    if (need > tok_cap) {
        HK_CUDA(cudaStreamSynchronize(st));
        cudaFree(tok_d);
        tok_cap = need * 2;
        tok_d = dalloc<uint64_t>(tok_cap);
    }
    HK_CUDA(cudaStreamSynchronize(st));
    HK_CUDA(cudaMemcpyAsync(tok_d, dev.data(), op_words * 8, cudaMemcpyHostToDevice, st));
    HK_CUDA(cudaMemcpyAsync(tok_d + op_words, keys.data(), keys.size() * 8, cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += (op_words + keys.size()) * 8;
    const int c = clock.begin(6, st);
    hkd::trie_apply(wk.trie, reinterpret_cast<const hkd::TrieOpDev*>(tok_d), tok_d + op_words,
                    static_cast<int>(dev.size()), st);
    clock.end(c, st);
    HK_CUDA(cudaStreamSynchronize(st));
}

void hk_engine::trie_lookup(int w, const std::vector<const std::vector<uint64_t>*>& prompts,
                            std::vector<std::vector<int>>& paths) {
    Worker& wk = workers[static_cast<size_t>(w)];
    const int n = static_cast<int>(prompts.size());
    std::vector<uint64_t> offs(static_cast<size_t>(n) + 1, 0);
    int stride = 1;
    for (int i = 0; i < n; ++i) {
        offs[static_cast<size_t>(i) + 1] = offs[static_cast<size_t>(i)] + prompts[static_cast<size_t>(i)]->size();
        stride = std::max(stride, static_cast<int>(prompts[static_cast<size_t>(i)]->size()) / wk.trie.block);
    }
    const size_t need = offs[static_cast<size_t>(n)] + offs.size();
    if (need > tok_cap) {
        HK_CUDA(cudaStreamSynchronize(st));
        cudaFree(tok_d);
        tok_cap = need * 2;
        tok_d = dalloc<uint64_t>(tok_cap);
    }
    const size_t mneed = static_cast<size_t>(n) * (1 + 2 * stride);
    if (mneed > match_cap) {
        HK_CUDA(cudaStreamSynchronize(st));
        cudaFree(match_d);
        match_cap = mneed * 2;
        match_d = dalloc<int32_t>(match_cap);
    }
    std::vector<uint64_t> flat;
    flat.reserve(offs[static_cast<size_t>(n)]);
    for (auto* p : prompts) flat.insert(flat.end(), p->begin(), p->end());
    HK_CUDA(cudaStreamSynchronize(st));
    HK_CUDA(cudaMemcpyAsync(tok_d, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st));
    HK_CUDA(cudaMemcpyAsync(tok_d + flat.size(), offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, st));
    int32_t* d_matched = match_d;
    int32_t* d_path = match_d + n;
    int32_t* d_pt = d_path + static_cast<size_t>(n) * stride;
    const int c = clock.begin(6, st);
    hkd::trie_match(wk.trie, tok_d, tok_d + flat.size(), n, d_matched, d_path, d_pt, stride, st);
    clock.end(c, st);
    std::vector<int32_t> hm(static_cast<size_t>(n)), hp(static_cast<size_t>(n) * stride);
    HK_CUDA(cudaMemcpyAsync(hm.data(), d_matched, hm.size() * 4, cudaMemcpyDeviceToHost, st));
    HK_CUDA(cudaMemcpyAsync(hp.data(), d_path, hp.size() * 4, cudaMemcpyDeviceToHost, st));
    HK_CUDA(cudaStreamSynchronize(st));
    stats.h2d_bytes += (flat.size() + offs.size()) * 8;
    stats.d2h_bytes += (hm.size() + hp.size()) * 4;
    paths.assign(static_cast<size_t>(n), {});
    for (int i = 0; i < n; ++i)
        paths[static_cast<size_t>(i)].assign(hp.begin() + static_cast<std::ptrdiff_t>(i) * stride,
                                             hp.begin() + static_cast<std::ptrdiff_t>(i) * stride + hm[static_cast<size_t>(i)]);
}

// ------------------------------------------------------------ device body
namespace hk {

class DeviceBody : public LlmBody {
  public:
    DeviceBody(hk_engine* e, const Plan& plan, const SimConfig& cfg, int only_worker) : e_(e) {
        // one pool per schedule worker; a single pool only serves a single device-driving
        // worker (W == 1, or only_worker mode) — two workers on one pool would hand out the
        // same page ids and device-trie node ids and overwrite each other's KV
        const bool one_driver = cfg.workers.size() == 1 || only_worker >= 0;
        if (cfg.workers.size() != e->workers.size() && !(e->workers.size() == 1 && one_driver))
            throw std::runtime_error("hk_simulate: engine has " + std::to_string(e->workers.size()) +
                                     " worker pools but the schedule has " + std::to_string(cfg.workers.size()) +
                                     " workers");
        for (const auto& w : cfg.workers)
            if (w.block != e->ec.block_tokens)
                throw std::runtime_error("hk_simulate: SimWorkerConfig::block differs from the engine page size");
        e_->sync();
        e_->reset_workers();
        e_->run_begin();
        (void)plan;
    }
    void begin_iteration(std::uint64_t, const std::vector<std::pair<int, LiveCall*>>&) override {
        e_->mark_pins_done();
        for (std::size_t w = 0; w < finished_slots_.size(); ++w) release_slots(static_cast<int>(w));
    }
    bool uses_pages() const override { return true; }
    int pages_per_worker(int) const override { return static_cast<int>(e_->ec.pages_per_worker); }
    bool device_lookup() const override { return e_->ec.use_device_trie != 0; }

    void precompute_pins(int w, const std::vector<TokenSeq>& pins, const std::vector<std::vector<int>>& pin_pages,
                         const std::vector<std::size_t>& first_new) override {
        const int block = static_cast<int>(e_->ec.block_tokens);
        const int role = e_->pin_fn ? e_->pin_role : 0;
        if (role != 2) {
            for (std::size_t i = 0; i < pins.size(); ++i) {
                const int start = static_cast<int>(first_new[i]) * block;
                const int len = static_cast<int>(pins[i].size());
                for (int c0 = start; c0 < len; c0 += e_->maxT) {
                    std::vector<hk_engine::SegIn> segs(1);
                    segs[0].slot = 0;
                    segs[0].start = c0;
                    segs[0].count = std::min(e_->maxT, len - c0);
                    segs[0].table = &pin_pages[i];
                    segs[0].prompt = &pins[i];
                    e_->step(pw(w), segs);
                }
            }
        }
        e_->sync();
        if (role == 0) return;
        // K6: the newly pinned pages, in pin / block order, leave (source) or
        // arrive (receiver) through one device buffer
        std::vector<int32_t> pages;
        for (std::size_t i = 0; i < pins.size(); ++i)
            for (std::size_t j = first_new[i]; j < pin_pages[i].size(); ++j) pages.push_back(pin_pages[i][j]);
        if (pages.empty()) return;
        const uint64_t bytes = static_cast<uint64_t>(pages.size()) * hk_engine_page_bytes(e_);
        // one exchange buffer per engine, kept across runs (no cudaMalloc/cudaFree in a timed run)
        if (e_->pin_xbuf_bytes < bytes) {
            e_->sync();
            cudaFree(e_->pin_xbuf);
            e_->pin_xbuf = nullptr;
            HK_CUDA(cudaMalloc(&e_->pin_xbuf, bytes));
            e_->pin_xbuf_bytes = bytes;
        }
        void* buf = e_->pin_xbuf;
        auto done = [&](int rc, const char* what) {
            if (rc != 0) {
                throw std::runtime_error(std::string("simulate: pin exchange ") + what + " failed for worker " +
                                         std::to_string(w) + (rc < 0 ? ": " + std::string(hk_last_error()) : ""));
            }
        };
        if (role == 1) {
            done(hk_pool_gather(e_, pw(w), pages.data(), pages.size(), buf), "gather");
            done(e_->pin_fn(e_->pin_user, w, buf, bytes), "callback");
        } else {
            done(e_->pin_fn(e_->pin_user, w, buf, bytes), "callback");
            done(hk_pool_scatter(e_, pw(w), buf, pages.data(), pages.size()), "scatter");
        }
        e_->sync();
    }
    void sync_trie(int w, KvTree& tree) override {
        e_->trie_sync(pw(w), tree.journal(), [&tree](int node) { return tree.node_key(node); });
    }
    void lookup_batch(int w, const std::vector<const TokenSeq*>& prompts, std::vector<std::vector<int>>& paths) override {
        e_->trie_lookup(pw(w), prompts, paths);
    }
    void on_admit(int w, LiveCall& lc) override { lc.slot = e_->alloc_slot(pw(w)); }
    void run_step(StepPlan& sp) override {
        std::vector<hk_engine::SegIn> segs;
        segs.reserve(sp.segs.size());
        for (auto& s : sp.segs) {
            hk_engine::SegIn in;
            in.slot = s.call->slot;
            in.start = static_cast<int>(s.start);
            in.count = static_cast<int>(s.count);
            in.from_prompt = s.from_prompt;
            in.write_kv = s.write_kv;
            in.sample = s.sample;
            in.group = s.group;
            in.group_pages = static_cast<int>(s.group_tokens / static_cast<std::size_t>(e_->ec.block_tokens));
            in.table = &s.table;
            in.prompt = &s.call->prompt;
            segs.push_back(in);
        }
        e_->step(pw(sp.worker), segs);
        release_slots(sp.worker);
    }
    TokenSeq take_output(int w, LiveCall& lc, double, bool) override {
        auto& toks = e_->workers[static_cast<size_t>(pw(w))].slot_tokens[static_cast<size_t>(lc.slot)];
        if (toks.size() < lc.out_len) e_->harvest(true);
        if (toks.size() < lc.out_len) {
            HK_CUDA(cudaStreamSynchronize(e_->st));
            e_->harvest(true);
        }
        TokenSeq out;
        out.reserve(lc.out_len);
        for (std::size_t i = 0; i < lc.out_len && i < toks.size(); ++i)
            out.push_back(gen_token(static_cast<std::uint32_t>(toks[i]), static_cast<std::uint32_t>(e_->V)));
        return out;
    }
    std::vector<float> take_logits(int w, LiveCall& lc) override {
        const auto& v = e_->workers[static_cast<size_t>(pw(w))].slot_logits[static_cast<size_t>(lc.slot)];
        return std::vector<float>(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(std::min(v.size(), lc.out_len)));
    }
    void on_finish(int w, LiveCall& lc) override {
        // The call's last decode token (it writes the KV of the final output
        // token, read back by the completion insert) is still in this
        // worker-iteration's step: keep its slot until that step is issued.
        if (lc.slot < 0) return;
        if (finished_slots_.size() <= static_cast<std::size_t>(w)) finished_slots_.resize(static_cast<std::size_t>(w) + 1);
        finished_slots_[static_cast<std::size_t>(w)].push_back(lc.slot);
    }
    void finish_run() override {
        e_->run_end();
        e_->sync();
    }

  private:
    // engine pool of schedule worker w (a single pool serves one-worker mode)
    int pw(int w) const { return e_->workers.size() == 1 ? 0 : w; }
    void release_slots(int w) {
        if (static_cast<std::size_t>(w) >= finished_slots_.size()) return;
        for (int s : finished_slots_[static_cast<std::size_t>(w)]) e_->free_slot(pw(w), s);
        finished_slots_[static_cast<std::size_t>(w)].clear();
    }
    hk_engine* e_;
    std::vector<std::vector<int>> finished_slots_;
};

std::unique_ptr<LlmBody> make_device_body(hk_engine* e, const Plan& plan, const SimConfig& cfg, int only_worker) {
    return std::make_unique<DeviceBody>(e, plan, cfg, only_worker);
}

}  // namespace hk

// ------------------------------------------------------------------ C-ABI
namespace {
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& ex) {
        hk::set_error(ex.what());
        return -1;
    }
}
}  // namespace

extern "C" {

hk_engine* hk_engine_create(const hk_model_config* m, const hk_engine_config* c) {
    try {
        if (!m || !c) throw std::runtime_error("hk_engine_create: null config");
        return new hk_engine(*m, *c);
    } catch (const std::exception& ex) {
        hk::set_error(ex.what());
        return nullptr;
    }
}

void hk_engine_destroy(hk_engine* e) { delete e; }

int hk_engine_set_graphs(hk_engine* e, int on) {
    return guarded([&] { e->use_graphs = on != 0 && std::getenv("HK_NO_GRAPHS") == nullptr; });
}

int hk_engine_set_pin_exchange(hk_engine* e, int role, hk_pin_exchange_fn fn, void* user) {
    return guarded([&] {
        if (role < 0 || role > 2) throw std::runtime_error("hk_engine_set_pin_exchange: role must be 0, 1 or 2");
        if (role != 0 && !fn) throw std::runtime_error("hk_engine_set_pin_exchange: roles 1 and 2 need a callback");
        e->pin_role = role;
        e->pin_fn = role ? fn : nullptr;
        e->pin_user = user;
    });
}

size_t hk_engine_page_bytes(const hk_engine* e) { return e ? e->page_bytes_layer * e->L : 0; }

int hk_engine_reset(hk_engine* e) {
    return guarded([&] {
        e->sync();
        e->reset_workers();
        e->clock.reset();
    });
}

int hk_pool_gather(hk_engine* e, int w, const int32_t* pages, size_t n, void* dst) {
    return guarded([&] {
        int32_t* dp = dalloc<int32_t>(n);
        HK_CUDA(cudaMemcpyAsync(dp, pages, n * 4, cudaMemcpyHostToDevice, e->st));
        const int c = e->clock.begin(7, e->st);
        hkd::pool_gather(e->workers.at(static_cast<size_t>(w)).kv, e->workers[static_cast<size_t>(w)].layer_stride,
                         e->L, e->page_bytes_layer, dp, static_cast<int>(n), dst, e->st);
        e->clock.end(c, e->st, 2.0 * n * e->page_bytes_layer * e->L);
        HK_CUDA(cudaStreamSynchronize(e->st));
        cudaFree(dp);
    });
}

int hk_pool_scatter(hk_engine* e, int w, const void* src, const int32_t* pages, size_t n) {
    return guarded([&] {
        int32_t* dp = dalloc<int32_t>(n);
        HK_CUDA(cudaMemcpyAsync(dp, pages, n * 4, cudaMemcpyHostToDevice, e->st));
        const int c = e->clock.begin(7, e->st);
        hkd::pool_scatter(e->workers.at(static_cast<size_t>(w)).kv, e->workers[static_cast<size_t>(w)].layer_stride,
                          e->L, e->page_bytes_layer, dp, static_cast<int>(n), src, e->st);
        e->clock.end(c, e->st, 2.0 * n * e->page_bytes_layer * e->L);
        HK_CUDA(cudaStreamSynchronize(e->st));
        cudaFree(dp);
    });
}

int hk_pool_copy(hk_engine* e, int w, const int32_t* src, const int32_t* dst, size_t n) {
    return guarded([&] {
        int32_t* dp = dalloc<int32_t>(2 * n);
        HK_CUDA(cudaMemcpyAsync(dp, src, n * 4, cudaMemcpyHostToDevice, e->st));
        HK_CUDA(cudaMemcpyAsync(dp + n, dst, n * 4, cudaMemcpyHostToDevice, e->st));
        const int c = e->clock.begin(7, e->st);
        hkd::pool_copy(e->workers.at(static_cast<size_t>(w)).kv, e->workers[static_cast<size_t>(w)].layer_stride, e->L,
                       e->page_bytes_layer, dp, dp + n, static_cast<int>(n), e->st);
        e->clock.end(c, e->st, 2.0 * n * e->page_bytes_layer * e->L);
        HK_CUDA(cudaStreamSynchronize(e->st));
        cudaFree(dp);
    });
}

int hk_trie_apply(hk_engine* e, int w, const hk_trie_op* ops, size_t n) {
    return guarded([&] {
        std::vector<hk::TrieOp> v;
        std::unordered_map<int, const uint64_t*> keys;
        for (size_t i = 0; i < n; ++i) {
            v.push_back(hk::TrieOp{ops[i].node, ops[i].parent, ops[i].page, ops[i].erase != 0, ops[i].phash});
            if (!ops[i].erase) keys[ops[i].node] = ops[i].key;
        }
        e->trie_sync(w, v, [&](int node) { return keys.at(node); });
    });
}

int hk_trie_match(hk_engine* e, int w, const uint64_t* tokens, const uint64_t* offsets, size_t n, int32_t* matched,
                  int32_t* node_path, int32_t* page_table, size_t stride) {
    return guarded([&] {
        std::vector<std::vector<uint64_t>> ps(n);
        std::vector<const std::vector<uint64_t>*> pp;
        for (size_t i = 0; i < n; ++i) {
            ps[i].assign(tokens + offsets[i], tokens + offsets[i + 1]);
            pp.push_back(&ps[i]);
        }
        std::vector<std::vector<int>> paths;
        e->trie_lookup(w, pp, paths);
        for (size_t i = 0; i < n; ++i) {
            matched[i] = static_cast<int32_t>(paths[i].size());
            for (size_t k = 0; k < paths[i].size() && k < stride; ++k) {
                node_path[i * stride + k] = paths[i][k];
                if (page_table) {
                    int32_t pg = 0;
                    HK_CUDA(cudaMemcpy(&pg, e->workers[static_cast<size_t>(w)].trie.page + paths[i][k], 4,
                                       cudaMemcpyDeviceToHost));
                    page_table[i * stride + k] = pg;
                }
            }
        }
    });
}

int hk_generate(hk_engine* e, const uint32_t* ids, size_t n, size_t n_new, uint32_t* out, float* logits) {
    return guarded([&] {
        if (n == 0) throw std::runtime_error("hk_generate: empty prompt");
        const int block = static_cast<int>(e->ec.block_tokens);
        const size_t total = n + n_new;
        if (static_cast<size_t>((total + block - 1) / block) > e->ec.pages_per_worker)
            throw std::runtime_error("hk_generate: sequence does not fit the page pool");
        std::vector<int> table;
        for (int p = 0; p < static_cast<int>((total + block - 1) / block); ++p) table.push_back(p);
        std::vector<uint32_t> seq(ids, ids + n);
        const int slot = e->alloc_slot(0);
        e->harvest(true);
        e->workers[0].slot_tokens[static_cast<size_t>(slot)].clear();
        const size_t V = static_cast<size_t>(e->V);
        // prefill in chunks; sample from the last prompt position
        for (size_t c0 = 0; c0 < n; c0 += static_cast<size_t>(e->maxT)) {
            std::vector<hk_engine::SegIn> segs(1);
            segs[0].slot = slot;
            segs[0].start = static_cast<int>(c0);
            segs[0].count = static_cast<int>(std::min(n - c0, static_cast<size_t>(e->maxT)));
            segs[0].table = &table;
            segs[0].ids = &seq;
            segs[0].sample = c0 + segs[0].count == n && n_new > 0;
            e->step(0, segs, segs[0].sample && logits ? logits : nullptr);
        }
        for (size_t k = 1; k < n_new; ++k) {
            std::vector<hk_engine::SegIn> segs(1);
            segs[0].slot = slot;
            segs[0].start = static_cast<int>(n + k - 1);
            segs[0].count = 1;
            segs[0].from_prompt = false;
            segs[0].sample = true;
            segs[0].table = &table;
            e->step(0, segs, logits ? logits + k * V : nullptr);
        }
        e->sync();
        auto& toks = e->workers[0].slot_tokens[static_cast<size_t>(slot)];
        for (size_t k = 0; k < n_new; ++k) out[k] = static_cast<uint32_t>(toks.at(k));
        e->free_slot(0, slot);
    });
}

// ---------------------------------------------------------- step-level C ABI
// one ragged forward of a worker (hk_step), pin prefill and the
// K6 page broadcast as stand-alone calls, for hosts that drive their own loop.
int hk_slot_alloc(hk_engine* e, int w) {
    try {
        if (w < 0 || w >= static_cast<int>(e->workers.size())) throw std::runtime_error("hk_slot_alloc: bad worker");
        const int slot = e->alloc_slot(w);
        e->harvest(true);
        e->workers[static_cast<size_t>(w)].slot_tokens[static_cast<size_t>(slot)].clear();
        e->workers[static_cast<size_t>(w)].slot_logits[static_cast<size_t>(slot)].clear();
        return slot;
    } catch (const std::exception& ex) {
        hk::set_error(ex.what());
        return -1;
    }
}

int hk_slot_free(hk_engine* e, int w, int slot) {
    return guarded([&] {
        if (w < 0 || w >= static_cast<int>(e->workers.size())) throw std::runtime_error("hk_slot_free: bad worker");
        if (slot < 0 || slot >= static_cast<int>(e->ec.max_calls)) throw std::runtime_error("hk_slot_free: bad slot");
        e->sync();
        e->free_slot(w, slot);
    });
}

int hk_step(hk_engine* e, int w, const hk_step_seg* in, size_t n, int32_t* sampled, float* logits) {
    return guarded([&] {
        if (w < 0 || w >= static_cast<int>(e->workers.size())) throw std::runtime_error("hk_step: bad worker");
        std::vector<std::vector<int>> tables(n);
        std::vector<std::vector<uint32_t>> ids(n);
        std::vector<hk_engine::SegIn> segs(n);
        std::vector<int> seen;
        for (size_t i = 0; i < n; ++i) {
            const hk_step_seg& g = in[i];
            if (g.count <= 0 || g.start < 0) throw std::runtime_error("hk_step: empty segment or negative start");
            if (!g.pages || g.n_pages <= 0) throw std::runtime_error("hk_step: segment without a block table");
            if (!g.ids && g.count != 1) throw std::runtime_error("hk_step: a decode segment (ids == NULL) has count 1");
            if ((g.sample || !g.ids) && g.slot < 0) throw std::runtime_error("hk_step: sampling / decode needs a call slot");
            if (g.sample) {
                if (std::find(seen.begin(), seen.end(), g.slot) != seen.end())
                    throw std::runtime_error("hk_step: a slot samples at most once per step");
                seen.push_back(g.slot);
            }
            tables[i].assign(g.pages, g.pages + g.n_pages);
            hk_engine::SegIn& s = segs[i];
            s.slot = g.slot;
            s.start = g.start;
            s.count = g.count;
            s.sample = g.sample != 0;
            s.write_kv = g.write_kv != 0;
            s.table = &tables[i];
            if (g.ids) {
                ids[i].assign(static_cast<size_t>(g.start) + g.count, 0u);
                std::copy(g.ids, g.ids + g.count, ids[i].begin() + g.start);
                s.ids = &ids[i];
                s.from_prompt = true;
            } else {
                s.from_prompt = false;
            }
        }
        const size_t V = static_cast<size_t>(e->V);
        std::vector<float> lg(logits ? seen.size() * V : 0);
        e->step(w, segs, logits && !seen.empty() ? lg.data() : nullptr);
        e->sync();
        auto& wk = e->workers[static_cast<size_t>(w)];
        for (size_t i = 0; i < n; ++i) {
            if (!in[i].sample) {
                if (sampled) sampled[i] = -1;
                continue;
            }
            const auto& toks = wk.slot_tokens[static_cast<size_t>(in[i].slot)];
            if (sampled) sampled[i] = toks.empty() ? -1 : static_cast<int32_t>(toks.back());
            if (logits) {
                const auto it = std::find(e->last_sslots.begin(), e->last_sslots.end(), in[i].slot);
                if (it == e->last_sslots.end()) throw std::runtime_error("hk_step: sampled row not found");
                std::copy_n(lg.begin() + static_cast<std::ptrdiff_t>((it - e->last_sslots.begin()) * V), V,
                            logits + i * V);
            }
        }
    });
}

int hk_pin_prefill(hk_engine* e, int w, const uint32_t* ids, size_t n, const int32_t* pages, size_t n_pages) {
    return guarded([&] {
        if (w < 0 || w >= static_cast<int>(e->workers.size())) throw std::runtime_error("hk_pin_prefill: bad worker");
        const size_t block = e->ec.block_tokens;
        if (n_pages * block < n) throw std::runtime_error("hk_pin_prefill: pages do not cover the sequence");
        std::vector<int> table(pages, pages + n_pages);
        std::vector<uint32_t> seq(ids, ids + n);
        for (size_t c0 = 0; c0 < n; c0 += static_cast<size_t>(e->maxT)) {
            std::vector<hk_engine::SegIn> segs(1);
            segs[0].slot = -1;
            segs[0].start = static_cast<int>(c0);
            segs[0].count = static_cast<int>(std::min(n - c0, static_cast<size_t>(e->maxT)));
            segs[0].table = &table;
            segs[0].ids = &seq;
            e->step(w, segs);
        }
        e->sync();
    });
}

int hk_kv_broadcast(hk_engine* e, int w, int role, const int32_t* pages, size_t n, hk_pin_exchange_fn fn, void* user) {
    return guarded([&] {
        if (role != 1 && role != 2) throw std::runtime_error("hk_kv_broadcast: role must be 1 (source) or 2 (receiver)");
        if (!fn) throw std::runtime_error("hk_kv_broadcast: no exchange function");
        if (n == 0) return;
        const uint64_t bytes = static_cast<uint64_t>(n) * hk_engine_page_bytes(e);
        if (e->pin_xbuf_bytes < bytes) {
            e->sync();
            cudaFree(e->pin_xbuf);
            e->pin_xbuf = nullptr;
            HK_CUDA(cudaMalloc(&e->pin_xbuf, bytes));
            e->pin_xbuf_bytes = bytes;
        }
        void* buf = e->pin_xbuf;
        auto check = [&](int rc, const char* what) {
            if (rc != 0) throw std::runtime_error(std::string("hk_kv_broadcast: ") + what + " failed");
        };
        if (role == 1) {
            check(hk_pool_gather(e, w, pages, n, buf), "gather");
            check(fn(user, w, buf, bytes), "exchange callback");
        } else {
            e->sync();
            check(fn(user, w, buf, bytes), "exchange callback");
            check(hk_pool_scatter(e, w, buf, pages, n), "scatter");
        }
        e->sync();
    });
}

double hk_engine_kernel_ms(const hk_engine* ce, const char* family, uint64_t* launches, double* bytes) {
    hk_engine* e = const_cast<hk_engine*>(ce);
    try {
        e->clock.collect();
    } catch (...) {
        return -1;
    }
    for (int i = 0; i < KernelClock::kFamilies; ++i)
        if (std::strcmp(e->clock.names[i], family) == 0) {
            if (launches) *launches = e->clock.launches[i];
            if (bytes) *bytes = e->clock.bytes[i];
            return e->clock.ms[i];
        }
    return -1;
}

int hk_engine_stats_get(const hk_engine* e, hk_engine_stats* out) {
    if (!e || !out) return -1;
    *out = e->stats;
    return 0;
}

int hk_engine_profile(hk_engine* e, int enable) {
    return guarded([&] {
        e->clock.reset();
        e->clock.enabled = enable != 0;
    });
}

}  // extern "C"
