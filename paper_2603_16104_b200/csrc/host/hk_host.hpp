// Host side of the B200 LLM-as-operator executor (C++ above the C-ABI).
//
// Restates the semantics of the reference's L4 execution layer
// (/root/reference/proj/src/simulator.cpp, evaluator.cpp, tokens.cpp) on a
// flattened plan (HKPLAN01, include/helium_b200.h) so it can be linked without
// the reference's planner types. The LLM body is pluggable: synthetic
// (synth_llm_output, evaluator.cpp:53-58) or the device transformer.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace hk {

using Token = std::uint64_t;
using TokenSeq = std::vector<Token>;
using NodeId = std::int64_t;

// ---------------------------------------------------------------- tokens.cpp
constexpr std::uint64_t kFnvOffset = 0xcbf29ce484222325ull;
std::uint64_t fnv1a64(const void* data, std::size_t len, std::uint64_t seed = kFnvOffset);
std::uint64_t hash_combine(std::uint64_t h, std::uint64_t v);
std::uint64_t hash_tokens(const Token* t, std::size_t n, std::uint64_t seed = kFnvOffset);
std::uint64_t splitmix64(std::uint64_t x);

std::size_t synth_output_len(const TokenSeq& prompt, double len_out, std::uint64_t seed, bool stochastic);
TokenSeq synth_output(const TokenSeq& prompt, double len_out, std::uint64_t seed, bool stochastic);
std::size_t synth_llm_len(const TokenSeq& prompt, double len_out, bool deterministic,
                          std::uint64_t seed, bool stochastic);
TokenSeq synth_llm_output(const TokenSeq& prompt, double len_out, bool deterministic,
                          std::uint64_t seed, bool stochastic);

// Model-mode token mapping (new definitions):
// prompt Token -> vocab id is tok % V; a generated vocab id maps to a Token in
// a tagged hash space whose residue mod V is the id itself, so generated text
// re-enters the model as the same id.
std::uint32_t vocab_of(Token t, std::uint32_t vocab);
Token gen_token(std::uint32_t id, std::uint32_t vocab);

// ------------------------------------------------------------------- plan
enum class Kind : std::uint32_t { kBound = 0, kOutput = 1, kLambda = 2, kFormat = 3, kLlm = 4 };

struct PlanNode {
    NodeId id = -1;
    Kind kind = Kind::kBound;
    bool deterministic = true;
    bool has_profile = false;
    double len_out = 0;
    std::vector<std::int64_t> a;  // kind-specific payload (see header doc)
};

struct TreePart {
    bool is_static = true;
    std::int64_t v = -1;  // span index (static) or source node (placeholder)
    std::int64_t q = -1;
};

struct TreeNode {
    int parent = -1;
    bool is_leaf = false;
    NodeId op = -1;
    int query = -1;
    std::vector<TreePart> parts;
    std::vector<int> preds;
};

struct CallId {
    NodeId op = -1;
    int query = 0;
    friend bool operator<(const CallId& a, const CallId& b) {
        return a.op != b.op ? a.op < b.op : a.query < b.query;
    }
    friend bool operator==(const CallId& a, const CallId& b) { return a.op == b.op && a.query == b.query; }
};

struct Plan {
    std::size_t batch = 1;
    std::vector<Token> pool;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> spans;
    std::map<NodeId, PlanNode> nodes;
    std::vector<NodeId> outputs;
    std::vector<TreeNode> tree;
    std::vector<int> leaves;
    std::map<CallId, int> leaf_index;
    std::vector<std::vector<CallId>> sigma;
    // Shared-prefix groups from the call-level TRT (trt.cpp:489-530), per tree
    // node: for a leaf, the deepest ancestor whose whole root path is static
    // text (-1: none) and the token length of that static path. Leaves with
    // the same group share those prompt tokens, hence (when cached) the same
    // KV pages: the decode-attention planner takes its prefix-shared groups
    // from here instead of rediscovering them from block tables every step.
    std::vector<int> static_group;
    std::vector<std::size_t> static_group_tokens;
    std::size_t sigma_offset = 0;  // byte offset of the schedule section in the blob
    std::size_t sig_offset = 0;    // byte offset after the schedule (optional signature section)
    // Optional HKSIG001 section: the reference's per-(node, query) content
    // signatures and taint flags (compute_signatures, signature.cpp:29-104),
    // the prompt-cache keys.
    bool has_sigs = false;
    std::map<NodeId, std::vector<std::uint64_t>> sig;
    std::map<NodeId, bool> tainted;

    const Token* span_ptr(std::int64_t s) const { return pool.data() + spans.at(static_cast<std::size_t>(s)).first; }
    std::size_t span_len(std::int64_t s) const { return spans.at(static_cast<std::size_t>(s)).second; }
    int leaf(NodeId op, int q) const {
        auto it = leaf_index.find(CallId{op, q});
        return it == leaf_index.end() ? -1 : it->second;
    }
    std::vector<int> path_from_root(int n) const;
};

Plan parse_plan(const std::uint8_t* data, std::size_t n);
// opt-in call-level partition of a plan over `workers` (diverges from the reference)
std::vector<std::uint8_t> partition_calls(const std::uint8_t* data, std::size_t n, int workers);
// native cache-aware planner (planner.cpp): partition_workflow + build_call_tree +
// plan_operators of the reference, over the plan's value graph, for `workers`
std::vector<std::uint8_t> replan(const std::uint8_t* data, std::size_t n, int workers,
                                 const std::vector<std::uint64_t>& capacities, double alpha);
struct PlanOutcome {
    std::vector<std::uint8_t> blob;                    // HKPLAN01 with the new call tree + schedule
    std::vector<std::vector<std::vector<NodeId>>> soft;  // SoftSchedule (inner sequences per worker)
    std::vector<std::vector<CallId>> sigma;
    std::uint64_t passes = 0, forced_emits = 0, emitted = 0;  // SchedulerStats
    double makespan = 0;                               // evaluate_schedule (cost_model.cpp:32-120)
};
PlanOutcome replan_full(const std::uint8_t* data, std::size_t n, int workers,
                        const std::vector<std::uint64_t>& capacities, double alpha);

// -------------------------------------------------------------- evaluator
class Evaluator {
  public:
    Evaluator(const Plan& p, std::uint64_t seed, bool stochastic, bool strict_llm)
        : plan_(&p), seed_(seed), stochastic_(stochastic), strict_(strict_llm) {}
    const TokenSeq& value(NodeId id, std::size_t q);
    TokenSeq prompt(NodeId llm, std::size_t q);
    void put_llm_output(NodeId llm, std::size_t q, TokenSeq out) { memo_[{llm, q}] = std::move(out); }
    double profile_len_out(NodeId llm) const;
    bool deterministic(NodeId llm) const { return plan_->nodes.at(llm).deterministic; }
    std::map<NodeId, std::vector<TokenSeq>> output_values();

  private:
    const Plan* plan_;
    std::uint64_t seed_;
    bool stochastic_, strict_;
    std::map<std::pair<NodeId, std::size_t>, TokenSeq> memo_;
};

// ---------------------------------------------------------- prompt cache
// class PromptCache (prompt_cache.hpp:15-40, prompt_cache.cpp:9-71): LRU map
// from operator signature to the token sequence that operator produced,
// serialised in the reference's JSON wire format byte for byte, so the
// reference's optimizer (substitute_cached, optimizer.cpp:71-95) can read a
// cache this executor harvested from device-generated outputs and the other
// way round.
class PromptCache {
  public:
    explicit PromptCache(std::size_t capacity = 4096);
    bool contains(std::uint64_t s) const { return index_.count(s) != 0; }
    const TokenSeq* lookup(std::uint64_t s);  // nullptr on miss; a hit refreshes recency
    void insert(std::uint64_t s, TokenSeq value);
    std::size_t size() const { return entries_.size(); }
    std::size_t capacity() const { return capacity_; }
    std::vector<std::uint64_t> keys_lru_first() const;
    std::string serialize() const;
    static PromptCache deserialize(const std::string& json_text);

  private:
    using Entry = std::pair<std::uint64_t, TokenSeq>;
    std::size_t capacity_;
    std::list<Entry> entries_;  // front = least recent
    std::unordered_map<std::uint64_t, std::list<Entry>::iterator> index_;
};
std::string sig_hex(std::uint64_t s);

struct SimMetrics;
// harvest_into_cache (optimizer.cpp:113-125) with the values of THIS run: every
// untainted format / lambda / llm node of the plan, every query, keyed by the
// plan's signatures, llm values = the tokens the LLM body generated (device
// transformer or synth), format / lambda values evaluated over them. Returns
// the number of entries inserted.
std::size_t harvest_into_cache(const Plan& plan, const SimMetrics& run, PromptCache& cache);

// ---------------------------------------------------------- page pool
// Physical KV pages of one worker. Frees are deferred to the next iteration so
// a page released while the current device step may still write it is never
// handed out inside the same step (DESIGN.md §KV pool).
class PagePool {
  public:
    explicit PagePool(int n_pages = 0) { reset(n_pages); }
    void reset(int n_pages);
    int alloc();
    void release(int page) { deferred_.push_back(page); }
    void flush_deferred();
    int capacity() const { return n_; }
    int in_use() const { return n_ - static_cast<int>(free_.size()) - static_cast<int>(deferred_.size()); }
    int high_water() const { return high_; }
    void mark_tree(int page, bool v) { tree_[static_cast<std::size_t>(page)] = v ? 1 : 0; }
    bool is_tree(int page) const { return tree_[static_cast<std::size_t>(page)] != 0; }

  private:
    int n_ = 0, high_ = 0;
    std::vector<int> free_, deferred_;
    std::vector<char> tree_;
};

// One journal entry for the device trie (create or erase of a tree node).
struct TrieOp {
    int node = 0;
    int parent = 0;
    int page = -1;
    bool erase = false;
    std::uint64_t phash = 0;
};

// ----------------------------------------------------------------- KvTree
// Per-worker radix tree of token blocks with exactly the semantics of the
// reference KvCache (simulator.cpp:14-128): same node numbering (root 0,
// LIFO free list), same LRU clock, holds, pins and store-what-fits rule.
// Eviction keeps an ordered set of evictable leaves instead of the O(N) scan
// (simulator.cpp:42-67); the victim is the same because clock values are unique.
// Each node additionally owns a physical KV page and a prefix hash
// H_k = hash_combine(H_{k-1}, fnv1a64(block_k)) used by the device trie.
struct KvOwner {  // a live call's block table, for adopt/dedupe on insert
    std::vector<int>* pages;
    PagePool* pool;
};

class KvTree {
  public:
    using Owner = KvOwner;

    KvTree(std::size_t capacity_tokens, std::size_t block_tokens);

    std::size_t capacity() const { return capacity_; }
    std::size_t block() const { return block_; }
    std::size_t used_tokens() const { return used_; }
    std::size_t pinned_tokens() const { return pinned_; }
    std::uint64_t evicted_tokens() const { return evicted_; }

    // simulator.cpp:69-87. path (optional) receives matched node ids.
    std::size_t lookup(const Token* seq, std::size_t n, std::uint64_t hold, std::vector<int>* path = nullptr);
    // Apply the side effects (touch/hold) of a lookup whose path was computed
    // elsewhere (the device trie), in path order.
    void apply_lookup(const int* path, std::size_t n_blocks, std::uint64_t hold);
    // Side-effect-free walk (used to verify device lookups).
    std::size_t peek(const Token* seq, std::size_t n, std::vector<int>* path) const;
    // simulator.cpp:89-121.
    std::size_t insert(const Token* seq, std::size_t n, std::size_t len, bool pinned, std::uint64_t hold,
                       Owner owner = Owner{nullptr, nullptr}, std::vector<int>* new_nodes = nullptr);
    void release(std::uint64_t hold);  // simulator.cpp:123-128

    int node_count() const { return static_cast<int>(nodes_.size()); }
    int node_page(int idx) const { return nodes_[static_cast<std::size_t>(idx)].page; }
    int node_parent(int idx) const { return nodes_[static_cast<std::size_t>(idx)].parent; }
    bool node_free(int idx) const { return nodes_[static_cast<std::size_t>(idx)].free; }
    std::uint64_t node_phash(int idx) const { return nodes_[static_cast<std::size_t>(idx)].phash; }
    const Token* node_key(int idx) const { return keys_.data() + static_cast<std::size_t>(idx) * block_; }

    void set_page_pool(PagePool* pool) { pool_ = pool; }
    std::vector<TrieOp>& journal() { return journal_; }
    bool journaling = false;

    std::uint64_t block_hash(const Token* blk) const { return fnv1a64(blk, block_ * sizeof(Token)); }

  private:
    struct Node {
        int parent = -1;
        int nkids = 0;
        bool pinned = false;
        int holds = 0;
        std::uint64_t last_use = 0;
        bool free = false;
        int page = -1;
        std::uint64_t phash = kFnvOffset;
        std::uint64_t bhash = 0;
    };
    struct ChildKey {
        int parent;
        std::uint64_t bhash;
        bool operator==(const ChildKey& o) const { return parent == o.parent && bhash == o.bhash; }
    };
    struct ChildKeyHash {
        std::size_t operator()(const ChildKey& k) const {
            return static_cast<std::size_t>(k.bhash ^ (static_cast<std::uint64_t>(k.parent) * 0x9e3779b97f4a7c15ull));
        }
    };

    int find_child(int parent, const Token* blk, std::uint64_t bh) const;
    int create_child(int parent, const Token* blk, std::uint64_t bh);
    bool evict_one();
    void touch(int idx);
    bool evictable(const Node& n) const { return !n.free && !n.pinned && n.holds == 0 && n.nkids == 0; }

    std::size_t capacity_ = 0, block_ = 0, used_ = 0, pinned_ = 0;
    std::uint64_t evicted_ = 0, clock_ = 0;
    std::vector<Node> nodes_;
    std::vector<Token> keys_;
    std::vector<int> free_;
    std::unordered_multimap<ChildKey, int, ChildKeyHash> kids_;
    std::set<std::pair<std::uint64_t, int>> evictable_;
    std::unordered_map<std::uint64_t, std::vector<int>> holds_;
    PagePool* pool_ = nullptr;
    std::vector<TrieOp> journal_;
};

// simulator.cpp:132-199 over the flattened call tree.
std::vector<TokenSeq> static_pin_prefixes(const Plan& p, int worker, std::size_t block,
                                          std::size_t threshold, std::size_t budget_tokens);

// --------------------------------------------------------------- simulate
struct SimWorkerConfig {
    std::size_t capacity = 4096, block = 16, prefill_budget = 0;
};

struct SimConfig {
    std::vector<SimWorkerConfig> workers;
    bool proactive_pin = true;
    std::size_t pin_threshold = 200;
    double pin_capacity_frac = 0.5;
    std::uint64_t seed = 0;
    bool stochastic = false;
    bool collect_trace = false;
    std::uint64_t max_iterations = 0;
};

struct SimIterRow {
    std::uint64_t iter = 0;
    int worker = 0, active = 0;
    std::size_t admitted = 0, prefill_tokens = 0, decode_tokens = 0;
};

struct SimCallRow {
    CallId call;
    int worker = 0;
    std::uint64_t admitted_iter = 0, prefill_done_iter = 0, completed_iter = 0;
    std::size_t prompt_tokens = 0, cached_tokens = 0, output_tokens = 0;
};

struct SimMetrics {
    std::uint64_t iterations = 0;
    std::size_t prompt_tokens = 0, cache_served_tokens = 0, prefill_computed_tokens = 0, decode_tokens = 0;
    double hit_rate_pct = 0;
    std::vector<std::size_t> pinned_tokens;
    std::vector<std::uint64_t> evicted_tokens;
    std::vector<SimCallRow> calls;
    std::vector<SimIterRow> trace;
    std::map<NodeId, std::vector<TokenSeq>> outputs;
    // B200 additions (not part of the reference report)
    std::map<CallId, TokenSeq> call_outputs;        // every llm call's generated tokens
    std::map<CallId, std::vector<float>> call_logits;  // device body: the logit of each generated token
    std::vector<std::uint64_t> pin_compute_tokens;  // per worker, pin precompute prefill
    std::uint64_t recompute_tokens = 0;             // fully-cached prompts: last position re-run
    double pin_seconds = 0, iter_seconds = 0;       // wall time: pin precompute, iteration loop
};

std::string sim_metrics_json(const SimMetrics& m);
std::string sim_calls_csv(const SimMetrics& m);
std::string sim_trace_csv(const SimMetrics& m);

// A running call (simulator.cpp:205-218) plus its block table.
struct LiveCall {
    CallId id;
    int leaf = -1;
    TokenSeq prompt;
    std::size_t out_len = 0, done = 0, decoded = 0;
    std::uint64_t hold = 0, prefill_done_iter = 0;
    std::size_t row = 0;
    bool finished = false;
    int slot = -1;            // device-side call slot
    int group = -1;           // TRT static group of the call's leaf (Plan::static_group)
    std::size_t group_tokens = 0;
    std::vector<int> pages;   // physical page per 16-token block (prompt + output)
    std::size_t remaining() const { return prompt.size() - done; }
};

// Work the device must do for one (iteration, worker). Built by the executor
// in reference order; run by an LlmBody.
struct StepPlan {
    struct Seg {
        LiveCall* call = nullptr;
        std::size_t start = 0;   // first position computed
        std::size_t count = 0;   // tokens computed
        bool from_prompt = true; // token ids come from prompt (else last sampled)
        bool write_kv = true;    // false for the recomputed last position of a fully cached prompt
        bool sample = false;     // produce the next token from the last position
        int group = -1;          // TRT static group (decode segs): rows of one group share its prefix pages
        std::size_t group_tokens = 0;
        std::vector<int> table;  // block table snapshot taken when the seg was planned
    };
    int worker = 0;
    std::uint64_t iter = 0;
    std::vector<Seg> segs;
};

// Pluggable LLM body. The synthetic body reproduces evaluator.cpp exactly;
// the device body runs the random-init transformer on the B200.
class LlmBody {
  public:
    virtual ~LlmBody() = default;
    virtual bool uses_pages() const { return false; }
    virtual int pages_per_worker(int /*w*/) const { return 0; }
    // Called once per worker after pins are inserted: compute KV of new pin blocks.
    virtual void precompute_pins(int /*w*/, const std::vector<TokenSeq>& /*pins*/,
                                 const std::vector<std::vector<int>>& /*pin_pages*/,
                                 const std::vector<std::size_t>& /*first_new_block*/) {}
    // Device trie: batched lookup of candidate prompts; returns matched node paths.
    virtual bool device_lookup() const { return false; }
    virtual void lookup_batch(int /*w*/, const std::vector<const TokenSeq*>& /*prompts*/,
                              std::vector<std::vector<int>>& /*paths*/) {}
    virtual void sync_trie(int /*w*/, KvTree& /*tree*/) {}
    // Start of iteration `iter`: `completing` lists every (worker, call) that
    // will complete with a non-empty output this iteration (multi-process
    // bodies exchange those outputs here, before any worker runs).
    virtual void begin_iteration(std::uint64_t /*iter*/,
                                 const std::vector<std::pair<int, LiveCall*>>& /*completing*/) {}
    virtual void on_admit(int /*w*/, LiveCall& /*lc*/) {}
    virtual void run_step(StepPlan& /*sp*/) {}
    virtual TokenSeq take_output(int w, LiveCall& lc, double len_out, bool det) = 0;
    // the logit of each token take_output returned (device body only; called right after it)
    virtual std::vector<float> take_logits(int /*w*/, LiveCall& /*lc*/) { return {}; }
    virtual void on_finish(int /*w*/, LiveCall& /*lc*/) {}
    virtual void finish_run() {}
};

class SyntheticBody : public LlmBody {
  public:
    SyntheticBody(std::uint64_t seed, bool stochastic) : seed_(seed), stochastic_(stochastic) {}
    TokenSeq take_output(int, LiveCall& lc, double len_out, bool det) override {
        return synth_llm_output(lc.prompt, len_out, det, seed_, stochastic_);
    }

  private:
    std::uint64_t seed_;
    bool stochastic_;
};

struct ExecOptions {
    bool verify_device_lookup = false;  // also walk the host tree and compare paths
    int only_worker = -1;  // >=0: this process owns one worker's device (others replayed)
    // Cross-worker dependencies with one process per worker (SURVEY §8(e)
    // exchange 2): with only_worker >= 0 and `exchange` set, every process
    // replays the host control plane of ALL workers and drives the body only
    // for its own; at every completion of every worker (in the same order on
    // all processes) exchange(worker, call, tokens) is called — the owning
    // process passes the generated ids, the others receive them (tokens is
    // pre-sized to the call's output length).
    std::function<void(int worker, const CallId& call, TokenSeq& tokens)> exchange;
};

SimMetrics simulate(const Plan& plan, const SimConfig& cfg, LlmBody& body, const ExecOptions& opts = {});

// ------------------------------------------------------- run_workflow (native)
// RunSpec (run_pipeline.hpp:16-38) and the documents of `helios run`
// (pipeline.cpp): parse -> bind -> rewrite -> plan -> simulate -> reports.
struct WorkflowSpec {
    int workers = 1;
    std::vector<std::uint64_t> capacities = {4096};
    std::string scheduler = "cache_aware";
    std::uint64_t seed = 0;
    bool stochastic = false;
    bool prune = true, merge_duplicates = true, cache_substitute = true;
    bool proactive_pin = true;
    std::size_t pin_threshold = 200;
    double pin_capacity_frac = 0.5;
    std::size_t block = 16, prefill_budget = 0;
    double alpha = 0;
    bool run_sim = true, collect_trace = false;
    std::uint64_t max_iterations = 0;
};
struct WorkflowRun {
    std::vector<std::uint8_t> plan;  // the planned HKPLAN01
    SimMetrics metrics;
    std::string report_json, calls_csv, trace_csv, outputs_json, schedule_json;
};
using BodyFactory = std::function<std::unique_ptr<LlmBody>(const Plan&, const SimConfig&)>;
WorkflowRun run_workflow(const std::string& workflow_json, const std::string& inputs_json,
                         const std::string& profile_json, const WorkflowSpec& spec, PromptCache* cache,
                         const BodyFactory& make_body);
// harvest_into_cache with the Evaluator's synthesized llm values (run_pipeline.cpp:74-79 as
// the reference does it): for runs whose LLM body did not run (run_sim = false)
std::size_t harvest_into_cache_synth(const Plan& plan, std::uint64_t seed, bool stochastic, PromptCache& cache);

}  // namespace hk
