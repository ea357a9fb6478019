// extern "C" entry points of include/helium_b200.h for the host side
// (executor, KvCache, pins, synth, hashes). Device entry points live in
// csrc/cuda/engine.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "../../../include/helium_b200.h"
#include "hk_host.hpp"

namespace hk {
thread_local std::string g_last_error;
void set_error(const std::string& s) { g_last_error = s; }
// Implemented in csrc/cuda/engine.cu.
std::unique_ptr<LlmBody> make_device_body(hk_engine* e, const Plan& plan, const SimConfig& cfg, int only_worker);
}  // namespace hk

struct hk_run {
    hk::SimMetrics m;
    std::string reports[3];
    std::string docs[3];            // hk_run_workflow: report json, outputs json, soft schedule json
    std::vector<uint8_t> plan;      // hk_run_workflow: the planned HKPLAN01
};

struct hk_pcache {
    hk::PromptCache c;
    explicit hk_pcache(hk::PromptCache x) : c(std::move(x)) {}
};

struct hk_kvcache {
    hk::KvTree tree;
    hk_kvcache(std::size_t c, std::size_t b) : tree(c, b) {}
};

namespace {

template <typename F>
auto guard(F&& f, decltype(f()) on_error) -> decltype(f()) {
    try {
        return f();
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return on_error;
    }
}

hk::SimConfig to_sim_config(const hk_sim_config* c) {
    if (!c) throw std::runtime_error("hk_simulate: null config");
    hk::SimConfig s;
    for (uint32_t w = 0; w < c->n_workers; ++w)
        s.workers.push_back(hk::SimWorkerConfig{c->capacity[w], c->block[w], c->prefill_budget[w]});
    s.proactive_pin = c->proactive_pin != 0;
    s.pin_threshold = c->pin_threshold;
    s.pin_capacity_frac = c->pin_capacity_frac;
    s.seed = c->seed;
    s.stochastic = c->stochastic != 0;
    s.collect_trace = c->collect_trace != 0;
    s.max_iterations = c->max_iterations;
    return s;
}

}  // namespace

extern "C" {

const char* hk_last_error(void) { return hk::g_last_error.c_str(); }
int hk_abi_version(void) { return HK_ABI_VERSION; }

hk_run* hk_simulate(const uint8_t* plan, size_t plan_len, const hk_sim_config* cfg, hk_engine* engine,
                    uint32_t flags) {
    return hk_simulate_ex(plan, plan_len, cfg, engine, flags, nullptr, nullptr);
}

hk_run* hk_simulate_ex(const uint8_t* plan, size_t plan_len, const hk_sim_config* cfg, hk_engine* engine,
                       uint32_t flags, hk_output_exchange_fn fn, void* user) {
    return guard(
        [&]() -> hk_run* {
            hk::Plan p = hk::parse_plan(plan, plan_len);
            hk::SimConfig sc = to_sim_config(cfg);
            auto run = std::make_unique<hk_run>();
            hk::ExecOptions eo;
            eo.verify_device_lookup = (flags & 1u) != 0;
            eo.only_worker = static_cast<int>((flags >> 8) & 0xFFFFu) - 1;
            if (fn) {
                eo.exchange = [fn, user](int w, const hk::CallId& c, hk::TokenSeq& t) {
                    if (fn(user, w, static_cast<int>(c.op), c.query, t.data(), t.size()) != 0)
                        throw std::runtime_error("simulate: output exchange failed for worker " + std::to_string(w) +
                                                 " call op " + std::to_string(c.op) + " q " + std::to_string(c.query));
                };
            }
            if (engine) {
                std::unique_ptr<hk::LlmBody> body = hk::make_device_body(engine, p, sc, eo.only_worker);
                run->m = hk::simulate(p, sc, *body, eo);
            } else {
                hk::SyntheticBody body(sc.seed, sc.stochastic);
                run->m = hk::simulate(p, sc, body, eo);
            }
            run->reports[0] = hk::sim_metrics_json(run->m);
            run->reports[1] = hk::sim_calls_csv(run->m);
            run->reports[2] = hk::sim_trace_csv(run->m);
            return run.release();
        },
        nullptr);
}

hk_run* hk_run_workflow(const char* workflow_json, const char* inputs_json, const char* profile_json,
                        const hk_workflow_spec* spec, hk_pcache* cache, hk_engine* engine) {
    return guard(
        [&]() -> hk_run* {
            if (!workflow_json || !inputs_json || !profile_json || !spec)
                throw std::runtime_error("hk_run_workflow: null argument");
            hk::WorkflowSpec ws;
            ws.workers = spec->workers;
            ws.capacities.assign(spec->capacities, spec->capacities + spec->n_capacities);
            ws.scheduler = spec->scheduler ? spec->scheduler : "cache_aware";
            ws.seed = spec->seed;
            ws.stochastic = spec->stochastic != 0;
            ws.prune = spec->prune != 0;
            ws.merge_duplicates = spec->merge_duplicates != 0;
            ws.cache_substitute = spec->cache_substitute != 0;
            ws.proactive_pin = spec->proactive_pin != 0;
            ws.pin_threshold = spec->pin_threshold;
            ws.pin_capacity_frac = spec->pin_capacity_frac;
            ws.block = spec->block;
            ws.prefill_budget = spec->prefill_budget;
            ws.alpha = spec->alpha;
            ws.run_sim = spec->run_sim != 0;
            ws.collect_trace = spec->collect_trace != 0;
            ws.max_iterations = spec->max_iterations;
            hk::BodyFactory mk = [engine](const hk::Plan& p, const hk::SimConfig& sc) -> std::unique_ptr<hk::LlmBody> {
                if (engine) return hk::make_device_body(engine, p, sc, -1);
                return std::make_unique<hk::SyntheticBody>(sc.seed, sc.stochastic);
            };
            hk::WorkflowRun wr = hk::run_workflow(workflow_json, inputs_json, profile_json, ws, cache ? &cache->c : nullptr, mk);
            auto run = std::make_unique<hk_run>();
            run->m = std::move(wr.metrics);
            run->reports[0] = hk::sim_metrics_json(run->m);
            run->reports[1] = wr.calls_csv;
            run->reports[2] = wr.trace_csv;
            run->docs[0] = wr.report_json;
            run->docs[1] = wr.outputs_json;
            run->docs[2] = wr.schedule_json;
            run->plan = std::move(wr.plan);
            return run.release();
        },
        static_cast<hk_run*>(nullptr));
}

size_t hk_run_document(const hk_run* r, int which, char* buf, size_t cap) {
    if (!r || which < 0 || which > 2) return 0;
    const std::string& s = r->docs[which];
    if (buf && cap) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return s.size() + 1;
}

size_t hk_run_plan(const hk_run* r, uint8_t* out, size_t cap) {
    if (!r) return 0;
    if (out) std::memcpy(out, r->plan.data(), std::min(cap, r->plan.size()));
    return r->plan.size();
}

int hk_run_metrics(const hk_run* r, hk_metrics* o) {
    if (!r || !o) return -1;
    o->iterations = r->m.iterations;
    o->prompt_tokens = r->m.prompt_tokens;
    o->cache_served_tokens = r->m.cache_served_tokens;
    o->prefill_computed_tokens = r->m.prefill_computed_tokens;
    o->decode_tokens = r->m.decode_tokens;
    o->hit_rate_pct = r->m.hit_rate_pct;
    o->calls = r->m.calls.size();
    o->recompute_tokens = r->m.recompute_tokens;
    o->pin_compute_tokens = 0;
    for (auto v : r->m.pin_compute_tokens) o->pin_compute_tokens += v;
    return 0;
}

size_t hk_run_worker_stat(const hk_run* r, int which, uint64_t* out, size_t cap) {
    if (!r) return 0;
    std::vector<uint64_t> v;
    if (which == 0)
        for (auto x : r->m.pinned_tokens) v.push_back(x);
    else if (which == 1)
        for (auto x : r->m.evicted_tokens) v.push_back(x);
    else
        for (auto x : r->m.pin_compute_tokens) v.push_back(x);
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    return v.size();
}

size_t hk_run_report(const hk_run* r, int which, char* buf, size_t cap) {
    if (!r || which < 0 || which > 2) return 0;
    const std::string& s = r->reports[which];
    if (buf && cap > 0) {
        size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return s.size() + 1;
}

size_t hk_run_outputs(const hk_run* r, uint64_t* out, size_t cap) {
    if (!r) return 0;
    std::vector<uint64_t> w;
    w.push_back(r->m.outputs.size());
    for (const auto& [id, vals] : r->m.outputs) {
        w.push_back(static_cast<uint64_t>(id));
        w.push_back(vals.size());
        for (const auto& v : vals) {
            w.push_back(v.size());
            w.insert(w.end(), v.begin(), v.end());
        }
    }
    for (size_t i = 0; i < w.size() && i < cap; ++i) out[i] = w[i];
    return w.size();
}

size_t hk_run_call_outputs(const hk_run* r, uint64_t* out, size_t cap) {
    if (!r) return 0;
    std::vector<uint64_t> w;
    w.push_back(r->m.call_outputs.size());
    for (const auto& [cid, toks] : r->m.call_outputs) {
        w.push_back(static_cast<uint64_t>(cid.op));
        w.push_back(static_cast<uint64_t>(cid.query));
        w.push_back(toks.size());
        w.insert(w.end(), toks.begin(), toks.end());
    }
    for (size_t i = 0; i < w.size() && i < cap; ++i) out[i] = w[i];
    return w.size();
}

size_t hk_run_call_logits(const hk_run* r, float* out, size_t cap) {
    if (!r) return 0;
    size_t n = 0;
    for (const auto& [cid, toks] : r->m.call_outputs) {
        auto it = r->m.call_logits.find(cid);
        for (size_t i = 0; i < toks.size(); ++i, ++n)
            if (n < cap) out[n] = it != r->m.call_logits.end() && i < it->second.size() ? it->second[i] : NAN;
    }
    return n;
}

int hk_run_timing(const hk_run* r, double out[2]) {
    if (!r) return -1;
    out[0] = r->m.pin_seconds;
    out[1] = r->m.iter_seconds;
    return 0;
}

void hk_run_free(hk_run* r) { delete r; }

hk_kvcache* hk_kv_create(size_t cap, size_t block) {
    return guard([&]() -> hk_kvcache* { return new hk_kvcache(cap, block); }, nullptr);
}
size_t hk_kv_lookup(hk_kvcache* c, const uint64_t* s, size_t n, uint64_t hold) {
    return c->tree.lookup(s, n, hold);
}
size_t hk_kv_insert(hk_kvcache* c, const uint64_t* s, size_t n, size_t len, int pinned, uint64_t hold) {
    return c->tree.insert(s, n, len, pinned != 0, hold);
}
void hk_kv_release(hk_kvcache* c, uint64_t hold) { c->tree.release(hold); }
void hk_kv_counters(const hk_kvcache* c, uint64_t out[3]) {
    out[0] = c->tree.used_tokens();
    out[1] = c->tree.pinned_tokens();
    out[2] = c->tree.evicted_tokens();
}
void hk_kv_destroy(hk_kvcache* c) { delete c; }

int64_t hk_static_pin_prefixes(const uint8_t* plan, size_t plan_len, int worker, size_t block, size_t threshold,
                               size_t budget, uint64_t* tokens, size_t cap, uint64_t* lens, size_t lens_cap) {
    return guard(
        [&]() -> int64_t {
            hk::Plan p = hk::parse_plan(plan, plan_len);
            std::vector<hk::TokenSeq> pins = hk::static_pin_prefixes(p, worker, block, threshold, budget);
            size_t off = 0;
            for (size_t i = 0; i < pins.size(); ++i) {
                if (i < lens_cap) lens[i] = pins[i].size();
                for (uint64_t t : pins[i]) {
                    if (off < cap) tokens[off] = t;
                    ++off;
                }
            }
            return static_cast<int64_t>(pins.size());
        },
        int64_t{-1});
}

int64_t hk_plan_partition_calls(const uint8_t* plan, size_t plan_len, int workers, uint8_t* out, size_t cap) {
    return guard(
        [&]() -> int64_t {
            const std::vector<std::uint8_t> b = hk::partition_calls(plan, plan_len, workers);
            if (out) std::memcpy(out, b.data(), std::min(cap, b.size()));
            return static_cast<int64_t>(b.size());
        },
        int64_t{-1});
}

int64_t hk_plan_schedule(const uint8_t* plan, size_t plan_len, int workers, const uint64_t* capacities, size_t n_caps,
                         double alpha, uint8_t* out, size_t cap) {
    return guard(
        [&]() -> int64_t {
            const std::vector<uint8_t> b =
                hk::replan(plan, plan_len, workers, std::vector<uint64_t>(capacities, capacities + n_caps), alpha);
            if (out) std::memcpy(out, b.data(), std::min(cap, b.size()));
            return static_cast<int64_t>(b.size());
        },
        int64_t{-1});
}

int64_t hk_plan_call_groups(const uint8_t* plan, size_t plan_len, int64_t* op, int32_t* query, int32_t* group,
                            uint64_t* tokens, size_t cap) {
    return guard(
        [&]() -> int64_t {
            hk::Plan p = hk::parse_plan(plan, plan_len);
            size_t i = 0;
            for (const auto& [cid, leaf] : p.leaf_index) {
                if (i < cap) {
                    op[i] = cid.op;
                    query[i] = cid.query;
                    group[i] = p.static_group[static_cast<size_t>(leaf)];
                    tokens[i] = p.static_group_tokens[static_cast<size_t>(leaf)];
                }
                ++i;
            }
            return static_cast<int64_t>(i);
        },
        int64_t{-1});
}

hk_pcache* hk_pcache_create(size_t capacity) {
    return guard([&]() { return new hk_pcache(hk::PromptCache(capacity)); }, static_cast<hk_pcache*>(nullptr));
}
hk_pcache* hk_pcache_load(const char* json, size_t len) {
    return guard(
        [&]() {
            if (!json) throw std::runtime_error("prompt cache json: null document");
            return new hk_pcache(hk::PromptCache::deserialize(std::string(json, len)));
        },
        static_cast<hk_pcache*>(nullptr));
}
size_t hk_pcache_save(const hk_pcache* c, char* buf, size_t cap) {
    return guard(
        [&]() -> size_t {
            const std::string s = c->c.serialize();
            if (buf && cap) {
                const size_t n = std::min(cap - 1, s.size());
                std::memcpy(buf, s.data(), n);
                buf[n] = 0;
            }
            return s.size() + 1;
        },
        size_t{0});
}
size_t hk_pcache_size(const hk_pcache* c) { return c ? c->c.size() : 0; }
size_t hk_pcache_capacity(const hk_pcache* c) { return c ? c->c.capacity() : 0; }
int hk_pcache_contains(const hk_pcache* c, uint64_t sig) { return c && c->c.contains(sig) ? 1 : 0; }
int64_t hk_pcache_lookup(hk_pcache* c, uint64_t sig, uint64_t* out, size_t cap) {
    return guard(
        [&]() -> int64_t {
            const hk::TokenSeq* v = c->c.lookup(sig);
            if (!v) return -1;
            for (size_t i = 0; i < v->size() && i < cap; ++i) out[i] = (*v)[i];
            return static_cast<int64_t>(v->size());
        },
        int64_t{-2});
}
int hk_pcache_insert(hk_pcache* c, uint64_t sig, const uint64_t* tokens, size_t n) {
    return guard(
        [&]() {
            c->c.insert(sig, hk::TokenSeq(tokens, tokens + n));
            return 0;
        },
        -1);
}
size_t hk_pcache_keys(const hk_pcache* c, uint64_t* out, size_t cap) {
    if (!c) return 0;
    const std::vector<uint64_t> k = c->c.keys_lru_first();
    for (size_t i = 0; i < k.size() && i < cap; ++i) out[i] = k[i];
    return k.size();
}
int64_t hk_pcache_harvest(hk_pcache* c, const uint8_t* plan, size_t plan_len, const hk_run* run) {
    return guard(
        [&]() -> int64_t {
            if (!c || !run) throw std::runtime_error("harvest_into_cache: null cache or run");
            const hk::Plan p = hk::parse_plan(plan, plan_len);
            return static_cast<int64_t>(hk::harvest_into_cache(p, run->m, c->c));
        },
        int64_t{-1});
}
int64_t hk_pcache_harvest_calls(hk_pcache* c, const uint8_t* plan, size_t plan_len, const uint64_t* calls,
                                size_t n_words) {
    return guard(
        [&]() -> int64_t {
            if (!c || !calls) throw std::runtime_error("harvest_into_cache: null cache or call outputs");
            const hk::Plan p = hk::parse_plan(plan, plan_len);
            hk::SimMetrics m;
            size_t i = 0;
            auto word = [&]() {
                if (i >= n_words) throw std::runtime_error("harvest_into_cache: truncated call outputs");
                return calls[i++];
            };
            const uint64_t n = word();
            for (uint64_t k = 0; k < n; ++k) {
                hk::CallId cid;
                cid.op = static_cast<hk::NodeId>(word());
                cid.query = static_cast<int>(word());
                const uint64_t len = word();
                hk::TokenSeq t(len);
                for (auto& x : t) x = word();
                m.call_outputs[cid] = std::move(t);
            }
            return static_cast<int64_t>(hk::harvest_into_cache(p, m, c->c));
        },
        int64_t{-1});
}
void hk_pcache_destroy(hk_pcache* c) { delete c; }

size_t hk_synth_llm_len(const uint64_t* p, size_t n, double len_out, int det, uint64_t seed, int stochastic) {
    return guard([&]() { return hk::synth_llm_len(hk::TokenSeq(p, p + n), len_out, det != 0, seed, stochastic != 0); },
                 size_t{0});
}

size_t hk_synth_llm_output(const uint64_t* p, size_t n, double len_out, int det, uint64_t seed, int stochastic,
                           uint64_t* out, size_t cap) {
    return guard(
        [&]() {
            hk::TokenSeq o = hk::synth_llm_output(hk::TokenSeq(p, p + n), len_out, det != 0, seed, stochastic != 0);
            for (size_t i = 0; i < o.size() && i < cap; ++i) out[i] = o[i];
            return o.size();
        },
        size_t{0});
}

uint64_t hk_fnv1a64(const void* d, size_t n, uint64_t seed) { return hk::fnv1a64(d, n, seed); }
uint64_t hk_hash_combine(uint64_t h, uint64_t v) { return hk::hash_combine(h, v); }
uint32_t hk_vocab_of(uint64_t t, uint32_t v) { return hk::vocab_of(t, v); }
uint64_t hk_gen_token(uint32_t id, uint32_t v) { return hk::gen_token(id, v); }

}  // extern "C"
