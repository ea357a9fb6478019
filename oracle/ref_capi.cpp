// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI wrapper around the UNMODIFIED reference library (built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Python tests,
// tests/golden/make_golden.py and bench.py's reference arm load
// oracle/_ref/libhelios_ref.so through ctypes to obtain:
//   * reference SimMetrics / call rows / outputs for a workflow
//     (the same pipeline as run_workflow, run_pipeline.cpp:47-81, with the
//     planning capacity separable from the simulated one so the
//     test_simulator.cpp SimFixture (:27-42) can be reproduced),
//   * the flattened executor plan (integration/plan_export.hpp),
//   * direct access to KvCache (simulator.cpp:14-128), static_pin_prefixes
//     (:132-199), synth_llm_len/output (evaluator.cpp:46-58) and the token
//     hashes (tokens.cpp) for differential tests.
#include <chrono>
#include <memory>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "json.hpp"
#include "helios/baselines.hpp"
#include "helios/evaluator.hpp"
#include "helios/optimizer.hpp"
#include "helios/run_pipeline.hpp"
#include "helios/scheduler.hpp"
#include "helios/simulator.hpp"
#include "helios/tokens.hpp"
#include "helios/workflow_io.hpp"
#include "helios/workload_gen.hpp"
#include "../integration/plan_export.hpp"

using nlohmann::json;
using namespace helios;

namespace {
thread_local std::string g_err;

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

struct Pipeline {
    CompiledGraph compiled;
    ProfileStats profile;
    TemplatedRadixTree tree;
    Schedule sigma;
    SimConfig cfg;
    std::unique_ptr<PromptCache> cache;  // spec "prompt_cache": cross-run cache document
    OptimizeReport rewrite;
};

// bind -> optimize -> partition -> plan -> call tree -> schedule, exactly as
// run_workflow does (run_pipeline.cpp:47-69); spec keys mirror RunSpec.
Pipeline build(const std::string& wf, const std::string& in, const std::string& prof,
               const json& spec) {
    Pipeline p;
    WorkflowGraph g = parse_workflow(wf);
    InputBatch inputs = parse_inputs(in);
    p.profile = parse_profile(prof);
    p.compiled = helios::bind(g, inputs);
    OptimizeOptions oo;
    oo.prune = spec.value("prune", true);
    oo.merge_duplicates = spec.value("merge_duplicates", true);
    oo.cache_substitute = spec.value("cache_substitute", true);
    if (spec.contains("prompt_cache"))
        p.cache = std::make_unique<PromptCache>(PromptCache::deserialize(spec.at("prompt_cache").get<std::string>()));
    p.rewrite = optimize(p.compiled, p.profile, p.cache.get(), oo);

    const int W = spec.value("workers", 1);
    std::vector<std::size_t> caps = spec.value("capacities", std::vector<std::size_t>{4096});
    std::vector<std::size_t> plan_caps = spec.value("plan_capacities", caps);
    auto cap_of = [&](const std::vector<std::size_t>& v, int w) {
        return v.size() == 1 ? v[0] : v.at(static_cast<std::size_t>(w));
    };
    CostParams params;
    for (int w = 0; w < W; ++w)
        params.workers.push_back(
            WorkerParams{static_cast<double>(cap_of(plan_caps, w)), spec.value("alpha", 0.0)});
    Partition part = partition_workflow(p.compiled, p.profile, W);
    if (spec.contains("worker_of")) {
        part.worker_of.clear();
        for (auto& [k, v] : spec.at("worker_of").items()) part.worker_of[std::stoll(k)] = v.get<int>();
    }
    const std::string sched = spec.value("scheduler", std::string("cache_aware"));
    p.tree = build_call_tree(p.compiled, p.profile, part.worker_of);
    if (spec.contains("sigma")) {
        for (const json& wq : spec.at("sigma")) {
            WorkerSequence s;
            for (const json& c : wq) s.push_back(CallId{c.at(0).get<NodeId>(), c.at(1).get<int>()});
            p.sigma.push_back(s);
        }
    } else if (sched == "cache_aware") {
        SoftSchedule soft = plan_operators(p.compiled, p.profile, params, part);
        p.sigma = expand_soft_schedule(soft, p.compiled.batch);
    } else {
        p.sigma = baseline_schedule(scheduler_kind_from_name(sched), p.compiled, p.profile, p.tree,
                                    W, spec.value("seed", std::uint64_t{0}));
    }
    for (int w = 0; w < static_cast<int>(p.sigma.size()); ++w)
        p.cfg.workers.push_back(SimWorkerConfig{cap_of(caps, w), spec.value("block", std::size_t{16}),
                                                spec.value("prefill_budget", std::size_t{0})});
    p.cfg.proactive_pin = spec.value("proactive_pin", true);
    p.cfg.pin_threshold = spec.value("pin_threshold", std::size_t{200});
    p.cfg.pin_capacity_frac = spec.value("pin_capacity_frac", 0.5);
    p.cfg.seed = spec.value("seed", std::uint64_t{0});
    p.cfg.stochastic = spec.value("stochastic", false);
    p.cfg.collect_trace = spec.value("collect_trace", false);
    p.cfg.max_iterations = spec.value("max_iterations", std::uint64_t{0});
    return p;
}

json sim_json(const SimMetrics& m) {
    json j;
    j["metrics_json"] = sim_metrics_json(m);
    j["calls_csv"] = sim_calls_csv(m);
    j["trace_csv"] = sim_trace_csv(m);
    json outs = json::object();
    for (const auto& [id, vals] : m.outputs) outs[std::to_string(id)] = vals;
    j["outputs"] = outs;
    return j;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// Runs the reference pipeline + simulate. Returns 0 on success.
//   *out_json : {"metrics_json","calls_csv","trace_csv","outputs","sigma","sim_seconds"}
//   *plan/*plan_len : flattened HKPLAN01 blob (malloc'd) when plan != NULL
int ref_run(const char* wf, const char* in, const char* prof, const char* spec_json,
            char** out_json, std::uint8_t** plan, std::size_t* plan_len) {
    try {
        json spec = json::parse(spec_json);
        Pipeline p = build(wf, in, prof, spec);
        json j;
        const int reps = spec.value("skip_sim", false) ? 0 : spec.value("time_reps", 1);
        double best = 0;
        SimMetrics m;
        for (int r = 0; r < reps; ++r) {
            if (r == 0) best = 1e30;
            auto t0 = std::chrono::steady_clock::now();
            m = simulate(p.compiled, p.profile, p.tree, p.sigma, p.cfg);
            auto t1 = std::chrono::steady_clock::now();
            best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
        }
        j = sim_json(m);
        j["sim_seconds"] = best;
        json sj = json::array();
        for (const auto& wq : p.sigma) {
            json s = json::array();
            for (const CallId& c : wq) s.push_back({c.op, c.query});
            sj.push_back(s);
        }
        j["sigma"] = sj;
        j["rewrite"] = {{"pruned", p.rewrite.pruned}, {"merged", p.rewrite.merged},
                        {"substituted", p.rewrite.substituted}};
        if (spec.value("harvest", false)) {
            // run_workflow's harvest (run_pipeline.cpp:74-79): the evaluator's
            // synthesized values into the (possibly fresh) cache
            if (!p.cache) p.cache = std::make_unique<PromptCache>(spec.value("cache_capacity", std::size_t{4096}));
            Evaluator ev(p.compiled, p.profile, EvalOptions{p.cfg.seed, p.cfg.stochastic, false});
            j["harvested"] = harvest_into_cache(p.compiled, p.profile, ev, *p.cache);
            j["prompt_cache_out"] = p.cache->serialize();
        }
        *out_json = dup(j.dump());
        if (plan) {
            std::vector<std::uint8_t> b = helium_b200::export_plan(p.compiled, p.profile, p.tree, p.sigma);
            *plan = static_cast<std::uint8_t*>(std::malloc(b.size()));
            std::memcpy(*plan, b.data(), b.size());
            *plan_len = b.size();
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Wall seconds of the whole reference run_workflow (best of reps) — the
// CPU path the reference ships, used as bench.py's reference arm.
int ref_time_run_workflow(const char* wf, const char* in, const char* prof, const char* spec_json,
                          int reps, double* best_s, char** metrics_json) {
    try {
        json spec = json::parse(spec_json);
        WorkflowGraph g = parse_workflow(wf);
        InputBatch inputs = parse_inputs(in);
        ProfileStats profile = parse_profile(prof);
        RunSpec rs;
        rs.workers = spec.value("workers", 1);
        rs.capacities = spec.value("capacities", std::vector<std::size_t>{4096});
        rs.block = spec.value("block", std::size_t{16});
        rs.prefill_budget = spec.value("prefill_budget", std::size_t{0});
        rs.proactive_pin = spec.value("proactive_pin", true);
        rs.pin_threshold = spec.value("pin_threshold", std::size_t{200});
        rs.seed = spec.value("seed", std::uint64_t{0});
        double best = 1e30;
        RunResult r;
        for (int k = 0; k < reps; ++k) {
            auto t0 = std::chrono::steady_clock::now();
            r = run_workflow(g, inputs, profile, rs, nullptr);
            auto t1 = std::chrono::steady_clock::now();
            best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
        }
        *best_s = best;
        *metrics_json = dup(sim_metrics_json(r.sim));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_generate_workload(const char* spec_json, int random, char** wf, char** in, char** prof) {
    try {
        json s = json::parse(spec_json);
        SynthWorkload w;
        if (random) {
            RandomSpec rs;
            rs.llm_ops = s.value("llm_ops", 3);
            rs.batch = s.value("batch", std::size_t{2});
            rs.allow_nondeterminism = s.value("allow_nondeterminism", true);
            rs.seed = s.value("seed", std::uint64_t{0});
            w = generate_random_workflow(rs);
        } else {
            SynthSpec ss;
            ss.pattern = s.value("pattern", std::string("mapred"));
            ss.agents = s.value("agents", 3);
            ss.rounds = s.value("rounds", 2);
            ss.batch = s.value("batch", std::size_t{2});
            ss.system_tokens = s.value("system_tokens", 120);
            ss.context_tokens = s.value("context_tokens", 60);
            ss.question_tokens = s.value("question_tokens", 12);
            ss.len_out = s.value("len_out", 8.0);
            ss.len_jitter = s.value("len_jitter", true);
            ss.seed = s.value("seed", std::uint64_t{0});
            w = generate_workload(ss);
        }
        *wf = dup(serialize_workflow(w.graph));
        *in = dup(serialize_inputs(w.inputs));
        *prof = dup(serialize_profile(w.profile));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// --- KvCache ----------------------------------------------------------------
void* ref_kv_new(std::size_t cap, std::size_t block) {
    try {
        return new KvCache(cap, block);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_kv_free(void* h) { delete static_cast<KvCache*>(h); }
std::size_t ref_kv_lookup(void* h, const std::uint64_t* s, std::size_t n, std::uint64_t hold) {
    return static_cast<KvCache*>(h)->lookup(TokenSeq(s, s + n), hold);
}
std::size_t ref_kv_insert(void* h, const std::uint64_t* s, std::size_t n, std::size_t len, int pinned,
                          std::uint64_t hold) {
    return static_cast<KvCache*>(h)->insert(TokenSeq(s, s + n), len, pinned != 0, hold);
}
void ref_kv_release(void* h, std::uint64_t hold) { static_cast<KvCache*>(h)->release(hold); }
void ref_kv_counters(void* h, std::uint64_t out[3]) {
    auto* c = static_cast<KvCache*>(h);
    out[0] = c->used_tokens();
    out[1] = c->pinned_tokens();
    out[2] = c->evicted_tokens();
}

// --- pins / synth / tokens -----------------------------------------------------
// Returns pins as JSON [[tok,...],...] for the pipeline's call tree and sigma.
int ref_static_pins(const char* wf, const char* in, const char* prof, const char* spec_json,
                    int worker, std::size_t block, std::size_t threshold, std::size_t budget,
                    char** out) {
    try {
        Pipeline p = build(wf, in, prof, json::parse(spec_json));
        std::vector<TokenSeq> pins = static_pin_prefixes(p.tree, p.sigma, worker, block, threshold, budget);
        *out = dup(json(pins).dump());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

std::size_t ref_synth_llm_len(const std::uint64_t* p, std::size_t n, double len_out, int det,
                              std::uint64_t seed, int stochastic) {
    return synth_llm_len(TokenSeq(p, p + n), len_out, det != 0, EvalOptions{seed, stochastic != 0, false});
}
std::size_t ref_synth_llm_output(const std::uint64_t* p, std::size_t n, double len_out, int det,
                                 std::uint64_t seed, int stochastic, std::uint64_t* out,
                                 std::size_t cap) {
    TokenSeq o = synth_llm_output(TokenSeq(p, p + n), len_out, det != 0,
                                  EvalOptions{seed, stochastic != 0, false});
    for (std::size_t k = 0; k < o.size() && k < cap; ++k) out[k] = o[k];
    return o.size();
}
// `helios run` (tools/helios_main.cpp:83-115) with the reference simulate(),
// for the command-line drop-in test: spec keys are the CLI flags
// (workers, capacity list, scheduler, seed, stochastic, no_prune, no_cse,
// no_prompt_cache, no_proactive_kv, block, prefill_budget, pin_threshold,
// alpha, trace, no_sim, cache: prompt-cache document or absent).
// Returns {"report","calls_csv","trace_csv","outputs_json","schedule_json","cache_out"}.
int ref_cli_run(const char* wf, const char* in, const char* prof, const char* spec_json, char** out_json) {
    try {
        json a = json::parse(spec_json);
        WorkflowGraph g = parse_workflow(wf);
        InputBatch inputs = parse_inputs(in);
        ProfileStats profile = parse_profile(prof);
        RunSpec spec;
        spec.workers = a.value("workers", 1);
        if (a.contains("capacity")) spec.capacities = a.at("capacity").get<std::vector<std::size_t>>();
        spec.scheduler = scheduler_kind_from_name(a.value("scheduler", std::string("cache_aware")));
        spec.seed = a.value("seed", std::uint64_t{0});
        spec.stochastic = a.value("stochastic", false);
        spec.prune = !a.value("no_prune", false);
        spec.merge_duplicates = !a.value("no_cse", false);
        spec.cache_substitute = !a.value("no_prompt_cache", false);
        spec.proactive_pin = !a.value("no_proactive_kv", false);
        spec.block = a.value("block", std::size_t{16});
        spec.prefill_budget = a.value("prefill_budget", std::size_t{0});
        spec.pin_threshold = a.value("pin_threshold", std::size_t{200});
        spec.alpha = a.value("alpha", 0.0);
        spec.collect_trace = a.value("trace", false);
        spec.run_sim = !a.value("no_sim", false);
        PromptCache cache(65536);
        PromptCache* cp = nullptr;
        if (a.contains("cache") && spec.cache_substitute) {
            if (!a.at("cache").is_null()) cache = PromptCache::deserialize(a.at("cache").get<std::string>());
            cp = &cache;
        }
        RunResult r = run_workflow(g, inputs, profile, spec, cp);
        json oj = json::object();
        for (const auto& [node, per_query] : r.sim.outputs) {
            json arr = json::array();
            for (const TokenSeq& v : per_query) arr.push_back(v);
            oj[std::to_string(node)] = std::move(arr);
        }
        json j{{"report", run_report_json(r, spec) + "\n"}, {"calls_csv", sim_calls_csv(r.sim)},
               {"trace_csv", sim_trace_csv(r.sim)}, {"outputs_json", oj.dump(2) + "\n"},
               {"schedule_json", soft_schedule_json(r.soft) + "\n"},
               {"cache_out", cp ? json(cache.serialize()) : json(nullptr)}};
        *out_json = dup(j.dump());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// reference PromptCache (prompt_cache.cpp) for differential tests
void* ref_pcache_new(std::size_t capacity) {
    try {
        return new PromptCache(capacity);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void* ref_pcache_load(const char* json) {
    try {
        return new PromptCache(PromptCache::deserialize(json));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_pcache_free(void* h) { delete static_cast<PromptCache*>(h); }
void ref_pcache_insert(void* h, std::uint64_t sig, const std::uint64_t* t, std::size_t n) {
    static_cast<PromptCache*>(h)->insert(sig, TokenSeq(t, t + n));
}
long long ref_pcache_lookup(void* h, std::uint64_t sig) {
    const TokenSeq* v = static_cast<PromptCache*>(h)->lookup(sig);
    return v ? static_cast<long long>(v->size()) : -1;
}
char* ref_pcache_save(void* h) { return dup(static_cast<PromptCache*>(h)->serialize()); }

std::uint64_t ref_fnv1a64(const void* d, std::size_t n, std::uint64_t seed) { return fnv1a64(d, n, seed); }
std::uint64_t ref_hash_combine(std::uint64_t h, std::uint64_t v) { return hash_combine(h, v); }
std::size_t ref_tokenize(const char* text, std::uint64_t* out, std::size_t cap) {
    TokenSeq t = tokenize(text);
    for (std::size_t k = 0; k < t.size() && k < cap; ++k) out[k] = t[k];
    return t.size();
}
std::uint64_t ref_role_marker(int role) { return role_marker(static_cast<MsgRole>(role)); }

}  // extern "C"
