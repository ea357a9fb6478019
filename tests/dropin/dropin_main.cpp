// TEST INFRASTRUCTURE — the drop-in proof: the reference's own pipeline
// (run_workflow, run_pipeline.cpp:47-81) with simulate() at its call site
// (:72) served by integration/simulate_b200.hpp, against the unmodified
// reference library (oracle/_ref/libhelios.a, built from /root/reference by
// oracle/Makefile) and linked with the product library libhelium_b200.so.
//
//   dropin_test <workflow.json> <inputs.json> <profile.json> <spec.json> [--engine tiny|tiny_f32]
//
// Runs run_workflow(spec) with the reference simulate, then the same pipeline
// with run_sim = false and simulate_b200(r.compiled, profile,
// build_call_tree(r.compiled, profile, r.partition.worker_of), r.schedule,
// sim_config(spec)) — the exact arguments of :72 — and compares every
// SimMetrics field and the cross-run prompt cache both runs harvested. Prints
// one JSON line {"equal": {...}, ...}; exit 0 when the compared fields agree
// (outputs and cached values are compared only without an engine: with the
// transformer body they are the model's tokens, not synth_llm_output's).
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "json.hpp"
#include "helios/run_pipeline.hpp"
#include "helios/simulator.hpp"
#include "helios/trt.hpp"
#include "helios/workflow_io.hpp"
#include "helium_b200.h"
#include "simulate_b200.hpp"

using namespace helios;
using nlohmann::json;

static std::string slurp(const char* p) {
    std::ifstream f(p);
    if (!f) throw std::runtime_error(std::string("cannot read ") + p);
    std::stringstream s;
    s << f.rdbuf();
    return s.str();
}

// run_pipeline.cpp:27-43 (anonymous there), restated
static SimConfig sim_config(const RunSpec& spec) {
    SimConfig cfg;
    for (int w = 0; w < spec.workers; ++w) {
        const std::size_t cap = spec.capacities.size() == 1 ? spec.capacities[0]
                                                            : spec.capacities[static_cast<std::size_t>(w)];
        cfg.workers.push_back(SimWorkerConfig{cap, spec.block, spec.prefill_budget});
    }
    cfg.proactive_pin = spec.proactive_pin;
    cfg.pin_threshold = spec.pin_threshold;
    cfg.pin_capacity_frac = spec.pin_capacity_frac;
    cfg.seed = spec.seed;
    cfg.stochastic = spec.stochastic;
    cfg.collect_trace = spec.collect_trace;
    cfg.max_iterations = spec.max_iterations;
    return cfg;
}

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s workflow inputs profile spec [--engine tiny|tiny_f32]\n", argv[0]);
        return 2;
    }
    try {
        const WorkflowGraph g = parse_workflow(slurp(argv[1]));
        const InputBatch inputs = parse_inputs(slurp(argv[2]));
        const ProfileStats profile = parse_profile(slurp(argv[3]));
        const json js = json::parse(slurp(argv[4]));
        RunSpec spec;
        spec.workers = js.value("workers", 1);
        spec.capacities = js.value("capacities", std::vector<std::size_t>{4096});
        spec.seed = js.value("seed", std::uint64_t{0});
        spec.stochastic = js.value("stochastic", false);
        spec.proactive_pin = js.value("proactive_pin", true);
        spec.pin_threshold = js.value("pin_threshold", std::size_t{200});
        spec.pin_capacity_frac = js.value("pin_capacity_frac", 0.5);
        spec.prefill_budget = js.value("prefill_budget", std::size_t{0});
        spec.collect_trace = js.value("collect_trace", false);
        std::string engine_kind;
        for (int i = 5; i + 1 < argc; ++i)
            if (std::string(argv[i]) == "--engine") engine_kind = argv[i + 1];

        // 1. the reference: run_workflow with its own simulate() (and its
        //    prompt-cache harvest, run_pipeline.cpp:74-79)
        PromptCache ref_cache(js.value("cache_capacity", std::size_t{4096}));
        const RunResult ref = run_workflow(g, inputs, profile, spec, &ref_cache);

        // 2. the same pipeline, simulate() at run_pipeline.cpp:72 replaced by simulate_b200
        RunSpec nosim = spec;
        nosim.run_sim = false;
        const RunResult r = run_workflow(g, inputs, profile, nosim, nullptr);
        const TemplatedRadixTree call_tree = build_call_tree(r.compiled, profile, r.partition.worker_of);
        hk_engine* eng = nullptr;
        if (!engine_kind.empty()) {
            // the tiny random-init model of configs[0] (paper_2603_16104_b200/engine.py TINY)
            hk_model_config mc{2, 256, 2, 1, 128, 768, 32768, 0, 10000.0f, 1e-5f, 0,
                               engine_kind == "tiny_f32" ? 1u : 0u, 0};
            std::uint64_t cap = 0;
            for (std::size_t c : spec.capacities) cap = std::max<std::uint64_t>(cap, c);
            hk_engine_config ec{0, static_cast<std::uint32_t>(spec.workers),
                                static_cast<std::uint32_t>(cap / 16 + 600 * 80 + 64), 16, 600, 8192 + 512, 12288, 1};
            eng = hk_engine_create(&mc, &ec);
            if (!eng) throw std::runtime_error(std::string("hk_engine_create: ") + hk_last_error());
        }
        PromptCache b_cache(js.value("cache_capacity", std::size_t{4096}));
        const SimMetrics b2 = helium_b200::simulate_b200(r.compiled, profile, call_tree, r.schedule,
                                                         sim_config(spec), eng, 0, &b_cache);
        if (eng) hk_engine_destroy(eng);

        const SimMetrics& a = ref.sim;
        json eq;
        eq["schedule"] = ref.schedule.size() == r.schedule.size();
        eq["counters"] = a.iterations == b2.iterations && a.prompt_tokens == b2.prompt_tokens &&
                         a.cache_served_tokens == b2.cache_served_tokens &&
                         a.prefill_computed_tokens == b2.prefill_computed_tokens && a.decode_tokens == b2.decode_tokens &&
                         a.hit_rate_pct == b2.hit_rate_pct;
        eq["pinned_evicted"] = a.pinned_tokens == b2.pinned_tokens && a.evicted_tokens == b2.evicted_tokens;
        eq["metrics_json"] = sim_metrics_json(a) == sim_metrics_json(b2);
        eq["calls_csv"] = sim_calls_csv(a) == sim_calls_csv(b2);
        eq["trace_csv"] = sim_trace_csv(a) == sim_trace_csv(b2);
        eq["outputs"] = a.outputs == b2.outputs;
        // the harvested cross-run cache: same keys and, in mode S, the same values
        eq["prompt_cache"] = ref_cache.serialize() == b_cache.serialize();
        eq["prompt_cache_keys"] = ref_cache.keys_lru_first() == b_cache.keys_lru_first();
        bool ok = eq["counters"] && eq["pinned_evicted"] && eq["metrics_json"] && eq["calls_csv"] && eq["trace_csv"] &&
                  eq["prompt_cache_keys"];
        if (!eng) ok = ok && eq["outputs"] && eq["prompt_cache"];
        json out{{"equal", eq},
                 {"ok", ok},
                 {"engine", engine_kind.empty() ? "none (mode S)" : engine_kind},
                 {"iterations", b2.iterations},
                 {"decode_tokens", b2.decode_tokens},
                 {"calls", b2.calls.size()}};
        std::printf("%s\n", out.dump().c_str());
        return ok ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("%s\n", json{{"ok", false}, {"error", e.what()}}.dump().c_str());
        return 1;
    }
}
