// The reference-side drop-in: helios::simulate served by the B200 executor.
//
//   SimMetrics simulate(const CompiledGraph&, const ProfileStats&,
//                       const TemplatedRadixTree& call_tree, const Schedule& sigma,
//                       const SimConfig& cfg);            (simulator.hpp:128-130)
//
// simulate_b200 has the same arguments, result type and error behaviour
// (std::runtime_error with the reference's "simulate: ..." messages,
// simulator.cpp:226-244, :286) plus the device engine: with engine == nullptr
// the LLM body is the reference's synth_llm_output (mode S, byte-identical to
// helios::simulate), with an engine it is the B200 transformer. A maintainer
// compiles this header next to simulator.cpp and replaces the call at
// run_pipeline.cpp:72; tests/dropin/dropin_main.cpp does exactly that against
// the unmodified reference library and checks every SimMetrics field.
#pragma once

#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "helios/prompt_cache.hpp"
#include "helios/simulator.hpp"
#include "helium_b200.h"
#include "plan_export.hpp"

namespace helium_b200 {

namespace detail {
inline std::string report(const hk_run* run, int which) {
    std::string s(hk_run_report(run, which, nullptr, 0), '\0');
    hk_run_report(run, which, s.data(), s.size());
    if (!s.empty() && s.back() == '\0') s.pop_back();
    return s;
}
inline std::vector<std::uint64_t> worker_stat(const hk_run* run, int which) {
    std::vector<std::uint64_t> v(hk_run_worker_stat(run, which, nullptr, 0));
    hk_run_worker_stat(run, which, v.data(), v.size());
    return v;
}
inline std::vector<std::vector<std::uint64_t>> csv_rows(const std::string& csv) {
    std::vector<std::vector<std::uint64_t>> rows;
    std::istringstream in(csv);
    std::string line;
    std::getline(in, line);  // header
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::vector<std::uint64_t> r;
        std::istringstream ls(line);
        std::string cell;
        while (std::getline(ls, cell, ','))
            r.push_back(static_cast<std::uint64_t>(std::stoll(cell)));
        rows.push_back(std::move(r));
    }
    return rows;
}
}  // namespace detail

// harvest_into (optional): the cross-run PromptCache of run_workflow
// (run_pipeline.cpp:74-79). run_workflow fills it with the Evaluator's
// synthesized values; under an engine the values the run GENERATED are the
// transformer's, so this harvests them from the run itself
// (hk_pcache_harvest, optimizer.cpp:113-125 with the same signatures) and the
// next submission's substitute_cached fetches device tokens.
inline helios::SimMetrics simulate_b200(const helios::CompiledGraph& g, const helios::ProfileStats& prof,
                                        const helios::TemplatedRadixTree& tree, const helios::Schedule& sigma,
                                        const helios::SimConfig& cfg, hk_engine* engine = nullptr,
                                        std::uint32_t flags = 0, helios::PromptCache* harvest_into = nullptr) {
    const std::vector<std::uint8_t> plan = export_plan(g, prof, tree, sigma);
    std::vector<std::uint64_t> cap, blk, bud;
    for (const auto& w : cfg.workers) {
        cap.push_back(w.capacity);
        blk.push_back(w.block);
        bud.push_back(w.prefill_budget);
    }
    hk_sim_config c{static_cast<std::uint32_t>(cfg.workers.size()), cap.data(), blk.data(), bud.data(),
                    cfg.proactive_pin ? 1 : 0, cfg.pin_threshold, cfg.pin_capacity_frac, cfg.seed,
                    cfg.stochastic ? 1 : 0, cfg.collect_trace ? 1 : 0, cfg.max_iterations};
    hk_run* run = hk_simulate(plan.data(), plan.size(), &c, engine, flags);
    if (!run) throw std::runtime_error(hk_last_error());  // keeps the "simulate: ..." wording
    helios::SimMetrics out;
    hk_metrics m{};
    hk_run_metrics(run, &m);
    out.iterations = m.iterations;
    out.prompt_tokens = m.prompt_tokens;
    out.cache_served_tokens = m.cache_served_tokens;
    out.prefill_computed_tokens = m.prefill_computed_tokens;
    out.decode_tokens = m.decode_tokens;
    out.hit_rate_pct = m.hit_rate_pct;
    for (std::uint64_t v : detail::worker_stat(run, 0)) out.pinned_tokens.push_back(static_cast<std::size_t>(v));
    out.evicted_tokens = detail::worker_stat(run, 1);
    // call rows (admission order) and the per-(iteration, worker) trace
    for (const auto& r : detail::csv_rows(detail::report(run, 1))) {
        helios::SimCallRow row;
        row.call = helios::CallId{static_cast<helios::NodeId>(static_cast<std::int64_t>(r.at(0))), static_cast<int>(r.at(1))};
        row.worker = static_cast<int>(r.at(2));
        row.admitted_iter = r.at(3);
        row.prefill_done_iter = r.at(4);
        row.completed_iter = r.at(5);
        row.prompt_tokens = r.at(6);
        row.cached_tokens = r.at(7);
        row.output_tokens = r.at(8);
        out.calls.push_back(row);
    }
    if (cfg.collect_trace)
        for (const auto& r : detail::csv_rows(detail::report(run, 2)))
            out.trace.push_back(helios::SimIterRow{r.at(0), static_cast<int>(r.at(1)), static_cast<int>(r.at(2)),
                                                   r.at(3), r.at(4), r.at(5)});
    // workflow outputs: n_nodes, {node, batch, {len, tokens[len]}[batch]}[n_nodes]
    std::vector<std::uint64_t> w(hk_run_outputs(run, nullptr, 0));
    hk_run_outputs(run, w.data(), w.size());
    std::size_t i = 1;
    for (std::uint64_t n = 0; !w.empty() && n < w[0]; ++n) {
        const helios::NodeId id = static_cast<helios::NodeId>(static_cast<std::int64_t>(w[i++]));
        const std::uint64_t batch = w[i++];
        std::vector<helios::TokenSeq>& vals = out.outputs[id];
        for (std::uint64_t b = 0; b < batch; ++b) {
            const std::uint64_t len = w[i++];
            vals.emplace_back(w.begin() + static_cast<std::ptrdiff_t>(i), w.begin() + static_cast<std::ptrdiff_t>(i + len));
            i += len;
        }
    }
    if (harvest_into) {
        const std::string doc = harvest_into->serialize();
        hk_pcache* pc = hk_pcache_load(doc.data(), doc.size());
        if (!pc) {
            hk_run_free(run);
            throw std::runtime_error(hk_last_error());
        }
        const bool ok = hk_pcache_harvest(pc, plan.data(), plan.size(), run) >= 0;
        std::string saved(ok ? hk_pcache_save(pc, nullptr, 0) : 0, '\0');
        if (ok) hk_pcache_save(pc, saved.data(), saved.size());
        hk_pcache_destroy(pc);
        if (!ok) {
            hk_run_free(run);
            throw std::runtime_error(hk_last_error());
        }
        saved.pop_back();  // NUL
        *harvest_into = helios::PromptCache::deserialize(saved);
    }
    hk_run_free(run);
    return out;
}

}  // namespace helium_b200
