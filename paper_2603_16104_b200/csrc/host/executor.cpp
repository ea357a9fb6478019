// The LLM-as-operator executor: simulate() restated from the reference
// (simulator.cpp:222-389) with the LLM body and the KV block pool made real.
//
// Control-plane semantics are kept bit-exact with the reference:
//   * validation messages (simulator.cpp:225-244),
//   * pin planning + pinned insert per worker (:250-265),
//   * per-iteration, per-worker admission in schedule order with the
//     backlog/budget rule and dependency readiness (:295-327),
//   * chunked prefill in admission order with per-chunk inserts (:331-343),
//   * one decode per running call whose prefill finished in an EARLIER
//     iteration, completion insert of prompt||output and hold release (:347-374),
//   * same-iteration visibility of completions to later workers (:287-379).
// Device work for each (iteration, worker) is described as a StepPlan and run
// by the LlmBody; see DESIGN.md §Executor for the mapping of reference
// iterations onto transformer forward passes.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <sstream>

#include "hk_host.hpp"

namespace hk {

namespace {

void ensure_pages(LiveCall& lc, std::size_t upto_tokens, std::size_t block, PagePool* pool) {
    if (!pool) return;
    const std::size_t need = (upto_tokens + block - 1) / block;
    while (lc.pages.size() < need) lc.pages.push_back(pool->alloc());
}

}  // namespace

SimMetrics simulate(const Plan& plan, const SimConfig& cfg, LlmBody& body, const ExecOptions& opts) {
    const std::size_t W = plan.sigma.size();
    if (W == 0) throw std::runtime_error("simulate: no workers");
    if (cfg.workers.size() != W) throw std::runtime_error("simulate: worker config count does not match schedule");

    std::map<CallId, int> seen;
    std::size_t total = 0;
    for (const auto& wq : plan.sigma) {
        for (const CallId& c : wq) {
            if (plan.leaf(c.op, c.query) < 0) throw std::runtime_error("simulate: scheduled call is not a tree leaf");
            if (seen.count(c)) throw std::runtime_error("simulate: call scheduled twice");
            seen[c] = 1;
            ++total;
        }
    }
    if (total != plan.leaves.size()) throw std::runtime_error("simulate: schedule does not cover all calls");

    // One-worker mode (one process per GPU): this process runs only worker
    // `only` of the schedule. Exact whenever no call of that worker waits on a
    // call of another worker (then its timeline is independent of the others).
    const int only = opts.only_worker;
    if (only >= static_cast<int>(W)) throw std::runtime_error("simulate: only_worker out of range");
    // replay: every worker's control plane runs here, outputs of other workers
    // arrive through opts.exchange (cross-worker dependencies allowed)
    const bool replay = only >= 0 && static_cast<bool>(opts.exchange);
    if (only >= 0 && !replay) {
        std::map<CallId, int> wof;
        for (std::size_t w = 0; w < W; ++w)
            for (const CallId& c : plan.sigma[w]) wof[c] = static_cast<int>(w);
        total = plan.sigma[static_cast<std::size_t>(only)].size();
        for (const CallId& c : plan.sigma[static_cast<std::size_t>(only)])
            for (int p : plan.tree[static_cast<std::size_t>(plan.leaf(c.op, c.query))].preds) {
                const TreeNode& pn = plan.tree[static_cast<std::size_t>(p)];
                if (wof[CallId{pn.op, pn.query}] != only)
                    throw std::runtime_error(
                        "simulate: only_worker mode cannot serve a cross-worker dependency (run all workers)");
            }
    }
    auto active = [&](std::size_t w) { return only < 0 || static_cast<int>(w) == only; };
    // host control plane of worker w runs in this process
    auto simulated = [&](std::size_t w) { return replay || active(w); };

    Evaluator ev(plan, cfg.seed, cfg.stochastic, /*strict_llm=*/true);

    SimMetrics m;
    const bool paged = body.uses_pages();
    std::vector<std::unique_ptr<KvTree>> caches;
    std::vector<std::unique_ptr<PagePool>> pools;
    std::vector<std::size_t> budgets(W, 0);
    const auto t_pin0 = std::chrono::steady_clock::now();
    m.pin_compute_tokens.assign(W, 0);
    for (std::size_t w = 0; w < W; ++w) {
        const SimWorkerConfig& wc = cfg.workers[w];
        caches.push_back(std::make_unique<KvTree>(wc.capacity, wc.block));
        pools.push_back(std::make_unique<PagePool>(paged && active(w) ? body.pages_per_worker(static_cast<int>(w)) : 0));
        if (paged && active(w)) {
            caches[w]->set_page_pool(pools[w].get());
            caches[w]->journaling = body.device_lookup();
        }
        budgets[w] = wc.prefill_budget > 0 ? wc.prefill_budget : std::max<std::size_t>(wc.capacity / 8, wc.block);
        if (cfg.proactive_pin && simulated(w)) {
            const auto budget = static_cast<std::size_t>(cfg.pin_capacity_frac * static_cast<double>(wc.capacity));
            std::vector<TokenSeq> pins = static_pin_prefixes(plan, static_cast<int>(w), wc.block, cfg.pin_threshold, budget);
            std::vector<std::vector<int>> pin_pages;
            std::vector<std::size_t> first_new;
            for (const TokenSeq& p : pins) {
                std::vector<int> created;
                caches[w]->insert(p.data(), p.size(), p.size(), true, 0, {}, &created);
                std::vector<int> path;
                caches[w]->peek(p.data(), p.size(), &path);
                std::vector<int> pages;
                for (int nd : path) pages.push_back(caches[w]->node_page(nd));
                // created nodes are the tail of the path (a pin extends earlier pins)
                const std::size_t fn = path.size() - created.size();
                m.pin_compute_tokens[w] += created.size() * wc.block;
                pin_pages.push_back(std::move(pages));
                first_new.push_back(fn);
            }
            if (paged && active(w)) body.precompute_pins(static_cast<int>(w), pins, pin_pages, first_new);
        }
        m.pinned_tokens.push_back(caches[w]->pinned_tokens());
    }

    m.pin_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_pin0).count();
    const auto t_iter0 = std::chrono::steady_clock::now();
    std::vector<char> leaf_done(plan.tree.size(), 0);
    auto ready = [&](int leaf) {
        for (int p : plan.tree[static_cast<std::size_t>(leaf)].preds)
            if (!leaf_done[static_cast<std::size_t>(p)]) return false;
        return true;
    };

    std::vector<std::vector<char>> admitted(W);
    for (std::size_t w = 0; w < W; ++w) admitted[w].assign(plan.sigma[w].size(), 0);
    std::vector<std::vector<std::unique_ptr<LiveCall>>> live(W);
    std::vector<std::size_t> backlog(W, 0);

    const std::uint64_t guard = cfg.max_iterations > 0 ? cfg.max_iterations : 10'000'000ull;
    std::uint64_t holdc = 0;
    std::size_t completed = 0;
    std::uint64_t iter = 0;
    std::vector<std::pair<int, LiveCall*>> completing;

    while (completed < total) {
        ++iter;
        if (iter > guard) throw std::runtime_error("simulate: iteration guard tripped");

        // Calls that will complete this iteration with a non-empty output are
        // already determined: running decoders one token short of out_len.
        completing.clear();
        for (std::size_t w = 0; w < W; ++w)
            for (auto& lcp : live[w]) {
                if (!active(w)) break;  // (replay: other workers' calls are host-only)
                LiveCall& lc = *lcp;
                if (lc.out_len > 0 && lc.remaining() == 0 && lc.prefill_done_iter < iter && lc.decoded + 1 == lc.out_len)
                    completing.emplace_back(static_cast<int>(w), &lc);
            }
        body.begin_iteration(iter, completing);

        for (std::size_t w = 0; w < W; ++w) {
            if (!simulated(w)) continue;
            const bool dev = active(w);            // this worker's body (device) runs here
            const bool wpaged = paged && dev;
            const bool dlook = dev && body.device_lookup();
            KvTree& cache = *caches[w];
            PagePool* pool = wpaged ? pools[w].get() : nullptr;
            if (pool) pool->flush_deferred();
            SimIterRow row;
            row.iter = iter;
            row.worker = static_cast<int>(w);
            StepPlan sp;
            sp.worker = static_cast<int>(w);
            sp.iter = iter;

            // ---- admission (simulator.cpp:295-327) ----
            // Candidates are ready, not-yet-admitted calls in schedule order.
            // Lookups of one admission burst do not observe each other (no
            // inserts happen between them), so a device body matches them as a
            // batch; the budget rule then decides how many are admitted and
            // only those get their touches/holds applied, in order.
            std::size_t qi = 0;
            bool stop = false;
            while (!stop) {
                std::vector<std::size_t> cand;
                std::vector<TokenSeq> prompts;
                const std::size_t max_batch = dlook ? 1024 : 1;
                std::size_t scan = qi;
                for (; scan < plan.sigma[w].size() && cand.size() < max_batch; ++scan) {
                    if (admitted[w][scan]) continue;
                    const CallId call = plan.sigma[w][scan];
                    if (!ready(plan.leaf(call.op, call.query))) continue;
                    cand.push_back(scan);
                    prompts.push_back(ev.prompt(call.op, static_cast<std::size_t>(call.query)));
                }
                if (cand.empty()) break;
                std::vector<std::vector<int>> paths;
                if (dlook) {
                    if (backlog[w] >= budgets[w]) break;
                    body.sync_trie(static_cast<int>(w), cache);
                    std::vector<const TokenSeq*> pp;
                    for (auto& p : prompts) pp.push_back(&p);
                    body.lookup_batch(static_cast<int>(w), pp, paths);
                }
                std::size_t k = 0;
                for (; k < cand.size(); ++k) {
                    if (backlog[w] >= budgets[w]) {
                        stop = true;
                        break;
                    }
                    const std::size_t idx = cand[k];
                    const CallId call = plan.sigma[w][idx];
                    admitted[w][idx] = 1;
                    auto lcp = std::make_unique<LiveCall>();
                    LiveCall& lc = *lcp;
                    lc.id = call;
                    lc.leaf = plan.leaf(call.op, call.query);
                    lc.group = plan.static_group[static_cast<std::size_t>(lc.leaf)];
                    lc.group_tokens = plan.static_group_tokens[static_cast<std::size_t>(lc.leaf)];
                    lc.prompt = std::move(prompts[k]);
                    lc.out_len = synth_llm_len(lc.prompt, ev.profile_len_out(call.op), ev.deterministic(call.op),
                                               cfg.seed, cfg.stochastic);
                    lc.hold = ++holdc;
                    std::vector<int> path;
                    if (dlook) {
                        path = paths[k];
                        if (opts.verify_device_lookup) {
                            std::vector<int> hp;
                            cache.peek(lc.prompt.data(), lc.prompt.size(), &hp);
                            if (hp != path)
                                throw std::runtime_error("device trie lookup diverged from the host tree for call op " +
                                                         std::to_string(call.op) + " q " + std::to_string(call.query));
                        }
                        cache.apply_lookup(path.data(), path.size(), lc.hold);
                        lc.done = path.size() * cache.block();
                    } else {
                        lc.done = cache.lookup(lc.prompt.data(), lc.prompt.size(), lc.hold, pool ? &path : nullptr);
                    }
                    if (pool)
                        for (int nd : path) lc.pages.push_back(cache.node_page(nd));
                    if (lc.remaining() == 0) lc.prefill_done_iter = iter;
                    backlog[w] += lc.remaining();

                    SimCallRow cr;
                    cr.call = call;
                    cr.worker = static_cast<int>(w);
                    cr.admitted_iter = iter;
                    cr.prompt_tokens = lc.prompt.size();
                    cr.cached_tokens = lc.done;
                    lc.row = m.calls.size();
                    m.prompt_tokens += lc.prompt.size();
                    m.cache_served_tokens += lc.done;
                    m.calls.push_back(cr);
                    if (dev) body.on_admit(static_cast<int>(w), lc);
                    if (lc.remaining() == 0 && lc.out_len > 0 && wpaged) {
                        // Fully cached prompt: the model still needs the logits of
                        // the last prompt position to produce output token 1. Re-run
                        // that position without rewriting its (shared) KV.
                        StepPlan::Seg s;
                        s.call = &lc;
                        s.start = lc.prompt.empty() ? 0 : lc.prompt.size() - 1;
                        s.count = 1;
                        s.write_kv = false;
                        s.sample = true;
                        s.table = lc.pages;
                        sp.segs.push_back(std::move(s));
                        m.recompute_tokens += 1;
                    }
                    live[w].push_back(std::move(lcp));
                    ++row.admitted;
                }
                if (k < cand.size()) break;
                qi = scan;
                if (!dlook) {
                    // host path admits one candidate at a time; continue scanning
                    if (scan >= plan.sigma[w].size()) break;
                }
            }
            row.active = static_cast<int>(live[w].size());

            // ---- chunked prefill (simulator.cpp:331-343) ----
            std::size_t left = budgets[w];
            for (auto& lcp : live[w]) {
                LiveCall& lc = *lcp;
                if (left == 0) break;
                if (lc.remaining() == 0) continue;
                const std::size_t chunk = std::min(left, lc.remaining());
                if (wpaged) {
                    ensure_pages(lc, lc.done + chunk, cache.block(), pool);
                    StepPlan::Seg s;
                    s.call = &lc;
                    s.start = lc.done;
                    s.count = chunk;
                    s.sample = (lc.done + chunk == lc.prompt.size()) && lc.out_len > 0;
                    s.table = lc.pages;
                    sp.segs.push_back(std::move(s));
                }
                lc.done += chunk;
                left -= chunk;
                backlog[w] -= chunk;
                m.prefill_computed_tokens += chunk;
                row.prefill_tokens += chunk;
                cache.insert(lc.prompt.data(), lc.prompt.size(), lc.done, false, lc.hold,
                             KvTree::Owner{pool ? &lc.pages : nullptr, pool});
                if (lc.remaining() == 0) lc.prefill_done_iter = iter;
            }

            // ---- decode / complete (simulator.cpp:347-374) ----
            for (auto& lcp : live[w]) {
                LiveCall& lc = *lcp;
                if (lc.finished || lc.remaining() > 0) continue;
                if (lc.out_len > 0) {
                    if (lc.prefill_done_iter >= iter) continue;
                    ++lc.decoded;
                    ++row.decode_tokens;
                    ++m.decode_tokens;
                    if (wpaged) {
                        // decode #k feeds output token k at position |prompt|+k-1
                        const std::size_t pos = lc.prompt.size() + lc.decoded - 1;
                        ensure_pages(lc, pos + 1, cache.block(), pool);
                        StepPlan::Seg s;
                        s.call = &lc;
                        s.start = pos;
                        s.count = 1;
                        s.from_prompt = false;
                        s.sample = lc.decoded < lc.out_len;
                        s.group = lc.group;
                        s.group_tokens = lc.group_tokens;
                        s.table = lc.pages;
                        sp.segs.push_back(std::move(s));
                    }
                    if (lc.decoded < lc.out_len) continue;
                }
                const double len_out = ev.profile_len_out(lc.id.op);
                const bool det = ev.deterministic(lc.id.op);
                TokenSeq out;
                if (dev) {
                    out = lc.out_len > 0 ? body.take_output(static_cast<int>(w), lc, len_out, det) : TokenSeq{};
                    if (lc.out_len > 0) {
                        std::vector<float> lv = body.take_logits(static_cast<int>(w), lc);
                        if (!lv.empty()) m.call_logits[lc.id] = std::move(lv);
                    }
                    if (replay && lc.out_len > 0) opts.exchange(static_cast<int>(w), lc.id, out);  // send
                } else if (lc.out_len > 0) {
                    out.assign(lc.out_len, 0);
                    opts.exchange(static_cast<int>(w), lc.id, out);  // receive from the owning process
                }
                if (out.size() != lc.out_len) throw std::logic_error("simulate: output length drifted from plan");
                ev.put_llm_output(lc.id.op, static_cast<std::size_t>(lc.id.query), out);
                m.call_outputs[lc.id] = out;
                TokenSeq full = lc.prompt;
                full.insert(full.end(), out.begin(), out.end());
                cache.insert(full.data(), full.size(), full.size(), false, 0,
                             KvTree::Owner{pool ? &lc.pages : nullptr, pool});
                cache.release(lc.hold);
                if (pool) {
                    for (int pg : lc.pages)
                        if (pg >= 0 && !pool->is_tree(pg)) pool->release(pg);
                    lc.pages.clear();
                }
                if (dev) body.on_finish(static_cast<int>(w), lc);
                leaf_done[static_cast<std::size_t>(lc.leaf)] = 1;
                SimCallRow& cr = m.calls[lc.row];
                cr.prefill_done_iter = lc.prefill_done_iter;
                cr.completed_iter = iter;
                cr.output_tokens = out.size();
                lc.finished = true;
                ++completed;
            }
            if (wpaged && !sp.segs.empty()) body.run_step(sp);
            // finished calls stay alive until their step was issued (segs point at them)
            live[w].erase(std::remove_if(live[w].begin(), live[w].end(),
                                         [](const std::unique_ptr<LiveCall>& lc) { return lc->finished; }),
                          live[w].end());
            if (cfg.collect_trace) m.trace.push_back(row);
        }
    }
    body.finish_run();
    m.iter_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_iter0).count();

    m.iterations = iter;
    for (std::size_t w = 0; w < W; ++w) m.evicted_tokens.push_back(caches[w]->evicted_tokens());
    m.hit_rate_pct = m.prompt_tokens > 0
                         ? 100.0 * static_cast<double>(m.cache_served_tokens) / static_cast<double>(m.prompt_tokens)
                         : 0.0;
    if (only < 0 || replay) {
        m.outputs = ev.output_values();
    } else {
        // one-worker mode: only outputs whose llm calls all ran here
        for (NodeId id : plan.outputs) {
            try {
                std::vector<TokenSeq> vals;
                for (std::size_t b = 0; b < plan.batch; ++b) vals.push_back(ev.value(id, b));
                m.outputs[id] = std::move(vals);
            } catch (const std::runtime_error&) {
            }
        }
    }
    return m;
}

// ------------------------------------------------------------------ reports
namespace {

// nlohmann::json's number formatting (shortest round-trip, ".0" for integral
// values) so reports are byte-identical with simulator.cpp:393-405.
std::string json_double(double v) {
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, res.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    // nlohmann prints exponents as e+XX / e-XX
    auto e = s.find('e');
    if (e != std::string::npos && s[e + 1] != '-' && s[e + 1] != '+') s.insert(e + 1, "+");
    return s;
}

template <typename T>
std::string json_uint_array(const std::vector<T>& v) {
    // the reference's json.hpp prints these unsigned arrays compactly: [a,b]
    std::ostringstream os;
    os << "[";
    for (std::size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << v[i];
    os << "]";
    return os.str();
}

}  // namespace

std::string sim_metrics_json(const SimMetrics& m) {
    std::ostringstream os;
    os << "{\n";
    os << "  \"cache_served_tokens\": " << m.cache_served_tokens << ",\n";
    os << "  \"calls\": " << m.calls.size() << ",\n";
    os << "  \"decode_tokens\": " << m.decode_tokens << ",\n";
    os << "  \"evicted_tokens\": " << json_uint_array(m.evicted_tokens) << ",\n";
    os << "  \"hit_rate_pct\": " << json_double(m.hit_rate_pct) << ",\n";
    os << "  \"iterations\": " << m.iterations << ",\n";
    os << "  \"pinned_tokens\": " << json_uint_array(m.pinned_tokens) << ",\n";
    os << "  \"prefill_computed_tokens\": " << m.prefill_computed_tokens << ",\n";
    os << "  \"prompt_tokens\": " << m.prompt_tokens << "\n";
    os << "}";
    return os.str();
}

std::string sim_calls_csv(const SimMetrics& m) {
    std::ostringstream os;
    os << "op,query,worker,admitted_iter,prefill_done_iter,completed_iter,prompt_tokens,cached_tokens,output_tokens\n";
    for (const SimCallRow& r : m.calls)
        os << r.call.op << ',' << r.call.query << ',' << r.worker << ',' << r.admitted_iter << ','
           << r.prefill_done_iter << ',' << r.completed_iter << ',' << r.prompt_tokens << ',' << r.cached_tokens
           << ',' << r.output_tokens << '\n';
    return os.str();
}

std::string sim_trace_csv(const SimMetrics& m) {
    std::ostringstream os;
    os << "iter,worker,active,admitted,prefill_tokens,decode_tokens\n";
    for (const SimIterRow& r : m.trace)
        os << r.iter << ',' << r.worker << ',' << r.active << ',' << r.admitted << ',' << r.prefill_tokens << ','
           << r.decode_tokens << '\n';
    return os.str();
}

}  // namespace hk
