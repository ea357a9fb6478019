// Flattens the reference's executor inputs into the HKPLAN01 blob that
// hk_simulate() (include/helium_b200.h) consumes.
//
// This is the reference-side half of the drop-in boundary: it is compiled
// against the reference's own headers (helios/*.hpp) and is what a maintainer
// adds next to simulator.cpp so that
//   simulate(compiled, profile, call_tree, sigma, cfg)   (simulator.hpp:128-130)
// can be served by the B200 executor. It walks exactly the structures
// simulate() reads:
//   * CompiledGraph / Operator  -> value graph used by Evaluator::prompt/value
//                                  (evaluator.cpp:79-157)
//   * ProfileStats              -> per-llm len_out (evaluator.cpp:74-78)
//   * TemplatedRadixTree        -> parents, static segments, leaves, preds
//                                  (trt.hpp:83-96; read by simulator.cpp:140-172, :268-272)
//   * Schedule                  -> per-worker call order (cost_model.hpp:31-32)
// Blob layout is documented in include/helium_b200.h.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "helios/cost_model.hpp"
#include "helios/evaluator.hpp"
#include "helios/signature.hpp"
#include "helios/trt.hpp"
#include "helios/workflow.hpp"

namespace helium_b200 {

class PlanWriter {
  public:
    std::vector<std::uint64_t> words;

    void u(std::uint64_t v) { words.push_back(v); }
    void i(std::int64_t v) { words.push_back(static_cast<std::uint64_t>(v)); }
    void f(double v) {
        std::uint64_t b;
        std::memcpy(&b, &v, 8);
        words.push_back(b);
    }
};

// Interns token runs into one pool so shared system prompts are stored once.
class SpanPool {
  public:
    std::vector<std::uint64_t> tokens;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> spans;

    std::uint64_t intern(const helios::TokenSeq& t) {
        auto it = index_.find(t);
        if (it != index_.end()) return it->second;
        std::uint64_t id = spans.size();
        spans.emplace_back(tokens.size(), t.size());
        tokens.insert(tokens.end(), t.begin(), t.end());
        index_.emplace(t, id);
        return id;
    }

  private:
    std::map<helios::TokenSeq, std::uint64_t> index_;
};

enum : std::uint64_t { kBound = 0, kOutput = 1, kLambda = 2, kFormat = 3, kLlm = 4 };

// with_signatures appends the HKSIG001 section: compute_signatures
// (signature.cpp:29-104) of every node, the keys of the prompt cache
// (hk_pcache_harvest; optimizer.cpp:113-125 harvests with the same keys).
inline std::vector<std::uint8_t> export_plan(const helios::CompiledGraph& c,
                                             const helios::ProfileStats& profile,
                                             const helios::TemplatedRadixTree& tree,
                                             const helios::Schedule& sigma,
                                             bool with_signatures = true) {
    using namespace helios;
    SpanPool pool;
    struct NodeRec {
        std::int64_t id;
        std::uint64_t kind, flags;
        double len_out;
        std::vector<std::int64_t> a;
    };
    std::vector<NodeRec> nodes;
    for (const auto& [id, n] : c.graph.nodes) {
        NodeRec r{id, 0, 0, std::nan(""), {}};
        switch (n.kind) {
            case OpKind::kInput:
            case OpKind::kData:
            case OpKind::kCacheFetch: {
                r.kind = kBound;
                auto it = c.bound.find(id);
                if (it != c.bound.end())
                    for (const TokenSeq& v : it->second)
                        r.a.push_back(static_cast<std::int64_t>(pool.intern(v)));
                break;
            }
            case OpKind::kOutput:
                r.kind = kOutput;
                r.a.push_back(c.graph.inputs_of(id).at(0));
                break;
            case OpKind::kLambda: {
                r.kind = kLambda;
                const std::string& fn = n.fn;
                if (fn == "identity") {
                    r.a = {0, 0};
                } else if (fn == "concat") {
                    r.a = {1, 0};
                } else if (fn.rfind("truncate:", 0) == 0) {
                    r.a = {2, static_cast<std::int64_t>(std::stoul(fn.substr(9)))};
                } else {
                    throw std::runtime_error("export_plan: unknown lambda fn '" + fn + "'");
                }
                for (NodeId in : c.graph.inputs_of(id)) r.a.push_back(in);
                break;
            }
            case OpKind::kFormat: {
                // Same literal/slot split as Evaluator::value kFormat (evaluator.cpp:122-143).
                r.kind = kFormat;
                std::vector<NodeId> ins = c.graph.inputs_of(id);
                const std::string& t = n.template_text;
                std::string lit;
                auto flush = [&] {
                    TokenSeq toks = tokenize(lit);
                    lit.clear();
                    if (toks.empty()) return;
                    r.a.push_back(0);
                    r.a.push_back(static_cast<std::int64_t>(pool.intern(toks)));
                };
                for (std::size_t k = 0; k < t.size(); ++k) {
                    if (t[k] == '{') {
                        std::size_t close = t.find('}', k);
                        int slot = std::stoi(t.substr(k + 1, close - k - 1));
                        flush();
                        r.a.push_back(1);
                        r.a.push_back(ins.at(static_cast<std::size_t>(slot)));
                        k = close;
                    } else {
                        lit.push_back(t[k]);
                    }
                }
                flush();
                break;
            }
            case OpKind::kLlm: {
                // Prompt template in Evaluator::prompt order (evaluator.cpp:79-99):
                // roles system, assistant, user; each message = marker + parts.
                r.kind = kLlm;
                r.flags = n.deterministic ? 1u : 0u;
                auto pit = profile.find(id);
                if (pit != profile.end()) {
                    r.flags |= 2u;
                    r.len_out = pit->second.len_out;
                }
                for (int role = 0; role < 3; ++role) {
                    for (const Message& m : n.messages) {
                        if (static_cast<int>(m.role) != role) continue;
                        r.a.push_back(0);
                        r.a.push_back(static_cast<std::int64_t>(pool.intern({role_marker(m.role)})));
                        for (const MessagePart& p : m.parts) {
                            if (p.is_ref) {
                                r.a.push_back(1);
                                r.a.push_back(p.ref);
                            } else {
                                TokenSeq toks = tokenize(p.text);
                                if (toks.empty()) continue;
                                r.a.push_back(0);
                                r.a.push_back(static_cast<std::int64_t>(pool.intern(toks)));
                            }
                        }
                    }
                }
                break;
            }
        }
        nodes.push_back(std::move(r));
    }

    PlanWriter w;
    w.u(0x31304e414c504b48ull);  // "HKPLAN01"
    w.u(c.batch);
    // tree statics are interned before the pool is written
    struct TPart {
        std::uint64_t is_static;
        std::int64_t v, q;
    };
    std::vector<std::vector<TPart>> tparts(tree.node_count());
    for (std::size_t k = 0; k < tree.node_count(); ++k) {
        for (const SegmentPart& p : tree.node(static_cast<int>(k)).seg.parts) {
            if (p.is_static)
                tparts[k].push_back({1, static_cast<std::int64_t>(pool.intern(p.tokens)), -1});
            else
                tparts[k].push_back({0, p.source, p.query});
        }
    }
    w.u(pool.tokens.size());
    for (std::uint64_t t : pool.tokens) w.u(t);
    w.u(pool.spans.size());
    for (auto& [off, len] : pool.spans) {
        w.u(off);
        w.u(len);
    }
    w.u(nodes.size());
    for (const NodeRec& r : nodes) {
        w.i(r.id);
        w.u(r.kind);
        w.u(r.flags);
        w.f(r.len_out);
        w.u(r.a.size());
        for (std::int64_t v : r.a) w.i(v);
    }
    w.u(c.graph.outputs.size());
    for (NodeId o : c.graph.outputs) w.i(o);
    w.u(tree.node_count());
    for (std::size_t k = 0; k < tree.node_count(); ++k) {
        const TrtNode& n = tree.node(static_cast<int>(k));
        w.i(n.parent);
        w.u(n.is_leaf ? 1 : 0);
        w.i(n.is_leaf ? n.leaf.op : -1);
        w.i(n.is_leaf ? n.leaf.query : -1);
        w.u(tparts[k].size());
        for (const TPart& p : tparts[k]) {
            w.u(p.is_static);
            w.i(p.v);
            w.i(p.q);
        }
        w.u(n.preds.size());
        for (int p : n.preds) w.i(p);
    }
    w.u(sigma.size());
    for (const auto& wq : sigma) {
        w.u(wq.size());
        for (const CallId& cid : wq) {
            w.i(cid.op);
            w.i(cid.query);
        }
    }
    if (with_signatures) {
        const SignatureSet sigs = compute_signatures(c, profile);
        w.u(0x3130304749534b48ull);  // "HKSIG001"
        w.u(sigs.sig.size());
        for (const auto& [id, v] : sigs.sig) {
            w.i(id);
            w.u(sigs.tainted.at(id) ? 1 : 0);
            for (std::uint64_t x : v) w.u(x);
        }
    }
    std::vector<std::uint8_t> bytes(w.words.size() * 8);
    std::memcpy(bytes.data(), w.words.data(), bytes.size());
    return bytes;
}

}  // namespace helium_b200
