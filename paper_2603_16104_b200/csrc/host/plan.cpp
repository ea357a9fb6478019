// HKPLAN01 parser and the prompt evaluator.
// Evaluator restates Evaluator::prompt / value (evaluator.cpp:79-157) and
// apply_lambda (workflow.cpp:258-273) over the flattened value graph.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "hk_host.hpp"

namespace hk {

namespace {

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }

class Reader {
  public:
    Reader(const std::uint8_t* d, std::size_t n) : d_(d), n_(n) {}
    std::uint64_t u() {
        if (pos_ + 8 > n_) fail("plan: truncated blob");
        std::uint64_t v;
        std::memcpy(&v, d_ + pos_, 8);
        pos_ += 8;
        return v;
    }
    std::int64_t i() { return static_cast<std::int64_t>(u()); }
    double f() {
        std::uint64_t b = u();
        double v;
        std::memcpy(&v, &b, 8);
        return v;
    }
    std::size_t count(std::size_t max_elems_per_word = 1) {
        std::uint64_t c = u();
        if (c > (n_ - pos_) / 8 * max_elems_per_word + 1) fail("plan: corrupt count");
        return static_cast<std::size_t>(c);
    }
    bool done() const { return pos_ == n_; }
    std::size_t pos() const { return pos_; }

  private:
    const std::uint8_t* d_;
    std::size_t n_, pos_ = 0;
};

}  // namespace

std::vector<int> Plan::path_from_root(int n) const {
    std::vector<int> path;
    for (int cur = n; cur >= 0; cur = tree[static_cast<std::size_t>(cur)].parent) path.push_back(cur);
    std::reverse(path.begin(), path.end());
    return path;
}

Plan parse_plan(const std::uint8_t* data, std::size_t n) {
    if (!data || n < 16 || n % 8) fail("plan: blob must be a non-empty multiple of 8 bytes");
    Reader r(data, n);
    if (r.u() != 0x31304e414c504b48ull) fail("plan: bad magic (expected HKPLAN01)");
    Plan p;
    p.batch = r.u();
    std::size_t nt = r.count();
    p.pool.resize(nt);
    for (auto& t : p.pool) t = r.u();
    std::size_t ns = r.count();
    p.spans.resize(ns);
    for (auto& s : p.spans) {
        s.first = r.u();
        s.second = r.u();
        if (s.first + s.second > nt) fail("plan: span out of range");
    }
    std::size_t nn = r.count();
    for (std::size_t k = 0; k < nn; ++k) {
        PlanNode nd;
        nd.id = r.i();
        std::uint64_t kind = r.u();
        if (kind > 4) fail("plan: bad node kind");
        nd.kind = static_cast<Kind>(kind);
        std::uint64_t flags = r.u();
        nd.deterministic = (flags & 1u) != 0;
        nd.has_profile = (flags & 2u) != 0;
        nd.len_out = r.f();
        std::size_t na = r.count();
        nd.a.resize(na);
        for (auto& v : nd.a) v = r.i();
        p.nodes[nd.id] = std::move(nd);
    }
    std::size_t no = r.count();
    for (std::size_t k = 0; k < no; ++k) p.outputs.push_back(r.i());
    std::size_t ntn = r.count();
    p.tree.resize(ntn);
    for (std::size_t k = 0; k < ntn; ++k) {
        TreeNode& t = p.tree[k];
        t.parent = static_cast<int>(r.i());
        t.is_leaf = r.u() != 0;
        t.op = r.i();
        t.query = static_cast<int>(r.i());
        std::size_t np = r.count();
        t.parts.resize(np);
        for (auto& pt : t.parts) {
            pt.is_static = r.u() != 0;
            pt.v = r.i();
            pt.q = r.i();
        }
        std::size_t npred = r.count();
        for (std::size_t j = 0; j < npred; ++j) t.preds.push_back(static_cast<int>(r.i()));
        if (t.is_leaf) {
            p.leaves.push_back(static_cast<int>(k));
            p.leaf_index[CallId{t.op, t.query}] = static_cast<int>(k);
        }
    }
    p.sigma_offset = r.pos();
    std::size_t nw = r.count();
    p.sigma.resize(nw);
    for (auto& wq : p.sigma) {
        std::size_t nc = r.count();
        for (std::size_t j = 0; j < nc; ++j) {
            CallId c;
            c.op = r.i();
            c.query = static_cast<int>(r.i());
            wq.push_back(c);
        }
    }
    p.sig_offset = r.pos();
    if (!r.done()) {
        // optional: per-node content signatures (signature.cpp:29-104) for the prompt cache
        if (r.u() != 0x3130304749534b48ull) fail("plan: trailing bytes");
        std::size_t nsig = r.count();
        for (std::size_t k = 0; k < nsig; ++k) {
            const NodeId id = r.i();
            p.tainted[id] = r.u() != 0;
            std::vector<std::uint64_t>& v = p.sig[id];
            v.resize(p.batch);
            for (auto& x : v) x = r.u();
        }
        p.has_sigs = true;
        if (!r.done()) fail("plan: trailing bytes");
    }
    // TRT static groups (see Plan::static_group)
    p.static_group.assign(p.tree.size(), -1);
    p.static_group_tokens.assign(p.tree.size(), 0);
    std::vector<int> leaves_under(p.tree.size(), 0);
    for (int lf : p.leaves)
        for (int v = lf; v >= 0; v = p.tree[static_cast<std::size_t>(v)].parent) ++leaves_under[static_cast<std::size_t>(v)];
    for (int lf : p.leaves) {
        // the deepest branching node (>= 2 calls below it) whose root path is all static text
        std::size_t toks = 0, best_toks = 0;
        int best = -1;
        for (int v : p.path_from_root(p.tree[static_cast<std::size_t>(lf)].parent)) {
            const TreeNode& t = p.tree[static_cast<std::size_t>(v)];
            bool all_static = true;
            for (const TreePart& pt : t.parts) {
                if (!pt.is_static) {
                    all_static = false;
                    break;
                }
                toks += p.span_len(pt.v);
            }
            if (!all_static) break;
            if (leaves_under[static_cast<std::size_t>(v)] >= 2 && toks > 0) {
                best = v;
                best_toks = toks;
            }
        }
        p.static_group[static_cast<std::size_t>(lf)] = best;
        p.static_group_tokens[static_cast<std::size_t>(lf)] = best_toks;
    }
    return p;
}

// Call-level partition (opt-in). DIVERGES from the reference,
// whose partition_workflow places whole operators on workers (scheduler.cpp:
// 59-115), so a one-operator workflow (configs[1]) can only ever use one
// worker there. Here every operator's calls are dealt round-robin over
// `workers` in the plan's schedule order (which each worker keeps); the
// blob's value graph and call tree are unchanged, only the schedule section
// (the blob's tail) is rewritten.
std::vector<std::uint8_t> partition_calls(const std::uint8_t* data, std::size_t n, int workers) {
    if (workers < 1) fail("partition_calls: workers must be positive");
    Plan p = parse_plan(data, n);
    std::vector<std::vector<CallId>> sigma(static_cast<std::size_t>(workers));
    std::map<NodeId, int> next;
    for (const auto& wq : p.sigma)
        for (const CallId& c : wq) sigma[static_cast<std::size_t>(next[c.op]++ % workers)].push_back(c);
    std::vector<std::uint64_t> tail;
    tail.push_back(static_cast<std::uint64_t>(workers));
    for (const auto& wq : sigma) {
        tail.push_back(wq.size());
        for (const CallId& c : wq) {
            tail.push_back(static_cast<std::uint64_t>(c.op));
            tail.push_back(static_cast<std::uint64_t>(static_cast<std::int64_t>(c.query)));
        }
    }
    std::vector<std::uint8_t> out(data, data + p.sigma_offset);
    const std::size_t head = out.size();
    out.resize(head + tail.size() * 8);
    std::memcpy(out.data() + head, tail.data(), tail.size() * 8);
    out.insert(out.end(), data + p.sig_offset, data + n);  // signature section, if any
    return out;
}

// ---------------------------------------------------------------- evaluator

double Evaluator::profile_len_out(NodeId llm) const {
    const PlanNode& n = plan_->nodes.at(llm);
    if (!n.has_profile) fail("no profile entry for llm node " + std::to_string(llm));
    return n.len_out;
}

TokenSeq Evaluator::prompt(NodeId llm, std::size_t q) {
    auto it = plan_->nodes.find(llm);
    if (it == plan_->nodes.end() || it->second.kind != Kind::kLlm)
        fail("node " + std::to_string(llm) + " is not an llm");
    const PlanNode& n = it->second;
    TokenSeq out;
    for (std::size_t k = 0; k + 1 < n.a.size(); k += 2) {
        if (n.a[k] == 0) {
            const Token* s = plan_->span_ptr(n.a[k + 1]);
            out.insert(out.end(), s, s + plan_->span_len(n.a[k + 1]));
        } else {
            const TokenSeq& v = value(n.a[k + 1], q);
            out.insert(out.end(), v.begin(), v.end());
        }
    }
    return out;
}

const TokenSeq& Evaluator::value(NodeId id, std::size_t q) {
    auto key = std::make_pair(id, q);
    auto mit = memo_.find(key);
    if (mit != memo_.end()) return mit->second;
    auto nit = plan_->nodes.find(id);
    if (nit == plan_->nodes.end()) fail("unknown node " + std::to_string(id));
    const PlanNode& n = nit->second;
    TokenSeq v;
    switch (n.kind) {
        case Kind::kBound: {
            if (n.a.empty()) fail("node " + std::to_string(id) + " has no bound value");
            if (q >= n.a.size()) fail("query index out of range for node " + std::to_string(id));
            const Token* s = plan_->span_ptr(n.a[q]);
            v.assign(s, s + plan_->span_len(n.a[q]));
            break;
        }
        case Kind::kOutput:
            v = value(n.a.at(0), q);
            break;
        case Kind::kLambda: {
            std::vector<TokenSeq> ins;
            for (std::size_t k = 2; k < n.a.size(); ++k) ins.push_back(value(n.a[k], q));
            if (ins.empty()) fail("lambda: no inputs");
            if (n.a[0] == 0) {
                v = ins[0];
            } else if (n.a[0] == 1) {
                for (const TokenSeq& s : ins) v.insert(v.end(), s.begin(), s.end());
            } else {
                v = ins[0];
                if (v.size() > static_cast<std::size_t>(n.a[1])) v.resize(static_cast<std::size_t>(n.a[1]));
            }
            break;
        }
        case Kind::kFormat: {
            for (std::size_t k = 0; k + 1 < n.a.size(); k += 2) {
                if (n.a[k] == 0) {
                    const Token* s = plan_->span_ptr(n.a[k + 1]);
                    v.insert(v.end(), s, s + plan_->span_len(n.a[k + 1]));
                } else {
                    const TokenSeq& sub = value(n.a[k + 1], q);
                    v.insert(v.end(), sub.begin(), sub.end());
                }
            }
            break;
        }
        case Kind::kLlm: {
            if (strict_)
                fail("llm node " + std::to_string(id) + " query " + std::to_string(q) +
                     " evaluated before its call completed");
            TokenSeq pr = prompt(id, q);
            v = synth_llm_output(pr, profile_len_out(id), n.deterministic, seed_, stochastic_);
            break;
        }
    }
    return memo_[key] = std::move(v);
}

std::map<NodeId, std::vector<TokenSeq>> Evaluator::output_values() {
    std::map<NodeId, std::vector<TokenSeq>> out;
    for (NodeId id : plan_->outputs) {
        std::vector<TokenSeq> vals;
        for (std::size_t b = 0; b < plan_->batch; ++b) vals.push_back(value(id, b));
        out[id] = std::move(vals);
    }
    return out;
}

}  // namespace hk
