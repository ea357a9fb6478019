// Native cache-aware planner: the reference's partitioner,
// templated radix tree and operator scheduler, restated over the flattened
// plan (HKPLAN01) so a plan can be (re)scheduled for any worker count without
// the reference library:
//   partition_workflow         scheduler.cpp:22-115
//   TemplatedRadixTree         trt.cpp:12-260 (insert / split / dependencies / weights)
//   prefix_template, estimated_len, llm_ops_topo, llm_dependencies, build_*_tree
//                              trt.cpp:318-530, workflow.cpp:172-193 (topo_sort), :275-286 (lambda_estimate)
//   plan_operators             scheduler.cpp:117-561 (cache-aware operator scheduling)
//   expand_soft_schedule       scheduler.cpp:563-571
//   cost model                 cost_model.cpp:20-30
// Its outputs must equal the reference planner's bit for bit (the schedule
// decides which prefix is cached when), so the algorithm — including every
// tie-break and the floating-point cost arithmetic — follows the reference
// step by step; tests/test_planner_cpu.py compares call trees, schedules and
// simulate() reports against the reference on the committed plans and on
// random workflow DAGs.
#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <cstring>
#include <limits>
#include <queue>

#include "hk_host.hpp"

namespace hk {

namespace {

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kEps = 1e-9;

// ------------------------------------------------------------- graph view
// Node inputs in slot order, from the plan payloads (the exported graph is
// already bound and rewritten).
struct GraphView {
    const Plan& p;
    std::map<NodeId, std::vector<NodeId>> ins;
    std::vector<NodeId> topo;
    std::map<NodeId, bool> llm_up;  // value depends on an llm output

    explicit GraphView(const Plan& plan) : p(plan) {
        for (const auto& [id, n] : p.nodes) {
            std::vector<NodeId>& v = ins[id];
            switch (n.kind) {
                case Kind::kBound: break;
                case Kind::kOutput: v.push_back(n.a.at(0)); break;
                case Kind::kLambda:
                    for (std::size_t k = 2; k < n.a.size(); ++k) v.push_back(n.a[k]);
                    break;
                case Kind::kFormat:
                case Kind::kLlm:
                    for (std::size_t k = 0; k + 1 < n.a.size(); k += 2)
                        if (n.a[k] == 1) v.push_back(n.a[k + 1]);
                    break;
            }
        }
        // workflow.cpp:172-193: Kahn's algorithm, smallest ready id first
        std::map<NodeId, int> indeg;
        std::map<NodeId, std::set<NodeId>> succ;
        for (const auto& [id, n] : p.nodes) indeg[id] = 0;
        for (const auto& [id, v] : ins)
            for (NodeId from : v)
                if (succ[from].insert(id).second) ++indeg[id];
        std::priority_queue<NodeId, std::vector<NodeId>, std::greater<NodeId>> ready;
        for (const auto& [id, d] : indeg)
            if (d == 0) ready.push(id);
        while (!ready.empty()) {
            NodeId id = ready.top();
            ready.pop();
            topo.push_back(id);
            for (NodeId s : succ[id])
                if (--indeg[s] == 0) ready.push(s);
        }
        if (topo.size() != p.nodes.size()) fail("workflow graph has a cycle");
        for (NodeId id : topo) {  // trt.cpp:322-330
            bool v = p.nodes.at(id).kind == Kind::kLlm;
            for (NodeId in : ins.at(id)) v = v || llm_up.at(in);
            llm_up[id] = v;
        }
    }
    const PlanNode& op(NodeId id) const { return p.nodes.at(id); }
    std::vector<NodeId> llm_ops_topo() const {
        std::vector<NodeId> out;
        for (NodeId id : topo)
            if (op(id).kind == Kind::kLlm) out.push_back(id);
        return out;
    }
    // trt.cpp:454-472: nearest upstream llm operators through non-llm nodes
    std::map<NodeId, std::vector<NodeId>> llm_dependencies() const {
        std::map<NodeId, std::set<NodeId>> nearest;
        std::map<NodeId, std::vector<NodeId>> deps;
        for (NodeId id : topo) {
            std::set<NodeId> up;
            for (NodeId in : ins.at(id)) up.insert(nearest.at(in).begin(), nearest.at(in).end());
            if (op(id).kind == Kind::kLlm) {
                deps[id] = {up.begin(), up.end()};
                nearest[id] = {id};
            } else {
                nearest[id] = std::move(up);
            }
        }
        return deps;
    }
    TokenSeq span(std::int64_t s) const { return TokenSeq(p.span_ptr(s), p.span_ptr(s) + p.span_len(s)); }
};

// trt.cpp:406-449 (lambda_estimate: workflow.cpp:275-286)
double estimated_len(const GraphView& g, NodeId id, int query) {
    const PlanNode& n = g.op(id);
    switch (n.kind) {
        case Kind::kBound: {
            if (n.a.empty()) fail("node " + std::to_string(id) + " has no bound value");
            if (query >= 0) return static_cast<double>(g.p.span_len(n.a.at(static_cast<std::size_t>(query))));
            double s = 0;
            for (std::int64_t sp : n.a) s += static_cast<double>(g.p.span_len(sp));
            return s / static_cast<double>(n.a.size());
        }
        case Kind::kLlm:
            if (!n.has_profile) fail("no profile entry for llm node " + std::to_string(id));
            return n.len_out;
        case Kind::kOutput:
            return estimated_len(g, n.a.at(0), query);
        case Kind::kFormat: {
            double total = 0;
            for (std::size_t k = 0; k + 1 < n.a.size(); k += 2)
                total += n.a[k] == 0 ? static_cast<double>(g.p.span_len(n.a[k + 1])) : estimated_len(g, n.a[k + 1], query);
            return total;
        }
        case Kind::kLambda: {
            std::vector<double> in;
            for (std::size_t k = 2; k < n.a.size(); ++k) in.push_back(estimated_len(g, n.a[k], query));
            if (in.empty()) fail("lambda: no inputs");
            if (n.a[0] == 0) return in[0];
            if (n.a[0] == 1) {
                double s = 0;
                for (double v : in) s += v;
                return s;
            }
            return std::min(in[0], static_cast<double>(n.a[1]));
        }
    }
    fail("bad kind");
}

// ---------------------------------------------------------------- segments
struct SegPart {
    bool is_static = true;
    TokenSeq tokens;
    NodeId source = -1;
    int query = -1;
    double est_len = 0;
    double weight() const { return is_static ? static_cast<double>(tokens.size()) : est_len; }
    bool same_placeholder(const SegPart& o) const {
        return !is_static && !o.is_static && source == o.source && query == o.query;
    }
};

struct Seg {
    std::vector<SegPart> parts;
    double weight() const {
        double w = 0;
        for (const SegPart& p : parts) w += p.weight();
        return w;
    }
    bool all_static() const {
        return std::all_of(parts.begin(), parts.end(), [](const SegPart& p) { return p.is_static; });
    }
    void normalize() {  // merge adjacent statics, drop empty statics
        std::vector<SegPart> out;
        for (SegPart& p : parts) {
            if (p.is_static && p.tokens.empty()) continue;
            if (p.is_static && !out.empty() && out.back().is_static)
                out.back().tokens.insert(out.back().tokens.end(), p.tokens.begin(), p.tokens.end());
            else
                out.push_back(std::move(p));
        }
        parts = std::move(out);
    }
};

Seg slice_from(const std::vector<SegPart>& parts, std::size_t j, std::size_t jo) {
    Seg s;
    for (std::size_t k = j; k < parts.size(); ++k) {
        SegPart p = parts[k];
        if (k == j && p.is_static && jo > 0)
            p.tokens.assign(parts[k].tokens.begin() + static_cast<std::ptrdiff_t>(jo), parts[k].tokens.end());
        s.parts.push_back(std::move(p));
    }
    s.normalize();
    return s;
}

Seg slice_prefix(const std::vector<SegPart>& parts, std::size_t i, std::size_t io) {
    Seg s;
    for (std::size_t k = 0; k < i; ++k) s.parts.push_back(parts[k]);
    if (io > 0) {
        SegPart p = parts[i];
        p.tokens.assign(parts[i].tokens.begin(), parts[i].tokens.begin() + static_cast<std::ptrdiff_t>(io));
        s.parts.push_back(std::move(p));
    }
    s.normalize();
    return s;
}

// trt.cpp:336-402: the prompt template of one llm operator (query -1) or call
Seg prefix_template(const GraphView& g, Evaluator& ev, NodeId llm, int query) {
    Seg seg;
    auto add_static = [&](TokenSeq t) {
        if (!t.empty()) seg.parts.push_back(SegPart{true, std::move(t), -1, -1, 0});
    };
    std::function<void(NodeId)> expand_ref = [&](NodeId id) {
        const PlanNode& n = g.op(id);
        if (query >= 0 && !g.llm_up.at(id)) {  // concrete pre-run value: inline as statics
            add_static(ev.value(id, static_cast<std::size_t>(query)));
            return;
        }
        if (n.kind == Kind::kOutput) {
            expand_ref(n.a.at(0));
            return;
        }
        if (n.kind == Kind::kFormat) {
            for (std::size_t k = 0; k + 1 < n.a.size(); k += 2) {
                if (n.a[k] == 0)
                    add_static(g.span(n.a[k + 1]));
                else
                    expand_ref(n.a[k + 1]);
            }
            return;
        }
        seg.parts.push_back(SegPart{false, {}, id, query, estimated_len(g, id, query)});
    };
    const PlanNode& n = g.op(llm);
    if (n.kind != Kind::kLlm) fail("prefix_template: not an llm node");
    for (std::size_t k = 0; k + 1 < n.a.size(); k += 2) {
        if (n.a[k] == 0)
            add_static(g.span(n.a[k + 1]));
        else
            expand_ref(n.a[k + 1]);
    }
    seg.normalize();
    return seg;
}

// ------------------------------------------------------------ radix tree
struct TLeaf {
    NodeId op = -1;
    int query = -1;
    int worker = 0;
    double len_out = 0;
    bool deterministic = true;
};
struct TNode {
    int id = 0, parent = -1, depth = 0;
    Seg seg;
    std::vector<int> children;
    bool is_leaf = false;
    TLeaf leaf;
    std::vector<int> preds, succs;
};

class Trt {
  public:
    Trt() { pool_.emplace_back(); }
    const TNode& node(int i) const { return pool_[static_cast<std::size_t>(i)]; }
    std::size_t size() const { return pool_.size(); }
    const std::vector<int>& leaves() const { return leaves_; }
    int root() const { return 0; }
    int leaf_index(NodeId op, int q) const {
        auto it = leaf_index_.find({op, q});
        return it == leaf_index_.end() ? -1 : it->second;
    }

    // trt.cpp:77-203
    int insert(Seg path, const TLeaf& payload) {
        path.normalize();
        int cur = root();
        std::size_t j = 0, jo = 0;
        while (true) {
            if (j == path.parts.size()) {
                const int lf = new_node();
                TNode& l = pool_[static_cast<std::size_t>(lf)];
                l.parent = cur;
                l.depth = pool_[static_cast<std::size_t>(cur)].depth + 1;
                l.is_leaf = true;
                l.leaf = payload;
                pool_[static_cast<std::size_t>(cur)].children.push_back(lf);
                leaves_.push_back(lf);
                if (!leaf_index_.emplace(std::make_pair(payload.op, payload.query), lf).second)
                    fail("duplicate leaf for op " + std::to_string(payload.op));
                return lf;
            }
            const SegPart& head = path.parts[j];
            int match = -1;
            for (int ch : pool_[static_cast<std::size_t>(cur)].children) {
                const TNode& c = pool_[static_cast<std::size_t>(ch)];
                if (c.is_leaf || c.seg.parts.empty()) continue;
                const SegPart& first = c.seg.parts[0];
                const bool hit = head.is_static ? (first.is_static && first.tokens[0] == head.tokens[jo])
                                                : first.same_placeholder(head);
                if (hit) {
                    match = ch;
                    break;
                }
            }
            if (match < 0) {
                const int mid = new_node();
                TNode& m = pool_[static_cast<std::size_t>(mid)];
                m.parent = cur;
                m.depth = pool_[static_cast<std::size_t>(cur)].depth + 1;
                m.seg = slice_from(path.parts, j, jo);
                pool_[static_cast<std::size_t>(cur)].children.push_back(mid);
                cur = mid;
                j = path.parts.size();
                jo = 0;
                continue;
            }
            const std::vector<SegPart>& cp = pool_[static_cast<std::size_t>(match)].seg.parts;
            std::size_t i = 0, io = 0;
            while (i < cp.size() && j < path.parts.size()) {
                const SegPart& a = cp[i];
                const SegPart& b = path.parts[j];
                if (a.is_static && b.is_static) {
                    std::size_t n = 0;
                    while (io + n < a.tokens.size() && jo + n < b.tokens.size() && a.tokens[io + n] == b.tokens[jo + n]) ++n;
                    io += n;
                    jo += n;
                    const bool a_end = io == a.tokens.size(), b_end = jo == b.tokens.size();
                    if (a_end) {
                        ++i;
                        io = 0;
                    }
                    if (b_end) {
                        ++j;
                        jo = 0;
                    }
                    if (!a_end && !b_end) break;
                } else if (a.same_placeholder(b)) {
                    ++i;
                    ++j;
                } else {
                    break;
                }
            }
            if (i == cp.size()) {
                cur = match;
                continue;
            }
            Seg head_seg = slice_prefix(cp, i, io);
            Seg tail_seg = slice_from(cp, i, io);
            const int pre = new_node();
            TNode& child = pool_[static_cast<std::size_t>(match)];
            TNode& prefix = pool_[static_cast<std::size_t>(pre)];
            prefix.seg = std::move(head_seg);
            prefix.parent = child.parent;
            prefix.depth = child.depth;
            prefix.children.push_back(match);
            TNode& parent = pool_[static_cast<std::size_t>(child.parent)];
            *std::find(parent.children.begin(), parent.children.end(), match) = pre;
            child.seg = std::move(tail_seg);
            child.parent = pre;
            std::vector<int> stack{match};
            while (!stack.empty()) {
                const int x = stack.back();
                stack.pop_back();
                pool_[static_cast<std::size_t>(x)].depth++;
                for (int ch : pool_[static_cast<std::size_t>(x)].children) stack.push_back(ch);
            }
            cur = pre;
        }
    }
    void add_dependency(NodeId from_op, int from_q, NodeId to_op, int to_q) {  // trt.cpp:205-216
        const int a = leaf_index(from_op, from_q), b = leaf_index(to_op, to_q);
        if (a < 0 || b < 0) fail("dependency references unknown leaf");
        TNode& na = pool_[static_cast<std::size_t>(a)];
        TNode& nb = pool_[static_cast<std::size_t>(b)];
        if (std::find(na.succs.begin(), na.succs.end(), b) == na.succs.end()) {
            na.succs.push_back(b);
            nb.preds.push_back(a);
        }
    }
    double node_weight(int i) const { return node(i).seg.weight(); }
    double weight_below(int ancestor, int n) const {
        double w = 0;
        for (int cur = n; cur != ancestor; cur = node(cur).parent) {
            if (cur < 0) fail("weight_below: not an ancestor");
            w += node_weight(cur);
        }
        return w;
    }
    int lca(int a, int b) const {
        while (node(a).depth > node(b).depth) a = node(a).parent;
        while (node(b).depth > node(a).depth) b = node(b).parent;
        while (a != b) {
            a = node(a).parent;
            b = node(b).parent;
        }
        return a;
    }
    double prefill_weight(int prev_leaf, int leaf) const {
        return prev_leaf < 0 ? weight_below(root(), leaf) : weight_below(lca(prev_leaf, leaf), leaf);
    }
    std::vector<int> path_from_root(int n) const {
        std::vector<int> path;
        for (int cur = n; cur >= 0; cur = node(cur).parent) path.push_back(cur);
        std::reverse(path.begin(), path.end());
        return path;
    }

  private:
    int new_node() {
        const int id = static_cast<int>(pool_.size());
        pool_.emplace_back();
        pool_.back().id = id;
        return id;
    }
    std::vector<TNode> pool_;
    std::vector<int> leaves_;
    std::map<std::pair<NodeId, int>, int> leaf_index_;
};

// trt.cpp:476-521
Trt build_tree(const GraphView& g, const std::map<NodeId, int>& worker_of, bool call_level) {
    Trt tree;
    Evaluator ev(g.p, 0, false, /*strict_llm=*/true);
    const std::vector<NodeId> ops = g.llm_ops_topo();
    const std::map<NodeId, std::vector<NodeId>> deps = g.llm_dependencies();
    const int queries = call_level ? static_cast<int>(g.p.batch) : 1;
    for (NodeId op : ops) {
        auto wit = worker_of.find(op);
        if (wit == worker_of.end()) fail("no worker assignment for llm op " + std::to_string(op));
        const PlanNode& n = g.op(op);
        for (int q = 0; q < queries; ++q) {
            const int query = call_level ? q : -1;
            TLeaf leaf;
            leaf.op = op;
            leaf.query = query;
            leaf.worker = wit->second;
            leaf.len_out = estimated_len(g, op, query);
            leaf.deterministic = n.deterministic;
            tree.insert(prefix_template(g, ev, op, query), leaf);
        }
    }
    for (NodeId op : ops)
        for (NodeId pr : deps.at(op))
            for (int q = 0; q < queries; ++q) {
                const int query = call_level ? q : -1;
                tree.add_dependency(pr, query, op, query);
            }
    return tree;
}

// cost_model.cpp:20-30
double decode_usage(double len_out) { return 0.5 * len_out * (len_out + 1.0); }
double total_usage(double alpha, double len_out, double u_p) { return alpha * (len_out * u_p + decode_usage(len_out)); }
double precedence_delay(double alpha, double capacity, double len_out) { return alpha * capacity * len_out; }

struct WorkerParams {
    double capacity = 0, alpha = 0;
    double resolved_alpha() const { return alpha > 0 ? alpha : 1.0 / capacity; }
};

// ------------------------------------------------------------ partition
struct Cluster {
    int tree_node = 0;
    std::vector<int> leaves;
    double load = 0;
    NodeId min_op = 0;
};

Cluster make_cluster(const Trt& tree, int node) {  // scheduler.cpp:32-55
    Cluster cl;
    cl.tree_node = node;
    std::vector<int> stack{node};
    cl.min_op = std::numeric_limits<NodeId>::max();
    double unique_weight = 0, len_sum = 0, decode_sum = 0;
    while (!stack.empty()) {
        const int n = stack.back();
        stack.pop_back();
        const TNode& t = tree.node(n);
        unique_weight += t.seg.weight();
        if (t.is_leaf) {
            cl.leaves.push_back(n);
            len_sum += t.leaf.len_out;
            decode_sum += decode_usage(t.leaf.len_out);
            cl.min_op = std::min(cl.min_op, t.leaf.op);
        }
        for (int ch : t.children) stack.push_back(ch);
    }
    const double mean_len = cl.leaves.empty() ? 0.0 : len_sum / static_cast<double>(cl.leaves.size());
    cl.load = mean_len * unique_weight + decode_sum;
    return cl;
}

std::map<NodeId, int> partition_workflow(const GraphView& g, int workers) {  // scheduler.cpp:59-115
    if (workers < 1) fail("need at least one worker");
    std::map<NodeId, int> worker_of;
    const std::vector<NodeId> ops = g.llm_ops_topo();
    if (workers == 1 || ops.size() <= 1) {
        for (NodeId op : ops) worker_of[op] = 0;
        return worker_of;
    }
    std::map<NodeId, int> all_zero;
    for (NodeId op : ops) all_zero[op] = 0;
    const Trt tree = build_tree(g, all_zero, false);
    std::vector<Cluster> clusters;
    for (int ch : tree.node(tree.root()).children) clusters.push_back(make_cluster(tree, ch));
    std::vector<double> load(static_cast<std::size_t>(workers), 0.0);
    std::map<int, int> cluster_worker;
    while (true) {
        std::sort(clusters.begin(), clusters.end(), [](const Cluster& a, const Cluster& b) {
            if (a.load != b.load) return a.load > b.load;
            return a.min_op < b.min_op;
        });
        std::fill(load.begin(), load.end(), 0.0);
        cluster_worker.clear();
        for (const Cluster& cl : clusters) {
            std::size_t w = 0;
            for (std::size_t i = 1; i < load.size(); ++i)
                if (load[i] < load[w] - kEps) w = i;
            cluster_worker[cl.tree_node] = static_cast<int>(w);
            load[w] += cl.load;
        }
        const double mx = *std::max_element(load.begin(), load.end());
        const double mn = *std::min_element(load.begin(), load.end());
        if (mx <= 1.5 * mn + kEps) break;
        std::ptrdiff_t pick = -1;
        for (std::size_t i = 0; i < clusters.size(); ++i) {
            if (clusters[i].leaves.size() < 2) continue;
            if (tree.node(clusters[i].tree_node).is_leaf) continue;
            if (pick < 0 || clusters[i].load > clusters[static_cast<std::size_t>(pick)].load)
                pick = static_cast<std::ptrdiff_t>(i);
        }
        if (pick < 0) break;
        const Cluster split = clusters[static_cast<std::size_t>(pick)];
        clusters.erase(clusters.begin() + pick);
        for (int ch : tree.node(split.tree_node).children) clusters.push_back(make_cluster(tree, ch));
    }
    for (const Cluster& cl : clusters)
        for (int lf : cl.leaves) worker_of[tree.node(lf).leaf.op] = cluster_worker.at(cl.tree_node);
    return worker_of;
}

// --------------------------------------------------- operator scheduling
struct GroupKey {
    int worker = 0;
    long long key = 0;  // tree node id, or -(op+2) for singleton groups
    friend bool operator<(const GroupKey& a, const GroupKey& b) {
        return a.worker != b.worker ? a.worker < b.worker : a.key < b.key;
    }
    friend bool operator==(const GroupKey& a, const GroupKey& b) { return a.worker == b.worker && a.key == b.key; }
};
struct GroupState {
    std::size_t total = 0, flushed = 0;
    std::vector<int> emitted;
};
struct LogEntry {
    int leaf = 0;
    GroupKey group;
    bool flushed = false;
};
using InnerSeq = std::vector<NodeId>;

// scheduler.cpp:144-470
struct Planner {
    const Trt& tree;
    const std::vector<WorkerParams>& params;
    std::size_t batch;

    std::map<NodeId, std::set<NodeId>> reach;
    std::map<int, std::vector<int>> paths;
    std::map<NodeId, bool> varies;
    std::map<int, GroupKey> group_of;

    std::vector<bool> emitted;
    std::vector<double> complete, delay;
    std::vector<int> unemitted_under;
    std::vector<double> frontier;
    std::vector<int> prev_leaf;
    std::map<GroupKey, GroupState> groups;
    std::vector<std::vector<LogEntry>> log;
    std::vector<std::vector<InnerSeq>> out;
    bool force_active = false;
    std::size_t emitted_count = 0;
    std::uint64_t passes = 0, forced_emits = 0;  // SchedulerStats (scheduler.hpp:33-40)

    Planner(const Trt& t, const std::vector<WorkerParams>& p, std::size_t b) : tree(t), params(p), batch(b) {}

    double es(int leaf) const {
        double v = 0;
        for (int p : tree.node(leaf).preds) {
            if (!emitted[static_cast<std::size_t>(p)]) return kInf;
            v = std::max(v, complete[static_cast<std::size_t>(p)] + delay[static_cast<std::size_t>(p)]);
        }
        return v;
    }
    bool forceable(int leaf) const {
        for (int p : tree.node(leaf).preds)
            if (!emitted[static_cast<std::size_t>(p)]) return false;
        return true;
    }
    double vary_weight(int leaf) const {
        double w = 0;
        for (int n : paths.at(leaf))
            for (const SegPart& p : tree.node(n).seg.parts)
                if (!p.is_static && varies.at(p.source)) w += p.est_len;
        return w;
    }
    void emit(int leaf) {
        const TLeaf& l = tree.node(leaf).leaf;
        const auto w = static_cast<std::size_t>(l.worker);
        const WorkerParams& wp = params[w];
        const double alpha = wp.resolved_alpha();
        const double u_p = tree.prefill_weight(prev_leaf[w], leaf);
        double usage = total_usage(alpha, l.len_out, u_p);
        if (batch > 1) usage += static_cast<double>(batch - 1) * total_usage(alpha, l.len_out, vary_weight(leaf));
        const double begin = std::max(frontier[w], es(leaf));
        const double c = begin + usage;
        emitted[static_cast<std::size_t>(leaf)] = true;
        complete[static_cast<std::size_t>(leaf)] = c;
        delay[static_cast<std::size_t>(leaf)] = precedence_delay(alpha, wp.capacity, l.len_out);
        frontier[w] = c;
        prev_leaf[w] = leaf;
        for (int n : paths.at(leaf)) unemitted_under[static_cast<std::size_t>(n)]--;
        ++emitted_count;
        if (force_active) {
            force_active = false;
            ++forced_emits;
        }
        const GroupKey gk = group_of.at(leaf);
        GroupState& g = groups.at(gk);
        g.emitted.push_back(leaf);
        log[w].push_back(LogEntry{leaf, gk, false});
        if (g.emitted.size() == g.total) release(gk);
    }
    void release(const GroupKey& gk) {
        GroupState& g = groups.at(gk);
        std::vector<int> pending(g.emitted.begin() + static_cast<std::ptrdiff_t>(g.flushed), g.emitted.end());
        if (pending.empty()) return;
        std::set<NodeId> targets;
        for (int lf : pending) targets.insert(tree.node(lf).leaf.op);
        const auto wi = static_cast<std::size_t>(gk.worker);
        std::vector<bool> needed(log[wi].size(), false);
        for (std::size_t i = 0; i < log[wi].size(); ++i) {
            const LogEntry& e = log[wi][i];
            if (e.flushed || e.group == gk) continue;
            auto rit = reach.find(tree.node(e.leaf).leaf.op);
            if (rit == reach.end()) continue;
            for (NodeId t : targets)
                if (rit->second.count(t)) {
                    needed[i] = true;
                    break;
                }
        }
        std::map<GroupKey, std::size_t> last_needed;
        for (std::size_t i = 0; i < log[wi].size(); ++i)
            if (needed[i]) last_needed[log[wi][i].group] = i;
        std::vector<std::size_t> to_flush;
        for (std::size_t i = 0; i < log[wi].size(); ++i) {
            const LogEntry& e = log[wi][i];
            if (e.flushed || e.group == gk) continue;
            auto it = last_needed.find(e.group);
            if (it != last_needed.end() && i <= it->second) to_flush.push_back(i);
        }
        std::size_t k = 0;
        while (k < to_flush.size()) {
            std::size_t kk = k;
            const GroupKey run = log[wi][to_flush[k]].group;
            InnerSeq seq;
            while (kk < to_flush.size() && log[wi][to_flush[kk]].group == run) {
                LogEntry& e = log[wi][to_flush[kk]];
                e.flushed = true;
                groups.at(e.group).flushed++;
                seq.push_back(tree.node(e.leaf).leaf.op);
                ++kk;
            }
            out[wi].push_back(std::move(seq));
            k = kk;
        }
        InnerSeq seq;
        for (int lf : pending) seq.push_back(tree.node(lf).leaf.op);
        for (LogEntry& e : log[wi])
            if (!e.flushed && e.group == gk) e.flushed = true;
        g.flushed = g.emitted.size();
        out[wi].push_back(std::move(seq));
    }
    void flush_remaining() {
        for (std::size_t wi = 0; wi < log.size(); ++wi) {
            std::size_t k = 0;
            while (k < log[wi].size()) {
                if (log[wi][k].flushed) {
                    ++k;
                    continue;
                }
                const GroupKey run = log[wi][k].group;
                InnerSeq seq;
                while (k < log[wi].size() && !log[wi][k].flushed && log[wi][k].group == run) {
                    log[wi][k].flushed = true;
                    groups.at(run).flushed++;
                    seq.push_back(tree.node(log[wi][k].leaf).leaf.op);
                    ++k;
                }
                out[wi].push_back(std::move(seq));
            }
        }
    }
    std::vector<int> select_children(int u) {
        std::vector<int> live;
        for (int ch : tree.node(u).children)
            if (unemitted_under[static_cast<std::size_t>(ch)] > 0) live.push_back(ch);
        const std::size_t k = live.size();
        if (k <= 1) return live;
        std::vector<double> min_es(k, kInf);
        std::vector<NodeId> min_op(k, std::numeric_limits<NodeId>::max());
        std::map<int, std::size_t> which;
        for (std::size_t i = 0; i < k; ++i) which[live[i]] = i;
        auto child_of = [&](int leaf) -> int {
            const std::vector<int>& path = paths.at(leaf);
            const auto d = static_cast<std::size_t>(tree.node(u).depth) + 1;
            return d < path.size() ? path[d] : -1;
        };
        std::vector<std::vector<int>> child_leaves(k);
        for (int lf : tree.leaves()) {
            if (emitted[static_cast<std::size_t>(lf)]) continue;
            auto it = which.find(child_of(lf));
            if (it == which.end()) continue;
            const std::size_t i = it->second;
            child_leaves[i].push_back(lf);
            min_op[i] = std::min(min_op[i], tree.node(lf).leaf.op);
            if (forceable(lf)) min_es[i] = std::min(min_es[i], es(lf));
        }
        if (force_active) {
            std::vector<int> order = live;
            std::sort(order.begin(), order.end(), [&](int a, int b) {
                const std::size_t ia = which[a], ib = which[b];
                if (min_es[ia] != min_es[ib]) return min_es[ia] < min_es[ib];
                return min_op[ia] < min_op[ib];
            });
            return order;
        }
        std::vector<std::vector<bool>> adj(k, std::vector<bool>(k, false));
        for (std::size_t i = 0; i < k; ++i)
            for (int lf : child_leaves[i])
                for (int s : tree.node(lf).succs) {
                    if (emitted[static_cast<std::size_t>(s)]) continue;
                    auto it = which.find(child_of(s));
                    if (it != which.end() && it->second != i) adj[i][it->second] = true;
                }
        std::vector<std::vector<bool>> rc = adj;
        for (std::size_t m = 0; m < k; ++m)
            for (std::size_t i = 0; i < k; ++i)
                for (std::size_t j = 0; j < k; ++j)
                    if (rc[i][m] && rc[m][j]) rc[i][j] = true;
        std::vector<std::size_t> comp(k, k);
        std::size_t ncomp = 0;
        for (std::size_t i = 0; i < k; ++i) {
            if (comp[i] != k) continue;
            comp[i] = ncomp;
            for (std::size_t j = i + 1; j < k; ++j)
                if (rc[i][j] && rc[j][i]) comp[j] = ncomp;
            ++ncomp;
        }
        std::vector<std::set<std::size_t>> cpred(ncomp);
        for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = 0; j < k; ++j)
                if (adj[i][j] && comp[i] != comp[j]) cpred[comp[j]].insert(comp[i]);
        std::vector<int> depth_of(ncomp, 0);
        for (bool changed = true; changed;) {
            changed = false;
            for (std::size_t cc = 0; cc < ncomp; ++cc)
                for (std::size_t p : cpred[cc])
                    if (depth_of[p] + 1 > depth_of[cc]) {
                        depth_of[cc] = depth_of[p] + 1;
                        changed = true;
                    }
        }
        std::vector<double> comp_es(ncomp, kInf);
        std::vector<NodeId> comp_op(ncomp, std::numeric_limits<NodeId>::max());
        for (std::size_t i = 0; i < k; ++i) {
            comp_es[comp[i]] = std::min(comp_es[comp[i]], min_es[i]);
            comp_op[comp[i]] = std::min(comp_op[comp[i]], min_op[i]);
        }
        std::vector<std::size_t> remaining(ncomp, 0), comp_order;
        for (std::size_t cc = 0; cc < ncomp; ++cc) remaining[cc] = cpred[cc].size();
        std::vector<bool> done(ncomp, false);
        for (std::size_t round = 0; round < ncomp; ++round) {
            std::size_t best = ncomp;
            for (std::size_t cc = 0; cc < ncomp; ++cc) {
                if (done[cc] || remaining[cc] > 0) continue;
                if (best == ncomp) {
                    best = cc;
                    continue;
                }
                if (depth_of[cc] != depth_of[best]) {
                    if (depth_of[cc] > depth_of[best]) best = cc;
                } else if (comp_es[cc] != comp_es[best]) {
                    if (comp_es[cc] < comp_es[best]) best = cc;
                } else if (comp_op[cc] < comp_op[best]) {
                    best = cc;
                }
            }
            if (best == ncomp) fail("child ordering failed (cyclic condensation)");
            done[best] = true;
            comp_order.push_back(best);
            for (std::size_t cc = 0; cc < ncomp; ++cc)
                if (!done[cc] && cpred[cc].count(best)) remaining[cc]--;
        }
        std::vector<int> order;
        for (std::size_t cc : comp_order) {
            std::vector<std::size_t> members;
            for (std::size_t i = 0; i < k; ++i)
                if (comp[i] == cc) members.push_back(i);
            std::sort(members.begin(), members.end(), [&](std::size_t a, std::size_t b) {
                if (min_es[a] != min_es[b]) return min_es[a] < min_es[b];
                return min_op[a] < min_op[b];
            });
            for (std::size_t i : members) order.push_back(live[i]);
        }
        return order;
    }
    bool recurse(int u) {
        const TNode& n = tree.node(u);
        if (n.is_leaf) {
            if (emitted[static_cast<std::size_t>(u)] || !forceable(u)) return false;
            const double start = es(u);
            const auto w = static_cast<std::size_t>(n.leaf.worker);
            if (!force_active && start > frontier[w] + kEps) return false;
            emit(u);
            return true;
        }
        bool any = false;
        for (int ch : select_children(u)) {
            if (unemitted_under[static_cast<std::size_t>(ch)] == 0) continue;
            if (recurse(ch)) any = true;
        }
        return any;
    }
};

struct Scheduled {
    std::vector<std::vector<InnerSeq>> soft;
    std::vector<std::vector<CallId>> sigma;
    std::uint64_t passes = 0, forced_emits = 0, emitted = 0;
};

// scheduler.cpp:474-561 + expand_soft_schedule (:563-571)
Scheduled plan_operators(const GraphView& g, const std::vector<WorkerParams>& params,
                         const std::map<NodeId, int>& worker_of) {
    const Trt tree = build_tree(g, worker_of, false);
    for (const auto& [op, w] : worker_of)
        if (w < 0 || w >= static_cast<int>(params.size()))
            fail("operator " + std::to_string(op) + " assigned to missing worker " + std::to_string(w));
    Planner pl(tree, params, g.p.batch);
    const std::map<NodeId, std::vector<NodeId>> deps = g.llm_dependencies();
    const std::vector<NodeId> ops = g.llm_ops_topo();
    std::map<NodeId, std::set<NodeId>> succs;
    for (const auto& [op, ds] : deps)
        for (NodeId d : ds) succs[d].insert(op);
    for (auto it = ops.rbegin(); it != ops.rend(); ++it) {
        std::set<NodeId>& r = pl.reach[*it];
        for (NodeId s : succs[*it]) {
            r.insert(s);
            r.insert(pl.reach[s].begin(), pl.reach[s].end());
        }
    }
    for (NodeId id : g.topo) {
        const PlanNode& n = g.op(id);
        bool v = false;
        if (n.kind == Kind::kBound) {  // c.bound: data / input / cache_fetch values
            for (std::size_t b = 1; b < n.a.size(); ++b)
                if (g.span(n.a[b]) != g.span(n.a[0])) v = true;
        } else {
            for (NodeId in : g.ins.at(id)) v = v || pl.varies.at(in);
        }
        pl.varies[id] = v;
    }
    pl.emitted.assign(tree.size(), false);
    pl.complete.assign(tree.size(), 0);
    pl.delay.assign(tree.size(), 0);
    pl.unemitted_under.assign(tree.size(), 0);
    for (int lf : tree.leaves()) {
        pl.paths[lf] = tree.path_from_root(lf);
        for (int n : pl.paths[lf]) pl.unemitted_under[static_cast<std::size_t>(n)]++;
    }
    pl.frontier.assign(params.size(), 0.0);
    pl.prev_leaf.assign(params.size(), -1);
    pl.log.resize(params.size());
    pl.out.resize(params.size());
    for (int lf : tree.leaves()) {
        const std::vector<int>& path = pl.paths[lf];
        int deepest = tree.root();
        for (std::size_t i = 1; i + 1 < path.size(); ++i) {
            if (!tree.node(path[i]).seg.all_static()) break;
            deepest = path[i];
        }
        GroupKey gk;
        gk.worker = tree.node(lf).leaf.worker;
        gk.key = deepest == tree.root() ? -(tree.node(lf).leaf.op + 2) : static_cast<long long>(deepest);
        pl.group_of[lf] = gk;
        pl.groups[gk].total++;
    }
    const std::size_t total = tree.leaves().size();
    while (pl.emitted_count < total) {
        ++pl.passes;
        pl.force_active = false;
        if (pl.recurse(tree.root())) continue;
        pl.force_active = true;
        ++pl.passes;
        if (!pl.recurse(tree.root())) fail("scheduling stalled: dependency cycle among llm operators");
    }
    pl.flush_remaining();
    Scheduled r;
    r.sigma.resize(pl.out.size());
    for (std::size_t w = 0; w < pl.out.size(); ++w)
        for (const InnerSeq& seq : pl.out[w])
            for (NodeId op : seq)
                for (std::size_t b = 0; b < g.p.batch; ++b) r.sigma[w].push_back(CallId{op, static_cast<int>(b)});
    r.soft = std::move(pl.out);
    r.passes = pl.passes;
    r.forced_emits = pl.forced_emits;
    r.emitted = pl.emitted_count;
    return r;
}

// evaluate_schedule (cost_model.cpp:32-120): replay sigma against the analytic
// model over the call tree; returns the makespan
double evaluate_schedule(const Trt& tree, const std::vector<std::vector<CallId>>& sigma,
                         const std::vector<WorkerParams>& params) {
    std::size_t total = 0;
    for (const auto& wq : sigma) total += wq.size();
    if (total != tree.leaves().size())
        fail("schedule covers " + std::to_string(total) + " of " + std::to_string(tree.leaves().size()) + " calls");
    std::map<int, double> complete_at, delay_of;
    std::vector<std::size_t> next(sigma.size(), 0);
    std::vector<double> frontier(sigma.size(), 0.0);
    std::vector<int> prev_leaf(sigma.size(), -1);
    double makespan = 0;
    std::size_t placed = 0;
    bool progress = true;
    while (placed < total && progress) {
        progress = false;
        for (std::size_t w = 0; w < sigma.size(); ++w) {
            while (next[w] < sigma[w].size()) {
                const CallId& c = sigma[w][next[w]];
                const int lf = tree.leaf_index(c.op, c.query);
                if (lf < 0) fail("schedule names unknown call");
                const TNode& leaf = tree.node(lf);
                double ready = 0.0;
                bool blocked = false;
                for (int p : leaf.preds) {
                    auto it = complete_at.find(p);
                    if (it == complete_at.end()) {
                        blocked = true;
                        break;
                    }
                    ready = std::max(ready, it->second + delay_of.at(p));
                }
                if (blocked) break;
                const WorkerParams& wp = params[w];
                const double alpha = wp.resolved_alpha();
                const double u_p = tree.prefill_weight(prev_leaf[w], lf);
                const double usage = total_usage(alpha, leaf.leaf.len_out, u_p);
                const double begin = std::max(frontier[w], ready);
                const double complete = begin + usage;
                complete_at[lf] = complete;
                delay_of[lf] = precedence_delay(alpha, wp.capacity, leaf.leaf.len_out);
                frontier[w] = complete;
                prev_leaf[w] = lf;
                makespan = std::max(makespan, complete);
                ++next[w];
                ++placed;
                progress = true;
            }
        }
    }
    if (placed < total) fail("schedule deadlock");
    return makespan;
}

// ---------------------------------------------------------------- writer
class Writer {
  public:
    std::vector<std::uint64_t> w;
    void u(std::uint64_t v) { w.push_back(v); }
    void i(std::int64_t v) { w.push_back(static_cast<std::uint64_t>(v)); }
    void f(double v) {
        std::uint64_t b;
        std::memcpy(&b, &v, 8);
        w.push_back(b);
    }
};

}  // namespace

// HKPLAN01 with the planner's own call tree and schedule: the plan's value
// graph, outputs and signatures are kept; the call tree is rebuilt for the new
// partition (build_call_tree, trt.cpp:527-530) and the schedule comes from
// plan_operators over the capacities (run_pipeline.cpp:47-69, cache-aware).
PlanOutcome replan_full(const std::uint8_t* data, std::size_t n, int workers,
                        const std::vector<std::uint64_t>& capacities, double alpha) {
    const Plan p = parse_plan(data, n);
    if (workers < 1) fail("workers must be positive");
    if (capacities.empty()) fail("no worker capacities given");
    if (capacities.size() != 1 && capacities.size() != static_cast<std::size_t>(workers))
        fail("capacity list must have one entry or one per worker");
    std::vector<WorkerParams> params;
    for (int w = 0; w < workers; ++w)
        params.push_back(WorkerParams{static_cast<double>(capacities.size() == 1 ? capacities[0]
                                                                                 : capacities[static_cast<std::size_t>(w)]),
                                      alpha});
    const GraphView g(p);
    const std::map<NodeId, int> worker_of = partition_workflow(g, workers);
    Scheduled sch = plan_operators(g, params, worker_of);
    const std::vector<std::vector<CallId>>& sigma = sch.sigma;
    const Trt tree = build_tree(g, worker_of, true);
    PlanOutcome res;
    res.makespan = evaluate_schedule(tree, sigma, params);
    res.passes = sch.passes;
    res.forced_emits = sch.forced_emits;
    res.emitted = sch.emitted;
    res.soft = sch.soft;
    res.sigma = sigma;

    // re-serialise: token pool + spans (the plan's, then the tree's new static runs)
    Writer wr;
    std::vector<Token> pool = p.pool;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> spans = p.spans;
    std::map<TokenSeq, std::size_t> index;
    for (std::size_t s = 0; s < spans.size(); ++s)
        index.emplace(TokenSeq(pool.begin() + static_cast<std::ptrdiff_t>(spans[s].first),
                               pool.begin() + static_cast<std::ptrdiff_t>(spans[s].first + spans[s].second)),
                      s);
    auto intern = [&](const TokenSeq& t) {
        auto it = index.find(t);
        if (it != index.end()) return it->second;
        spans.emplace_back(pool.size(), t.size());
        pool.insert(pool.end(), t.begin(), t.end());
        return index[t] = spans.size() - 1;
    };
    std::vector<std::vector<std::array<std::int64_t, 3>>> tparts(tree.size());
    for (std::size_t k = 0; k < tree.size(); ++k)
        for (const SegPart& sp : tree.node(static_cast<int>(k)).seg.parts)
            tparts[k].push_back(sp.is_static ? std::array<std::int64_t, 3>{1, static_cast<std::int64_t>(intern(sp.tokens)), -1}
                                             : std::array<std::int64_t, 3>{0, sp.source, sp.query});
    wr.u(0x31304e414c504b48ull);
    wr.u(p.batch);
    wr.u(pool.size());
    for (Token t : pool) wr.u(t);
    wr.u(spans.size());
    for (const auto& [off, len] : spans) {
        wr.u(off);
        wr.u(len);
    }
    wr.u(p.nodes.size());
    for (const auto& [id, nd] : p.nodes) {
        wr.i(id);
        wr.u(static_cast<std::uint64_t>(nd.kind));
        wr.u((nd.deterministic ? 1u : 0u) | (nd.has_profile ? 2u : 0u));
        wr.f(nd.has_profile ? nd.len_out : std::nan(""));
        wr.u(nd.a.size());
        for (std::int64_t v : nd.a) wr.i(v);
    }
    wr.u(p.outputs.size());
    for (NodeId o : p.outputs) wr.i(o);
    wr.u(tree.size());
    for (std::size_t k = 0; k < tree.size(); ++k) {
        const TNode& t = tree.node(static_cast<int>(k));
        wr.i(t.parent);
        wr.u(t.is_leaf ? 1 : 0);
        wr.i(t.is_leaf ? t.leaf.op : -1);
        wr.i(t.is_leaf ? t.leaf.query : -1);
        wr.u(tparts[k].size());
        for (const auto& pt : tparts[k]) {
            wr.u(static_cast<std::uint64_t>(pt[0]));
            wr.i(pt[1]);
            wr.i(pt[2]);
        }
        wr.u(t.preds.size());
        for (int pr : t.preds) wr.i(pr);
    }
    wr.u(sigma.size());
    for (const auto& wq : sigma) {
        wr.u(wq.size());
        for (const CallId& c : wq) {
            wr.i(c.op);
            wr.i(c.query);
        }
    }
    std::vector<std::uint8_t>& out = res.blob;
    out.resize(wr.w.size() * 8);
    std::memcpy(out.data(), wr.w.data(), out.size());
    out.insert(out.end(), data + p.sig_offset, data + n);  // signature section, if any
    return res;
}

std::vector<std::uint8_t> replan(const std::uint8_t* data, std::size_t n, int workers,
                                 const std::vector<std::uint64_t>& capacities, double alpha) {
    return replan_full(data, n, workers, capacities, alpha).blob;
}

}  // namespace hk
