// Native `run_workflow`: the reference's workflow / inputs /
// profile JSON (workflow_io.cpp:88-216), validate + bind (workflow.cpp:103-255),
// content signatures (signature.cpp:29-104), the rewrite passes
// (optimizer.cpp:39-110: prune, fold duplicates, prompt-cache substitution),
// then the native planner (planner.cpp), the executor and the reports of
// run_report_json (run_pipeline.cpp:85-112), soft_schedule_json
// (scheduler.cpp:573-581) and the CLI's outputs json (helios_main.cpp:26-34) —
// so `helios run` needs no reference library at all. Every report is
// byte-identical to the reference's (tests/test_cli_cpu.py runs both CLIs).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>

#include "hk_host.hpp"
#include "json.hpp"

namespace hk {

namespace {

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }

enum class OpKind { kData, kInput, kOutput, kFormat, kLambda, kLlm, kCacheFetch };
enum class Role { kSystem, kAssistant, kUser };

const char* kind_name(OpKind k) {
    static const char* n[] = {"data", "input", "output", "format", "lambda", "llm", "cache_fetch"};
    return n[static_cast<int>(k)];
}
OpKind kind_from(const std::string& s) {
    static const char* n[] = {"data", "input", "output", "format", "lambda", "llm", "cache_fetch"};
    for (int k = 0; k < 7; ++k)
        if (s == n[k]) return static_cast<OpKind>(k);
    fail("unknown operator kind '" + s + "'");
}
Role role_from(const std::string& s) {
    if (s == "system") return Role::kSystem;
    if (s == "assistant") return Role::kAssistant;
    if (s == "user") return Role::kUser;
    fail("unknown message role '" + s + "'");
}

struct ValueSpec {
    bool synthetic = false;
    std::string text;
    std::size_t token_count = 0;
};
struct Part {
    bool is_ref = false;
    std::string text;
    NodeId ref = -1;
};
struct Msg {
    Role role = Role::kUser;
    std::vector<Part> parts;
};
struct Op {
    NodeId id = -1;
    OpKind kind = OpKind::kData;
    std::vector<ValueSpec> values;
    std::string input_name, template_text, fn;
    std::vector<Msg> messages;
    bool deterministic = true;
    std::vector<std::uint64_t> keys;
    std::vector<TokenSeq> fetched;
};
struct Edge {
    NodeId from = -1, to = -1;
    int slot = 0;
};
struct Graph {
    std::map<NodeId, Op> nodes;
    std::vector<Edge> edges;
    std::vector<NodeId> outputs;
    const Op& op(NodeId id) const {
        auto it = nodes.find(id);
        if (it == nodes.end()) fail("no node " + std::to_string(id));
        return it->second;
    }
    bool has(NodeId id) const { return nodes.count(id) != 0; }
    std::vector<NodeId> inputs_of(NodeId id) const {  // workflow.cpp:86-94
        int max_slot = -1;
        for (const Edge& e : edges)
            if (e.to == id) max_slot = std::max(max_slot, e.slot);
        std::vector<NodeId> in(static_cast<std::size_t>(max_slot + 1), -1);
        for (const Edge& e : edges)
            if (e.to == id) in[static_cast<std::size_t>(e.slot)] = e.from;
        return in;
    }
};
using Inputs = std::map<std::string, std::vector<ValueSpec>>;
using Profile = std::map<NodeId, double>;

// tokens.cpp:28-67
std::uint64_t hash_str(const std::string& s, std::uint64_t h) {
    h = fnv1a64(s.data(), s.size(), h);
    const unsigned char end = 0xff;
    return fnv1a64(&end, 1, h);
}
TokenSeq tokenize(const std::string& text) {
    TokenSeq out;
    std::size_t i = 0;
    while (i < text.size()) {
        while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
        const std::size_t st = i;
        while (i < text.size() && !std::isspace(static_cast<unsigned char>(text[i]))) ++i;
        if (i > st) out.push_back(fnv1a64(text.data() + st, i - st));
    }
    return out;
}
TokenSeq synthetic_tokens(std::size_t count, std::uint64_t& counter) {
    TokenSeq out;
    out.reserve(count);
    for (std::size_t i = 0; i < count; ++i) {
        std::uint64_t h = kFnvOffset;
        const unsigned char tag = 0x01;
        h = fnv1a64(&tag, 1, h);
        const std::uint64_t c = counter++;
        h = fnv1a64(&c, sizeof(c), h);
        out.push_back(h);
    }
    return out;
}
Token role_marker(Role r) {  // evaluator.cpp:60-67
    const char* w = r == Role::kSystem ? "<|system|>" : r == Role::kAssistant ? "<|assistant|>" : "<|user|>";
    return fnv1a64(w, std::strlen(w));
}
bool lambda_known(const std::string& fn) {
    if (fn == "identity" || fn == "concat") return true;
    if (fn.rfind("truncate:", 0) == 0) {
        const std::string n = fn.substr(9);
        return !n.empty() && n.find_first_not_of("0123456789") == std::string::npos;
    }
    return false;
}

std::vector<NodeId> topo_sort(const Graph& g) {  // workflow.cpp:172-193
    std::map<NodeId, int> indeg;
    std::map<NodeId, std::set<NodeId>> succ;
    for (const auto& [id, n] : g.nodes) indeg[id] = 0;
    for (const Edge& e : g.edges)
        if (succ[e.from].insert(e.to).second) ++indeg[e.to];
    std::priority_queue<NodeId, std::vector<NodeId>, std::greater<NodeId>> ready;
    for (const auto& [id, d] : indeg)
        if (d == 0) ready.push(id);
    std::vector<NodeId> order;
    while (!ready.empty()) {
        const NodeId id = ready.top();
        ready.pop();
        order.push_back(id);
        for (NodeId s : succ[id])
            if (--indeg[s] == 0) ready.push(s);
    }
    if (order.size() != g.nodes.size()) fail("workflow graph has a cycle");
    return order;
}

std::set<int> template_slots(const std::string& t, NodeId id) {  // workflow.cpp:17-31
    std::set<int> slots;
    for (std::size_t i = 0; i < t.size(); ++i) {
        if (t[i] != '{') continue;
        const std::size_t close = t.find('}', i);
        if (close == std::string::npos) fail("format node " + std::to_string(id) + ": unbalanced '{'");
        const std::string inner = t.substr(i + 1, close - i - 1);
        if (inner.empty() || inner.find_first_not_of("0123456789") != std::string::npos)
            fail("format node " + std::to_string(id) + ": bad slot '{" + inner + "}'");
        slots.insert(std::stoi(inner));
        i = close;
    }
    return slots;
}

void validate(const Graph& g) {  // workflow.cpp:103-170
    for (const auto& [id, n] : g.nodes) {
        if (id < 0) fail("negative node id " + std::to_string(id));
        if (n.id != id) fail("node " + std::to_string(id) + ": id field mismatch");
    }
    std::map<NodeId, std::set<int>> seen;
    for (const Edge& e : g.edges) {
        if (!g.has(e.from)) fail("edge from missing node " + std::to_string(e.from));
        if (!g.has(e.to)) fail("edge to missing node " + std::to_string(e.to));
        if (e.slot < 0) fail("edge into " + std::to_string(e.to) + ": negative slot");
        if (!seen[e.to].insert(e.slot).second)
            fail("node " + std::to_string(e.to) + ": duplicate input slot " + std::to_string(e.slot));
    }
    for (const auto& [id, slots] : seen)
        if (*slots.rbegin() != static_cast<int>(slots.size()) - 1)
            fail("node " + std::to_string(id) + ": input slots not dense");
    for (const auto& [id, n] : g.nodes) {
        const std::vector<NodeId> ins = g.inputs_of(id);
        const std::string where = std::string(kind_name(n.kind)) + " node " + std::to_string(id);
        switch (n.kind) {
            case OpKind::kData:
                if (!ins.empty()) fail(where + ": takes no inputs");
                if (n.values.empty()) fail(where + ": empty value batch");
                break;
            case OpKind::kInput:
                if (!ins.empty()) fail(where + ": takes no inputs");
                if (n.input_name.empty()) fail(where + ": missing name");
                break;
            case OpKind::kCacheFetch:
                if (!ins.empty()) fail(where + ": takes no inputs");
                if (n.fetched.empty() || n.keys.size() != n.fetched.size()) fail(where + ": keys/values mismatch");
                break;
            case OpKind::kOutput:
                if (ins.size() != 1) fail(where + ": needs exactly one input");
                break;
            case OpKind::kFormat:
                for (int s : template_slots(n.template_text, id))
                    if (s >= static_cast<int>(ins.size()))
                        fail(where + ": template slot {" + std::to_string(s) + "} has no edge");
                break;
            case OpKind::kLambda:
                if (!lambda_known(n.fn)) fail(where + ": unknown fn '" + n.fn + "'");
                if (ins.empty()) fail(where + ": needs at least one input");
                break;
            case OpKind::kLlm: {
                if (n.messages.empty()) fail(where + ": no messages");
                std::vector<NodeId> refs;
                for (const Msg& m : n.messages)
                    for (const Part& p : m.parts)
                        if (p.is_ref) refs.push_back(p.ref);
                if (refs != ins) fail(where + ": message refs do not match input edges");
                break;
            }
        }
    }
    for (NodeId out : g.outputs) {
        if (!g.has(out)) fail("outputs list names missing node " + std::to_string(out));
        if (g.op(out).kind != OpKind::kOutput) fail("outputs list entry " + std::to_string(out) + " is not an output node");
    }
    topo_sort(g);
}

ValueSpec value_spec(const json::Value& j) {  // workflow_io.cpp:17-28
    ValueSpec v;
    if (j.is_string()) {
        v.text = j.as_string();
    } else if (j.is_object() && j.contains("token_count")) {
        v.synthetic = true;
        v.token_count = static_cast<std::size_t>(j.at("token_count").as_uint());
    } else {
        fail("value entry must be a string or {\"token_count\": N}");
    }
    return v;
}

json::Value parse_doc(const std::string& text, const char* what) {
    try {
        return json::parse(text);
    } catch (const std::exception& e) {
        fail(std::string(what) + " json: " + e.what());
    }
}

Graph parse_workflow(const std::string& text) {  // workflow_io.cpp:134-167
    const json::Value j = parse_doc(text, "workflow");
    Graph g;
    for (const json::Value& jn : j.at("nodes").arr) {
        Op n;
        n.id = jn.at("id").as_int();
        n.kind = kind_from(jn.at("kind").as_string());
        const json::Value a = jn.contains("args") ? jn.at("args") : json::Value::object();
        switch (n.kind) {  // workflow_io.cpp:88-131
            case OpKind::kData:
                for (const json::Value& v : a.at("values").arr) n.values.push_back(value_spec(v));
                break;
            case OpKind::kInput: n.input_name = a.at("name").as_string(); break;
            case OpKind::kOutput: break;
            case OpKind::kFormat: n.template_text = a.at("template").as_string(); break;
            case OpKind::kLambda: n.fn = a.at("fn").as_string(); break;
            case OpKind::kLlm:
                for (const json::Value& jm : a.at("messages").arr) {
                    Msg m;
                    m.role = role_from(jm.at("role").as_string());
                    for (const json::Value& jp : jm.at("parts").arr) {
                        Part p;
                        if (jp.contains("ref")) {
                            p.is_ref = true;
                            p.ref = jp.at("ref").as_int();
                        } else {
                            p.text = jp.at("text").as_string();
                        }
                        m.parts.push_back(std::move(p));
                    }
                    n.messages.push_back(std::move(m));
                }
                n.deterministic = a.contains("deterministic") ? a.at("deterministic").as_bool() : true;
                break;
            case OpKind::kCacheFetch:
                for (const json::Value& k : a.at("keys").arr) n.keys.push_back(std::stoull(k.as_string(), nullptr, 16));
                for (const json::Value& v : a.at("tokens").arr) {
                    TokenSeq t;
                    for (const json::Value& x : v.arr) t.push_back(x.as_uint());
                    n.fetched.push_back(std::move(t));
                }
                break;
        }
        if (g.nodes.count(n.id)) fail("duplicate node id " + std::to_string(n.id));
        g.nodes[n.id] = std::move(n);
    }
    if (j.contains("edges"))
        for (const json::Value& je : j.at("edges").arr)
            g.edges.push_back(Edge{je.at("from").as_int(), je.at("to").as_int(),
                                   je.contains("slot") ? static_cast<int>(je.at("slot").as_int()) : 0});
    for (auto& [id, n] : g.nodes) {  // llm edges from message refs when the file has none
        if (n.kind != OpKind::kLlm) continue;
        bool has = false;
        for (const Edge& e : g.edges)
            if (e.to == id) has = true;
        if (has) continue;
        int slot = 0;
        for (const Msg& m : n.messages)
            for (const Part& p : m.parts)
                if (p.is_ref) g.edges.push_back(Edge{p.ref, id, slot++});
    }
    if (j.contains("outputs"))
        for (const json::Value& o : j.at("outputs").arr) g.outputs.push_back(o.as_int());
    validate(g);
    return g;
}

Inputs parse_inputs(const std::string& text) {  // workflow_io.cpp:181-193
    const json::Value j = parse_doc(text, "inputs");
    Inputs in;
    for (const auto& [name, vals] : j.obj) {
        if (!vals.is_array()) fail("input '" + name + "': expected an array");
        for (const json::Value& v : vals.arr) in[name].push_back(value_spec(v));
    }
    return in;
}

Profile parse_profile(const std::string& text) {  // workflow_io.cpp:205-216
    const json::Value j = parse_doc(text, "profile");
    Profile p;
    for (const auto& [key, val] : j.obj) {
        const NodeId id = std::stoll(key);
        p[id] = val.at("len_out").as_double();
        if (p[id] < 0) fail("profile for node " + key + ": negative len_out");
    }
    return p;
}

struct Compiled {
    Graph graph;
    std::size_t batch = 1;
    std::map<NodeId, std::vector<TokenSeq>> bound;
};

Compiled bind(const Graph& g, const Inputs& inputs) {  // workflow.cpp:202-255
    validate(g);
    Compiled c;
    c.graph = g;
    std::size_t batch = 0;
    for (const auto& [name, vals] : inputs) {
        if (vals.empty()) fail("input '" + name + "': empty batch");
        if (batch == 0) batch = vals.size();
        if (vals.size() != batch) fail("input '" + name + "': batch size mismatch");
    }
    if (batch == 0) batch = 1;
    c.batch = batch;
    std::uint64_t mint = 0;
    auto resolve = [&](const ValueSpec& v) { return v.synthetic ? synthetic_tokens(v.token_count, mint) : tokenize(v.text); };
    for (const auto& [id, n] : g.nodes) {
        switch (n.kind) {
            case OpKind::kInput: {
                auto it = inputs.find(n.input_name);
                if (it == inputs.end()) fail("no binding for input '" + n.input_name + "'");
                std::vector<TokenSeq> vals;
                for (const ValueSpec& v : it->second) vals.push_back(resolve(v));
                c.bound[id] = std::move(vals);
                break;
            }
            case OpKind::kData: {
                if (n.values.size() != 1 && n.values.size() != batch)
                    fail("data node " + std::to_string(id) + ": batch size " + std::to_string(n.values.size()) +
                         " incompatible with " + std::to_string(batch));
                std::vector<TokenSeq> vals;
                for (std::size_t b = 0; b < batch; ++b) vals.push_back(resolve(n.values[n.values.size() == 1 ? 0 : b]));
                c.bound[id] = std::move(vals);
                break;
            }
            case OpKind::kCacheFetch:
                if (n.fetched.size() != batch) fail("cache_fetch node " + std::to_string(id) + ": batch size mismatch");
                c.bound[id] = n.fetched;
                break;
            default: break;
        }
    }
    return c;
}

struct Sigs {
    std::map<NodeId, std::vector<std::uint64_t>> sig;
    std::map<NodeId, bool> tainted;
    std::uint64_t node_sig(NodeId id) const {
        std::uint64_t h = kFnvOffset;
        for (std::uint64_t s : sig.at(id)) h = hash_combine(h, s);
        return h;
    }
};

Sigs compute_signatures(const Compiled& c, const Profile& profile) {  // signature.cpp:29-104
    const Graph& g = c.graph;
    Sigs out;
    for (NodeId id : topo_sort(g)) {
        const Op& n = g.op(id);
        const std::vector<NodeId> ins = g.inputs_of(id);
        bool taint = false;
        for (NodeId in : ins) taint = taint || out.tainted.at(in);
        if (n.kind == OpKind::kLlm && !n.deterministic) taint = true;
        out.tainted[id] = taint;
        std::vector<std::uint64_t>& sigs = out.sig[id];
        for (std::size_t b = 0; b < c.batch; ++b) {
            std::uint64_t h = hash_combine(kFnvOffset, 0x100 + static_cast<std::uint64_t>(n.kind));
            switch (n.kind) {
                case OpKind::kInput:
                case OpKind::kData: {
                    const TokenSeq& v = c.bound.at(id).at(b);
                    h = hash_combine(h, hash_tokens(v.data(), v.size()));
                    break;
                }
                case OpKind::kCacheFetch: h = n.keys[b]; break;
                case OpKind::kOutput: h = hash_combine(h, out.sig.at(ins[0])[b]); break;
                case OpKind::kFormat:
                    h = hash_str(n.template_text, h);
                    for (NodeId in : ins) h = hash_combine(h, out.sig.at(in)[b]);
                    break;
                case OpKind::kLambda:
                    h = hash_str(n.fn, h);
                    for (NodeId in : ins) h = hash_combine(h, out.sig.at(in)[b]);
                    break;
                case OpKind::kLlm: {
                    if (!n.deterministic) {
                        h = hash_combine(h, 0xdeadull);
                        h = hash_combine(h, static_cast<std::uint64_t>(id));
                        h = hash_combine(h, b);
                        break;
                    }
                    auto it = profile.find(id);
                    if (it == profile.end()) fail("no profile entry for llm node " + std::to_string(id));
                    h = hash_combine(h, static_cast<std::uint64_t>(it->second * 1024.0));
                    std::size_t ref_slot = 0;
                    for (const Msg& m : n.messages) {
                        h = hash_combine(h, static_cast<std::uint64_t>(m.role));
                        for (const Part& p : m.parts) {
                            if (p.is_ref) {
                                h = hash_combine(h, 0x7265f);
                                h = hash_combine(h, out.sig.at(ins[ref_slot])[b]);
                                ++ref_slot;
                            } else {
                                h = hash_str(p.text, h);
                            }
                        }
                    }
                    break;
                }
            }
            sigs.push_back(h);
        }
    }
    return out;
}

// optimizer.cpp:14-31, :39-110
void erase_node(Compiled& c, NodeId id) {
    c.graph.nodes.erase(id);
    c.bound.erase(id);
    auto& e = c.graph.edges;
    e.erase(std::remove_if(e.begin(), e.end(), [&](const Edge& x) { return x.from == id || x.to == id; }), e.end());
}
void rewire_producer(Compiled& c, NodeId from, NodeId to) {
    for (Edge& e : c.graph.edges)
        if (e.from == from) e.from = to;
    for (auto& [id, n] : c.graph.nodes)
        for (Msg& m : n.messages)
            for (Part& p : m.parts)
                if (p.is_ref && p.ref == from) p.ref = to;
}
bool substitutable(OpKind k) { return k == OpKind::kFormat || k == OpKind::kLambda || k == OpKind::kLlm; }

std::size_t prune_unreachable(Compiled& c) {
    std::set<NodeId> live(c.graph.outputs.begin(), c.graph.outputs.end());
    std::vector<NodeId> stack(live.begin(), live.end());
    while (!stack.empty()) {
        const NodeId id = stack.back();
        stack.pop_back();
        for (const Edge& e : c.graph.edges)
            if (e.to == id && live.insert(e.from).second) stack.push_back(e.from);
    }
    std::vector<NodeId> dead;
    for (const auto& [id, n] : c.graph.nodes)
        if (!live.count(id)) dead.push_back(id);
    for (NodeId id : dead) erase_node(c, id);
    return dead.size();
}
std::size_t fold_duplicates(Compiled& c, const Profile& profile) {
    const Sigs sigs = compute_signatures(c, profile);
    std::map<std::uint64_t, std::vector<NodeId>> groups;
    for (const auto& [id, n] : c.graph.nodes) {
        if (n.kind == OpKind::kOutput) continue;
        groups[sigs.node_sig(id)].push_back(id);
    }
    std::size_t merged = 0;
    for (auto& [s, ids] : groups) {
        if (ids.size() < 2) continue;
        const NodeId survivor = ids.front();
        for (std::size_t i = 1; i < ids.size(); ++i) {
            rewire_producer(c, ids[i], survivor);
            erase_node(c, ids[i]);
            ++merged;
        }
    }
    return merged;
}
std::size_t substitute_cached(Compiled& c, const Profile& profile, PromptCache& cache) {
    const Sigs sigs = compute_signatures(c, profile);
    std::size_t substituted = 0;
    for (auto& [id, n] : c.graph.nodes) {
        if (!substitutable(n.kind) || sigs.tainted.at(id)) continue;
        const std::vector<std::uint64_t>& keys = sigs.sig.at(id);
        if (!std::all_of(keys.begin(), keys.end(), [&](std::uint64_t s) { return cache.contains(s); })) continue;
        std::vector<TokenSeq> values;
        for (std::uint64_t s : keys) values.push_back(*cache.lookup(s));
        n.kind = OpKind::kCacheFetch;
        n.keys = keys;
        n.fetched = values;
        n.messages.clear();
        n.template_text.clear();
        n.fn.clear();
        n.values.clear();
        c.bound[id] = std::move(values);
        auto& e = c.graph.edges;
        const NodeId nid = id;
        e.erase(std::remove_if(e.begin(), e.end(), [&](const Edge& x) { return x.to == nid; }), e.end());
        ++substituted;
    }
    return substituted;
}

// The compiled graph as HKPLAN01 (integration/plan_export.hpp's node encoding),
// with no call tree / schedule yet (the planner adds them) and the signatures.
std::vector<std::uint8_t> to_plan(const Compiled& c, const Profile& profile) {
    std::vector<Token> pool;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> spans;
    std::map<TokenSeq, std::size_t> index;
    auto intern = [&](const TokenSeq& t) -> std::int64_t {
        auto it = index.find(t);
        if (it != index.end()) return static_cast<std::int64_t>(it->second);
        spans.emplace_back(pool.size(), t.size());
        pool.insert(pool.end(), t.begin(), t.end());
        index[t] = spans.size() - 1;
        return static_cast<std::int64_t>(spans.size() - 1);
    };
    struct Rec {
        NodeId id;
        std::uint64_t kind, flags;
        double len_out;
        std::vector<std::int64_t> a;
    };
    std::vector<Rec> recs;
    for (const auto& [id, n] : c.graph.nodes) {
        Rec r{id, 0, 0, std::nan(""), {}};
        switch (n.kind) {
            case OpKind::kInput:
            case OpKind::kData:
            case OpKind::kCacheFetch: {
                auto it = c.bound.find(id);
                if (it != c.bound.end())
                    for (const TokenSeq& v : it->second) r.a.push_back(intern(v));
                break;
            }
            case OpKind::kOutput:
                r.kind = 1;
                r.a.push_back(c.graph.inputs_of(id).at(0));
                break;
            case OpKind::kLambda: {
                r.kind = 2;
                if (n.fn == "identity") r.a = {0, 0};
                else if (n.fn == "concat") r.a = {1, 0};
                else r.a = {2, static_cast<std::int64_t>(std::stoul(n.fn.substr(9)))};
                for (NodeId in : c.graph.inputs_of(id)) r.a.push_back(in);
                break;
            }
            case OpKind::kFormat: {
                r.kind = 3;
                const std::vector<NodeId> ins = c.graph.inputs_of(id);
                const std::string& t = n.template_text;
                std::string lit;
                auto flush = [&] {
                    const TokenSeq toks = tokenize(lit);
                    lit.clear();
                    if (toks.empty()) return;
                    r.a.push_back(0);
                    r.a.push_back(intern(toks));
                };
                for (std::size_t k = 0; k < t.size(); ++k) {
                    if (t[k] == '{') {
                        const std::size_t close = t.find('}', k);
                        const int slot = std::stoi(t.substr(k + 1, close - k - 1));
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
                r.kind = 4;
                r.flags = n.deterministic ? 1u : 0u;
                auto pit = profile.find(id);
                if (pit != profile.end()) {
                    r.flags |= 2u;
                    r.len_out = pit->second;
                }
                for (int role = 0; role < 3; ++role)
                    for (const Msg& m : n.messages) {
                        if (static_cast<int>(m.role) != role) continue;
                        r.a.push_back(0);
                        r.a.push_back(intern({role_marker(m.role)}));
                        for (const Part& p : m.parts) {
                            if (p.is_ref) {
                                r.a.push_back(1);
                                r.a.push_back(p.ref);
                            } else {
                                const TokenSeq toks = tokenize(p.text);
                                if (toks.empty()) continue;
                                r.a.push_back(0);
                                r.a.push_back(intern(toks));
                            }
                        }
                    }
                break;
            }
        }
        recs.push_back(std::move(r));
    }
    std::vector<std::uint64_t> w;
    auto f = [&](double v) {
        std::uint64_t b;
        std::memcpy(&b, &v, 8);
        w.push_back(b);
    };
    w.push_back(0x31304e414c504b48ull);
    w.push_back(c.batch);
    w.push_back(pool.size());
    w.insert(w.end(), pool.begin(), pool.end());
    w.push_back(spans.size());
    for (const auto& [o, l] : spans) {
        w.push_back(o);
        w.push_back(l);
    }
    w.push_back(recs.size());
    for (const Rec& r : recs) {
        w.push_back(static_cast<std::uint64_t>(r.id));
        w.push_back(r.kind);
        w.push_back(r.flags);
        f(r.len_out);
        w.push_back(r.a.size());
        for (std::int64_t v : r.a) w.push_back(static_cast<std::uint64_t>(v));
    }
    w.push_back(c.graph.outputs.size());
    for (NodeId o : c.graph.outputs) w.push_back(static_cast<std::uint64_t>(o));
    w.push_back(0);  // call tree: the planner's
    w.push_back(0);  // schedule: the planner's
    const Sigs sigs = compute_signatures(c, profile);
    w.push_back(0x3130304749534b48ull);
    w.push_back(sigs.sig.size());
    for (const auto& [id, v] : sigs.sig) {
        w.push_back(static_cast<std::uint64_t>(id));
        w.push_back(sigs.tainted.at(id) ? 1 : 0);
        w.insert(w.end(), v.begin(), v.end());
    }
    std::vector<std::uint8_t> out(w.size() * 8);
    std::memcpy(out.data(), w.data(), out.size());
    return out;
}

json::Value u(std::uint64_t v) { return json::Value::uint(v); }

}  // namespace

// run_workflow + the CLI's documents (see the file header).
WorkflowRun run_workflow(const std::string& wf, const std::string& in, const std::string& prof, const WorkflowSpec& spec,
                         PromptCache* cache, const BodyFactory& make_body) {
    if (spec.scheduler != "cache_aware")
        fail("scheduler '" + spec.scheduler + "': only cache_aware is native (the baselines stay in the reference)");
    if (spec.workers < 1) fail("workers must be positive");
    if (spec.capacities.empty()) fail("no worker capacities given");
    if (spec.capacities.size() != 1 && spec.capacities.size() != static_cast<std::size_t>(spec.workers))
        fail("capacity list must have one entry or one per worker");
    const Graph g = parse_workflow(wf);
    const Inputs inputs = parse_inputs(in);
    const Profile profile = parse_profile(prof);
    Compiled c = bind(g, inputs);
    std::size_t pruned = 0, merged = 0, substituted = 0;  // optimize(), optimizer.cpp:98-107
    if (spec.prune) pruned += prune_unreachable(c);
    if (spec.merge_duplicates) merged = fold_duplicates(c, profile);
    if (spec.cache_substitute && cache) substituted = substitute_cached(c, profile, *cache);
    if (spec.prune) pruned += prune_unreachable(c);
    validate(c.graph);

    const std::vector<std::uint8_t> bare = to_plan(c, profile);
    PlanOutcome po = replan_full(bare.data(), bare.size(), spec.workers, spec.capacities, spec.alpha);
    WorkflowRun r;
    r.plan = po.blob;
    const Plan plan = parse_plan(r.plan.data(), r.plan.size());
    if (spec.run_sim) {
        SimConfig sc;
        for (int w = 0; w < spec.workers; ++w)
            sc.workers.push_back(SimWorkerConfig{
                static_cast<std::size_t>(spec.capacities.size() == 1 ? spec.capacities[0]
                                                                     : spec.capacities[static_cast<std::size_t>(w)]),
                spec.block, spec.prefill_budget});
        sc.proactive_pin = spec.proactive_pin;
        sc.pin_threshold = spec.pin_threshold;
        sc.pin_capacity_frac = spec.pin_capacity_frac;
        sc.seed = spec.seed;
        sc.stochastic = spec.stochastic;
        sc.collect_trace = spec.collect_trace;
        sc.max_iterations = spec.max_iterations;
        std::unique_ptr<LlmBody> body = make_body(plan, sc);
        r.metrics = simulate(plan, sc, *body, ExecOptions{});
    }
    if (cache) {  // run_pipeline.cpp:74-79, with this run's own values
        if (spec.run_sim)
            harvest_into_cache(plan, r.metrics, *cache);
        else
            harvest_into_cache_synth(plan, spec.seed, spec.stochastic, *cache);
    }

    // run_report_json (run_pipeline.cpp:85-112)
    json::Value j = json::Value::object();
    j["scheduler"] = json::Value::str(spec.scheduler);
    j["workers"] = json::Value::sint(spec.workers);
    j["batch"] = u(c.batch);
    j["rewrite"]["pruned"] = u(pruned);
    j["rewrite"]["merged"] = u(merged);
    j["rewrite"]["substituted"] = u(substituted);
    j["makespan"] = json::Value::dbl(po.makespan);
    std::size_t calls = 0;
    for (const auto& wq : po.sigma) calls += wq.size();
    j["calls"] = u(calls);
    json::Value sched = json::Value::array();
    for (const auto& wq : po.sigma) {
        json::Value seq = json::Value::array();
        for (const CallId& cid : wq) {
            json::Value o = json::Value::object();
            o["op"] = json::Value::sint(cid.op);
            o["query"] = json::Value::sint(cid.query);
            seq.push_back(std::move(o));
        }
        sched.push_back(std::move(seq));
    }
    j["schedule"] = std::move(sched);
    j["scheduler_stats"]["passes"] = u(po.passes);
    j["scheduler_stats"]["forced_emits"] = u(po.forced_emits);
    j["scheduler_stats"]["emitted"] = u(po.emitted);
    if (r.metrics.iterations > 0) j["sim"] = json::parse(sim_metrics_json(r.metrics));
    r.report_json = json::dump(j) + "\n";
    r.calls_csv = sim_calls_csv(r.metrics);
    r.trace_csv = sim_trace_csv(r.metrics);
    json::Value oj = json::Value::object();  // helios_main.cpp:26-34
    for (const auto& [node, per_query] : r.metrics.outputs) {
        json::Value arr = json::Value::array();
        for (const TokenSeq& v : per_query) {
            json::Value t = json::Value::array();
            for (Token x : v) t.push_back(u(x));
            arr.push_back(std::move(t));
        }
        oj[std::to_string(node)] = std::move(arr);
    }
    r.outputs_json = json::dump(oj) + "\n";
    json::Value sj = json::Value::object();  // soft_schedule_json (scheduler.cpp:573-581)
    json::Value ws = json::Value::array();
    for (const auto& seqs : po.soft) {
        json::Value jw = json::Value::array();
        for (const auto& seq : seqs) {
            json::Value s = json::Value::array();
            for (NodeId op : seq) s.push_back(json::Value::sint(op));
            jw.push_back(std::move(s));
        }
        ws.push_back(std::move(jw));
    }
    sj["workers"] = std::move(ws);
    r.schedule_json = json::dump(sj) + "\n\n";  // soft_schedule_json's newline + the CLI's (helios_main.cpp:110)
    return r;
}

}  // namespace hk
