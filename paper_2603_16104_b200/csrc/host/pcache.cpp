// Cross-run prompt cache: the reference's PromptCache
// (prompt_cache.hpp:15-40, prompt_cache.cpp:9-71) with its JSON wire format,
// and harvest_into_cache (optimizer.cpp:113-125) fed with the values the LLM
// body of a run actually generated — on the B200 that is the transformer's
// greedy output, so a warm resubmission planned by the reference's optimizer
// (substitute_cached, optimizer.cpp:71-95) fetches device-generated tokens.
#include <cctype>
#include <cstdio>
#include <cstring>

#include "hk_host.hpp"

namespace hk {

namespace {

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }

// Minimal JSON reader for the cache document ({"capacity": n, "entries":
// [{"sig": "hex", "tokens": [u64...]}...]}); other keys are skipped.
class Json {
  public:
    explicit Json(const std::string& s) : s_(s) {}
    void ws() {
        while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
    }
    bool peek(char c) {
        ws();
        return p_ < s_.size() && s_[p_] == c;
    }
    void expect(char c) {
        ws();
        if (p_ >= s_.size() || s_[p_] != c) err(std::string("expected '") + c + "'");
        ++p_;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (p_ < s_.size() && s_[p_] != '"') {
            if (s_[p_] == '\\') {
                if (++p_ >= s_.size()) break;
                const char e = s_[p_];
                out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e);
            } else {
                out.push_back(s_[p_]);
            }
            ++p_;
        }
        if (p_ >= s_.size()) err("unterminated string");
        ++p_;
        return out;
    }
    std::uint64_t uint() {
        ws();
        if (p_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[p_]))) err("expected an unsigned integer");
        std::uint64_t v = 0;
        while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) {
            const std::uint64_t d = static_cast<std::uint64_t>(s_[p_] - '0');
            if (v > (UINT64_MAX - d) / 10) err("integer out of range");
            v = v * 10 + d;
            ++p_;
        }
        return v;
    }
    void skip() {  // any value
        ws();
        if (p_ >= s_.size()) err("unexpected end of input");
        const char c = s_[p_];
        if (c == '"') {
            str();
        } else if (c == '{' || c == '[') {
            const char close = c == '{' ? '}' : ']';
            ++p_;
            if (peek(close)) {
                ++p_;
                return;
            }
            for (;;) {
                if (c == '{') {
                    str();
                    expect(':');
                }
                skip();
                if (peek(',')) {
                    ++p_;
                    continue;
                }
                expect(close);
                return;
            }
        } else {
            while (p_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[p_])) || s_[p_] == '-' ||
                                      s_[p_] == '+' || s_[p_] == '.'))
                ++p_;
        }
    }
    // iterate the members of an object: fn(key) consumes the value
    template <class F>
    void object(F fn) {
        expect('{');
        if (peek('}')) {
            ++p_;
            return;
        }
        for (;;) {
            const std::string k = str();
            expect(':');
            fn(k);
            if (peek(',')) {
                ++p_;
                continue;
            }
            expect('}');
            return;
        }
    }
    template <class F>
    void array(F fn) {
        expect('[');
        if (peek(']')) {
            ++p_;
            return;
        }
        for (;;) {
            fn();
            if (peek(',')) {
                ++p_;
                continue;
            }
            expect(']');
            return;
        }
    }
    void end() {
        ws();
        if (p_ != s_.size()) err("trailing characters");
    }
    [[noreturn]] void err(const std::string& what) const {
        fail("prompt cache json: " + what + " at byte " + std::to_string(p_));
    }

  private:
    const std::string& s_;
    std::size_t p_ = 0;
};

}  // namespace

std::string sig_hex(std::uint64_t s) {
    char buf[17];
    std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(s));
    return buf;
}

PromptCache::PromptCache(std::size_t capacity) : capacity_(capacity) {
    if (capacity == 0) fail("prompt cache capacity must be positive");
}

const TokenSeq* PromptCache::lookup(std::uint64_t s) {
    auto it = index_.find(s);
    if (it == index_.end()) return nullptr;
    entries_.splice(entries_.end(), entries_, it->second);  // most recent
    return &it->second->second;
}

void PromptCache::insert(std::uint64_t s, TokenSeq value) {
    auto it = index_.find(s);
    if (it != index_.end()) {
        it->second->second = std::move(value);
        entries_.splice(entries_.end(), entries_, it->second);
        return;
    }
    entries_.emplace_back(s, std::move(value));
    index_[s] = std::prev(entries_.end());
    while (entries_.size() > capacity_) {
        index_.erase(entries_.front().first);
        entries_.pop_front();
    }
}

std::vector<std::uint64_t> PromptCache::keys_lru_first() const {
    std::vector<std::uint64_t> out;
    out.reserve(entries_.size());
    for (const Entry& e : entries_) out.push_back(e.first);
    return out;
}

// The document prompt_cache.cpp:47-53 writes (nlohmann dump(2): object keys
// in sorted order, 2-space indent; each token array on one line), plus the
// trailing newline.
std::string PromptCache::serialize() const {
    std::string o = "{\n  \"capacity\": " + std::to_string(capacity_) + ",\n  \"entries\": ";
    if (entries_.empty()) {
        o += "[]";
    } else {
        o += "[\n";
        std::size_t k = 0;
        for (const Entry& e : entries_) {
            o += "    {\n      \"sig\": \"" + sig_hex(e.first) + "\",\n      \"tokens\": ";
            o += '[';  // the reference's token arrays come out on one line, no spaces
            for (std::size_t i = 0; i < e.second.size(); ++i) {
                if (i) o += ',';
                o += std::to_string(e.second[i]);
            }
            o += ']';
            o += ++k < entries_.size() ? "\n    },\n" : "\n    }\n";
        }
        o += "  ]";
    }
    o += "\n}\n";
    return o;
}

// prompt_cache.cpp:56-67: capacity first (it bounds the inserts), entries in
// file order (least recent first), so a round trip is exact.
PromptCache PromptCache::deserialize(const std::string& json_text) {
    Json j(json_text);
    std::size_t capacity = 0;
    bool has_cap = false, has_entries = false;
    std::vector<Entry> entries;
    j.object([&](const std::string& k) {
        if (k == "capacity") {
            capacity = static_cast<std::size_t>(j.uint());
            has_cap = true;
        } else if (k == "entries") {
            has_entries = true;
            j.array([&] {
                Entry e{0, {}};
                bool has_sig = false, has_tok = false;
                j.object([&](const std::string& ek) {
                    if (ek == "sig") {
                        const std::string h = j.str();
                        if (h.empty() || h.size() > 16 || h.find_first_not_of("0123456789abcdefABCDEF") != std::string::npos)
                            j.err("bad signature '" + h + "'");
                        e.first = std::stoull(h, nullptr, 16);
                        has_sig = true;
                    } else if (ek == "tokens") {
                        j.array([&] { e.second.push_back(j.uint()); });
                        has_tok = true;
                    } else {
                        j.skip();
                    }
                });
                if (!has_sig || !has_tok) j.err("entry needs sig and tokens");
                entries.push_back(std::move(e));
            });
        } else {
            j.skip();
        }
    });
    j.end();
    if (!has_cap) j.err("key 'capacity' not found");
    if (!has_entries) j.err("key 'entries' not found");
    PromptCache c(capacity);
    for (Entry& e : entries) c.insert(e.first, std::move(e.second));
    return c;
}

namespace {
std::size_t harvest(const Plan& plan, Evaluator& ev, PromptCache& cache);
}  // namespace

std::size_t harvest_into_cache(const Plan& plan, const SimMetrics& run, PromptCache& cache) {
    if (!plan.has_sigs) fail("harvest_into_cache: the plan carries no signatures (export it with them)");
    Evaluator ev(plan, 0, false, /*strict_llm=*/true);
    for (const auto& [cid, toks] : run.call_outputs) ev.put_llm_output(cid.op, static_cast<std::size_t>(cid.query), toks);
    return harvest(plan, ev, cache);
}

std::size_t harvest_into_cache_synth(const Plan& plan, std::uint64_t seed, bool stochastic, PromptCache& cache) {
    if (!plan.has_sigs) fail("harvest_into_cache: the plan carries no signatures (export it with them)");
    Evaluator ev(plan, seed, stochastic, /*strict_llm=*/false);
    return harvest(plan, ev, cache);
}

namespace {
std::size_t harvest(const Plan& plan, Evaluator& ev, PromptCache& cache) {
    std::size_t inserted = 0;
    for (const auto& [id, n] : plan.nodes) {  // ascending ids: the reference's map order
        if (n.kind != Kind::kFormat && n.kind != Kind::kLambda && n.kind != Kind::kLlm) continue;
        auto t = plan.tainted.find(id);
        auto s = plan.sig.find(id);
        if (t == plan.tainted.end() || s == plan.sig.end())
            fail("harvest_into_cache: no signature for node " + std::to_string(id));
        if (t->second) continue;
        for (std::size_t b = 0; b < plan.batch; ++b) {
            cache.insert(s->second[b], ev.value(id, b));
            ++inserted;
        }
    }
    return inserted;
}
}  // namespace

}  // namespace hk
