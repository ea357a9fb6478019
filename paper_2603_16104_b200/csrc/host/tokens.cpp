// Hash primitives and the synthetic LLM body.
// Restates tokens.cpp:7-65 and evaluator.cpp:13-58 of the reference
// (/root/reference/proj/src); the golden vectors of test_tokens.cpp:10-15 are
// checked in tests/test_host_cpu.py.
#include <cmath>

#include "hk_host.hpp"

namespace hk {

std::uint64_t fnv1a64(const void* data, std::size_t len, std::uint64_t seed) {
    const auto* p = static_cast<const unsigned char*>(data);
    std::uint64_t h = seed;
    for (std::size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// tokens.cpp:17-22: spread the seed, then fold the 8 bytes of v.
std::uint64_t hash_combine(std::uint64_t h, std::uint64_t v) {
    h = (h ^ 0x9e3779b97f4a7c15ull) * 0x100000001b3ull;
    return fnv1a64(&v, sizeof(v), h);
}

std::uint64_t hash_tokens(const Token* t, std::size_t n, std::uint64_t seed) {
    return fnv1a64(t, n * sizeof(Token), seed);
}

std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

namespace {
// evaluator.cpp:20-25
std::uint64_t output_digest(const TokenSeq& prompt, std::uint64_t seed) {
    std::uint64_t h = hash_tokens(prompt.data(), prompt.size());
    h = hash_combine(h, seed);
    unsigned char tag = 0x02;
    return fnv1a64(&tag, 1, h);
}
}  // namespace

// evaluator.cpp:29-35
std::size_t synth_output_len(const TokenSeq& prompt, double len_out, std::uint64_t seed, bool stochastic) {
    if (len_out < 0) throw std::runtime_error("negative len_out");
    auto base = static_cast<std::size_t>(std::llround(len_out));
    if (!stochastic) return base;
    std::uint64_t h = splitmix64(hash_combine(output_digest(prompt, seed), 0x6c656e));
    return h % (2 * base + 1);
}

// evaluator.cpp:37-44
TokenSeq synth_output(const TokenSeq& prompt, double len_out, std::uint64_t seed, bool stochastic) {
    std::size_t n = synth_output_len(prompt, len_out, seed, stochastic);
    std::uint64_t d = output_digest(prompt, seed);
    TokenSeq out;
    out.reserve(n);
    for (std::size_t i = 0; i < n; ++i) out.push_back(splitmix64(hash_combine(d, i)));
    return out;
}

// evaluator.cpp:46-58: deterministic ops ignore the run seed.
std::size_t synth_llm_len(const TokenSeq& prompt, double len_out, bool deterministic, std::uint64_t seed,
                          bool stochastic) {
    return synth_output_len(prompt, len_out, deterministic ? 0 : seed, stochastic);
}

TokenSeq synth_llm_output(const TokenSeq& prompt, double len_out, bool deterministic, std::uint64_t seed,
                          bool stochastic) {
    return synth_output(prompt, len_out, deterministic ? 0 : seed, stochastic);
}

std::uint32_t vocab_of(Token t, std::uint32_t vocab) { return static_cast<std::uint32_t>(t % vocab); }

Token gen_token(std::uint32_t id, std::uint32_t vocab) {
    unsigned char buf[5] = {0x03, static_cast<unsigned char>(id), static_cast<unsigned char>(id >> 8),
                            static_cast<unsigned char>(id >> 16), static_cast<unsigned char>(id >> 24)};
    std::uint64_t h = fnv1a64(buf, sizeof(buf));
    return h - h % vocab + id;  // wraps mod 2^64 in the (2^-47) top-of-range case
}

}  // namespace hk
