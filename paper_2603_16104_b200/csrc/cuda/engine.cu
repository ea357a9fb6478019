// Device engine (placeholder until the kernels land).
#include <memory>
#include <stdexcept>

#include "helium_b200.h"
#include "hk_host.hpp"

namespace hk {
void set_error(const std::string& s);
std::unique_ptr<LlmBody> make_device_body(hk_engine*, const Plan&, const SimConfig&) {
    throw std::runtime_error("device engine not built");
}
}  // namespace hk

extern "C" {
hk_engine* hk_engine_create(const hk_model_config*, const hk_engine_config*) {
    hk::set_error("not implemented");
    return nullptr;
}
void hk_engine_destroy(hk_engine*) {}
size_t hk_engine_page_bytes(const hk_engine*) { return 0; }
int hk_engine_reset(hk_engine*) { return -1; }
int hk_pool_gather(hk_engine*, int, const int32_t*, size_t, void*) { return -1; }
int hk_pool_scatter(hk_engine*, int, const void*, const int32_t*, size_t) { return -1; }
int hk_pool_copy(hk_engine*, int, const int32_t*, const int32_t*, size_t) { return -1; }
int hk_trie_apply(hk_engine*, int, const hk_trie_op*, size_t) { return -1; }
int hk_trie_match(hk_engine*, int, const uint64_t*, const uint64_t*, size_t, int32_t*, int32_t*, int32_t*, size_t) {
    return -1;
}
int hk_generate(hk_engine*, const uint32_t*, size_t, size_t, uint32_t*, float*) { return -1; }
double hk_engine_kernel_ms(const hk_engine*, const char*, uint64_t*, double*) { return -1; }
int hk_engine_profile(hk_engine*, int) { return -1; }
}
