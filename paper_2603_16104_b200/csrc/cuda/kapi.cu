// Kernel-level C-ABI (include/helium_b200_kernels.h).
#include <string>
#include <vector>

#include <algorithm>
#include "common.cuh"
#include "helium_b200_kernels.h"
#include "kernels.cuh"

namespace hk {
void set_error(const std::string& s);
}

namespace {
unsigned long long* g_trace = nullptr;  // hkx_decode_attention_trace target (device)
float* g_ws = nullptr;
size_t g_ws_floats = 0;

float* workspace(size_t n) {
    if (n > g_ws_floats) {
        cudaFree(g_ws);
        HK_CUDA(cudaMalloc(&g_ws, n * sizeof(float)));
        g_ws_floats = n;
    }
    return g_ws;
}

void init_sms() {
    static bool done = false;
    if (done) return;
    int dev = 0, sms = 0;
    HK_CUDA(cudaGetDevice(&dev));
    HK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    hkd::g_num_sms = sms;
    done = true;
}
}  // namespace

extern "C" {

int hkx_gemm_bf16(const void* W, const void* X, void* out, int N, int K, int T, int epi, const void* bias, int splits,
                  void* stream) {
    try {
        init_sms();
        const size_t ws = static_cast<size_t>(32) * (T + 256) * N;
        const int ldo = epi == hkd::kEpiSwiGLU ? N / 2 : N;
        hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, ldo,
                       static_cast<const hkd::bf16*>(bias), workspace(ws), ws, static_cast<cudaStream_t>(stream),
                       splits, 64);
        return 0;
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return -1;
    }
}

double hkx_gemm_bench(const void* W, const void* X, void* out, int N, int K, int T, int epi, int splits, int iters) {
    try {
        init_sms();
        const size_t ws = static_cast<size_t>(32) * (T + 256) * N;
        float* w = workspace(ws);
        cudaEvent_t a, b;
        HK_CUDA(cudaEventCreate(&a));
        HK_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 3; ++i)
            hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, N,
                           nullptr, w, ws, nullptr, splits);
        HK_CUDA(cudaEventRecord(a));
        for (int i = 0; i < iters; ++i)
            hkd::gemm_bf16(static_cast<const hkd::bf16*>(W), static_cast<const hkd::bf16*>(X), N, K, T, epi, out, N,
                           nullptr, w, ws, nullptr, splits);
        HK_CUDA(cudaEventRecord(b));
        HK_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        HK_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms / iters;
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return -1;
    }
}

double hkx_decode_attention(const void* qkv, const void* kv, int n_pages, int n_rows, int H, int Hkv,
                            const int32_t* tables, const int32_t* offs, const int32_t* pos, const int32_t* group_rows,
                            const int32_t* group_shared_pages, int n_groups, void* out, int iters) {
    void* bufs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    try {
        init_sms();
        constexpr int kMaxParts = 32;
        std::vector<hkd::DecodeRowIn> rows(static_cast<size_t>(n_rows));
        for (int r = 0; r < n_rows; ++r) {
            rows[static_cast<size_t>(r)] = hkd::DecodeRowIn{offs[r], pos[r]};
            if ((pos[r] + 16) / 16 > offs[r + 1] - offs[r]) throw std::runtime_error("hkx_decode_attention: short table");
            for (int k = offs[r]; k < offs[r + 1]; ++k)
                if (tables[k] < 0 || tables[k] >= n_pages) throw std::runtime_error("hkx_decode_attention: bad page");
        }
        std::vector<hkd::DecodeGroupIn> groups;
        int r0 = 0;
        for (int g = 0; g < n_groups; ++g) {
            groups.push_back(hkd::DecodeGroupIn{r0, group_rows[g], group_shared_pages[g]});
            r0 += group_rows[g];
        }
        if (r0 != n_rows) throw std::runtime_error("hkx_decode_attention: groups do not cover the rows");
        hkd::DecodePlan plan;
        hkd::plan_decode_attention(rows, groups, H, Hkv, kMaxParts, hkd::g_num_sms, plan);
        const size_t n_tab = static_cast<size_t>(offs[n_rows]);
        const size_t b_tab = n_tab * 4, b_sh = plan.sh.size() * sizeof(hkd::ShItem),
                     b_pv = plan.pv.size() * sizeof(hkd::PvItem), b_np = plan.n_parts.size() * 4;
        HK_CUDA(cudaMalloc(&bufs[0], b_tab + b_sh + b_pv + b_np + 64));
        uint8_t* m = static_cast<uint8_t*>(bufs[0]);
        HK_CUDA(cudaMemcpy(m, tables, b_tab, cudaMemcpyHostToDevice));
        const size_t o_sh = (b_tab + 15) / 16 * 16, o_pv = o_sh + b_sh, o_np = o_pv + b_pv;
        if (b_sh) HK_CUDA(cudaMemcpy(m + o_sh, plan.sh.data(), b_sh, cudaMemcpyHostToDevice));
        if (b_pv) HK_CUDA(cudaMemcpy(m + o_pv, plan.pv.data(), b_pv, cudaMemcpyHostToDevice));
        HK_CUDA(cudaMemcpy(m + o_np, plan.n_parts.data(), b_np, cudaMemcpyHostToDevice));
        const size_t n_part = static_cast<size_t>(n_rows) * H * kMaxParts;
        HK_CUDA(cudaMalloc(&bufs[1], n_part * 128 * 4));
        HK_CUDA(cudaMalloc(&bufs[2], n_part * 8));
        // arrival counters [rows][Hkv], then queue state (head, exits, grid arrival) for the
        // first call and for each of the 10 launches of the timing graph: a launch may
        // claim queue items before griddepcontrol.wait, so back-to-back launches never
        // share a queue head (as the engine's layers do not)
        const size_t ctr_n = static_cast<size_t>(n_rows) * Hkv + 4 * 11;
        HK_CUDA(cudaMalloc(&bufs[3], ctr_n * 4));
        HK_CUDA(cudaMemset(bufs[3], 0, ctr_n * 4));
        int32_t* ctr = static_cast<int32_t*>(bufs[3]);
        const CUtensorMap tm = hkd::make_tmap_2d_bf16(kv, static_cast<uint64_t>(n_pages) * 2 * Hkv * 16, 128, 64, 16);
        hkd::DecodeAttnArgs a{static_cast<const hkd::bf16*>(qkv), nullptr, H, Hkv, (H + 2 * Hkv) * 128,
                              static_cast<const hkd::bf16*>(kv), 0, reinterpret_cast<const int32_t*>(m),
                              reinterpret_cast<const hkd::ShItem*>(m + o_sh), static_cast<int>(plan.sh.size()), plan.sh_cluster,
                              reinterpret_cast<const hkd::PvItem*>(m + o_pv), static_cast<int>(plan.pv.size()),
                              static_cast<float*>(bufs[1]), static_cast<float2*>(bufs[2]), kMaxParts,
                              reinterpret_cast<const int32_t*>(m + o_np), ctr, n_rows,
                              [&] {
                                  const int mx = plan.n_parts.empty() ? 0 : *std::max_element(plan.n_parts.begin(), plan.n_parts.end());
                                  return mx > 1 ? mx : 0;
                              }(),
                              ctr + static_cast<size_t>(n_rows) * Hkv,
                              ctr + static_cast<size_t>(n_rows) * Hkv + 1, ctr + static_cast<size_t>(n_rows) * Hkv + 2,
                              0, 0,
                              static_cast<hkd::bf16*>(out), 1.4426950408889634f / sqrtf(128.f), g_trace, nullptr, 0};
        hkd::decode_attention(a, tm, nullptr);
        HK_CUDA(cudaDeviceSynchronize());
        double ms = 0;
        if (iters > 0) {
            // time graph replays (as the engine runs decode steps), 10 calls per graph
            cudaStream_t cs;
            HK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t g;
            HK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            for (int i = 0; i < 10; ++i) {
                hkd::DecodeAttnArgs ai = a;
                ai.pv_next = ctr + static_cast<size_t>(n_rows) * Hkv + 4 * (i + 1);
                ai.pv_done = ai.pv_next + 1;
                ai.grid_arrive = ai.pv_next + 2;
                hkd::decode_attention(ai, tm, cs);
            }
            HK_CUDA(cudaStreamEndCapture(cs, &g));
            cudaGraphExec_t ge;
            HK_CUDA(cudaGraphInstantiate(&ge, g, 0));
            HK_CUDA(cudaGraphLaunch(ge, cs));  // warm
            cudaEvent_t e0, e1;
            HK_CUDA(cudaEventCreate(&e0));
            HK_CUDA(cudaEventCreate(&e1));
            const int reps = (iters + 9) / 10;
            HK_CUDA(cudaEventRecord(e0, cs));
            for (int i = 0; i < reps; ++i) HK_CUDA(cudaGraphLaunch(ge, cs));
            HK_CUDA(cudaEventRecord(e1, cs));
            HK_CUDA(cudaEventSynchronize(e1));
            float t = 0;
            HK_CUDA(cudaEventElapsedTime(&t, e0, e1));
            ms = t / (reps * 10);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
            cudaStreamDestroy(cs);
        }
        for (void* b : bufs) cudaFree(b);
        return ms;
    } catch (const std::exception& e) {
        for (void* b : bufs) cudaFree(b);
        hk::set_error(e.what());
        return -1;
    }
}

/* Phase timestamps (%globaltimer ns) of the next hkx_decode_attention calls:
 * [n_sh + n_pv CTAs][8] into a device buffer of `words` u64 (NULL = off). */
int hkx_span_trace(int on) {
    try {
        hkd::span_trace_reset(on != 0);
        return 0;
    } catch (...) {
        return -1;
    }
}

int hkx_gemm_trace_dump(const char* path) {
    try {
        return hkd::gemm_trace_dump(path);
    } catch (...) {
        return -1;
    }
}

int hkx_decode_attention_trace(void* device_buf) {
    g_trace = static_cast<unsigned long long*>(device_buf);
    return 0;
}

/* algorithmic bytes of the same call (shared KV once per group + private KV + q/o) */
double hkx_decode_attention_bytes(int n_rows, int H, int Hkv, const int32_t* offs, const int32_t* pos,
                                  const int32_t* group_rows, const int32_t* group_shared_pages, int n_groups) {
    std::vector<hkd::DecodeRowIn> rows(static_cast<size_t>(n_rows));
    for (int r = 0; r < n_rows; ++r) rows[static_cast<size_t>(r)] = hkd::DecodeRowIn{offs[r], pos[r]};
    std::vector<hkd::DecodeGroupIn> groups;
    int r0 = 0;
    for (int g = 0; g < n_groups; ++g) {
        groups.push_back(hkd::DecodeGroupIn{r0, group_rows[g], group_shared_pages[g]});
        r0 += group_rows[g];
    }
    hkd::DecodePlan plan;
    try {
        hkd::plan_decode_attention(rows, groups, H, Hkv, 32, 148, plan);
    } catch (const std::exception& e) {
        hk::set_error(e.what());
        return -1;
    }
    return plan.shared_bytes + plan.private_bytes;
}

/* Several causal prefill segments in ONE launch, planned exactly as the engine
 * plans a step (plan_prefill_attention with the page-id arena): segment s has
 * seg_count[s] tokens at batch rows seg_tok0[s].., positions seg_start[s]..,
 * and its block table at arena[seg_ptab[s]..]. Adjacent single-tile segments
 * that share >= 8 leading pages are paired (common pages multicast). */
int hkx_prefill_attention_segs(const void* qkv, const void* kv, int n_pages, int n_segs, const int32_t* seg_tok0,
                               const int32_t* seg_count, const int32_t* seg_start, const int32_t* seg_ptab, int H,
                               int Hkv, const int32_t* arena, int arena_len, int n_tok, void* out) {
    void* bufs[2] = {nullptr, nullptr};
    try {
        init_sms();
        hkd::DecodePlan plan;
        std::vector<hkd::PrefillSegIn> segs;
        std::vector<int32_t> pos(static_cast<size_t>(n_tok), 0);
        for (int s = 0; s < n_segs; ++s) {
            if (seg_tok0[s] + seg_count[s] > n_tok) throw std::runtime_error("hkx_prefill_attention_segs: rows");
            if (seg_ptab[s] + (seg_start[s] + seg_count[s] + 15) / 16 > arena_len)
                throw std::runtime_error("hkx_prefill_attention_segs: short table");
            segs.push_back(hkd::PrefillSegIn{seg_tok0[s], seg_count[s], seg_start[s], seg_ptab[s]});
            for (int i = 0; i < seg_count[s]; ++i) pos[static_cast<size_t>(seg_tok0[s] + i)] = seg_start[s] + i;
        }
        for (int i = 0; i < arena_len; ++i)
            if (arena[i] < 0 || arena[i] >= n_pages) throw std::runtime_error("hkx_prefill_attention_segs: bad page");
        hkd::plan_prefill_attention(segs, H, Hkv, plan, arena);
        const int32_t* table = arena;
        const int table_len = arena_len;
        const size_t b_tab = static_cast<size_t>(table_len) * 4, b_pos = pos.size() * 4,
                     b_sh = plan.sh.size() * sizeof(hkd::ShItem);
        const size_t o_pos = (b_tab + 15) / 16 * 16, o_sh = o_pos + (b_pos + 15) / 16 * 16;
        HK_CUDA(cudaMalloc(&bufs[0], o_sh + b_sh + 64));
        uint8_t* m = static_cast<uint8_t*>(bufs[0]);
        HK_CUDA(cudaMemcpy(m, table, b_tab, cudaMemcpyHostToDevice));
        HK_CUDA(cudaMemcpy(m + o_pos, pos.data(), b_pos, cudaMemcpyHostToDevice));
        HK_CUDA(cudaMemcpy(m + o_sh, plan.sh.data(), b_sh, cudaMemcpyHostToDevice));
        HK_CUDA(cudaMalloc(&bufs[1], 64));
        HK_CUDA(cudaMemset(bufs[1], 0, 64));
        int32_t* ctr = static_cast<int32_t*>(bufs[1]);
        const CUtensorMap tm = hkd::make_tmap_2d_bf16(kv, static_cast<uint64_t>(n_pages) * 2 * Hkv * 16, 128, 64, 16);
        hkd::DecodeAttnArgs a{static_cast<const hkd::bf16*>(qkv), reinterpret_cast<const int32_t*>(m + o_pos), H, Hkv,
                              (H + 2 * Hkv) * 128, static_cast<const hkd::bf16*>(kv), 0,
                              reinterpret_cast<const int32_t*>(m), reinterpret_cast<const hkd::ShItem*>(m + o_sh),
                              static_cast<int>(plan.sh.size()), 1, nullptr, 0, nullptr, nullptr, 32, nullptr, ctr, 0, 0,
                              ctr + 4, ctr + 5, ctr + 6, 0, n_tok, static_cast<hkd::bf16*>(out),
                              1.4426950408889634f / sqrtf(128.f), nullptr, nullptr, 0};
        hkd::decode_attention(a, tm, nullptr);
        HK_CUDA(cudaDeviceSynchronize());
        for (void* b : bufs) cudaFree(b);
        return 0;
    } catch (const std::exception& e) {
        for (void* b : bufs) cudaFree(b);
        hk::set_error(e.what());
        return -1;
    }
}

int hkx_prefill_attention(const void* qkv, const void* kv, int n_pages, int n_tok, int start, int H, int Hkv,
                          const int32_t* table, int table_len, void* out) {
    if ((start + n_tok + 15) / 16 > table_len) {
        hk::set_error("hkx_prefill_attention: short table");
        return -1;
    }
    const int32_t zero = 0;
    return hkx_prefill_attention_segs(qkv, kv, n_pages, 1, &zero, &n_tok, &start, &zero, H, Hkv, table,
                                      (start + n_tok + 15) / 16, n_tok, out);
}

}  // extern "C"
