// K2: batched prefix-trie match + block-table construction on device.
//
// The device trie mirrors one worker's KvTree (kvtree.cpp, itself bit-exact
// with the reference KvCache, simulator.cpp:14-128). Nodes are addressed by
// the host's node ids; an open-addressing table maps the PREFIX hash
//   H_0 = FNV offset,  H_k = hash_combine(H_{k-1}, fnv1a64(block_k bytes))
// to node ids, so every block of a prompt is probed independently (no
// pointer chase). A hit is accepted only if the node's stored block tokens
// equal the prompt's block and its parent is the node matched for block k-1;
// the matched length is the first failing k. That reproduces
// KvCache::lookup's walk exactly (hash collisions can only cause a miss to be
// re-checked, never a false hit).
#include "common.cuh"
#include "kernels.cuh"

namespace hkd {

namespace {

constexpr uint64_t kEmpty = 0, kTomb = 1;
__device__ __forceinline__ uint64_t tab_key(uint64_t h) { return h < 2 ? h + 2 : h; }

__device__ __forceinline__ uint64_t fnv_bytes(const uint8_t* p, int n, uint64_t h) {
    for (int i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
__device__ __forceinline__ uint64_t fnv_u64(uint64_t v, uint64_t h) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h ^= (v >> (8 * i)) & 0xff;
        h *= 0x100000001b3ull;
    }
    return h;
}
__device__ __forceinline__ uint64_t hash_combine_d(uint64_t h, uint64_t v) {
    h = (h ^ 0x9e3779b97f4a7c15ull) * 0x100000001b3ull;
    return fnv_u64(v, h);
}

__global__ void trie_erase_kernel(DevTrie t, const TrieOpDev* ops, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !ops[i].erase) return;
    const uint64_t key = tab_key(ops[i].phash);
    const uint32_t mask = static_cast<uint32_t>(t.table_size - 1);
    uint32_t s = static_cast<uint32_t>(key) & mask;
    for (int probe = 0; probe < t.table_size; ++probe, s = (s + 1) & mask) {
        const uint64_t k = t.tab_key[s];
        if (k == kEmpty) break;
        if (k == key && t.tab_node[s] == ops[i].node) {
            t.tab_key[s] = kTomb;
            break;
        }
    }
    t.parent[ops[i].node] = -2;  // free
}

__global__ void trie_insert_kernel(DevTrie t, const TrieOpDev* ops, const uint64_t* keys, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || ops[i].erase) return;
    const TrieOpDev op = ops[i];
    t.parent[op.node] = op.parent;
    t.page[op.node] = op.page;
    t.phash[op.node] = op.phash;
    for (int j = 0; j < t.block; ++j) t.keys[static_cast<size_t>(op.node) * t.block + j] = keys[static_cast<size_t>(i) * t.block + j];
    const uint64_t key = tab_key(op.phash);
    const uint32_t mask = static_cast<uint32_t>(t.table_size - 1);
    uint32_t s = static_cast<uint32_t>(key) & mask;
    for (int probe = 0; probe < t.table_size; ++probe, s = (s + 1) & mask) {
        unsigned long long* slot = reinterpret_cast<unsigned long long*>(t.tab_key + s);
        unsigned long long prev = atomicCAS(slot, kEmpty, key);
        if (prev == kEmpty || (prev == kTomb && atomicCAS(slot, kTomb, key) == kTomb)) {
            t.tab_node[s] = op.node;
            break;
        }
    }
}

// One CTA per prompt. smem: bh/H [max_blocks] u64, cand [max_blocks] int.
__global__ void __launch_bounds__(256) trie_match_kernel(DevTrie t, const uint64_t* tokens, const uint64_t* offsets,
                                                        int32_t* matched, int32_t* node_path, int32_t* page_table,
                                                        int stride) {
    extern __shared__ uint64_t sh[];
    const int p = blockIdx.x;
    const uint64_t off = offsets[p];
    const int len = static_cast<int>(offsets[p + 1] - off);
    const int nb = min(len / t.block, stride);
    uint64_t* H = sh;
    int32_t* cand = reinterpret_cast<int32_t*>(sh + stride);
    __shared__ int first_fail;
    if (threadIdx.x == 0) first_fail = nb;
    // 1. per-block FNV of the block's bytes (parallel)
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
        H[k] = fnv_bytes(reinterpret_cast<const uint8_t*>(tokens + off + static_cast<uint64_t>(k) * t.block),
                         t.block * 8, 0xcbf29ce484222325ull);
    __syncthreads();
    // 2. prefix fold (serial; nb <= a few hundred)
    if (threadIdx.x == 0) {
        uint64_t h = 0xcbf29ce484222325ull;
        for (int k = 0; k < nb; ++k) {
            h = hash_combine_d(h, H[k]);
            H[k] = h;
        }
    }
    __syncthreads();
    // 3. independent probes with full-key verification
    const uint32_t mask = static_cast<uint32_t>(t.table_size - 1);
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const uint64_t key = tab_key(H[k]);
        const uint64_t* blk = tokens + off + static_cast<uint64_t>(k) * t.block;
        int found = -1;
        uint32_t s = static_cast<uint32_t>(key) & mask;
        for (int probe = 0; probe < t.table_size; ++probe, s = (s + 1) & mask) {
            const uint64_t tk = t.tab_key[s];
            if (tk == kEmpty) break;
            if (tk != key) continue;
            const int nd = t.tab_node[s];
            if (t.phash[nd] != H[k]) continue;
            bool eq = true;
            for (int j = 0; j < t.block && eq; ++j) eq = t.keys[static_cast<size_t>(nd) * t.block + j] == blk[j];
            if (eq) {
                found = nd;
                break;
            }
        }
        cand[k] = found;
    }
    __syncthreads();
    // 4. chain check: node k's parent must be node k-1 (root = 0)
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const int c = cand[k];
        const int want = k == 0 ? 0 : cand[k - 1];
        if (c < 0 || want < 0 || t.parent[c] != want) atomicMin(&first_fail, k);
    }
    __syncthreads();
    const int m = first_fail;
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        node_path[static_cast<size_t>(p) * stride + k] = cand[k];
        page_table[static_cast<size_t>(p) * stride + k] = t.page[cand[k]];
    }
    if (threadIdx.x == 0) matched[p] = m;
}

}  // namespace

void trie_apply(DevTrie& t, const TrieOpDev* ops, const uint64_t* keys, int n_ops, cudaStream_t st) {
    if (n_ops <= 0) return;
    const int blocks = (n_ops + 127) / 128;
    trie_erase_kernel<<<blocks, 128, 0, st>>>(t, ops, n_ops);
    trie_insert_kernel<<<blocks, 128, 0, st>>>(t, ops, keys, n_ops);
    HK_LAUNCHED(2);
}

void trie_match(const DevTrie& t, const uint64_t* tokens, const uint64_t* offsets, int n_prompts, int32_t* matched,
                int32_t* node_path, int32_t* page_table, int stride, cudaStream_t st) {
    if (n_prompts <= 0) return;
    const size_t sm = static_cast<size_t>(stride) * (8 + 4);
    if (sm > 48 * 1024) HK_CUDA(cudaFuncSetAttribute(trie_match_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     static_cast<int>(sm)));
    trie_match_kernel<<<n_prompts, 256, sm, st>>>(t, tokens, offsets, matched, node_path, page_table, stride);
    HK_LAUNCHED(1);
}

}  // namespace hkd
