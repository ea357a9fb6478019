// KvTree: the per-worker block radix tree with the reference KvCache's exact
// semantics (simulator.cpp:14-128), plus physical pages and device-trie
// journaling. Differentially fuzzed against the reference KvCache in
// tests/test_host_cpu.py::test_kvtree_matches_reference_fuzz.
#include <algorithm>

#include "hk_host.hpp"

namespace hk {

// ------------------------------------------------------------------ PagePool
void PagePool::reset(int n_pages) {
    n_ = n_pages;
    high_ = 0;
    free_.clear();
    deferred_.clear();
    tree_.assign(static_cast<std::size_t>(n_pages), 0);
    free_.reserve(static_cast<std::size_t>(n_pages));
    for (int p = n_pages - 1; p >= 0; --p) free_.push_back(p);  // hand out 0,1,2,...
}

int PagePool::alloc() {
    if (free_.empty()) {
        if (!deferred_.empty())
            throw std::runtime_error("kv page pool exhausted within one iteration (" + std::to_string(n_) +
                                     " pages); raise the private-page reserve");
        throw std::runtime_error("kv page pool exhausted (" + std::to_string(n_) + " pages)");
    }
    int p = free_.back();
    free_.pop_back();
    high_ = std::max(high_, in_use());
    return p;
}

void PagePool::flush_deferred() {
    for (auto it = deferred_.rbegin(); it != deferred_.rend(); ++it) free_.push_back(*it);
    deferred_.clear();
}

// -------------------------------------------------------------------- KvTree
KvTree::KvTree(std::size_t capacity_tokens, std::size_t block_tokens)
    : capacity_(capacity_tokens), block_(block_tokens) {
    if (block_ == 0) throw std::runtime_error("kv block size must be positive");
    if (capacity_ < block_) throw std::runtime_error("kv capacity below one block");
    nodes_.push_back(Node{});  // root sentinel, never evicted
    keys_.resize(block_, 0);
}

int KvTree::find_child(int parent, const Token* blk, std::uint64_t bh) const {
    auto range = kids_.equal_range(ChildKey{parent, bh});
    for (auto it = range.first; it != range.second; ++it) {
        const Token* k = node_key(it->second);
        if (std::equal(blk, blk + block_, k)) return it->second;
    }
    return -1;
}

void KvTree::touch(int idx) {
    Node& n = nodes_[static_cast<std::size_t>(idx)];
    if (evictable(n)) evictable_.erase({n.last_use, idx});
    n.last_use = ++clock_;
    if (evictable(n)) evictable_.insert({n.last_use, idx});
}

int KvTree::create_child(int parent, const Token* blk, std::uint64_t bh) {
    // phash comes from the parent before any reuse of its slot (see the
    // self-parent corner case in DESIGN.md §KvTree).
    const std::uint64_t ph = hash_combine(nodes_[static_cast<std::size_t>(parent)].phash, bh);
    int idx;
    if (!free_.empty()) {
        idx = free_.back();
        free_.pop_back();
        nodes_[static_cast<std::size_t>(idx)] = Node{};
    } else {
        idx = static_cast<int>(nodes_.size());
        nodes_.push_back(Node{});
        keys_.resize(keys_.size() + block_);
    }
    Node& n = nodes_[static_cast<std::size_t>(idx)];
    n.parent = parent;
    n.phash = ph;
    n.bhash = bh;
    std::copy(blk, blk + block_, keys_.begin() + static_cast<std::ptrdiff_t>(static_cast<std::size_t>(idx) * block_));
    Node& p = nodes_[static_cast<std::size_t>(parent)];
    if (parent != 0 && evictable(p)) evictable_.erase({p.last_use, parent});
    p.nkids++;
    kids_.emplace(ChildKey{parent, bh}, idx);
    // a fresh node is childless/unpinned/unheld but last_use 0; it is touched
    // right after creation by insert(), which files it in the evictable set.
    return idx;
}

bool KvTree::evict_one() {
    if (evictable_.empty()) return false;
    const int victim = evictable_.begin()->second;
    evictable_.erase(evictable_.begin());
    Node& v = nodes_[static_cast<std::size_t>(victim)];
    const int parent = v.parent;
    auto range = kids_.equal_range(ChildKey{parent, v.bhash});
    for (auto it = range.first; it != range.second; ++it) {
        if (it->second == victim) {
            kids_.erase(it);
            break;
        }
    }
    Node& p = nodes_[static_cast<std::size_t>(parent)];
    p.nkids--;
    v.free = true;
    free_.push_back(victim);
    used_ -= block_;
    evicted_ += block_;
    if (v.page >= 0 && pool_) {
        pool_->mark_tree(v.page, false);
        pool_->release(v.page);
    }
    if (journaling) journal_.push_back(TrieOp{victim, parent, v.page, true, v.phash});
    v.page = -1;
    if (parent != 0 && parent != victim && evictable(p)) evictable_.insert({p.last_use, parent});
    return true;
}

std::size_t KvTree::lookup(const Token* seq, std::size_t n, std::uint64_t hold, std::vector<int>* path) {
    std::size_t matched = 0;
    int cur = 0;
    for (std::size_t off = 0; off + block_ <= n; off += block_) {
        const Token* blk = seq + off;
        int next = find_child(cur, blk, block_hash(blk));
        if (next < 0) break;
        touch(next);
        if (hold != 0) {
            Node& nn = nodes_[static_cast<std::size_t>(next)];
            if (evictable(nn)) evictable_.erase({nn.last_use, next});
            nn.holds++;
            holds_[hold].push_back(next);
        }
        if (path) path->push_back(next);
        matched += block_;
        cur = next;
    }
    return matched;
}

std::size_t KvTree::peek(const Token* seq, std::size_t n, std::vector<int>* path) const {
    std::size_t matched = 0;
    int cur = 0;
    for (std::size_t off = 0; off + block_ <= n; off += block_) {
        int next = find_child(cur, seq + off, block_hash(seq + off));
        if (next < 0) break;
        if (path) path->push_back(next);
        matched += block_;
        cur = next;
    }
    return matched;
}

void KvTree::apply_lookup(const int* path, std::size_t n_blocks, std::uint64_t hold) {
    for (std::size_t k = 0; k < n_blocks; ++k) {
        const int next = path[k];
        touch(next);
        if (hold != 0) {
            Node& nn = nodes_[static_cast<std::size_t>(next)];
            if (evictable(nn)) evictable_.erase({nn.last_use, next});
            nn.holds++;
            holds_[hold].push_back(next);
        }
    }
}

std::size_t KvTree::insert(const Token* seq, std::size_t n, std::size_t len, bool pinned, std::uint64_t hold,
                           Owner owner, std::vector<int>* new_nodes) {
    len = std::min(len, n);
    std::size_t stored = 0;
    int cur = 0;
    for (std::size_t off = 0; off + block_ <= len; off += block_) {
        const Token* blk = seq + off;
        const std::uint64_t bh = block_hash(blk);
        const std::size_t bi = off / block_;
        int next = find_child(cur, blk, bh);
        if (next < 0) {
            // Make room before allocating; if nothing is evictable, stop here.
            while (used_ + block_ > capacity_) {
                if (!evict_one()) return stored;
            }
            next = create_child(cur, blk, bh);
            used_ += block_;
            stored += block_;
            Node& nn = nodes_[static_cast<std::size_t>(next)];
            if (owner.pages) {
                // adopt the call's page for this block: zero-copy ownership transfer
                nn.page = (*owner.pages)[bi];
            } else if (pool_) {
                nn.page = pool_->alloc();  // pins: fresh page, KV computed by pin precompute
            }
            if (nn.page >= 0 && pool_) pool_->mark_tree(nn.page, true);
            if (new_nodes) new_nodes->push_back(next);
            if (journaling) journal_.push_back(TrieOp{next, cur, nn.page, false, nn.phash});
        } else if (owner.pages) {
            // content-identical block already in the tree: share its page and
            // drop the call's private copy (deferred free)
            int tp = nodes_[static_cast<std::size_t>(next)].page;
            int& mine = (*owner.pages)[bi];
            if (tp >= 0 && mine != tp) {
                if (mine >= 0 && owner.pool) owner.pool->release(mine);
                mine = tp;
            }
        }
        Node& nd = nodes_[static_cast<std::size_t>(next)];
        if (pinned && !nd.pinned) {
            if (evictable(nd)) evictable_.erase({nd.last_use, next});
            nd.pinned = true;
            pinned_ += block_;
        }
        touch(next);
        if (hold != 0) {
            if (evictable(nd)) evictable_.erase({nd.last_use, next});
            nd.holds++;
            holds_[hold].push_back(next);
        }
        cur = next;
    }
    return stored;
}

void KvTree::release(std::uint64_t hold) {
    auto it = holds_.find(hold);
    if (it == holds_.end()) return;
    for (int idx : it->second) {
        Node& n = nodes_[static_cast<std::size_t>(idx)];
        n.holds--;
        if (evictable(n)) evictable_.insert({n.last_use, idx});
    }
    holds_.erase(it);
}

// ------------------------------------------------------------ pin planning
// simulator.cpp:132-199, over the flattened call tree.
std::vector<TokenSeq> static_pin_prefixes(const Plan& p, int worker, std::size_t block, std::size_t threshold,
                                          std::size_t budget_tokens) {
    if (block == 0) throw std::runtime_error("kv block size must be positive");
    std::map<CallId, int> place;
    for (std::size_t w = 0; w < p.sigma.size(); ++w)
        for (const CallId& c : p.sigma[w]) place[c] = static_cast<int>(w);

    std::vector<int> cnt(p.tree.size(), 0);
    for (int lf : p.leaves) {
        const TreeNode& L = p.tree[static_cast<std::size_t>(lf)];
        auto it = place.find(CallId{L.op, L.query});
        if (it == place.end() || it->second != worker) continue;
        for (int v = lf; v >= 0; v = p.tree[static_cast<std::size_t>(v)].parent) ++cnt[static_cast<std::size_t>(v)];
    }

    auto all_static = [&](const TreeNode& t) {
        for (const TreePart& pt : t.parts)
            if (!pt.is_static) return false;
        return true;
    };
    std::vector<TokenSeq> cands;
    for (std::size_t i = 1; i < p.tree.size(); ++i) {
        if (cnt[i] < 2) continue;
        const TreeNode& n = p.tree[i];
        TokenSeq prefix;
        bool concrete = true;
        for (int anc : p.path_from_root(n.parent)) {
            const TreeNode& a = p.tree[static_cast<std::size_t>(anc)];
            if (!all_static(a)) {
                concrete = false;
                break;
            }
            for (const TreePart& pt : a.parts)
                prefix.insert(prefix.end(), p.span_ptr(pt.v), p.span_ptr(pt.v) + p.span_len(pt.v));
        }
        if (!concrete) continue;
        for (const TreePart& pt : n.parts) {
            if (!pt.is_static) break;
            prefix.insert(prefix.end(), p.span_ptr(pt.v), p.span_ptr(pt.v) + p.span_len(pt.v));
        }
        prefix.resize(prefix.size() - prefix.size() % block);
        if (prefix.size() < threshold || prefix.empty()) continue;
        cands.push_back(std::move(prefix));
    }
    std::sort(cands.begin(), cands.end(), [](const TokenSeq& a, const TokenSeq& b) {
        if (a.size() != b.size()) return a.size() > b.size();
        return a < b;
    });
    cands.erase(std::unique(cands.begin(), cands.end()), cands.end());

    // longest-first under the budget, counting each distinct block prefix once
    std::set<TokenSeq> chosen;
    std::vector<TokenSeq> out;
    std::size_t total = 0;
    for (const TokenSeq& cand : cands) {
        std::size_t marginal = 0;
        for (std::size_t off = 0; off + block <= cand.size(); off += block)
            if (!chosen.count(TokenSeq(cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(off + block))))
                marginal += block;
        if (total + marginal > budget_tokens) continue;
        for (std::size_t off = 0; off + block <= cand.size(); off += block)
            chosen.insert(TokenSeq(cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(off + block)));
        total += marginal;
        out.push_back(cand);
    }
    return out;
}

}  // namespace hk
