// alloc.cpp -- buddy partition allocator and first-fit sub-allocator (host).
//
// Buddy: SPEC.md:214-229 (power-of-two, size-aligned partitions carved from
// one reserved pool).  Sub-allocator: SPEC.md:230-245
// (first fit, 256-byte alignment, exact-address free).
#include "arena.h"

namespace gd {

void Buddy::init(uint64_t arena_size, unsigned min_order) {
    min_order_ = min_order;
    max_order_ = 0;
    while ((1ull << max_order_) < arena_size) max_order_++;
    free_.assign(max_order_ + 1, {});
    free_[max_order_].insert(0);
}

bool Buddy::alloc(unsigned order, uint64_t *off) {
    if (order < min_order_) order = min_order_;
    if (order > max_order_) return false;
    unsigned j = order;
    while (j <= max_order_ && free_[j].empty()) j++;
    if (j > max_order_) return false;
    uint64_t o = *free_[j].begin();
    free_[j].erase(free_[j].begin());
    while (j > order) {                 // split, keep the lower half
        j--;
        free_[j].insert(o + (1ull << j));
    }
    *off = o;
    return true;
}

void Buddy::free(uint64_t off, unsigned order) {
    while (order < max_order_) {
        const uint64_t buddy = off ^ (1ull << order);
        auto it = free_[order].find(buddy);
        if (it == free_[order].end()) break;
        free_[order].erase(it);
        off = off < buddy ? off : buddy;
        order++;
    }
    free_[order].insert(off);
}

namespace {
// Split [lo, hi) into maximal aligned power-of-two blocks, ascending.
template <typename F>
void aligned_pieces(uint64_t lo, uint64_t hi, unsigned max_order, F f) {
    while (lo < hi) {
        unsigned k = lo ? (unsigned)__builtin_ctzll(lo) : max_order;
        if (k > max_order) k = max_order;
        while ((1ull << k) > hi - lo) k--;
        f(lo, k);
        lo += 1ull << k;
    }
}
}  // namespace

bool Buddy::alloc_exact(uint64_t bytes, uint64_t *off) {
    unsigned order = min_order_;
    while ((1ull << order) < bytes) order++;
    if (order > max_order_ || !alloc(order, off)) return false;
    aligned_pieces(*off + bytes, *off + (1ull << order), max_order_, [this](uint64_t o, unsigned k) { free(o, k); });
    return true;
}

void Buddy::free_exact(uint64_t off, uint64_t bytes) {
    aligned_pieces(off, off + bytes, max_order_, [this](uint64_t o, unsigned k) { free(o, k); });
}

uint64_t Buddy::free_bytes() const {
    uint64_t s = 0;
    for (unsigned k = 0; k < free_.size(); k++) s += (uint64_t)free_[k].size() << k;
    return s;
}

void SubAlloc::init(uint64_t size) {
    free_.clear();
    live_.clear();
    free_[0] = size;
}

bool SubAlloc::alloc(uint64_t bytes, uint64_t *off) {
    if (bytes == 0) return false;
    const uint64_t len = (bytes + 255) & ~255ull;
    if (len < bytes) return false;
    for (auto it = free_.begin(); it != free_.end(); ++it) {
        if (it->second >= len) {                // extents start 256-aligned
            const uint64_t o = it->first, rest = it->second - len;
            free_.erase(it);
            if (rest) free_[o + len] = rest;
            live_[o] = len;
            *off = o;
            return true;
        }
    }
    return false;
}

bool SubAlloc::free(uint64_t off) {
    auto it = live_.find(off);
    if (it == live_.end()) return false;
    uint64_t o = it->first, len = it->second;
    live_.erase(it);
    auto nx = free_.lower_bound(o);
    if (nx != free_.end() && nx->first == o + len) {
        len += nx->second;
        nx = free_.erase(nx);
    }
    if (nx != free_.begin()) {
        auto pv = std::prev(nx);
        if (pv->first + pv->second == o) {
            pv->second += len;
            return true;
        }
    }
    free_[o] = len;
    return true;
}

}  // namespace gd
