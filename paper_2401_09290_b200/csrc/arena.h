// arena.h -- partition manager internals.
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <shared_mutex>
#include <vector>

#include "guardian.h"

namespace gd {

// Buddy allocator over [0, arena_size) in units of 2^min_order bytes
// ("base allocated by buddy allocation (guarantees
// alignment)").  Offsets of order-k blocks are multiples of 2^k; free blocks
// are coalesced eagerly, so any fully free aligned 2^k region lies inside a
// single free block of order >= k.  Lowest-address-first within an order.
class Buddy {
public:
    void init(uint64_t arena_size, unsigned min_order);
    // returns false when no block of 2^order bytes is free
    bool alloc(unsigned order, uint64_t *off);
    void free(uint64_t off, unsigned order);
    // Exact-size extent (bytes a multiple of 2^min_order): take the block of
    // next_pow2(bytes) and give its tail back as aligned sub-blocks; freeing
    // returns the extent's aligned sub-blocks, which coalesce with the tail.
    bool alloc_exact(uint64_t bytes, uint64_t *off);
    void free_exact(uint64_t off, uint64_t bytes);
    uint64_t free_bytes() const;
    unsigned max_order() const { return max_order_; }
    unsigned min_order() const { return min_order_; }

private:
    unsigned min_order_ = 12, max_order_ = 12;
    std::vector<std::set<uint64_t>> free_;   // free_[order] = offsets
};

// First-fit sub-allocator inside one partition, 256-byte
// alignment, exact-address frees.
class SubAlloc {
public:
    void init(uint64_t size);
    bool alloc(uint64_t bytes, uint64_t *off);
    bool free(uint64_t off);
private:
    std::map<uint64_t, uint64_t> free_;      // offset -> length, disjoint, coalesced
    std::map<uint64_t, uint64_t> live_;      // offset -> length
};

struct Partition {
    bool live = false;
    uint64_t base = 0, size = 0;
    unsigned order = 0;
    bool pow2 = true;              // false: exact-size partition (modulo / check / none modes)
    uint64_t gen = 0;              // allocation generation (captured graphs check it)
    SubAlloc sub;
};

struct HostCounters {
    uint64_t launches = 0, bytes = 0, flops = 0;
};

struct Chunk {                      // one physical VMM allocation mapped in the arena
    unsigned long long handle = 0;  // CUmemGenericAllocationHandle
    uint64_t size = 0;
    uint32_t refs = 0;
};

}  // namespace gd

struct gd_arena {
    int device = -1;                 // -1: virtual (bookkeeping only)
    bool vmm = false;                // VA reserved / physical memory mapped by us
    uint64_t base = 0, size = 0;     // the arena: size pow2, base % size == 0
    uint64_t reserve_va = 0, reserve_size = 0, gran = 0;
    std::map<uint64_t, gd::Chunk> chunks;   // chunk VA -> mapping
    gd::Buddy buddy;
    gd::Partition parts[GD_MAX_TENANTS];
    gd::HostCounters host[GD_MAX_TENANTS][GD_NUM_KINDS];
    unsigned long long *d_stats = nullptr;  // u64[GD_MAX_TENANTS][GD_NUM_KINDS], outside the arena
    uint64_t d_zero = 0;             // trusted all-zero 256-byte block after the counters (FenceDesc::zero)
    void *zero_buf = nullptr;        // trusted zero row for operands with no rows (gemm.cu)
    uint64_t zero_bytes = 0;
    std::vector<void *> zero_retired;  // outgrown zero rows: captured graphs may still read them (freed at destroy)
    int sms = 148;
    uint64_t next_gen = 1;
    bool native_when_solo = false;   // a tenant alone runs the native kernel
    uint64_t epoch = 0;              // bumped by every carve / free / native_when_solo change
    std::mutex mu;                   // bounds table, allocators, counters
    // Launch guard: every path that snapshots partition bounds and enqueues
    // work with them (launches, checked transfers, fills, graph replays)
    // holds it shared from the snapshot until the work is enqueued; carve and
    // free hold it exclusively, so bounds never change between a snapshot and
    // its enqueue (free then synchronises before it unmaps).  Taken before mu.
    std::shared_mutex launch_mu;
};
