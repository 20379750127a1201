// fence_desc.h -- launch-time partition descriptor shared by host and device.
#pragma once
#include <cstdint>

namespace gd {

enum Mode : int { kNone = 0, kMask = 1, kCheck = 2, kModulo = 3, kMaskCount = 4, kClamp = 5,
                  // internal: MASK on a kBig partition (Fence::addr_big, one LOP3), chosen by the
                  // launchers of the streaming kernels from FenceDesc::flags; never an API mode
                  kMaskBig = 6 };

// modes that count accesses outside the partition (the trusted counter)
constexpr bool counts(int m) { return m == kCheck || m == kMaskCount || m == kClamp; }
// modes whose fence is the identity, with nothing counted, for every access
// inside the partition: a tile wholly inside may run the unfenced body (R-hoist)
constexpr bool hoistable(int m) { return m == kCheck || m == kModulo || m == kMaskCount || m == kClamp; }

// Launch-time partition descriptor.  Built on the host
// from an immutable snapshot of the bounds-table row.
struct FenceDesc {
    uint64_t base;                 // partition base (size-aligned for pow2 partitions)
    uint64_t mask;                 // size - 1 (the mask-mode fence; pow2 partitions only)
    uint64_t mask16, mask4;        // mask_w = (size - 1) & ~(w - 1) for w = 16 / 4 (reading A3), so the
                                   // mask fence of a w-byte access is one LOP3 per 32-bit half
    uint64_t size;                 // partition size in bytes (check / modulo)
    uint64_t inv;                  // floor(2^64 / size): modulo-mode reciprocal
    unsigned long long *viol;      // trusted counter (outside every partition)
    uint64_t zero;                 // trusted all-zero 256-byte block outside every partition: a load the
                                   // check predicate refuses reads here instead (it reads 0, reading A1)
    uint32_t flags;                // kNoHoist: check / modulo fence every access (no tile-level range test)
    uint32_t pad_;
};

constexpr uint32_t kNoHoist = 1u;
// a power-of-two, size-aligned partition of at least 4 GiB: an address lies
// in it iff its high 32 bits agree with the base's above log2(size) (one
// LOP3 and one compare instead of a 64-bit subtract and compare)
constexpr uint32_t kBig = 2u;

// floor(2^64 / s) for s >= 2
inline uint64_t recip64(uint64_t s) {
    const uint64_t q = ~0ull / s, r = ~0ull % s;
    return r == s - 1 ? q + 1 : q;
}

}  // namespace gd
