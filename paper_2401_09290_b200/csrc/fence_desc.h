// fence_desc.h -- launch-time partition descriptor shared by host and device.
#pragma once
#include <cstdint>

namespace gd {

enum Mode : int { kNone = 0, kMask = 1, kCheck = 2 };

// Launch-time partition descriptor.  Built on the host
// from an immutable snapshot of the bounds-table row.
struct FenceDesc {
    uint64_t base;                 // partition base, size-aligned
    uint64_t mask;                 // size - 1
    unsigned long long *viol;      // trusted counter (outside every partition)
};

}  // namespace gd
