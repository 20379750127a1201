// fence.cuh -- the per-access fence of Guardian (arXiv 2401.09290), sm_100a.
//
// One device function per mode, applied to the FINAL effective address of
// every global access (base+offset forms are materialised first, PAPER.md:232
// §4.3 second addressing mode).  The partition descriptor reaches the kernel
// by value as a __grid_constant__ parameter, i.e. in constant bank 0: the
// paper's "mask and the base partition address" parameters (PAPER.md:175
// §4.2.3, Listing 1 lines 5-7 and 17-18, reading A12).
//
//   MASK  : f = (a & mask_w) | base        Listing 1 lines 26-28 (and.b64, or.b64)
//           mask_w = (size-1) & ~(w-1)      reading A3 (keeps w-alignment)
//           -> on sm_100 one LOP3 per 32-bit half, operands uniform.
//           Needs a power-of-two, size-aligned partition.
//   MODULO: f = base + (((a - base) mod size) & ~(w-1))     PAPER.md:238-244 §4.4
//           the 64-bit modulo inline with the reciprocal parameter
//           inv = floor(2^64 / size) ("an extra parameter holding the
//           1/partition_size"): q = mulhi(off, inv) is off/size
//           or one less, so one conditional subtract finishes it.  Works for
//           any partition size that is a multiple of 16.
//   CHECK : ok = (a - base) <= size - w  and  a % w == 0
//           PAPER.md:175 ("partition base and ending addresses"), 236; A1, A2.
//           A refused load yields 0, a refused store/atomic is dropped, and
//           the refusal is counted (aggregated per thread, then per CTA).
//   NONE  : identity (the unfenced twin, "native kernel").
#pragma once
#include <cstdint>

#include "fence_desc.h"

namespace gd {

// Per-width precomputation, hoisted out of every loop (uniform values).
template <int MODE, int W>
struct Fence {
    uint64_t base, keep, size, inv, lim;
    __device__ __forceinline__ explicit Fence(const FenceDesc &fd)
        : base(fd.base), keep(fd.mask & ~(uint64_t)(W - 1)), size(fd.size), inv(fd.inv), lim(fd.size - W) {}
    // address the access really uses (MASK / MODULO: fenced; CHECK / NONE: unchanged)
    __device__ __forceinline__ uint64_t addr(uint64_t a) const {
        if constexpr (MODE == kMask) {
            return (a & keep) | base;
        } else if constexpr (MODE == kModulo) {
            const uint64_t off = a - base;
            uint64_t r = off - __umul64hi(off, inv) * size;
            if (r >= size) r -= size;
            return base + (r & ~(uint64_t)(W - 1));
        } else {
            return a;
        }
    }
    // may the access be performed?
    __device__ __forceinline__ bool ok(uint64_t a) const {
        if constexpr (MODE == kCheck) return (a - base) <= lim && (a & (uint64_t)(W - 1)) == 0;
        else return true;
    }
    // ok() for an address the caller has proven W-aligned (aligned operand
    // bases and W-multiple strides): the alignment half of the test is known true
    __device__ __forceinline__ bool ok_aligned(uint64_t a) const {
        if constexpr (MODE == kCheck) return (a - base) <= lim;
        else return true;
    }
};

// Check-mode hoisting: true iff every byte of [a, a+len) lies in the
// partition (no 64-bit wraparound).  A CTA whose whole tile passes this test
// performs exactly the accesses the per-access check would allow (all of
// them) and refuses none, so it may run the unchecked body; only tiles that
// touch or cross the partition edge pay for per-access checks.
__device__ __forceinline__ bool range_in(const FenceDesc &fd, uint64_t a, uint64_t len) {
    const uint64_t off = a - fd.base;
    return !(fd.flags & kNoHoist) && len <= fd.size && off <= fd.size - len;
}

// Sum a per-thread refusal count over the CTA and add it to the trusted
// counter with one atomic per CTA.  All threads of the
// CTA must call it.
__device__ __forceinline__ void flush_violations(uint32_t nv_thread, unsigned long long *viol) {
    if (!__syncthreads_or(nv_thread != 0)) return;    // common case: nothing refused in this CTA
    __shared__ unsigned long long warp_sums[32];
    uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long nv = nv_thread;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
    if (lane == 0) warp_sums[warp] = nv;
    __syncthreads();
    if (warp == 0) {
        uint32_t nw = (blockDim.x + 31u) >> 5;
        unsigned long long s = lane < nw ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && s) atomicAdd(viol, s);
    }
}

}  // namespace gd
