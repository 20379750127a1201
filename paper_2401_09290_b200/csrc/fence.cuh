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
//   MASK_COUNT: the mask fence, plus a count of the accesses the check
//           predicate refuses ("GD_FLAG_COUNT").
//   CLAMP : north_star's "compare, clamp and set a violation flag" (A1's
//           saturating variant): the access goes to the largest w-aligned
//           address of the partition at or below it (base when there is
//           none) and is counted when the check predicate refuses it.
//   NONE  : identity (the unfenced twin, "native kernel").
#pragma once
#include <cstdint>

#include "fence_desc.h"

// Refused check / clamp loads read the trusted zero block (Fence::ld_at)
// instead of being predicated off; 0 restores predicated loads (A/B builds).
#ifndef GD_ZERO_REDIRECT
#define GD_ZERO_REDIRECT 1
#endif
// Modulo fence: with 1, offsets below 2 size take one conditional subtract
// instead of the reciprocal (Fence::addr).  Off: the per-access branch cost
// more than the reciprocal it saves (tools/r02_iter12.sh: row gather D = 32
// per access +1.8 -> +9.6 %, scatter-add +4.8 -> +6.1 %, L2 saxpy +12 -> +16 %).
#ifndef GD_MODULO_FAST
#define GD_MODULO_FAST 0
#endif

namespace gd {

// Per-width precomputation, hoisted out of every loop (uniform values).
template <int MODE, int W>
struct Fence {
    uint64_t base, keep, size, inv, lim, zero, size2;
    uint32_t mask_hi;              // high word of size - 1 (= of keep for every W <= 16)
    __device__ __forceinline__ explicit Fence(const FenceDesc &fd)
        : base(fd.base), keep(W == 16 ? fd.mask16 : W == 4 ? fd.mask4 : fd.mask & ~(uint64_t)(W - 1)), size(fd.size),
          inv(fd.inv), lim(fd.size - W), zero(fd.zero), size2(2 * fd.size), mask_hi((uint32_t)(fd.mask >> 32)) {}
    // The address a load reads when `ok` may refuse it (check / clamp
    // predicate, or a dead lane): refused -> the trusted zero block, which
    // reads 0 exactly as a refused check-mode load must (reading A1).  An
    // unpredicated load from a selected address keeps every load of a batch
    // free of predicates (a predicated load's destination must be zeroed
    // first and ties the scheduler to that order).  W <= 16.
    __device__ __forceinline__ uint64_t ld_at(uint64_t a, bool ok) const { return ok ? a : zero; }
    // address the access really uses (MASK / MODULO / CLAMP: fenced; CHECK / NONE: unchanged)
    __device__ __forceinline__ uint64_t addr(uint64_t a) const {
        if constexpr (MODE == kMask || MODE == kMaskCount) {
            return (a & keep) | base;
        } else if constexpr (MODE == kMaskBig) {      // a W-aligned (the call sites' vectors and tails)
            return addr_big(a);
        } else if constexpr (MODE == kModulo) {
            const uint64_t off = a - base;
#if GD_MODULO_FAST
            // an offset below 2 size (every access inside the partition, and
            // every one up to a partition past its end) needs one conditional
            // subtract; only the others take the reciprocal (exact either
            // way: the u64 remainder of A10)
            if (off < size2) return base + ((off >= size ? off - size : off) & ~(uint64_t)(W - 1));
#endif
            uint64_t r = off - __umul64hi(off, inv) * size;
            if (r >= size) r -= size;
            return base + (r & ~(uint64_t)(W - 1));
        } else if constexpr (MODE == kClamp) {
            const uint64_t down = a & ~(uint64_t)(W - 1);            // base is W-aligned
            return a < base ? base : (a - base > lim ? base + lim : down);
        } else {
            return a;
        }
    }
    // MODULO, strength-reduced along a walk known not to wrap (every address
    // of the walk on one side of base, so the u64 offsets a - base do not
    // cross 2^64 (A10), and d < size): the fence of a_prev + d / of
    // a_next - d from the fence of a_prev / a_next, one add and one select,
    // equal to addr() (the residues stay W-aligned when base, the addresses,
    // d and size are).
    __device__ __forceinline__ uint64_t step_up(uint64_t f_prev, uint64_t d) const {
        const uint64_t r = (f_prev - base) + d;
        return base + (r >= size ? r - size : r);
    }
    __device__ __forceinline__ uint64_t step_down(uint64_t f_next, uint64_t d) const {
        const uint64_t r = f_next - base;
        return base + (r >= d ? r - d : r + (size - d));
    }
    // the check predicate: every byte in the partition, a W-aligned
    __device__ __forceinline__ bool inside(uint64_t a) const {
        return (a - base) <= lim && (a & (uint64_t)(W - 1)) == 0;
    }
    // may the access be performed?
    __device__ __forceinline__ bool ok(uint64_t a) const {
        if constexpr (MODE == kCheck) return inside(a);
        else return true;
    }
    // ok(), and add k to the thread's count when the mode counts this access
    __device__ __forceinline__ bool go(uint64_t a, uint32_t &nv, uint32_t k) const {
        if constexpr (MODE == kCheck) {
            const bool o = inside(a);
            if (!o) nv += k;
            return o;
        } else if constexpr (counts(MODE)) {
            if (!inside(a)) nv += k;
            return true;
        } else {
            return true;
        }
    }
    // ok() / go() for an address the caller has proven W-aligned (aligned
    // operand bases and W-multiple strides): the alignment half of the test is known true
    __device__ __forceinline__ bool ok_aligned(uint64_t a) const {
        if constexpr (MODE == kCheck) return (a - base) <= lim;
        else return true;
    }
    __device__ __forceinline__ bool go_aligned(uint64_t a, uint32_t &nv, uint32_t k) const {
        if constexpr (MODE == kCheck) {
            const bool o = (a - base) <= lim;
            if (!o) nv += k;
            return o;
        } else if constexpr (counts(MODE)) {
            if ((a - base) > lim) nv += k;
            return true;
        } else {
            return true;
        }
    }
    // MASK / MASK_COUNT on a kBig partition (FenceDesc::flags: power of two,
    // >= 4 GiB, size-aligned, so base's low word is 0 and keep's low word is
    // all ones above the W alignment) for a W-aligned address: the fence
    // leaves the low word as it is, so it is one LOP3 on the high word --
    // equal to addr(a).  The high words of keep and base are the same for
    // every W, so the 4- and 16-byte fences of a kernel share their operands.
    __device__ __forceinline__ uint64_t addr_big(uint64_t a) const {
        const uint32_t hi = ((uint32_t)(a >> 32) & mask_hi) | (uint32_t)(base >> 32);
        return ((uint64_t)hi << 32) | (uint64_t)(uint32_t)a;
    }
    // inside(a) for an address the caller has proven W-aligned
    __device__ __forceinline__ bool ok_aligned_in(uint64_t a) const { return (a - base) <= lim; }
    // the same for a kBig partition (FenceDesc::flags): equal high bits
    __device__ __forceinline__ bool in_big(uint64_t a) const {
        return (((uint32_t)(a >> 32) ^ (uint32_t)(base >> 32)) & ~(uint32_t)((size - 1) >> 32)) == 0;
    }
    // CLAMP, for a 16-byte vector of four logical 4-byte elements wholly
    // outside the partition: the word every one of its elements clamps to
    __device__ __forceinline__ uint64_t edge4(uint64_t a) const { return a < base ? base : base + size - 4; }
};

// A 16-byte-aligned vector at a holding four logical 4-byte accesses
// (a, a+4, a+8, a+12).  Every mode but CLAMP fences it as one 16-byte access:
// with base and size multiples of 16 the vector is wholly inside or wholly
// outside the partition, and the mask / modulo fence of a+4k is F16(a)+4k.
// CLAMP sends all four elements of an outside vector to one edge word, so the
// vector is that word four times (a store keeps the last element, element
// order).  Counted 4 per vector.  LD16 / LD4 / ST16 / ST4 are the cache
// operators of the call site.  Precondition: a is 16-byte aligned (every
// call site indexes a 16-byte-aligned buffer in 16-byte steps; the API
// refuses misaligned buffers), so the alignment half of the check predicate
// is known true.
template <int MODE, typename LD16, typename LD4>
__device__ __forceinline__ uint4 vld4(const Fence<MODE, 16> &f, uint64_t a, uint32_t &nv, LD16 ld16, LD4 ld4) {
    if constexpr (MODE == kClamp) {
        if (f.ok_aligned_in(a)) return ld16(a);
        nv += 4;
        const uint32_t w = ld4(f.edge4(a));
        return make_uint4(w, w, w, w);
    } else {
        if (f.go_aligned(a, nv, 4)) return ld16(f.addr(a));
        return make_uint4(0, 0, 0, 0);
    }
}

// (ALIGNED = false: the alignment half of the predicate is tested anyway --
// identical results, a different register allocation; see k_gatherR)
template <int MODE, typename ST16, typename ST4, bool ALIGNED = true>
__device__ __forceinline__ void vst4(const Fence<MODE, 16> &f, uint64_t a, uint4 v, uint32_t &nv, ST16 st16,
                                     ST4 st4) {
    if constexpr (MODE == kClamp) {
        if (ALIGNED ? f.ok_aligned_in(a) : f.inside(a)) {
            st16(a, v);
        } else {
            nv += 4;
            st4(f.edge4(a), v.w);
        }
    } else {
        if (ALIGNED ? f.go_aligned(a, nv, 4) : f.go(a, nv, 4)) st16(f.addr(a), v);
    }
}

// Hoisting (R-hoist): true iff every byte of [a, a+len) lies in the
// partition (no 64-bit wraparound).  A CTA whose whole tile passes this test
// performs exactly the accesses the per-access check would allow (all of
// them), refuses and counts none, and every modulo / clamp / mask fence of it
// is the identity, so it may run the unfenced body; only tiles that touch or
// cross the partition edge pay for per-access fencing.
__device__ __forceinline__ bool range_in(const FenceDesc &fd, uint64_t a, uint64_t len) {
    const uint64_t off = a - fd.base;
    return !(fd.flags & kNoHoist) && len <= fd.size && off <= fd.size - len;
}

// Add the refusal counts of a warp to the trusted counter: nothing when no
// lane counted (the common case, one vote), else a warp reduction and one
// 64-bit atomic from lane 0 (warp-level aggregation of
// the violation counters).  No CTA-wide barrier, so warps that finish early
// are not held back.  Every lane of a full warp must call it (the per-thread
// counts are small: their warp sum fits 32 bits).
__device__ __forceinline__ void flush_violations(uint32_t nv_thread, unsigned long long *viol) {
    if (!__any_sync(0xffffffffu, nv_thread != 0)) return;
    const uint32_t s = __reduce_add_sync(0xffffffffu, nv_thread);
    if ((threadIdx.x & 31u) == 0) atomicAdd(viol, (unsigned long long)s);
}

// The CTA-wide variant (a barrier vote, a shared-memory reduction, one
// atomic per CTA), kept for the row gather: with it ptxas keeps every mode
// of k_gatherR inside 40 registers without local memory (6 CTAs per SM).
__device__ __forceinline__ void flush_violations_cta(uint32_t nv_thread, unsigned long long *viol) {
    if (!__syncthreads_or(nv_thread != 0)) return;
    __shared__ unsigned long long warp_sums[32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t s = __reduce_add_sync(0xffffffffu, nv_thread);
    if (lane == 0) warp_sums[warp] = s;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = (blockDim.x + 31u) >> 5;
        unsigned long long t = lane < nw ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0 && t) atomicAdd(viol, t);
    }
}

}  // namespace gd
