// k_stencil.cu -- fenced 2-D 5-point Jacobi sweep for
// sm_100a.
//
// out[r][c] = fmaf(c1, (N + S) + (W + E), c0 * C) over interior points, fp32,
// every operation rounded as written.
//
// Layout: each thread owns a 4-column vector (16 bytes) of a column strip and
// walks kRows rows of it, keeping the rows above / at / below in registers and
// loading G new rows per step (G 128-bit loads in flight).  The west / east
// neighbours that fall outside the thread's vector are 32-bit loads (L1
// hits: the neighbouring lanes load the same lines).  Every physical access
// is fenced at its own width; the values a point uses are exactly the values
// its five logical loads would read (a 16-byte-aligned vector is wholly
// inside or wholly outside a pow2 partition, and F(a+4k,4) = F(a,16)+4k).
// Refusals / detections are counted per logical access: 5 loads + 1 store per
// interior point, as in the oracle, each when its load is issued (with the
// number of strip points that use the loaded vector).  The hoistable modes
// (check, modulo, mask-count, clamp) take one conservative range test per
// thread strip (fence.cuh range_in): strips wholly inside the partition run
// the unfenced body, the rest the per-access fenced body.  With hoisting off
// (GD_CHECK_PER_ACCESS=1) k_stencil_pa fences every access of every strip.
#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kRows = 16;     // rows per CTA strip (a multiple of the rows loaded per step)

__device__ __forceinline__ void st_v(uint64_t a, uint4 v) { __stcs(reinterpret_cast<uint4 *>(a), v); }
__device__ __forceinline__ void st_w(uint64_t a, uint32_t v) { __stcs(reinterpret_cast<unsigned int *>(a), v); }

// One thread's strip: rows [r0, r1) of the 4-column vector at column c
// (r1 - r0 <= ROWS), kG rows of loads in flight.  FULL: r1 - r0 == ROWS and
// every lane of the warp holds four interior points (the common case: no
// row guards, one 16-byte store per row).  The row loop is unrolled at
// compile time, addresses advance by one row pitch per row, and every
// access is fenced at its own address.
template <int MODE, int kG, int ROWS, bool FULL, bool WALK = false, bool BIG = false>
__device__ __forceinline__ void strip(const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t W, uint64_t pitch,
                                      float c0, float c1, uint64_t c, uint32_t r0, uint32_t r1, uint32_t &nv) {
    static_assert(ROWS % kG == 0 && ROWS + 2 <= 32, "strip rows");
    // Every lane of the warp runs this (the W / E words travel by shuffle):
    // a lane past the grid's width (c >= W) loads nothing and stores nothing.
    const Fence<MODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    // the mask fence of a 16- / 4-aligned address (BIG: one LOP3, Fence::addr_big)
    constexpr bool kMaskBig = BIG && (MODE == kMask || MODE == kMaskCount);
    // MASK on a kBig partition walks fenced pointers: F(F(a) + s) = F(a + s)
    // for the mask fence (the low words and the carry out of them are the
    // same, and base's bits lie above the mask's), so a row's fenced address
    // is the previous row's plus the row step, fenced in place (adv: one LOP3
    // and no copy of the unfenced pointer); fa16 / fa4 are then the identity
#ifndef GD_STENCIL_MASK_WALK
#define GD_STENCIL_MASK_WALK 1
#endif
    constexpr bool kMaskWalk = BIG && MODE == kMask && GD_STENCIL_MASK_WALK;
    auto fa16 = [&](uint64_t a) { return kMaskWalk ? a : kMaskBig ? f16.addr_big(a) : f16.addr(a); };
    auto fa4 = [&](uint64_t a) { return kMaskWalk ? a : kMaskBig ? f4.addr_big(a) : f4.addr(a); };
    // CHECK on a kBig partition: every load is issued, unpredicated, at its
    // mask-fenced address (inside the tenant's own partition), and a refused
    // load's value is replaced by 0 after its batch of loads (zerofix below,
    // the rare path): the values used are exactly the check fence's (refused
    // -> 0) and nothing outside the partition is read.  A predicated load ties
    // each destination to a zeroing move and let ptxas start the next batch
    // only after the previous one was consumed (ncu: +8 % time at 32768^2).
#ifndef GD_STENCIL_CHECK_MASKED
#define GD_STENCIL_CHECK_MASKED 1
#endif
    // (16-row strips, the HBM-size grids; at the L2-resident size's 8-row
    // strips the predicated form measured faster: +17 % vs +29 % per access)
    constexpr bool kCheckMasked = BIG && MODE == kCheck && ROWS >= 16 && GD_STENCIL_CHECK_MASKED;
    const uint32_t lane = threadIdx.x & 31u;
#ifndef GD_STENCIL_FULL_WARP
#define GD_STENCIL_FULL_WARP 1
#endif
    const bool active = (FULL && GD_STENCIL_FULL_WARP) || c < W;
    bool interior[4];
    bool all4 = true;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        interior[k] = (c + k >= 1) && (c + k + 2 <= W);
        all4 = all4 && interior[k];
    }
    const bool all4a = (FULL && GD_STENCIL_FULL_WARP) || all4;   // (all four interior implies c < W)
    // The W word of point k = 0 (column c-1) is word 3 of lane-1's vector of
    // the same row, the E word of point k = 3 (column c+4) word 0 of
    // lane+1's: F4(a-4) = F16(a-16)+12 and F4(a+16) = F16(a+16) in every
    // mode (base and size multiples of 16), a word is refused exactly when
    // its vector is, and a clamped outside vector is its edge word four
    // times, so the shuffled word is the value the point's own fenced 32-bit
    // load would return.  Only the warp's edge lanes load their halo word
    // (lane 0: column c-1, lane 31: column c+4), fenced at 4 bytes.
    const bool need_h = lane == 0 ? interior[0] : (lane == 31 ? interior[3] : false);
    // lane 0 / lane 31 take the halo word instead of the shuffled one; as
    // bit masks in general registers (one LOP3 each), not live predicates
    const uint32_t m0 = lane == 0 ? ~0u : 0u, m31 = lane == 31 ? ~0u : 0u;
    const uint64_t step = 4 * pitch;
    // A lane past the width loads the last vector of the row instead (never
    // used: a point needs lane+1's word only when lane+1 is inside the
    // width), so no load waits on a lane predicate; it stores nothing and
    // counts nothing (its weights below are zero).
    const uint64_t cl = active ? c : ((uint64_t)(W - 1) & ~3ull);
    uint64_t pv = in + 4 * ((uint64_t)(r0 - 1) * pitch + cl);                 // vector of row r0 - 1
    uint64_t ph = in + 4 * ((uint64_t)r0 * pitch + (lane == 0 ? c - 1 : c + 4));   // halo word of row r0
    uint64_t po = out + 4 * ((uint64_t)r0 * pitch + c);                       // output vector of row r0
    if constexpr (kMaskWalk) {
        pv = f16.addr_big(pv);
        ph = f16.addr_big(ph);
        po = f16.addr_big(po);
    }
    auto adv = [&](uint64_t &p) {                      // the pointer of the next row
        p += step;
        if constexpr (kMaskWalk) p = f16.addr_big(p);
    };
    // counting modes: bit b of refm = the vector of row r0 - 1 + b lies
    // outside the partition (one predicated OR per load, the bit a
    // compile-time constant); its refused logical accesses are weighted
    // after the loop by the points that use it (see below)
    uint32_t refm = 0;
    // modulo with WALK (no lane's strip straddles the base and a row step
    // is below the partition size): each vector's fence follows from the
    // previous row's (Fence::step_up), an edge lane's halo word from the
    // fence of the vector of the row below it (step_down) and each output
    // vector from the previous output row's; every access still gets its own
    // fenced address, equal to the full modulo.
    uint64_t fv = 0, fo = 0;
    auto ldv = [&](int b) {                            // the vector of row r0 - 1 + b, at pv
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (MODE == kModulo && WALK) {
            fv = b == 0 ? f16.addr(pv) : f16.step_up(fv, step);
            v = __ldg(reinterpret_cast<const float4 *>(fv));
        } else if constexpr (counts(MODE)) {
            const bool ok = BIG ? f16.in_big(pv) : (pv - f16.base) <= f16.lim;   // pv is 16-aligned (API)
            if (!ok) refm |= 1u << b;
            if constexpr (kCheckMasked) {
                v = __ldg(reinterpret_cast<const float4 *>(f16.addr_big(pv)));
            } else if constexpr (MODE == kCheck || MODE == kClamp) {
                // predicated: the destination is zeroed before the load (clamp:
                // an outside vector is fixed up after its batch of loads, clampfix).
                // (Reading a refused vector from the trusted zero block instead,
                // Fence::ld_at, measured 25 % slower per access at 32768^2.)
                if (ok) v = __ldg(reinterpret_cast<const float4 *>(pv));
            } else {
                v = __ldg(reinterpret_cast<const float4 *>(fa16(pv)));
            }
        } else {
            v = __ldg(reinterpret_cast<const float4 *>(fa16(pv)));
        }
        return v;
    };
    uint32_t hrefm = 0;                                // clamp / kCheckMasked: bit x of a halo word of row r0 + x outside
    auto ldh = [&](int hb) {                           // an edge lane's halo word of row r0 + hb, at ph (pv: the row below)
        float v = 0.f;
        if constexpr (MODE == kModulo && WALK) {
            if (need_h) v = __ldg(reinterpret_cast<const float *>(f4.step_down(fv, pv - ph)));
        } else if constexpr (counts(MODE)) {
            const uint64_t fh = fa4(ph);
            const bool ok = MODE == kMaskCount ? fh == ph : BIG ? f4.in_big(ph) : (ph - f4.base) <= f4.lim;
            if (need_h && !ok) nv++;
            if constexpr (MODE == kClamp || kCheckMasked) {
                if (need_h && !ok) hrefm |= 1u << hb;
            }
            if constexpr (kCheckMasked) {
                if (need_h) v = __ldg(reinterpret_cast<const float *>(f4.addr_big(ph)));
            } else if constexpr (MODE == kCheck || MODE == kClamp) {
                if (need_h && ok) v = __ldg(reinterpret_cast<const float *>(ph));
            } else {
                if (need_h) v = __ldg(reinterpret_cast<const float *>(fh));
            }
        } else {
            if (need_h) v = __ldg(reinterpret_cast<const float *>(fa4(ph)));
        }
        return v;
    };
    // clamp: an outside vector at a is its edge word four times (fence.cuh vld4)
    auto clampfix = [&](uint64_t a) {
        const float w = __ldg(reinterpret_cast<const float *>(f16.edge4(a)));
        return make_float4(w, w, w, w);
    };
    auto stv = [&](int row, const float (&o)[4]) {    // the output vector at po
        if constexpr (MODE == kModulo && WALK) {
            fo = row == 0 ? f16.addr(po) : f16.step_up(fo, step);             // F4(po + 4k) = F16(po) + 4k
            if (all4) {
                st_v(fo, make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                                    __float_as_uint(o[3])));
            } else {
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (interior[k]) *reinterpret_cast<float *>(fo + 4 * k) = o[k];
            }
        } else if (all4a) {                            // the common case: one 16-byte store
            const uint4 val = make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                                         __float_as_uint(o[3]));
            if constexpr (MODE == kMaskCount) {
                const uint64_t f = fa16(po);
                nv += f != po ? 4u : 0u;                // inside iff the fence is the identity
                st_v(f, val);
            } else if constexpr (MODE == kClamp) {     // (fence.cuh vst4, po 16-aligned)
                if (BIG ? f16.in_big(po) : (po - f16.base) <= f16.lim) {
                    st_v(po, val);
                } else {                               // rare: the last element wins the edge word
                    nv += 4;
                    st_w(f16.edge4(po), val.w);
                }
            } else {
                const bool ok = BIG ? f16.in_big(po) : (po - f16.base) <= f16.lim;    // po is 16-aligned
                if (counts(MODE) && !ok) nv += 4;
                if (MODE != kCheck || ok) st_v(fa16(po), val);
            }
        } else if (active) {                           // the grid's first / last columns
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (!interior[k]) continue;
                const uint64_t a = po + 4 * k;
                if (f4.go_aligned(a, nv, 1)) *reinterpret_cast<float *>(f4.addr(a)) = o[k];   // a is 4-aligned
            }
        }
    };
    float4 P = ldv(0);
    adv(pv);
    float4 Cv = ldv(1);
    adv(pv);
    if constexpr (MODE == kClamp) {
        if (refm & 1u) P = clampfix(pv - 2 * step);
        if (refm & 2u) Cv = clampfix(pv - step);
    }
    if constexpr (kCheckMasked) {
        if (refm & 1u) P = make_float4(0.f, 0.f, 0.f, 0.f);
        if (refm & 2u) Cv = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < ROWS; i += kG) {
        if (!FULL && r0 + i >= r1) break;              // uniform over the CTA
        float4 S[kG];
        float hv[kG];
#pragma unroll
        for (int g = 0; g < kG; g++) {
            S[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            hv[g] = 0.f;
            if (FULL || r0 + i + g < r1) {
                S[g] = ldv(i + g + 2);
                hv[g] = ldh(i + g);
                adv(pv);
                adv(ph);
            }
        }
        if constexpr (kCheckMasked) {                  // rare: refused loads of this batch read 0
            const uint32_t rows = (1u << kG) - 1u;
            if (((refm >> (i + 2)) & rows) | ((hrefm >> i) & rows)) {
#pragma unroll
                for (int g = 0; g < kG; g++) {
                    if (refm & (1u << (i + g + 2))) S[g] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (hrefm & (1u << (i + g))) hv[g] = 0.f;
                }
            }
        }
        if constexpr (MODE == kClamp) {                // rare: outside accesses of this batch, after its loads
            const uint32_t rows = (1u << kG) - 1u;
            if (((refm >> (i + 2)) & rows) | ((hrefm >> i) & rows)) {
#pragma unroll
                for (int g = 0; g < kG; g++) {
                    if (!(FULL || r0 + i + g < r1)) continue;
                    if (refm & (1u << (i + g + 2))) S[g] = clampfix(pv - (uint64_t)(kG - g) * step);
                    if (hrefm & (1u << (i + g))) {
                        const uint64_t a = ph - (uint64_t)(kG - g) * step;
                        hv[g] = __ldg(reinterpret_cast<const float *>(f4.addr(a)));
                    }
                }
            }
        }
#pragma unroll
        for (int g = 0; g < kG; g++) {
            if (FULL || r0 + i + g < r1) {
                const float4 N = (g == 0) ? P : ((g == 1) ? Cv : S[g >= 2 ? g - 2 : 0]);
                const float4 C = (g == 0) ? Cv : S[g >= 1 ? g - 1 : 0];
                const float wl = __shfl_up_sync(0xffffffffu, C.w, 1);
                const float er = __shfl_down_sync(0xffffffffu, C.x, 1);
                const float cn[4] = {N.x, N.y, N.z, N.w};
                const float cc[4] = {C.x, C.y, C.z, C.w};
                const float cs[4] = {S[g].x, S[g].y, S[g].z, S[g].w};
                float o[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const float w = (k == 0) ? __uint_as_float((__float_as_uint(wl) & ~m0) | (__float_as_uint(hv[g]) & m0))
                                             : cc[k - 1];
                    const float e = (k == 3) ? __uint_as_float((__float_as_uint(er) & ~m31) | (__float_as_uint(hv[g]) & m31))
                                             : cc[k + 1];
                    const float ns = __fadd_rn(cn[k], cs[k]);
                    const float we = __fadd_rn(w, e);
                    const float s = __fadd_rn(ns, we);
                    o[k] = __fmaf_rn(c1, s, __fmul_rn(c0, cc[k]));
                }
                stv(i + g, o);
                adv(po);
            }
        }
        // slide the window: rows r+kG-1 (new P) and r+kG (new C)
        if constexpr (kG >= 2) P = S[kG - 2];
        else P = Cv;
        Cv = S[kG - 1];
    }
    if constexpr (counts(MODE) && !(MODE == kModulo && WALK)) {
        // the vector of row x = r0 - 1 + b is loaded by the interior points of
        // row x + 1 as N (bits 0 .. n-1), of row x as C (each), W (k >= 1), E
        // (k <= 2), and as lane+1's W / lane-1's E within the warp (bits
        // 1 .. n), of row x - 1 as S (bits 2 .. n+1), n = r1 - r0 rows
        if (refm) {
            uint32_t ni = 0, nCv = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                ni += interior[k];
                nCv += interior[k] * (1u + (k >= 1) + (k <= 2));
            }
            nCv += (uint32_t)(lane < 31 && c + 6 <= W) + (uint32_t)(lane > 0 && active);
            const uint32_t m = (1u << (r1 - r0)) - 1u;
            nv += ni * (__popc(refm & m) + __popc(refm & (m << 2))) + nCv * __popc(refm & (m << 1));
        }
    }
}

// The strip of a warp's rows: full (ROWS rows, every lane interior: the common
// case) or not (the grid's last rows, its first / last columns).  Full strips
// on a kBig partition take the BIG variant (one-LOP3 partition test and mask
// fence), except mask-count: with 16-row strips ptxas spills at 64
// registers, and with 8-row strips it measured no faster (L2-resident 2048^2
// per access +23.9 % vs +22.6 %, tools/r02_iter14.sh; knob kept for A/B).
#ifndef GD_STENCIL_MC_BIG8
#define GD_STENCIL_MC_BIG8 0
#endif
template <int MODE, int kG, int ROWS, bool WALK = false>
__device__ __forceinline__ void strip_rows(const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t W,
                                           uint64_t pitch, float c0, float c1, uint64_t c, uint32_t r0, uint32_t r1,
                                           uint32_t &nv) {
    if (r1 - r0 == ROWS && (!GD_STENCIL_FULL_WARP || __all_sync(0xffffffffu, c >= 1 && c + 5 <= W))) {
        if (((counts(MODE) && (MODE != kMaskCount || (GD_STENCIL_MC_BIG8 && ROWS <= 8))) || MODE == kMask) && (fd.flags & kBig))
            strip<MODE, kG, ROWS, true, WALK, true>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
        else
            strip<MODE, kG, ROWS, true, WALK>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    } else {
        strip<MODE, kG, ROWS, false, WALK>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    }
}

// ROWS (rows per CTA strip) is a compile-time constant: 16-row strips at HBM
// sizes (the 2-row halo re-reads hit L2; measured 8 / 16 / 32 / 64 / 128 rows:
// 6.5 / 6.8 / 6.5 / 6.4 / 6.36 TB/s), 8 rows when that leaves fewer than 4
// CTAs per SM (L2-resident sizes); the row loop unrolls over it.
template <int MODE, int ROWS>
__global__ void __launch_bounds__(kThreads, 4) k_stencil(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                         uint64_t in, uint32_t H, uint32_t W, uint64_t pitch,
                                                         float c0, float c1) {
    uint32_t nv = 0;
    const uint64_t c = 4ull * ((uint64_t)blockIdx.x * kThreads + threadIdx.x);
    const uint32_t r0 = 1u + blockIdx.y * (uint32_t)ROWS;
    const uint32_t r1 = (r0 + ROWS < H - 1) ? r0 + ROWS : H - 1;
    if (r0 >= r1) return;                              // uniform over the CTA
    if constexpr (hoistable(MODE)) {
        // conservative extents of everything the CTA's strip touches (from
        // blockIdx only, so the test runs on the uniform datapath); inside the
        // partition the fence is the identity and nothing is counted, so the
        // whole CTA runs the unfenced body and skips the violation flush
        const uint64_t cb = 4ull * blockIdx.x * kThreads, ce = cb + 4ull * kThreads;
        const uint64_t lo_in = in + 4 * ((r0 - 1) * pitch + cb) - (cb ? 4 : 0);
        const uint64_t hi_in = in + 4 * (r1 * pitch + ce + 1);
        const uint64_t lo_out = out + 4 * (r0 * pitch + cb), hi_out = out + 4 * ((r1 - 1) * pitch + ce);
        if (lo_in < hi_in && lo_out < hi_out && range_in(fd, lo_in, hi_in - lo_in) &&
            range_in(fd, lo_out, hi_out - lo_out)) {
            strip_rows<kNone, 4, ROWS>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
            return;
        }
        strip<MODE, 1, ROWS, false>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    } else {
        strip_rows<MODE, 4, ROWS>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    }
#ifdef GD_STENCIL_CTA_FLUSH
    if constexpr (counts(MODE)) flush_violations_cta(nv, fd.viol);
#else
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
#endif
}

// Per-access fencing (GD_FENCE_PER_ACCESS, fd.flags & kNoHoist, the paper's
// instrumentation): no range test, every strip runs the fenced body with 4
// rows of loads in flight.
template <int MODE, int ROWS>
__global__ void __launch_bounds__(kThreads, 4) k_stencil_pa(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                            uint64_t in, uint32_t H, uint32_t W, uint64_t pitch,
                                                            float c0, float c1) {
    uint32_t nv = 0;
    const uint64_t c = 4ull * ((uint64_t)blockIdx.x * kThreads + threadIdx.x);
    const uint32_t r0 = 1u + blockIdx.y * (uint32_t)ROWS;
    const uint32_t r1 = (r0 + ROWS < H - 1) ? r0 + ROWS : H - 1;
    if (r0 >= r1) return;                              // uniform over the CTA
    if constexpr (MODE == kModulo) {
        // the walk recurrence holds when no operand range of the strip
        // straddles the base (the u64 offsets do not wrap) and a row step is
        // below the partition size; decided for the whole warp (shuffles)
        // (a lane past the width walks the loads of the row's last vector)
        const uint64_t cl = c < W ? c : ((uint64_t)(W - 1) & ~3ull);
        const uint64_t lo_in = in + 4 * ((r0 - 1) * pitch + cl) - (cl ? 4 : 0);
        const uint64_t hi_in = in + 4 * (r1 * pitch + cl + 5);
        const uint64_t lo_out = out + 4 * (r0 * pitch + cl), hi_out = out + 4 * ((r1 - 1) * pitch + cl + 4);
        const auto side = [&](uint64_t lo, uint64_t hi) { return lo <= hi && (hi <= fd.base || lo >= fd.base); };
        const bool walk = 4 * pitch < fd.size && side(lo_in, hi_in) && side(lo_out, hi_out);
        if (__all_sync(0xffffffffu, walk))
            strip_rows<MODE, 4, ROWS, true>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
        else
            strip<MODE, 4, ROWS, false>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    } else {
        strip_rows<MODE, 4, ROWS>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    }
#ifdef GD_STENCIL_CTA_FLUSH
    if constexpr (counts(MODE)) flush_violations_cta(nv, fd.viol);
#else
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
#endif
}

template <int MODE>
cudaError_t stencil_t(const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t H, uint32_t W, uint64_t pitch,
                      float c0, float c1, cudaStream_t s, int sms) {
    const uint64_t nvec = (W + 3ull) / 4, gx = (nvec + kThreads - 1) / kThreads;
    // long strips unless that leaves fewer than 4 CTAs per SM
    const bool pa = hoistable(MODE) && (fd.flags & kNoHoist);
    if (gx * ((H - 2ull + kRows - 1) / kRows) >= 4ull * (uint64_t)sms) {
        const dim3 grid((unsigned)gx, (unsigned)((H - 2ull + kRows - 1) / kRows));
        if (pa) k_stencil_pa<MODE, kRows><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
        else k_stencil<MODE, kRows><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
    } else {
#ifndef GD_STENCIL_SMALL_ROWS
#define GD_STENCIL_SMALL_ROWS 8
#endif
        constexpr int kSmall = GD_STENCIL_SMALL_ROWS;
        const dim3 grid((unsigned)gx, (unsigned)((H - 2ull + kSmall - 1) / kSmall));
        if (pa) k_stencil_pa<MODE, kSmall><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
        else k_stencil<MODE, kSmall><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stencil(int mode, const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                           uint64_t pitch, float c0, float c1, cudaStream_t s, const Geom &g) {
    if (H < 3 || W < 3) return cudaSuccess;        // no interior point
    switch (mode) {
        case kNone: return stencil_t<kNone>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
        case kMask: return stencil_t<kMask>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
        case kModulo: return stencil_t<kModulo>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
        case kMaskCount: return stencil_t<kMaskCount>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
        case kClamp: return stencil_t<kClamp>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
        default: return stencil_t<kCheck>(fd, out, in, H, W, pitch, c0, c1, s, g.sms);
    }
}

}  // namespace gd
