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

template <int MODE, int kG, bool WALK = false>
__device__ __forceinline__ void strip(const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t W, uint64_t pitch,
                                      float c0, float c1, uint64_t c, uint32_t r0, uint32_t r1, uint32_t &nv) {
    // row indices are 32-bit (H <= 2^19, api.cpp); addresses are 64-bit
    const Fence<MODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    bool interior[4];
    bool all4 = true;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        interior[k] = (c + k >= 1) && (c + k + 2 <= W);
        all4 = all4 && interior[k];
    }
    // refused-access weights (counting modes): the own vector of row x is
    // loaded by the interior points of row x as C (each), as W (k >= 1) and
    // as E (k <= 2), and by those of rows x-1 / x+1 as S / N (once each).
    // A refusal is counted when the vector is loaded, with the weight of the
    // strip rows [r0, r1) that use it, so no per-load flag stays live.
    uint32_t ni = 0, nCv = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        ni += interior[k];
        nCv += interior[k] * (1u + (k >= 1) + (k <= 2));
    }
    auto weight = [&](uint32_t x) {
        return ni * ((uint32_t)(x >= r0 + 1 && x <= r1) + (uint32_t)(x + 1 >= r0 && x + 1 < r1)) +
               nCv * (uint32_t)(x >= r0 && x < r1);
    };
    // modulo with WALK (the strip does not straddle the base and a row step
    // is below the partition size): the rows are loaded in increasing order,
    // so each vector's fence follows from the previous row's
    // (Fence::step_up), the W / E words of a row from the fence of the row
    // below it (step_down) and each output vector from the previous output
    // row's; every access still gets its own fenced address, equal to the
    // full modulo.  Without WALK every access takes the full modulo.
    uint64_t f_last = 0, fo_last = 0;
    // a clamped outside vector is its edge word four times (fence.cuh vld4)
    auto ldv = [&](uint32_t r) {
        const uint64_t a = in + 4 * ((uint64_t)r * pitch + c);
        if constexpr (MODE == kModulo && WALK) {
            f_last = r == r0 - 1 ? f16.addr(a) : f16.step_up(f_last, 4 * pitch);
            return __ldg(reinterpret_cast<const float4 *>(f_last));
        }
        const bool ok = counts(MODE) ? (a - f16.base) <= f16.lim : true;    // a is 16-aligned (API)
        if constexpr (counts(MODE)) nv += ok ? 0u : weight(r);
        if constexpr (MODE == kClamp) {
            if (ok) return __ldg(reinterpret_cast<const float4 *>(a));
            const float w = __ldg(reinterpret_cast<const float *>(f16.edge4(a)));
            return make_float4(w, w, w, w);
        } else if constexpr (MODE == kCheck) {
            // predicated: the destination is zeroed before the load, so
            // nothing consumes the loaded value until the stencil uses it
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) v = __ldg(reinterpret_cast<const float4 *>(a));
            return v;
        } else {
            return __ldg(reinterpret_cast<const float4 *>(f16.addr(a)));
        }
    };
    auto lds = [&](uint64_t e, uint64_t a_below) {     // one logical access of one point
        const uint64_t a = in + 4 * e;
        if constexpr (MODE == kModulo && WALK) {       // f_last: the fence of the vector of the row below
            return __ldg(reinterpret_cast<const float *>(f4.step_down(f_last, a_below - a)));
        }
        const bool ok = counts(MODE) ? (a - f4.base) <= f4.lim : true;      // a is 4-aligned
        if constexpr (counts(MODE)) nv += ok ? 0u : 1u;
        if constexpr (MODE == kCheck) {
            float v = 0.f;
            if (ok) v = __ldg(reinterpret_cast<const float *>(a));
            return v;
        } else {
            return __ldg(reinterpret_cast<const float *>(f4.addr(a)));
        }
    };
    float4 P = ldv(r0 - 1);
    float4 Cv = ldv(r0);
    for (uint32_t r = r0; r < r1; r += kG) {
        float4 S[kG];
        float wv[kG], ev[kG];
#pragma unroll
        for (int g = 0; g < kG; g++) {
            const uint32_t rr = r + g;
            S[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            wv[g] = ev[g] = 0.f;
            if (rr < r1) {
                S[g] = ldv(rr + 1);
                if (interior[0]) wv[g] = lds((uint64_t)rr * pitch + c - 1, in + 4 * ((uint64_t)(rr + 1) * pitch + c));
                if (interior[3]) ev[g] = lds((uint64_t)rr * pitch + c + 4, in + 4 * ((uint64_t)(rr + 1) * pitch + c));
            }
        }
#pragma unroll
        for (int g = 0; g < kG; g++) {
            const uint32_t rr = r + g;
            if (rr < r1) {
                const float4 N = (g == 0) ? P : ((g == 1) ? Cv : S[g >= 2 ? g - 2 : 0]);
                const float4 C = (g == 0) ? Cv : S[g >= 1 ? g - 1 : 0];
                const float cn[4] = {N.x, N.y, N.z, N.w};
                const float cc[4] = {C.x, C.y, C.z, C.w};
                const float cs[4] = {S[g].x, S[g].y, S[g].z, S[g].w};
                float o[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const float w = (k == 0) ? wv[g] : cc[k - 1];
                    const float e = (k == 3) ? ev[g] : cc[k + 1];
                    const float ns = __fadd_rn(cn[k], cs[k]);
                    const float we = __fadd_rn(w, e);
                    const float s = __fadd_rn(ns, we);
                    o[k] = __fmaf_rn(c1, s, __fmul_rn(c0, cc[k]));
                }
                const uint64_t ao = out + 4 * ((uint64_t)rr * pitch + c);
                if constexpr (MODE == kModulo && WALK) {
                    // F4(ao + 4k) = F16(ao) + 4k
                    fo_last = rr == r0 ? f16.addr(ao) : f16.step_up(fo_last, 4 * pitch);
                    if (all4) {
                        st_v(fo_last, make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                                                 __float_as_uint(o[3])));
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            if (interior[k]) *reinterpret_cast<float *>(fo_last + 4 * k) = o[k];
                    }
                } else if (all4) {
                    vst4(f16, ao,
                         make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                                    __float_as_uint(o[3])),
                         nv, st_v, st_w);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        if (!interior[k]) continue;
                        const uint64_t a = ao + 4 * k;
                        if (f4.go(a, nv, 1)) *reinterpret_cast<float *>(f4.addr(a)) = o[k];
                    }
                }
            }
        }
        // slide the window: rows r+kG-1 (new P) and r+kG (new C)
        if constexpr (kG >= 2) P = S[kG - 2];
        else P = Cv;
        Cv = S[kG - 1];
    }
}

// ROWS (rows per CTA strip) is a compile-time constant: 16-row strips at HBM
// sizes (the 2-row halo re-reads hit L2; measured 8 / 16 / 32 / 64 / 128 rows:
// 6.5 / 6.8 / 6.5 / 6.4 / 6.36 TB/s), 8 rows when that leaves fewer than 4
// CTAs per SM (L2-resident sizes); as a constant it also keeps the fenced
// variants (hoisted body + per-access body) inside 64 registers with no
// local memory.
template <int MODE, int ROWS>
__global__ void __launch_bounds__(kThreads, 4) k_stencil(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                         uint64_t in, uint32_t H, uint32_t W, uint64_t pitch,
                                                         float c0, float c1) {
    uint32_t nv = 0;
    const uint64_t c = 4ull * ((uint64_t)blockIdx.x * kThreads + threadIdx.x);
    const uint32_t r0 = 1u + blockIdx.y * (uint32_t)ROWS;
    const uint32_t r1 = (r0 + ROWS < H - 1) ? r0 + ROWS : H - 1;
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
            if (c < W && r0 < r1) strip<kNone, 4>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
            return;
        }
        if (c < W && r0 < r1) strip<MODE, 1>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    } else {
        if (c < W && r0 < r1) strip<MODE, 4>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
    }
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
}

// Per-access fencing (fd.flags & kNoHoist, GD_CHECK_PER_ACCESS=1, the
// paper's instrumentation): no range test, every strip runs the fenced body
// with 4 rows of loads in flight, inside 64 registers in every mode (the
// hoisted kernel's edge body keeps one row in flight next to its unfenced
// body).
template <int MODE, int ROWS>
__global__ void __launch_bounds__(kThreads, 4) k_stencil_pa(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                            uint64_t in, uint32_t H, uint32_t W, uint64_t pitch,
                                                            float c0, float c1) {
    uint32_t nv = 0;
    const uint64_t c = 4ull * ((uint64_t)blockIdx.x * kThreads + threadIdx.x);
    const uint32_t r0 = 1u + blockIdx.y * (uint32_t)ROWS;
    const uint32_t r1 = (r0 + ROWS < H - 1) ? r0 + ROWS : H - 1;
    if (c < W && r0 < r1) {
        if constexpr (MODE == kModulo) {
            // the walk recurrence holds when no operand range of the strip
            // straddles the base (the u64 offsets do not wrap) and a row step
            // is below the partition size
            const uint64_t lo_in = in + 4 * ((r0 - 1) * pitch + c) - (c ? 4 : 0);
            const uint64_t hi_in = in + 4 * (r1 * pitch + c + 5);
            const uint64_t lo_out = out + 4 * (r0 * pitch + c), hi_out = out + 4 * ((r1 - 1) * pitch + c + 4);
            const auto side = [&](uint64_t lo, uint64_t hi) { return lo <= hi && (hi <= fd.base || lo >= fd.base); };
            if (4 * pitch < fd.size && side(lo_in, hi_in) && side(lo_out, hi_out))
                strip<MODE, 4, true>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
            else
                strip<MODE, 4>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
        } else {
            strip<MODE, 4>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
        }
    }
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
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
        const dim3 grid((unsigned)gx, (unsigned)((H - 2ull + 7) / 8));
        if (pa) k_stencil_pa<MODE, 8><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
        else k_stencil<MODE, 8><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
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
