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
// interior point, as in the oracle.  The hoistable modes (check, modulo,
// mask-count, clamp) take one conservative range test per thread strip
// (fence.cuh range_in): strips wholly inside the partition run the unfenced
// body, the rest the per-access fenced body.
#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kRows = 16;     // rows per CTA strip (a multiple of the rows loaded per step)

__device__ __forceinline__ void st_v(uint64_t a, uint4 v) { __stcs(reinterpret_cast<uint4 *>(a), v); }
__device__ __forceinline__ void st_w(uint64_t a, uint32_t v) { __stcs(reinterpret_cast<unsigned int *>(a), v); }

template <int MODE, int kG>
__device__ __forceinline__ void strip(const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t W, uint64_t pitch,
                                      float c0, float c1, uint64_t c, uint64_t r0, uint64_t r1, uint32_t &nv) {
    const Fence<MODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    bool interior[4];
    bool all4 = true;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        interior[k] = (c + k >= 1) && (c + k + 2 <= W);
        all4 = all4 && interior[k];
    }
    // refused-access weights (check mode): loads of the own vector used by
    // the interior points as C (each), as W (k >= 1) and as E (k <= 2)
    uint32_t ni = 0, nCv = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        ni += interior[k];
        nCv += interior[k] * (1u + (k >= 1) + (k <= 2));
    }
    // ok = the vector's / word's accesses are not counted (check: performed);
    // a clamped outside vector is its edge word four times (fence.cuh vld4)
    auto ldv = [&](uint64_t r, bool &ok) {
        const uint64_t a = in + 4 * (r * pitch + c);
        ok = counts(MODE) ? f16.inside(a) : true;
        if constexpr (MODE == kClamp) {
            if (ok) return __ldg(reinterpret_cast<const float4 *>(a));
            const float w = __ldg(reinterpret_cast<const float *>(f16.edge4(a)));
            return make_float4(w, w, w, w);
        } else {
            return f16.ok(a) ? __ldg(reinterpret_cast<const float4 *>(f16.addr(a))) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto lds = [&](uint64_t e, bool &ok) {
        const uint64_t a = in + 4 * e;
        ok = counts(MODE) ? f4.inside(a) : true;
        return f4.ok(a) ? __ldg(reinterpret_cast<const float *>(f4.addr(a))) : 0.f;
    };
    bool okP, okC;
    float4 P = ldv(r0 - 1, okP);
    float4 Cv = ldv(r0, okC);
    for (uint64_t r = r0; r < r1; r += kG) {
        float4 S[kG];
        bool okS[kG];
        float wv[kG], ev[kG];
        bool okW[kG], okE[kG];
#pragma unroll
        for (int g = 0; g < kG; g++) {
            const uint64_t rr = r + g;
            okS[g] = okW[g] = okE[g] = true;
            S[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            wv[g] = ev[g] = 0.f;
            if (rr < r1) {
                S[g] = ldv(rr + 1, okS[g]);
                if (interior[0]) wv[g] = lds(rr * pitch + c - 1, okW[g]);
                if (interior[3]) ev[g] = lds(rr * pitch + c + 4, okE[g]);
            }
        }
#pragma unroll
        for (int g = 0; g < kG; g++) {
            const uint64_t rr = r + g;
            if (rr < r1) {
                const float4 N = (g == 0) ? P : ((g == 1) ? Cv : S[g >= 2 ? g - 2 : 0]);
                const float4 C = (g == 0) ? Cv : S[g >= 1 ? g - 1 : 0];
                const bool okN = (g == 0) ? okP : ((g == 1) ? okC : okS[g >= 2 ? g - 2 : 0]);
                const bool okCC = (g == 0) ? okC : okS[g >= 1 ? g - 1 : 0];
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
                if constexpr (counts(MODE)) {
                    // per interior point: N, S, C loads; W from the own vector
                    // unless k == 0; E from the own vector unless k == 3
                    nv += ni * ((uint32_t)!okN + (uint32_t)!okS[g]) + nCv * (uint32_t)!okCC +
                          (uint32_t)!okW[g] + (uint32_t)!okE[g];
                }
                const uint64_t ao = out + 4 * (rr * pitch + c);
                if (all4) {
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
        if constexpr (kG >= 2) {
            P = S[kG - 2];
            okP = okS[kG - 2];
        } else {
            P = Cv;
            okP = okC;
        }
        Cv = S[kG - 1];
        okC = okS[kG - 1];
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
    constexpr uint64_t rows = ROWS;
    uint32_t nv = 0;
    const uint64_t c = 4ull * ((uint64_t)blockIdx.x * kThreads + threadIdx.x);
    const uint64_t r0 = 1ull + (uint64_t)blockIdx.y * rows;
    const uint64_t r1 = (r0 + rows < (uint64_t)H - 1) ? r0 + rows : (uint64_t)H - 1;
    if (c < W && r0 < r1) {
        if constexpr (hoistable(MODE)) {
            // conservative extents of everything this strip touches; inside the
            // partition the fence is the identity and nothing is counted
            const uint64_t lo_in = in + 4 * ((r0 - 1) * pitch + c) - (c ? 4 : 0);
            const uint64_t hi_in = in + 4 * (r1 * pitch + c + 5);
            const uint64_t lo_out = out + 4 * (r0 * pitch + c), hi_out = out + 4 * ((r1 - 1) * pitch + c + 4);
            if (lo_in < hi_in && lo_out < hi_out && range_in(fd, lo_in, hi_in - lo_in) &&
                range_in(fd, lo_out, hi_out - lo_out))
                strip<kNone, 4>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
            else
                strip<MODE, 1>(fd, out, in, W, pitch, c0, c1, c, r0, r1, nv);
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
    if (gx * ((H - 2ull + kRows - 1) / kRows) >= 4ull * (uint64_t)sms) {
        const dim3 grid((unsigned)gx, (unsigned)((H - 2ull + kRows - 1) / kRows));
        k_stencil<MODE, kRows><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
    } else {
        const dim3 grid((unsigned)gx, (unsigned)((H - 2ull + 7) / 8));
        k_stencil<MODE, 8><<<grid, kThreads, 0, s>>>(fd, out, in, H, W, pitch, c0, c1);
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
