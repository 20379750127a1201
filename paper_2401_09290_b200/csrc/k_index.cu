// k_index.cu -- fenced embedding-style gather / scatter-add (SURVEY.md §2.7
// K3, K4) for sm_100a.
//
// The effective address of every indexed access is materialised first
// (table + 4 * sext(j), Listing 1 lines 20-23 `mul.wide.s32` + `add.s64`,
// PAPER.md:206-209) and only then fenced (second addressing
// mode) -- the fence never sees a partial address.
//
// D = 1 path: each CTA owns a contiguous chunk of kThreads x kU index
// vectors; per thread kU 128-bit index loads, then 4 kU independent fenced
// random 32-bit table loads (L1-bypassing, sector-granular), then kU 128-bit
// output stores.  In check mode the index and output streams are range-tested
// once per CTA chunk (fence.cuh range_in); the random table accesses are
// checked one by one.  D > 1 path: one warp per index row, lanes stride over
// the row; lane 0 loads the index once (one logical access, as in the
// oracle) and broadcasts it.
#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kU = 4;
constexpr uint64_t kChunk = (uint64_t)kThreads * kU;   // index vectors per CTA

__device__ __forceinline__ int4 ld_idx(uint64_t a) { return __ldcs(reinterpret_cast<const int4 *>(a)); }
__device__ __forceinline__ uint4 ld_u4(uint64_t a) { return __ldcs(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ uint32_t ld_tab(uint64_t a) { return __ldcg(reinterpret_cast<const uint32_t *>(a)); }
__device__ __forceinline__ void st_out(uint64_t a, uint4 v) { __stcs(reinterpret_cast<uint4 *>(a), v); }

__device__ __forceinline__ uint64_t row_addr(uint64_t table, int32_t j) {
    return table + (uint64_t)((int64_t)j * 4);        // sext, scale in 64 bits
}

template <int MODE>
__device__ __forceinline__ uint32_t fenced_tab(const Fence<MODE, 4> &f4, uint64_t table, int32_t j, uint32_t &nv) {
    const uint64_t a = row_addr(table, j);
    if (f4.ok(a)) return ld_tab(f4.addr(a));
    nv++;
    return 0u;
}

__device__ __forceinline__ uint64_t chunk_len(uint64_t nvec, uint64_t c0) {
    return nvec > c0 ? (nvec - c0 < kChunk ? nvec - c0 : kChunk) : 0;
}

// ---------------------------------------------------------------------------
// K3, D = 1: out[i] = table[sext(idx[i])]
// SMODE fences the index/output streams, TMODE the table accesses.
// ---------------------------------------------------------------------------
template <int SMODE, int TMODE>
__device__ __forceinline__ void gather_chunk(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                             uint64_t v0, uint64_t nvec, uint32_t &nv) {
    const Fence<SMODE, 16> f16(fd);
    const Fence<TMODE, 4> f4(fd);
    int4 j[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        j[u] = make_int4(0, 0, 0, 0);
        if (v < nvec) {
            const uint64_t a = idx + 16 * v;
            if (f16.ok(a)) j[u] = ld_idx(f16.addr(a));
            else nv += 4;
        }
    }
    uint4 r[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        if (v0 + u * kThreads < nvec) {
            r[u].x = fenced_tab<TMODE>(f4, table, j[u].x, nv);
            r[u].y = fenced_tab<TMODE>(f4, table, j[u].y, nv);
            r[u].z = fenced_tab<TMODE>(f4, table, j[u].z, nv);
            r[u].w = fenced_tab<TMODE>(f4, table, j[u].w, nv);
        }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        if (v < nvec) {
            const uint64_t a = out + 16 * v;
            if (f16.ok(a)) st_out(f16.addr(a), r[u]);
            else nv += 4;
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_gather1(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t nvec, uint32_t tail) {
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, v0 = c0 + threadIdx.x;
    if constexpr (MODE == kCheck || MODE == kModulo) {   // streams hoisted; random table accesses fenced
        const uint64_t cn = chunk_len(nvec, c0);
        if (cn && range_in(fd, idx + 16 * c0, 16 * cn) && range_in(fd, out + 16 * c0, 16 * cn))
            gather_chunk<kNone, MODE>(fd, out, table, idx, v0, nvec, nv);
        else
            gather_chunk<MODE, MODE>(fd, out, table, idx, v0, nvec, nv);
    } else {
        gather_chunk<MODE, MODE>(fd, out, table, idx, v0, nvec, nv);
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) {
        const Fence<MODE, 4> f4(fd);
        const uint64_t ai = idx + 16 * nvec + 4 * threadIdx.x, ao = out + 16 * nvec + 4 * threadIdx.x;
        int32_t j = 0;
        if (f4.ok(ai)) j = *reinterpret_cast<const int32_t *>(f4.addr(ai));
        else nv++;
        const uint32_t r = fenced_tab<MODE>(f4, table, j, nv);
        if (f4.ok(ao)) *reinterpret_cast<uint32_t *>(f4.addr(ao)) = r;
        else nv++;
    }
    if constexpr (MODE == kCheck) flush_violations(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K3, D > 1: out[i*D+d] = table[sext(idx[i])*D + d]; one warp per row i.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_gatherD(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t n, uint32_t D) {
    const Fence<MODE, 4> f4(fd);
    uint32_t nv = 0;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t W = (uint64_t)gridDim.x * (kThreads / 32);
    for (uint64_t i = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; i < n; i += W) {
        int32_t j = 0;
        if (lane == 0) {
            const uint64_t ai = idx + 4 * i;
            if (f4.ok(ai)) j = *reinterpret_cast<const int32_t *>(f4.addr(ai));
            else nv++;
        }
        j = __shfl_sync(0xffffffffu, j, 0);
        for (uint32_t d = lane; d < D; d += 32) {
            const uint64_t e = (uint64_t)((int64_t)j * (int64_t)D + (int64_t)d);
            const uint64_t at = table + e * 4;
            uint32_t r = 0;
            if (f4.ok(at)) r = ld_tab(f4.addr(at));
            else nv++;
            const uint64_t ao = out + 4 * (i * D + d);
            if (f4.ok(ao)) *reinterpret_cast<uint32_t *>(f4.addr(ao)) = r;
            else nv++;
        }
    }
    if constexpr (MODE == kCheck) flush_violations(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K3, D % 4 == 0 (16-byte-aligned rows): embedding rows moved as 128-bit
// vectors.  Vector e of the output is element group v = e % (D/4) of row
// i = e / (D/4): out + 16 e <- table + 4 (sext(j_i) D) + 16 v.  Every CTA owns
// kThreads x kU consecutive output vectors (coalesced stores; a row of D >= 32
// words is one or more whole 128-byte lines, so DRAM moves only useful bytes).
// Logical accesses as in the oracle: one index load per row (counted by the
// row's v == 0 vector), D table loads and D stores per row (4 per vector).
// ---------------------------------------------------------------------------
template <int SMODE, int TMODE>
__device__ __forceinline__ void gatherv_chunk(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                              uint64_t e0, uint64_t nv_total, uint32_t vpr, uint32_t &nv) {
    const Fence<SMODE, 4> fi(fd);
    const Fence<SMODE, 16> fo(fd);
    const Fence<TMODE, 16> ft(fd);
    uint4 r[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t e = e0 + u * kThreads;
        r[u] = make_uint4(0, 0, 0, 0);
        if (e < nv_total) {
            const uint64_t i = nv_total <= 0xFFFFFFFFull ? (uint64_t)((uint32_t)e / vpr) : e / vpr;
            const uint64_t v = e - i * vpr;
            const uint64_t ai = idx + 4 * i;
            int32_t j = 0;
            if (fi.ok(ai)) j = __ldg(reinterpret_cast<const int32_t *>(fi.addr(ai)));
            else nv += (v == 0);
            const uint64_t at = table + (uint64_t)((int64_t)j * (int64_t)vpr * 16) + 16 * v;
            if (ft.ok(at)) r[u] = __ldcg(reinterpret_cast<const uint4 *>(ft.addr(at)));
            else nv += 4;
        }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t e = e0 + u * kThreads;
        if (e < nv_total) {
            const uint64_t ao = out + 16 * e;
            if (fo.ok(ao)) st_out(fo.addr(ao), r[u]);
            else nv += 4;
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_gatherV(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t nv_total, uint32_t vpr) {
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, e0 = c0 + threadIdx.x;
    if constexpr (MODE == kCheck || MODE == kModulo) {   // streams hoisted; table rows fenced
        const uint64_t cn = chunk_len(nv_total, c0);
        const uint64_t r0 = c0 / vpr, r1 = (c0 + cn - 1) / vpr;       // rows this CTA touches
        if (cn && range_in(fd, idx + 4 * r0, 4 * (r1 - r0 + 1)) && range_in(fd, out + 16 * c0, 16 * cn))
            gatherv_chunk<kNone, MODE>(fd, out, table, idx, e0, nv_total, vpr, nv);
        else
            gatherv_chunk<MODE, MODE>(fd, out, table, idx, e0, nv_total, vpr, nv);
    } else {
        gatherv_chunk<MODE, MODE>(fd, out, table, idx, e0, nv_total, vpr, nv);
    }
    if constexpr (MODE == kCheck) flush_violations(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K4: table[sext(idx[i])] += src[i] (u32).  The read-modify-write is one
// fenced access (atomics instrumented like stores) issued as a
// no-return RED.E.ADD.
// ---------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void fenced_red(const Fence<MODE, 4> &f4, uint64_t table, int32_t j, uint32_t v,
                                           uint32_t &nv) {
    const uint64_t a = row_addr(table, j);
    if (f4.ok(a)) atomicAdd(reinterpret_cast<unsigned int *>(f4.addr(a)), v);
    else nv++;
}

template <int SMODE, int TMODE>
__device__ __forceinline__ void scatter_chunk(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src,
                                              uint64_t v0, uint64_t nvec, uint32_t &nv) {
    const Fence<SMODE, 16> f16(fd);
    const Fence<TMODE, 4> f4(fd);
    int4 j[kU];
    uint4 s[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        j[u] = make_int4(0, 0, 0, 0);
        s[u] = make_uint4(0, 0, 0, 0);
        if (v < nvec) {
            const uint64_t ai = idx + 16 * v, as = src + 16 * v;
            if (f16.ok(ai)) j[u] = ld_idx(f16.addr(ai));
            else nv += 4;
            if (f16.ok(as)) s[u] = ld_u4(f16.addr(as));
            else nv += 4;
        }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        if (v0 + u * kThreads < nvec) {
            fenced_red<TMODE>(f4, table, j[u].x, s[u].x, nv);
            fenced_red<TMODE>(f4, table, j[u].y, s[u].y, nv);
            fenced_red<TMODE>(f4, table, j[u].z, s[u].z, nv);
            fenced_red<TMODE>(f4, table, j[u].w, s[u].w, nv);
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_scatter(const __grid_constant__ FenceDesc fd, uint64_t table,
                                                      uint64_t idx, uint64_t src, uint64_t nvec, uint32_t tail) {
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, v0 = c0 + threadIdx.x;
    if constexpr (MODE == kCheck || MODE == kModulo) {   // streams hoisted; random RMWs fenced
        const uint64_t cn = chunk_len(nvec, c0);
        if (cn && range_in(fd, idx + 16 * c0, 16 * cn) && range_in(fd, src + 16 * c0, 16 * cn))
            scatter_chunk<kNone, MODE>(fd, table, idx, src, v0, nvec, nv);
        else
            scatter_chunk<MODE, MODE>(fd, table, idx, src, v0, nvec, nv);
    } else {
        scatter_chunk<MODE, MODE>(fd, table, idx, src, v0, nvec, nv);
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) {
        const Fence<MODE, 4> f4(fd);
        const uint64_t ai = idx + 16 * nvec + 4 * threadIdx.x, as = src + 16 * nvec + 4 * threadIdx.x;
        int32_t j = 0;
        uint32_t s = 0;
        if (f4.ok(ai)) j = *reinterpret_cast<const int32_t *>(f4.addr(ai));
        else nv++;
        if (f4.ok(as)) s = *reinterpret_cast<const uint32_t *>(f4.addr(as));
        else nv++;
        fenced_red<MODE>(f4, table, j, s, nv);
    }
    if constexpr (MODE == kCheck) flush_violations(nv, fd.viol);
}

template <typename K>
int blocks_per_sm(K kernel) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) b = 1;
    return b;
}

unsigned chunk_grid(uint64_t nvec) {
    const uint64_t g = (nvec + kChunk - 1) / kChunk;
    return (unsigned)(g ? g : 1);
}

template <int MODE>
cudaError_t gather_t(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx, uint64_t n, uint32_t D,
                     cudaStream_t s, const Geom &g) {
    if (D == 1) {
        k_gather1<MODE><<<chunk_grid(n / 4), kThreads, 0, s>>>(fd, out, table, idx, n / 4, (uint32_t)(n % 4));
    } else if (D % 4 == 0 && (table | out) % 16 == 0) {
        k_gatherV<MODE><<<chunk_grid(n * (D / 4)), kThreads, 0, s>>>(fd, out, table, idx, n * (D / 4), D / 4);
    } else {
        static const int bps = blocks_per_sm(k_gatherD<MODE>);
        const uint64_t want = (n * 32 + kThreads - 1) / kThreads, cap = (uint64_t)g.sms * bps;
        k_gatherD<MODE><<<(unsigned)(want < cap ? want : cap), kThreads, 0, s>>>(fd, out, table, idx, n, D);
    }
    return cudaGetLastError();
}

template <int MODE>
cudaError_t scatter_t(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n, cudaStream_t s) {
    k_scatter<MODE><<<chunk_grid(n / 4), kThreads, 0, s>>>(fd, table, idx, src, n / 4, (uint32_t)(n % 4));
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather(int mode, const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx, uint64_t n,
                          uint32_t D, cudaStream_t s, const Geom &g) {
    switch (mode) {
        case kNone: return gather_t<kNone>(fd, out, table, idx, n, D, s, g);
        case kMask: return gather_t<kMask>(fd, out, table, idx, n, D, s, g);
        case kModulo: return gather_t<kModulo>(fd, out, table, idx, n, D, s, g);
        default: return gather_t<kCheck>(fd, out, table, idx, n, D, s, g);
    }
}

cudaError_t launch_scatter(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n,
                           cudaStream_t s, const Geom &) {
    switch (mode) {
        case kNone: return scatter_t<kNone>(fd, table, idx, src, n, s);
        case kMask: return scatter_t<kMask>(fd, table, idx, src, n, s);
        case kModulo: return scatter_t<kModulo>(fd, table, idx, src, n, s);
        default: return scatter_t<kCheck>(fd, table, idx, src, n, s);
    }
}

}  // namespace gd
