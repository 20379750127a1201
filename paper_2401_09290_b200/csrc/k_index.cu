// k_index.cu -- fenced embedding-style gather / scatter-add (SURVEY.md §2.7
// K3, K4) for sm_100a.
//
// The effective address of every indexed access is materialised first
// (table + 4 * sext(j), Listing 1 lines 20-23 `mul.wide.s32` + `add.s64`,
// PAPER.md:206-209) and only then fenced (second addressing
// mode) -- the fence never sees a partial address.
//
// D = 1 path: 128-bit index loads, 4 independent fenced random 32-bit table
// loads per index vector, x2 unrolled (8 random loads in flight per thread),
// 128-bit output stores.  D > 1 path: one warp per index row, lanes stride
// over the row; lane 0 loads the index once (one logical access, as in the
// oracle) and broadcasts it.
#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 2;

__device__ __forceinline__ int4 ld_idx(uint64_t a) { return __ldcs(reinterpret_cast<const int4 *>(a)); }
__device__ __forceinline__ uint4 ld_u4(uint64_t a) { return __ldcs(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ uint32_t ld_tab(uint64_t a) { return __ldg(reinterpret_cast<const uint32_t *>(a)); }
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

// ---------------------------------------------------------------------------
// K3, D = 1: out[i] = table[sext(idx[i])]
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_gather1(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t nvec,
                                                      uint32_t tail) {
    const Fence<MODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    uint32_t nv = 0;
    const uint64_t T = (uint64_t)gridDim.x * kThreads;
    uint64_t v = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    for (; v + (kUnroll - 1) * T < nvec; v += kUnroll * T) {
        int4 j[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint64_t a = idx + 16 * (v + u * T);
            j[u] = make_int4(0, 0, 0, 0);
            if (f16.ok(a)) j[u] = ld_idx(f16.addr(a));
            else nv += 4;
        }
        uint4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            r[u].x = fenced_tab<MODE>(f4, table, j[u].x, nv);
            r[u].y = fenced_tab<MODE>(f4, table, j[u].y, nv);
            r[u].z = fenced_tab<MODE>(f4, table, j[u].z, nv);
            r[u].w = fenced_tab<MODE>(f4, table, j[u].w, nv);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint64_t a = out + 16 * (v + u * T);
            if (f16.ok(a)) st_out(f16.addr(a), r[u]);
            else nv += 4;
        }
    }
    for (; v < nvec; v += T) {
        const uint64_t ai = idx + 16 * v, ao = out + 16 * v;
        int4 j = make_int4(0, 0, 0, 0);
        if (f16.ok(ai)) j = ld_idx(f16.addr(ai));
        else nv += 4;
        uint4 r;
        r.x = fenced_tab<MODE>(f4, table, j.x, nv);
        r.y = fenced_tab<MODE>(f4, table, j.y, nv);
        r.z = fenced_tab<MODE>(f4, table, j.z, nv);
        r.w = fenced_tab<MODE>(f4, table, j.w, nv);
        if (f16.ok(ao)) st_out(f16.addr(ao), r);
        else nv += 4;
    }
    const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (tid < tail) {
        const uint64_t ai = idx + 16 * nvec + 4 * tid, ao = out + 16 * nvec + 4 * tid;
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

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_scatter(const __grid_constant__ FenceDesc fd, uint64_t table,
                                                      uint64_t idx, uint64_t src, uint64_t nvec, uint32_t tail) {
    const Fence<MODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    uint32_t nv = 0;
    const uint64_t T = (uint64_t)gridDim.x * kThreads;
    uint64_t v = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    for (; v + (kUnroll - 1) * T < nvec; v += kUnroll * T) {
        int4 j[kUnroll];
        uint4 s[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint64_t ai = idx + 16 * (v + u * T), as = src + 16 * (v + u * T);
            j[u] = make_int4(0, 0, 0, 0);
            s[u] = make_uint4(0, 0, 0, 0);
            if (f16.ok(ai)) j[u] = ld_idx(f16.addr(ai));
            else nv += 4;
            if (f16.ok(as)) s[u] = ld_u4(f16.addr(as));
            else nv += 4;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            fenced_red<MODE>(f4, table, j[u].x, s[u].x, nv);
            fenced_red<MODE>(f4, table, j[u].y, s[u].y, nv);
            fenced_red<MODE>(f4, table, j[u].z, s[u].z, nv);
            fenced_red<MODE>(f4, table, j[u].w, s[u].w, nv);
        }
    }
    for (; v < nvec; v += T) {
        const uint64_t ai = idx + 16 * v, as = src + 16 * v;
        int4 j = make_int4(0, 0, 0, 0);
        uint4 s = make_uint4(0, 0, 0, 0);
        if (f16.ok(ai)) j = ld_idx(f16.addr(ai));
        else nv += 4;
        if (f16.ok(as)) s = ld_u4(f16.addr(as));
        else nv += 4;
        fenced_red<MODE>(f4, table, j.x, s.x, nv);
        fenced_red<MODE>(f4, table, j.y, s.y, nv);
        fenced_red<MODE>(f4, table, j.z, s.z, nv);
        fenced_red<MODE>(f4, table, j.w, s.w, nv);
    }
    const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (tid < tail) {
        const uint64_t ai = idx + 16 * nvec + 4 * tid, as = src + 16 * nvec + 4 * tid;
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

uint64_t grid_for(uint64_t threads_wanted, int sms, int bps) {
    uint64_t want = (threads_wanted + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sms * (uint64_t)bps;
    if (want > cap) want = cap;
    return want ? want : 1;
}

template <int MODE>
cudaError_t gather_t(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx, uint64_t n, uint32_t D,
                     cudaStream_t s, const Geom &g) {
    if (D == 1) {
        static const int bps = blocks_per_sm(k_gather1<MODE>);
        const uint64_t nvec = n / 4;
        k_gather1<MODE><<<(unsigned)grid_for(nvec / kUnroll + 1, g.sms, bps), kThreads, 0, s>>>(
            fd, out, table, idx, nvec, (uint32_t)(n % 4));
    } else {
        static const int bps = blocks_per_sm(k_gatherD<MODE>);
        k_gatherD<MODE><<<(unsigned)grid_for(n * 32, g.sms, bps), kThreads, 0, s>>>(fd, out, table, idx, n, D);
    }
    return cudaGetLastError();
}

template <int MODE>
cudaError_t scatter_t(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n, cudaStream_t s,
                      const Geom &g) {
    static const int bps = blocks_per_sm(k_scatter<MODE>);
    const uint64_t nvec = n / 4;
    k_scatter<MODE><<<(unsigned)grid_for(nvec / kUnroll + 1, g.sms, bps), kThreads, 0, s>>>(fd, table, idx, src,
                                                                                           nvec, (uint32_t)(n % 4));
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather(int mode, const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx, uint64_t n,
                          uint32_t D, cudaStream_t s, const Geom &g) {
    switch (mode) {
        case kNone: return gather_t<kNone>(fd, out, table, idx, n, D, s, g);
        case kMask: return gather_t<kMask>(fd, out, table, idx, n, D, s, g);
        default: return gather_t<kCheck>(fd, out, table, idx, n, D, s, g);
    }
}

cudaError_t launch_scatter(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n,
                           cudaStream_t s, const Geom &g) {
    switch (mode) {
        case kNone: return scatter_t<kNone>(fd, table, idx, src, n, s, g);
        case kMask: return scatter_t<kMask>(fd, table, idx, src, n, s, g);
        default: return scatter_t<kCheck>(fd, table, idx, src, n, s, g);
    }
}

}  // namespace gd
