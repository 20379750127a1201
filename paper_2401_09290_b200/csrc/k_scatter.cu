// k_scatter.cu -- K4 v2: the fenced embedding-style scatter-add,
// table[sext(idx[i])] += src[i] (u32), radix-partitioned by partition slice
// for sm_100a (the per-access fence of PAPER.md:230).
//
// Why: a random 4-byte read-modify-write into a table far larger than L2
// costs two random DRAM transactions (the sector fill and, later, its dirty
// write-back).  tools/scatter_probe.cu measures 22.6 G random REDs/s into a
// 2 GiB table against 50.4 G random reads/s and 195 G REDs/s into an
// L2-resident (<= 64 MiB) table: the direct kernel (k_index.cu k_scatter) is
// bound by the DRAM's random-transaction rate, not by bytes.  Applying the
// updates one partition slice at a time keeps each slice's table lines in L2
// while they are updated, so the fills and write-backs of a slice happen
// close together in time and address.
//
//   A1  k_scatter_part<M, 0>  every index: its fenced address -> slice id;
//                             per-CTA shared histogram, one global atomic
//                             per non-empty slice
//   A2  k_scatter_scan        exclusive scan of the slice counts (one CTA)
//   A3  k_scatter_part<M, 1>  the same fence again, refusals counted (once,
//                             here), each update placed as (word offset,
//                             value) in its slice's run of the scratch
//   B   k_scatter_apply       the runs in slice order: RED.ADD.U32 at
//                             base + 4 * word (CTAs in flight cover about one
//                             slice, so its lines stay in L2)
//
// Every logical access is fenced exactly as in the direct kernel and as the
// oracle defines it (or_scatter_add): the index and source loads per access
// or per CTA tile (R-hoist), the read-modify-write at its own fenced address
// (one logical access), each refusal counted once.  u32 addition
// is commutative and associative, so the order of the updates does not
// change the result (reading A6).  Clamped RMWs of a CTA are summed per edge
// word and added by one atomic each (as in k_scatter).  In NONE mode an
// address outside the partition is updated directly, unfenced (the native
// twin).  The scratch (8 bytes per update) is trusted memory outside every
// partition, allocated stream-ordered (cudaMallocAsync) per launch, so
// concurrent tenants never share it; a placement past its slice's run (only
// possible if the tenant rewrites idx while its own launch runs) is dropped,
// never written outside the scratch.
#include <type_traits>

#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kU = 4;                                  // 16-byte index vectors per thread
constexpr uint64_t kChunk = (uint64_t)kThreads * kU;   // vectors (4 indices each) per CTA
#ifndef GD_SCATTER_SLICE_SHIFT
#define GD_SCATTER_SLICE_SHIFT 25
#endif
// 32 MiB slices: measured 784 GB/s against 746 (16 MiB) and 631 (64 MiB),
// and 689 without the L2 bulk prefetch (tools/r02_iter16.sh)
constexpr int kSliceShift = GD_SCATTER_SLICE_SHIFT;
constexpr uint32_t kMaxSlices = (uint32_t)((1ull << 34) >> kSliceShift);   // partitions up to 16 GiB (u32 word offsets)
static_assert(kMaxSlices >= kThreads && kMaxSlices % kThreads == 0 && kMaxSlices <= 1024, "slice count");

__device__ __forceinline__ uint4 ld_u4(uint64_t a) { return __ldcs(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ uint32_t ld_w(uint64_t a) { return __ldcs(reinterpret_cast<const unsigned int *>(a)); }

struct EdgeAcc {                                       // clamped RMWs of a thread, per edge word
    uint32_t lo = 0, hi = 0;
    bool alo = false, ahi = false;
};

__device__ __forceinline__ void edge_add(const FenceDesc &fd, const EdgeAcc &es) {
    __shared__ uint32_t sum[2], any[2];
    if (threadIdx.x < 2) sum[threadIdx.x] = any[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lo = __reduce_add_sync(0xffffffffu, es.lo), hi = __reduce_add_sync(0xffffffffu, es.hi);
    const bool alo = __any_sync(0xffffffffu, es.alo), ahi = __any_sync(0xffffffffu, es.ahi);
    if ((threadIdx.x & 31u) == 0) {
        if (alo) { atomicAdd(&sum[0], lo); any[0] = 1; }
        if (ahi) { atomicAdd(&sum[1], hi); any[1] = 1; }
    }
    __syncthreads();
    if (threadIdx.x == 0 && any[0]) atomicAdd(reinterpret_cast<unsigned int *>(fd.base), sum[0]);
    if (threadIdx.x == 1 && any[1]) atomicAdd(reinterpret_cast<unsigned int *>(fd.base + fd.size - 4), sum[1]);
}

// One RMW of the direct kernel's semantics, resolved: *word = partition word
// offset of the fenced address when it is to be bucketed (returns true);
// otherwise counted / clamped / (NONE, outside) applied directly in pass 1.
// NEAR (modulo, decided per launch: the table base lies in the partition and
// the partition is at least 2^33 bytes): every RMW offset a - base = (table -
// base) + 4 sext(j) lies in [-2^33, 2 size), so its u64 remainder (reading
// A10) needs at most one correction: s >= 0: s or s - size; s < 0: the u64
// value 2^64 + s has remainder (c + s) mod size with c = 2^64 mod size, i.e.
// c + s or c + s + size.  Exactly the full modulo, without the reciprocal.
template <int MODE, int PASS, bool NEAR = false>
__device__ __forceinline__ bool resolve(const Fence<MODE, 4> &f4, uint64_t table, int32_t j, uint32_t v,
                                        uint32_t &nv, EdgeAcc &es, uint64_t &word, uint64_t c64 = 0) {
    const uint64_t a = table + (uint64_t)((int64_t)j * 4);        // sext, scale in 64 bits (Listing 1 l.22)
    if constexpr (MODE == kModulo && NEAR) {
        const uint64_t off = a - f4.base;
        uint64_t r;
        if ((int64_t)off >= 0) {
            r = off >= f4.size ? off - f4.size : off;
        } else {
            const uint64_t x = off + c64;                            // c + s, as u64
            r = (int64_t)x < 0 ? x + f4.size : x;
        }
        word = r >> 2;                                               // (r & ~3) / 4: a is 4-aligned
        return true;
    } else if constexpr (MODE == kNone) {
        if (a - f4.base <= f4.lim && (a & 3) == 0) {
            word = (a - f4.base) >> 2;
            return true;
        }
        if (PASS == 1) atomicAdd(reinterpret_cast<unsigned int *>(a), v);   // the native twin: unfenced
        return false;
    } else if constexpr (MODE == kClamp) {
        if (f4.inside(a)) {
            word = (a - f4.base) >> 2;
            return true;
        }
        if (PASS == 1) {
            nv++;
            if (a < f4.base) {
                es.lo += v;
                es.alo = true;
            } else {
                es.hi += v;
                es.ahi = true;
            }
        }
        return false;
    } else {
        uint32_t c = 0;
        const bool ok = f4.go(a, c, 1);                               // check: refused; mask-count: counted
        if (PASS == 1) nv += c;
        if (!ok) return false;
        word = (f4.addr(a) - f4.base) >> 2;
        return true;
    }
}

// The 16 updates of one thread (A1 / A3): loads, fence, slice rank.
// SMODE fences the idx / src streams (kNone when the CTA's tiles of both lie
// in the partition: R-hoist), MODE the RMWs.  Bit k of *putm: update k is
// bucketed at partition word w[k], rank rk[k] in its slice's CTA histogram.
constexpr int kItems = 4 * kU;

template <int SMODE, int MODE, int PASS, bool NEAR = false>
__device__ __forceinline__ void items(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t v0,
                                      uint64_t nvec, uint32_t &nv, EdgeAcc &es, unsigned *hist,
                                      uint32_t (&w)[kItems], uint32_t (&rk)[kItems], uint32_t (&sv)[kItems],
                                      uint32_t &putm) {
    const Fence<SMODE, 16> f16(fd);
    const Fence<MODE, 4> f4(fd);
    const uint64_t c64 = NEAR ? 0ull - fd.inv * fd.size : 0ull;   // 2^64 mod size (inv = floor(2^64 / size))
    uint4 j[kU], s[kU];
    // Every load of the 2 kU is issued unconditionally, with no branch
    // between them (a branch per vector had made ptxas consume each loaded
    // index vector before issuing the next load: four serial DRAM round
    // trips, ncu: +26 % time for the mask pass A3): a dead vector (past
    // nvec) or a refused one (check) reads the trusted zero block, so it
    // reads 0 as a refused check-mode load must (reading A1); under clamp
    // an outside vector is then replaced by its edge word four times
    // (fence.cuh vld4), after every load has been issued.
    // MODULO walks each stream: a thread's kU vectors of a stream lie
    // kStep bytes apart, so unless the stream straddles the base each
    // fenced address follows from the previous one (Fence::step_up,
    // exactly the full modulo).
    constexpr uint64_t kStep = 16ull * kThreads;
    const auto walk_ok = [&](uint64_t lo) {
        const uint64_t hi = lo + kStep * (kU - 1) + 16;
        return SMODE == kModulo && kStep < fd.size && lo <= hi && (hi <= fd.base || lo >= fd.base);
    };
    const bool wi = walk_ok(idx + 16 * v0), ws = walk_ok(src + 16 * v0);
    uint64_t fi = 0, fs = 0;
    uint32_t outm = 0;                             // clamp: bit 2u / 2u+1 = idx / src vector u outside
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads, ai = idx + 16 * v, as = src + 16 * v;
        const bool live = v < nvec;
        fi = (u == 0 || !wi) ? f16.addr(ai) : f16.step_up(fi, kStep);
        fs = (u == 0 || !ws) ? f16.addr(as) : f16.step_up(fs, kStep);
        bool oki = true, oks = true;
        if constexpr (counts(SMODE)) {             // the check predicate (16-aligned vectors)
            oki = f16.ok_aligned_in(ai);
            oks = f16.ok_aligned_in(as);
            if (PASS == 1 && live) nv += (oki ? 0u : 4u) + (oks ? 0u : 4u);
        }
        constexpr bool kRefuse = SMODE == kCheck || SMODE == kClamp;
        if (SMODE == kClamp && live) outm |= (oki ? 0u : 1u << (2 * u)) | (oks ? 0u : 2u << (2 * u));
        j[u] = ld_u4(live && (!kRefuse || oki) ? (SMODE == kClamp ? ai : fi) : fd.zero);
        s[u] = make_uint4(0, 0, 0, 0);
        if (PASS == 1) s[u] = ld_u4(live && (!kRefuse || oks) ? (SMODE == kClamp ? as : fs) : fd.zero);
    }
    if constexpr (SMODE == kClamp) {
        if (outm) {                                // rare: outside vectors, edge word four times
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const uint64_t v = v0 + u * kThreads;
                if (outm & (1u << (2 * u))) {
                    const uint32_t x = ld_w(f16.edge4(idx + 16 * v));
                    j[u] = make_uint4(x, x, x, x);
                }
                if (PASS == 1 && (outm & (2u << (2 * u)))) {
                    const uint32_t x = ld_w(f16.edge4(src + 16 * v));
                    s[u] = make_uint4(x, x, x, x);
                }
            }
        }
    }
    putm = 0;
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const bool live = v0 + u * kThreads < nvec;
        const uint32_t jj[4] = {j[u].x, j[u].y, j[u].z, j[u].w}, ss[4] = {s[u].x, s[u].y, s[u].z, s[u].w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int k = 4 * u + q;
            uint64_t word = 0;
            const bool put = live && resolve<MODE, PASS, NEAR>(f4, table, (int32_t)jj[q], ss[q], nv, es, word, c64);
            w[k] = (uint32_t)word;
            sv[k] = ss[q];
            rk[k] = put ? atomicAdd(&hist[w[k] >> (kSliceShift - 2)], 1u) : 0u;
            putm |= (uint32_t)put << k;
        }
    }
}

template <int MODE, int PASS>
__global__ void __launch_bounds__(kThreads) k_scatter_part(const __grid_constant__ FenceDesc fd, uint64_t table,
                                                           uint64_t idx, uint64_t src, uint64_t nvec,
                                                           uint32_t nslices, unsigned *cnt, unsigned *cur,
                                                           const unsigned *lim, uint2 *pairs) {
    __shared__ unsigned hist[kMaxSlices];
    __shared__ unsigned gpos[kMaxSlices];
    for (uint32_t i = threadIdx.x; i < nslices; i += kThreads) hist[i] = 0;
    __syncthreads();
    uint32_t nv = 0, putm = 0;
    uint32_t w[kItems], rk[kItems], sv[kItems];
    EdgeAcc es;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, v0 = c0 + threadIdx.x;
    const auto run = [&](auto near_tag) {
        constexpr bool NEAR = decltype(near_tag)::value;
        if constexpr (hoistable(MODE)) {               // streams hoisted per CTA tile; RMWs fenced one by one
            const uint64_t cn = nvec > c0 ? (nvec - c0 < kChunk ? nvec - c0 : kChunk) : 0;
            if (cn && range_in(fd, idx + 16 * c0, 16 * cn) && range_in(fd, src + 16 * c0, 16 * cn))
                items<kNone, MODE, PASS, NEAR>(fd, table, idx, src, v0, nvec, nv, es, hist, w, rk, sv, putm);
            else
                items<MODE, MODE, PASS, NEAR>(fd, table, idx, src, v0, nvec, nv, es, hist, w, rk, sv, putm);
        } else {
            items<MODE, MODE, PASS, NEAR>(fd, table, idx, src, v0, nvec, nv, es, hist, w, rk, sv, putm);
        }
    };
#ifndef GD_SCATTER_MOD_NEAR
#define GD_SCATTER_MOD_NEAR 1
#endif
    if (MODE == kModulo && GD_SCATTER_MOD_NEAR && table - fd.base < fd.size && fd.size >= (1ull << 33))
        run(std::true_type{});
    else
        run(std::false_type{});
    __syncthreads();
    if constexpr (PASS == 0) {
        for (uint32_t i = threadIdx.x; i < nslices; i += kThreads)
            if (hist[i]) atomicAdd(&cnt[i], hist[i]);
    } else {
        // Reserve this CTA's run in every slice it updates, sort its updates
        // by slice in shared memory (exclusive scan of the histogram), then
        // write each run out with consecutive threads on consecutive pairs.
        __shared__ unsigned lstart[kMaxSlices];
        __shared__ unsigned wsum[kThreads / 32];
        __shared__ uint2 staged[kThreads * kItems];
        const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
        constexpr uint32_t SPT = kMaxSlices / kThreads;             // slices per thread
        uint32_t a[SPT], sum = 0;
#pragma unroll
        for (uint32_t q = 0; q < SPT; q++) {
            a[q] = SPT * t + q < nslices ? hist[SPT * t + q] : 0u;
            sum += a[q];
        }
        uint32_t run = sum;                            // inclusive scan, SPT slices per thread
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, run, o);
            if (lane >= (uint32_t)o) run += y;
        }
        if (lane == 31) wsum[warp] = run;
        for (uint32_t i = t; i < nslices; i += kThreads) gpos[i] = hist[i] ? atomicAdd(&cur[i], hist[i]) : 0u;
        __syncthreads();
        uint32_t pre = 0, total = 0;
#pragma unroll
        for (uint32_t k = 0; k < kThreads / 32; k++) {
            pre += k < warp ? wsum[k] : 0u;
            total += wsum[k];
        }
        uint32_t ex = pre + run - sum;
#pragma unroll
        for (uint32_t q = 0; q < SPT; q++) {
            if (SPT * t + q < nslices) lstart[SPT * t + q] = ex;
            ex += a[q];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; k++)
            if ((putm >> k) & 1u) staged[lstart[w[k] >> (kSliceShift - 2)] + rk[k]] = make_uint2(w[k], sv[k]);
        __syncthreads();
        for (uint32_t i = t; i < total; i += kThreads) {
            const uint2 p = staged[i];
            const uint32_t b = p.x >> (kSliceShift - 2);
            const uint32_t pos = gpos[b] + (i - lstart[b]);
            if (pos < lim[b]) pairs[pos] = p;
        }
        if constexpr (MODE == kClamp) edge_add(fd, es);
        if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
    }
}

// A2: exclusive scan of the slice counts -> run starts (cur) and ends (lim);
// total = updates placed.  One CTA of kMaxSlices threads.
__global__ void __launch_bounds__(kMaxSlices) k_scatter_scan(const unsigned *cnt, unsigned *cur, unsigned *lim,
                                                             unsigned *total, uint32_t nslices) {
    __shared__ unsigned sh[kMaxSlices];
    const uint32_t t = threadIdx.x;
    const unsigned c = t < nslices ? cnt[t] : 0u;
    sh[t] = c;
    __syncthreads();
    for (uint32_t o = 1; o < kMaxSlices; o <<= 1) {  // inclusive Hillis-Steele scan
        const unsigned add = t >= o ? sh[t - o] : 0u;
        __syncthreads();
        sh[t] += add;
        __syncthreads();
    }
    if (t < nslices) {
        cur[t] = sh[t] - c;
        lim[t] = sh[t];
    }
    if (t == kMaxSlices - 1) *total = sh[t];
}

// B: the placed updates in slice order.  word < words by construction (the
// word offset of a fenced address of the partition); tested anyway, so
// every address this kernel computes provably lies in the partition.  Each
// CTA also prefetches into L2 (one bulk prefetch, cp.async.bulk.prefetch.L2)
// its share of the NEXT updated slice, in proportion to its share of the
// current one: the CTAs of a slice stream the following slice into L2 ahead
// of its updates, so those REDs hit L2 and its lines are fetched (and later
// written back) in address order rather than one random sector at a time.
__global__ void __launch_bounds__(kThreads) k_scatter_apply(uint64_t base, uint64_t words, const uint2 *pairs,
                                                            const unsigned *total, const unsigned *cnt,
                                                            const unsigned *lim) {
    const uint64_t n = *total;
    const uint64_t c0 = (uint64_t)blockIdx.x * kThreads * 4;
#ifndef GD_SCATTER_PREFETCH
#define GD_SCATTER_PREFETCH 1
#endif
    if (GD_SCATTER_PREFETCH && threadIdx.x == 0 && c0 < n) {
        const uint32_t s = pairs[c0].x >> (kSliceShift - 2);             // the slice of the CTA's first update
        const uint64_t e = lim[s], c = cnt[s], st = e - c;
        const auto prefetch = [&](uint32_t sl, uint64_t from) {
            const uint64_t lo = ((c0 - st) << kSliceShift) / c & ~127ull;
            const uint64_t hi = (((c0 - st + (uint64_t)kThreads * 4) << kSliceShift) / c + 127) & ~127ull;
            const uint64_t slice0 = (uint64_t)sl << kSliceShift, wbytes = words * 4;
            uint64_t a = slice0 + lo, b = slice0 + (hi < (1ull << kSliceShift) ? hi : (1ull << kSliceShift));
            if (b > wbytes) b = wbytes;
            (void)from;
            if (a < b)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + a), "r"((uint32_t)(b - a))
                             : "memory");
        };
        // only dense slices (on average an update per 128-byte line or
        // more) are worth streaming in whole; sparse ones are left to their
        // REDs' own sector fills
        constexpr uint32_t kDense = (1u << kSliceShift) / 128;
        if (st == 0 && c >= kDense) prefetch(s, st);                     // the first slice: its own lines
        if (e < n) {
            const uint32_t s2 = pairs[e].x >> (kSliceShift - 2);         // the next updated slice
            if (cnt[s2] >= kDense) prefetch(s2, e);
        }
    }
    const uint64_t i0 = c0 + (uint64_t)threadIdx.x * 4;
    if (i0 >= n) return;
    uint2 p[4];
    if (i0 + 4 <= n) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(pairs + i0));
        const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(pairs + i0 + 2));
        p[0] = make_uint2(a.x, a.y);
        p[1] = make_uint2(a.z, a.w);
        p[2] = make_uint2(b.x, b.y);
        p[3] = make_uint2(b.z, b.w);
    } else {
#pragma unroll
        for (int q = 0; q < 4; q++) p[q] = i0 + q < n ? pairs[i0 + q] : make_uint2(0xFFFFFFFFu, 0u);
    }
#pragma unroll
    for (int q = 0; q < 4; q++)
        if (i0 + q < n && p[q].x < words) atomicAdd(reinterpret_cast<unsigned int *>(base + 4ull * p[q].x), p[q].y);
}

bool pool_ready() {
    // keep freed scratch in the device's default memory pool (stream-ordered
    // reuse, no release to the OS at every synchronisation)
    static const bool ok = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return false;
        uint64_t thr = ~0ull;
        return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess;
    }();
    return ok;
}

template <int MODE>
cudaError_t bucketed_t(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n, cudaStream_t s) {
    const uint64_t nvec = n / 4;
    const uint32_t nslices = (uint32_t)((fd.size + (1ull << kSliceShift) - 1) >> kSliceShift);
    const uint64_t meta = 4ull * (3 * kMaxSlices + 4);                 // cnt | cur | lim | total
    char *scratch = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&scratch), meta + 8 * (4 * nvec) + 16, s);
    if (e != cudaSuccess) return e;
    unsigned *cnt = reinterpret_cast<unsigned *>(scratch), *cur = cnt + kMaxSlices, *lim = cur + kMaxSlices;
    unsigned *total = lim + kMaxSlices;
    uint2 *pairs = reinterpret_cast<uint2 *>(scratch + meta);
    const unsigned grid = (unsigned)((nvec + kChunk - 1) / kChunk);
    e = cudaMemsetAsync(cnt, 0, 4ull * kMaxSlices, s);
    if (e == cudaSuccess) {
        k_scatter_part<MODE, 0><<<grid, kThreads, 0, s>>>(fd, table, idx, src, nvec, nslices, cnt, cur, lim, pairs);
        k_scatter_scan<<<1, kMaxSlices, 0, s>>>(cnt, cur, lim, total, nslices);
        k_scatter_part<MODE, 1><<<grid, kThreads, 0, s>>>(fd, table, idx, src, nvec, nslices, cnt, cur, lim, pairs);
        const unsigned gb = (unsigned)((4 * nvec + 4 * kThreads - 1) / (4 * kThreads));
        k_scatter_apply<<<gb, kThreads, 0, s>>>(fd.base, fd.size / 4, pairs, total, cnt, lim);
        e = cudaGetLastError();
    }
    const cudaError_t f = cudaFreeAsync(scratch, s);
    return e != cudaSuccess ? e : f;
}

}  // namespace

// The bucketed path for the update vectors (n / 4 * 4 of them; the caller
// issues the tail of n % 4 with the direct kernel).  cudaErrorNotSupported:
// not applicable (a partition above 16 GiB, or too few updates to gain),
// nothing issued.
cudaError_t launch_scatter_bucketed(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src,
                                    uint64_t n, cudaStream_t s) {
    static const bool off = [] {
        const char *e = getenv("GD_SCATTER_DIRECT");
        return e && e[0] == '1';
    }();
    if (off || n < (1ull << 20) || fd.size > (uint64_t)kMaxSlices << kSliceShift || fd.size < (4ull << kSliceShift) ||
        !pool_ready())
        return cudaErrorNotSupported;
    switch (mode) {
        case kNone: return bucketed_t<kNone>(fd, table, idx, src, n, s);
        case kMask: return bucketed_t<kMask>(fd, table, idx, src, n, s);
        case kModulo: return bucketed_t<kModulo>(fd, table, idx, src, n, s);
        case kMaskCount: return bucketed_t<kMaskCount>(fd, table, idx, src, n, s);
        case kClamp: return bucketed_t<kClamp>(fd, table, idx, src, n, s);
        default: return bucketed_t<kCheck>(fd, table, idx, src, n, s);
    }
}

}  // namespace gd
