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
// output stores.  In the hoistable modes (check, modulo, mask-count, clamp)
// the index and output streams are range-tested once per CTA chunk (fence.cuh
// range_in); the random table accesses are fenced one by one.  D % 4 == 0 with 16-byte-aligned table and output:
// row slots of 128-bit vectors (k_gatherR below).  Other D > 1: the n * D
// output words as one flat stream (k_gatherE below).
#include "fence.cuh"
#include "kernels.h"

namespace gd {
namespace {

constexpr int kThreads = 256;
constexpr int kU = 4;
constexpr uint64_t kChunk = (uint64_t)kThreads * kU;   // index vectors per CTA

__device__ __forceinline__ uint4 ld_u4(uint64_t a) { return __ldcs(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ uint32_t ld_w(uint64_t a) { return __ldcs(reinterpret_cast<const unsigned int *>(a)); }
__device__ __forceinline__ uint32_t ld_tab(uint64_t a) { return __ldcg(reinterpret_cast<const uint32_t *>(a)); }
__device__ __forceinline__ uint4 ld_row(uint64_t a) { return __ldcg(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ void st_out(uint64_t a, uint4 v) { __stcs(reinterpret_cast<uint4 *>(a), v); }
__device__ __forceinline__ void st_w(uint64_t a, uint32_t v) { __stcs(reinterpret_cast<unsigned int *>(a), v); }

__device__ __forceinline__ uint64_t row_addr(uint64_t table, int32_t j) {
    return table + (uint64_t)((int64_t)j * 4);        // sext, scale in 64 bits
}

// (A range-only table test, with the one-LOP3 form on >= 4 GiB partitions,
// measured slower at the L2-resident size: clamp +1.4 -> +11.3 %, per-access
// check +3.2 -> +4.1 %, tools/r02_iter15.sh; not used.)
// (table is 4-byte aligned (API) and 4 sext(j) a multiple of 4, so the
// alignment half of the check predicate is known true: go_aligned)
template <int MODE>
__device__ __forceinline__ uint32_t fenced_tab(const Fence<MODE, 4> &f4, uint64_t table, int32_t j, uint32_t &nv) {
    const uint64_t a = row_addr(table, j);
#if GD_ZERO_REDIRECT
    const bool o = f4.go_aligned(a, nv, 1);
    return ld_tab(f4.ld_at(f4.addr(a), o));           // refused: the trusted zero block
#else
    if (f4.go_aligned(a, nv, 1)) return ld_tab(f4.addr(a));
    return 0u;
#endif
}

// Check / mask-count on a >= 4 GiB power-of-two partition (FenceDesc kBig):
// the partition test is one LOP3 on the high address word (Fence::in_big), the
// mask fence another (Fence::addr_big); a refused check load reads the trusted
// zero block (Fence::ld_at: loading at the mask-fenced address and zeroing the
// value measured slower, and it moves refused reads to DRAM).  The refusal
// sets bit `bit` of refm (a compile-time bit: one predicated OR), counted
// once per chunk.
template <int MODE>
__device__ __forceinline__ uint32_t fenced_tab_big(const Fence<MODE, 4> &f4, uint64_t table, int32_t j,
                                                   uint32_t &refm, int bit) {
    static_assert(MODE == kCheck || MODE == kMaskCount, "counting mask-type modes");
    const uint64_t a = row_addr(table, j);
    const bool in = f4.in_big(a);
    if (!in) refm |= 1u << bit;
    if constexpr (MODE == kCheck) return ld_tab(f4.ld_at(a, in));
    else return ld_tab(f4.addr_big(a));
}

__device__ __forceinline__ uint64_t chunk_len(uint64_t nvec, uint64_t c0) {
    return nvec > c0 ? (nvec - c0 < kChunk ? nvec - c0 : kChunk) : 0;
}

// ---------------------------------------------------------------------------
// K3, D = 1: out[i] = table[sext(idx[i])]
// SMODE fences the index/output streams, TMODE the table accesses.
// ---------------------------------------------------------------------------
template <int SMODE, int TMODE, bool BIG = false>
__device__ __forceinline__ void gather_chunk(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                             uint64_t v0, uint64_t nvec, uint32_t &nv) {
    const Fence<SMODE, 16> f16(fd);
    const Fence<TMODE, 4> f4(fd);
    uint4 j[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        j[u] = make_uint4(0, 0, 0, 0);
        if (v < nvec) j[u] = vld4(f16, idx + 16 * v, nv, ld_u4, ld_w);
    }
    uint4 r[kU];
    if constexpr (BIG) {
        uint32_t refm = 0;
#pragma unroll
        for (int u = 0; u < kU; u++) {
            if (v0 + u * kThreads < nvec) {
                r[u].x = fenced_tab_big<TMODE>(f4, table, (int32_t)j[u].x, refm, 4 * u);
                r[u].y = fenced_tab_big<TMODE>(f4, table, (int32_t)j[u].y, refm, 4 * u + 1);
                r[u].z = fenced_tab_big<TMODE>(f4, table, (int32_t)j[u].z, refm, 4 * u + 2);
                r[u].w = fenced_tab_big<TMODE>(f4, table, (int32_t)j[u].w, refm, 4 * u + 3);
            }
        }
        nv += __popc(refm);
    } else {
#pragma unroll
        for (int u = 0; u < kU; u++) {
            if (v0 + u * kThreads < nvec) {
                r[u].x = fenced_tab<TMODE>(f4, table, (int32_t)j[u].x, nv);
                r[u].y = fenced_tab<TMODE>(f4, table, (int32_t)j[u].y, nv);
                r[u].z = fenced_tab<TMODE>(f4, table, (int32_t)j[u].z, nv);
                r[u].w = fenced_tab<TMODE>(f4, table, (int32_t)j[u].w, nv);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        if (v < nvec) vst4(f16, out + 16 * v, r[u], nv, st_out, st_w);
    }
}

// bit 0: mask-count, bit 1: check take fenced_tab_big on kBig partitions.
// Mask-count on: L2-resident 2^22 gather per access +1.4 -> +1.2 % (kernel
// bench), +8.6 -> -0.3 % inside bench.py's process.  Check: no faster (+3.2 %
// either way per access; loading at the mask-fenced address instead of the
// zero block: +3.4 -> +14.8 %, and refused reads reach DRAM), off
// (tools/r02_iter26.sh, r02_iter26b.sh).
#ifndef GD_GATHER1_BIG
#define GD_GATHER1_BIG 1
#endif
template <int MODE>
__global__ void __launch_bounds__(kThreads, 5) k_gather1(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t nvec, uint32_t tail) {
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, v0 = c0 + threadIdx.x;
    if constexpr (hoistable(MODE)) {     // streams hoisted; random table accesses fenced
        const uint64_t cn = chunk_len(nvec, c0);
        constexpr bool kBigTab = (MODE == kMaskCount && (GD_GATHER1_BIG & 1)) || (MODE == kCheck && (GD_GATHER1_BIG & 2));
        const bool inside = cn && range_in(fd, idx + 16 * c0, 16 * cn) && range_in(fd, out + 16 * c0, 16 * cn);
        if (kBigTab && (fd.flags & kBig)) {
            if (inside) gather_chunk<kNone, MODE, kBigTab>(fd, out, table, idx, v0, nvec, nv);
            else gather_chunk<MODE, MODE, kBigTab>(fd, out, table, idx, v0, nvec, nv);
        } else if (inside) {
            gather_chunk<kNone, MODE>(fd, out, table, idx, v0, nvec, nv);
        } else {
            gather_chunk<MODE, MODE>(fd, out, table, idx, v0, nvec, nv);
        }
    } else {
        gather_chunk<MODE, MODE>(fd, out, table, idx, v0, nvec, nv);
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) {
        const Fence<MODE, 4> f4(fd);
        const uint64_t ai = idx + 16 * nvec + 4 * threadIdx.x, ao = out + 16 * nvec + 4 * threadIdx.x;
        int32_t j = 0;
        if (f4.go(ai, nv, 1)) j = *reinterpret_cast<const int32_t *>(f4.addr(ai));
        const uint32_t r = fenced_tab<MODE>(f4, table, j, nv);
        if (f4.go(ao, nv, 1)) *reinterpret_cast<uint32_t *>(f4.addr(ao)) = r;
    }
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K3, D >= 2 outside the row-slot path (D % 4 != 0, or table / out not
// 16-byte aligned): out[e] = table[sext(idx[e / D]) * D + e % D] over the
// n * D output words as one flat stream.  Each thread takes kE words kThreads
// apart (every warp instruction covers 32 consecutive words: coalesced
// stores, and the table words of a row are contiguous), with every index
// load of the batch issued before the table loads and every table load
// before the stores.  The row and column of a thread's first word come from
// the reciprocal dinv = floor(2^64 / D) (mulhi is e / D or one less, one
// compare finishes it), the next ones by adding kThreads / D and
// kThreads % D.  Logical accesses as in the oracle (or_gather): one index
// load per row, counted by the row's d == 0 word (the other words of the row
// repeat the same fenced load and the same decision, uncounted), D table
// loads and D stores per row.  A refused or dead load reads the trusted zero
// block (Fence::ld_at), so no load of a batch waits on a branch.
// ---------------------------------------------------------------------------
constexpr int kE = 8;                                  // words per thread
constexpr uint64_t kEChunk = (uint64_t)kThreads * kE;  // words per CTA
// clamp holds each word's clamped table address until its load: 4 words per
// pass (two passes per chunk) keep it free of local memory.  GD_GATHERE_NARROW:
// the check / mask-count passes 4 words wide too, at 6 CTAs per SM instead of
// 8 words at 5 (D = 6, tools/r02_iter22.sh: check +1.8 -> +0.3 %, mask-count
// +5.1 -> +0.3 %, per access +6.4 -> +4.2 % / +12.8 -> +7.5 %), and modulo
// (its stream walk spills at 8 words in 40 registers)
#ifndef GD_GATHERE_NARROW
#define GD_GATHERE_NARROW 1
#endif
constexpr int ke_pass(int mode) {
    return (mode == kClamp || (GD_GATHERE_NARROW && (counts(mode) || mode == kModulo))) ? 4 : kE;
}

#ifndef GD_GATHERE_WALK
#define GD_GATHERE_WALK 1
#endif
// e / D from dinv = floor(2^64 / D), D >= 2 (no 64-bit division call)
__device__ __forceinline__ uint64_t div_d(uint64_t e, uint32_t D, uint64_t dinv) {
    const uint64_t q = __umul64hi(e, dinv);
    return e - q * D >= D ? q + 1 : q;
}

template <int SMODE, int TMODE, int KE>
__device__ __forceinline__ void gathere_pass(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                              uint64_t e0, uint64_t N, uint32_t D, uint64_t dinv, uint32_t qs,
                                              uint32_t rs, uint32_t &nv) {
    const Fence<SMODE, 4> fs(fd);
    const Fence<TMODE, 4> ft(fd);
    uint64_t i = div_d(e0, D, dinv);
    uint32_t d = (uint32_t)(e0 - i * D);
    int32_t j[KE];
    uint32_t dd[KE];
    // Modulo on the streams (per access, or a CTA range not inside): this
    // pass's index and output addresses increase with u, so when neither
    // range straddles the base nor spans the partition each access's fence
    // follows from the previous one's (Fence::step_up: one add and one
    // select, exactly the full modulo, reading A10); otherwise every access
    // takes the full modulo.
    bool walk = false;
    if constexpr (SMODE == kModulo && GD_GATHERE_WALK) {
        const uint64_t eL = e0 + (uint64_t)(KE - 1) * kThreads;
        const uint64_t lo_i = idx + 4 * i, hi_i = idx + 4 * div_d(eL, D, dinv) + 4;
        const uint64_t lo_o = out + 4 * e0, hi_o = out + 4 * eL + 4;
        const auto side = [&](uint64_t lo, uint64_t hi) {
            return lo <= hi && hi - lo < fd.size && (hi <= fd.base || lo >= fd.base);
        };
        walk = side(lo_i, hi_i) && side(lo_o, hi_o);
    }
    if (walk) {
        uint64_t fa = 0, aa = 0;
#pragma unroll
        for (int u = 0; u < KE; u++) {
            const bool live = e0 + (uint64_t)u * kThreads < N;
            const uint64_t ai = idx + 4 * i;
            fa = u == 0 ? fs.addr(ai) : fs.step_up(fa, ai - aa);
            aa = ai;
            j[u] = (int32_t)__ldg(reinterpret_cast<const unsigned int *>(fs.ld_at(fa, live)));
            dd[u] = d;
            i += qs;
            d += rs;
            if (d >= D) {
                d -= D;
                i++;
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < KE; u++) {
            const bool live = e0 + (uint64_t)u * kThreads < N;
            const uint64_t ai = idx + 4 * i;
            const bool o = fs.go(ai, nv, (live && d == 0) ? 1u : 0u);
            j[u] = (int32_t)__ldg(reinterpret_cast<const unsigned int *>(fs.ld_at(fs.addr(ai), o && live)));
            dd[u] = d;
            i += qs;
            d += rs;
            if (d >= D) {
                d -= D;
                i++;
            }
        }
    }
    uint32_t r[KE];
#pragma unroll
    for (int u = 0; u < KE; u++) {
        const bool live = e0 + (uint64_t)u * kThreads < N;
        const uint64_t at = table + (uint64_t)((int64_t)j[u] * (int64_t)D + (int64_t)dd[u]) * 4u;
        const bool o = ft.go(at, nv, live ? 1u : 0u);
        r[u] = ld_tab(ft.ld_at(ft.addr(at), o && live));
    }
    if (walk) {
        uint64_t fo = fs.addr(out + 4 * e0);
#pragma unroll
        for (int u = 0; u < KE; u++) {
            if (u) fo = fs.step_up(fo, 4 * kThreads);
            if (e0 + (uint64_t)u * kThreads < N) st_w(fo, r[u]);
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < KE; u++) {
        const uint64_t e = e0 + (uint64_t)u * kThreads;
        if (e < N) {
            const uint64_t ao = out + 4 * e;
            if (fs.go(ao, nv, 1)) st_w(fs.addr(ao), r[u]);
        }
    }
}

template <int SMODE, int TMODE>
__device__ __forceinline__ void gathere_chunk(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                              uint64_t e0, uint64_t N, uint32_t D, uint64_t dinv, uint32_t qs,
                                              uint32_t rs, uint32_t &nv) {
    constexpr int KE = ke_pass(TMODE);
#pragma unroll 1
    for (int p = 0; p < kE; p += KE)
        gathere_pass<SMODE, TMODE, KE>(fd, out, table, idx, e0 + (uint64_t)p * kThreads, N, D, dinv, qs, rs, nv);
}

// CTAs per SM: the most at which ptxas keeps the mode free of local memory
// (40 registers; clamp 48)
constexpr int gathere_minb(int mode) {
    return (mode == kClamp || (!GD_GATHERE_NARROW && counts(mode))) ? 5 : 6;
}
template <int MODE>
__global__ void __launch_bounds__(kThreads, gathere_minb(MODE)) k_gatherE(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t N, uint32_t D,
                                                      uint64_t dinv, uint32_t qs, uint32_t rs) {
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * kEChunk, e0 = c0 + threadIdx.x;
    if constexpr (hoistable(MODE)) {     // the index / output streams hoisted per CTA; table words fenced
        const uint64_t cn = N - c0 < kEChunk ? N - c0 : kEChunk;
        const uint64_t r0 = div_d(c0, D, dinv), r1 = div_d(c0 + cn - 1, D, dinv);   // rows this CTA touches
        if (range_in(fd, idx + 4 * r0, 4 * (r1 - r0 + 1)) && range_in(fd, out + 4 * c0, 4 * cn))
            gathere_chunk<kNone, MODE>(fd, out, table, idx, e0, N, D, dinv, qs, rs, nv);
        else
            gathere_chunk<MODE, MODE>(fd, out, table, idx, e0, N, D, dinv, qs, rs, nv);
    } else {
        gathere_chunk<MODE, MODE>(fd, out, table, idx, e0, N, D, dinv, qs, rs, nv);
    }
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K3, D % 4 == 0 (16-byte-aligned rows): embedding rows moved as 128-bit
// vectors in row slots.  A row of vpr = D/4 vectors is split into tpr = vpr/G
// slots of G vectors (G = 4, 2 or 1, dividing vpr); slot t of
// row i moves vectors t + tpr*g (g < G): table + 16 (sext(j_i) vpr + t + tpr g)
// -> out + 16 (i vpr + t + tpr g).  Consecutive threads take consecutive
// slots, so every warp instruction covers whole 16-byte pieces of contiguous
// runs (coalesced); the index load, the row address and the table fence of
// check / modulo mode are paid once per slot instead of once per vector: a
// row wholly inside the partition (check) or not wrapping around its end
// (modulo) needs no per-vector fence (same results, see range_in).  Each
// thread owns 4/G slots, i.e. 4 vectors (64 B) in flight.  G is chosen so
// that a row still has >= 8 slots (see gather_t).
// Logical accesses as in the oracle: one index load per row (counted by the
// row's t == 0 slot), D table loads and D stores per row (4 per vector).
// ---------------------------------------------------------------------------
// Code-generation choices of the row gather, measured per access at 1 GiB
// of gathered rows (tools/r02_iter5.sh; A/B with tools/build_variant.sh):
// CLAMP_SAFE: clamp's index loads read a safe word when the slot is dead, as
//   the other modes do (G = 1 with a power-of-two slot count, e.g. D = 32:
//   +8.4 -> -0.5 %; the non-power-of-two row index would spill; G >= 2 kept
//   predicated: D = 64 +5.8 -> +11.3 %, and G = 4 would spill);
// LIVE_REDIRECT: a dead slot's table vector is read from the trusted zero
//   block in none / mask / mask-count too, instead of a predicated load
//   (mask-count D = 64: +13.2 -> +0.3 %; modulo and clamp keep the
//   predicated load: 7-40 % slower with the selected address).
// (the clamp knobs are bit masks over G: bit G set = applied to slots of G
// vectors; CLAMP_SAFE needs a power-of-two slot count at G = 1)
#ifndef GD_GATHER_CLAMP_SAFE
#define GD_GATHER_CLAMP_SAFE 0x2
#endif
#ifndef GD_GATHER_CLAMP_SYNCWARP
#define GD_GATHER_CLAMP_SYNCWARP 0x16
#endif
#ifndef GD_GATHER_CLAMP_REDIRECT
#define GD_GATHER_CLAMP_REDIRECT 0x0
#endif
// CLAMP_BITS (bit G): step 3b takes each outside vector's edge word from a
// below-the-base bit instead of the vector's address, so the addresses die at
// their loads; with it the fix-up fits behind one branch (CLAMP_FIX_BRANCH)
// at G = 2 without local memory: D = 64 clamp +9.6-10.0 -> +0.0-0.1 %
// (tools/r02_iter28.sh; G = 4 measured no faster per access, G = 1 spills).
#ifndef GD_GATHER_CLAMP_BITS
#define GD_GATHER_CLAMP_BITS 0x4
#endif
#ifndef GD_GATHER_LIVE_REDIRECT
#define GD_GATHER_LIVE_REDIRECT 1
#endif
// Row of slot sl without a branch (a branch between the index loads would
// make the compiler consume each loaded index before the next load issues):
// a shift when the slots per row are a power of two (P2, dv = log2 tpr),
// else the reciprocal dv = floor(2^64 / tpr) (tpr >= 3): q = mulhi(sl, dv) is
// sl / tpr or one less, one predicated add finishes it.
template <bool P2>
__device__ __forceinline__ uint64_t row_of(uint64_t sl, uint64_t tpr, uint64_t dv) {
    if constexpr (P2) {
        return sl >> dv;
    } else {
        uint64_t q = __umul64hi(sl, dv);
        if (sl - q * tpr >= tpr) q++;
        return q;
    }
}

template <int SMODE, int TMODE, int G, bool P2>
__device__ __forceinline__ void gatherr_chunk(const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                                              uint64_t s0, uint64_t nslots, uint32_t tpr32, uint64_t dv,
                                              uint32_t &nv) {
    constexpr int S = 4 / G;
    constexpr bool kClampSafe = ((GD_GATHER_CLAMP_SAFE >> G) & 1) && (G > 1 || P2);
    const Fence<SMODE, 4> fi(fd);
    const Fence<SMODE, 16> fo(fd);
    const Fence<TMODE, 16> ft(fd);
    const uint64_t tpr = tpr32, vpr = tpr * G, rowbytes = 16 * vpr;
    // Every address here is aligned by construction (idx 4-, table and out
    // 16-aligned: gather_t and the API check), hence ok_aligned.
    // Phases keep every load of a kind in flight together: the fence's rare
    // per-vector path is a branch, and a branch between two loads would
    // serialise their latencies.
    bool live[S], okj[S];
    int32_t j[S];
    // A refused (or dead) index load reads a safe word instead -- the first
    // index of the launch when the streams are unfenced, else the partition's
    // base -- and its value is replaced by 0 only where it is used (step 2):
    // a predicated load would make the compiler consume each loaded index
    // (its sign extension) before the next load issues.
    const uint64_t safe = SMODE == kNone ? idx : fd.base;
    uint64_t ov[S], tv[S];
    // Per-access modulo on the streams (SMODE == kModulo: hoisting off): this
    // thread's index and output addresses increase with k (and g), so when
    // neither range straddles the base nor spans the partition, each access's
    // fence follows from the previous one's (Fence::step_up, exactly the full
    // modulo); otherwise every access takes the full modulo.
    bool walk = false;
    if constexpr (SMODE == kModulo) {
        const uint64_t sl0 = s0, sl1 = s0 + (uint64_t)(S - 1) * kThreads;
        const uint64_t i0 = row_of<P2>(sl0, tpr, dv), i1 = row_of<P2>(sl1, tpr, dv);
        const uint64_t lo_i = idx + 4 * i0, hi_i = idx + 4 * i1 + 4;
        const uint64_t lo_o = out + 16 * (i0 * vpr + (sl0 - i0 * tpr));
        const uint64_t hi_o = out + 16 * (i1 * vpr + (sl1 - i1 * tpr)) + 16 * tpr * (G - 1) + 16;
        const auto side = [&](uint64_t lo, uint64_t hi) {
            return lo <= hi && hi - lo < fd.size && (hi <= fd.base || lo >= fd.base);
        };
        walk = side(lo_i, hi_i) && side(lo_o, hi_o);
    }
    if constexpr (SMODE == kModulo) {
        uint64_t fa_prev = 0, aa_prev = 0;
#pragma unroll
        for (int k = 0; k < S; k++) {                       // 1. index loads (predicated, no branch:
            const uint64_t sl = s0 + (uint64_t)k * kThreads; //    a branch would serialise them)
            live[k] = sl < nslots;
            const uint64_t i = row_of<P2>(sl, tpr, dv);
            const uint64_t t = sl - i * tpr;
            const uint64_t ai = idx + 4 * i;
            uint32_t ci = 0;
            const bool oki = fi.go_aligned(ai, ci, 1) && live[k];        // ALU only: no branch
            const uint64_t fa = (k == 0 || !walk) ? fi.addr(ai) : fi.step_up(fa_prev, ai - aa_prev);
            fa_prev = fa;
            aa_prev = ai;
            okj[k] = oki;
            j[k] = __ldg(reinterpret_cast<const int32_t *>(oki ? fa : safe));
            if (live[k] && t == 0) nv += ci;                             // one index access per row
            ov[k] = out + 16 * (i * vpr + t);
            tv[k] = 16 * t;
        }
    } else {
#pragma unroll
        for (int k = 0; k < S; k++) {                       // 1. index loads (predicated, no branch:
            const uint64_t sl = s0 + (uint64_t)k * kThreads; //    a branch would serialise them)
            live[k] = sl < nslots;
            const uint64_t i = row_of<P2>(sl, tpr, dv);
            const uint64_t t = sl - i * tpr;
            const uint64_t ai = idx + 4 * i;
            uint32_t ci = 0;
            const bool oki = fi.go_aligned(ai, ci, 1) && live[k];        // ALU only: no branch
            okj[k] = oki;
            if constexpr (SMODE == kClamp && !kClampSafe) {   // (clamp: only dead slots are refused)
                j[k] = 0;
                if (oki) j[k] = __ldg(reinterpret_cast<const int32_t *>(fi.addr(ai)));
            } else {
                j[k] = __ldg(reinterpret_cast<const int32_t *>(oki ? fi.addr(ai) : safe));
            }
            if (live[k] && t == 0) nv += ci;                             // one index access per row
            ov[k] = out + 16 * (i * vpr + t);
            tv[k] = 16 * t;
        }
    }
    // (clamp: a warp-synchronising point after the index loads keeps ptxas
    // from consuming each loaded index before the next load issues)
    if constexpr (TMODE == kClamp && ((GD_GATHER_CLAMP_SYNCWARP >> G) & 1)) __syncwarp();
    uint64_t at[S][G];
    bool ok[S][G];
    uint32_t cnt[S];
    // clamp (GD_GATHER_CLAMP_BITS): bit k*G+g set when that vector lies below
    // the base, so step 3b needs only bits, not the vectors' addresses
    uint32_t below = 0;
#pragma unroll
    for (int k = 0; k < S; k++) {                       // 2. fenced table addresses (ALU only)
        const int32_t jk = ((SMODE == kClamp && !kClampSafe) || okj[k]) ? j[k] : 0;   // a refused index load reads 0
        const uint64_t rt = table + (uint64_t)((int64_t)jk * (int64_t)rowbytes) + tv[k];   // vector g = 0
        bool whole = false;                             // every vector of the slot in / unwrapped
        uint64_t fr = rt;
        cnt[k] = 0;
        if constexpr (G > 1 && (TMODE == kCheck || TMODE == kMaskCount || TMODE == kClamp)) {
            whole = range_in(fd, rt, 16 * tpr * (G - 1) + 16);
        } else if constexpr (G > 1 && TMODE == kModulo) {
            fr = ft.addr(rt);                           // rt is 16-aligned: fr - base = (rt - base) mod size
            const uint64_t span = 16 * tpr * (G - 1) + 16;
            whole = !(fd.flags & kNoHoist) && span <= fd.size && fr - fd.base <= fd.size - span;
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            const uint64_t a = rt + 16 * tpr * g;
            if constexpr (TMODE == kNone || TMODE == kMask) {
                at[k][g] = ft.addr(a);
                ok[k][g] = true;
            } else if (whole) {
                at[k][g] = fr + 16 * tpr * g;
                ok[k][g] = true;
            } else if constexpr (TMODE == kClamp) {
                // as check here (an outside vector is not loaded); step 3b
                // then gives it its edge word four times (fence.cuh vld4)
                at[k][g] = a;
                ok[k][g] = (a - fd.base) <= fd.size - 16;
                cnt[k] += ok[k][g] ? 0u : 4u;
                if (((GD_GATHER_CLAMP_BITS >> G) & 1) && a < fd.base) below |= 1u << (k * G + g);
            } else {
                at[k][g] = ft.addr(a);
                ok[k][g] = ft.go_aligned(a, cnt[k], 4);
            }
        }
    }
    uint4 r[S][G];
#pragma unroll
    for (int k = 0; k < S; k++) {                       // 3. table loads
#pragma unroll
        for (int g = 0; g < G; g++) {
            if constexpr (GD_ZERO_REDIRECT && (TMODE == kCheck || (TMODE == kClamp && ((GD_GATHER_CLAMP_REDIRECT >> G) & 1)) ||
                                               (GD_GATHER_LIVE_REDIRECT && (TMODE == kNone ||
                                                  TMODE == kMask || TMODE == kMaskCount)))) {
                // refused / dead: the trusted zero block (per access at D = 32:
                // +3.8 -> +1.1 %; the predicated form stays for the other
                // modes, where the selected address measured 7-40 % slower)
                r[k][g] = ld_row(ft.ld_at(at[k][g], live[k] && ok[k][g]));
            } else {
                r[k][g] = make_uint4(0, 0, 0, 0);
                if (live[k] && ok[k][g]) r[k][g] = ld_row(at[k][g]);
            }
        }
        if (live[k]) nv += cnt[k];
    }
    if constexpr (TMODE == kClamp) {                    // 3b. rare: outside vectors, after every load issued
#ifndef GD_GATHER_CLAMP_FIX_BRANCH
#define GD_GATHER_CLAMP_FIX_BRANCH 0x4
#endif
        // (bit G of CLAMP_FIX_BRANCH: one branch around the whole fix-up, taken
        // only when some vector of the thread lies outside; else predicated
        // edge-word loads per vector, which every warp issues.  On at G = 2
        // with CLAMP_BITS (without them ptxas spills within the 6-CTA
        // register budget); off at G = 1 (spills).  Before it the D = 64 clamp
        // gather stayed +6-11 % over its twin: index loads from a safe word,
        // no warp sync, table loads from the zero block all measured 6-47 %,
        // tools/r02_iter11.sh)
        bool anyout = !((GD_GATHER_CLAMP_FIX_BRANCH >> G) & 1);
#pragma unroll
        for (int k = 0; k < S; k++)
#pragma unroll
            for (int g = 0; g < G; g++) anyout = anyout || (live[k] && !ok[k][g]);
        if (anyout) {
#pragma unroll
            for (int k = 0; k < S; k++) {
#pragma unroll
                for (int g = 0; g < G; g++) {
                    if (live[k] && !ok[k][g]) {
                        const uint64_t e = ((GD_GATHER_CLAMP_BITS >> G) & 1)
                                               ? (((below >> (k * G + g)) & 1u) ? fd.base : fd.base + fd.size - 4)
                                               : ft.edge4(at[k][g]);
                        const uint32_t w = ld_tab(e);
                        r[k][g] = make_uint4(w, w, w, w);
                    }
                }
            }
        }
    }
    uint64_t fo_prev = 0, ao_prev = 0;
#pragma unroll
    for (int k = 0; k < S; k++) {                       // 4. output stores
        if (live[k]) {
            if constexpr (SMODE == kModulo) {
                // live[] is a prefix, so k == 0 is the first store of the walk
                const uint64_t f0 = (k == 0 || !walk) ? fo.addr(ov[k]) : fo.step_up(fo_prev, ov[k] - ao_prev);
                fo_prev = f0;
                ao_prev = ov[k];
#pragma unroll
                for (int g = 0; g < G; g++)
                    st_out(g == 0 ? f0 : (walk ? fo.step_up(f0, 16 * tpr * g) : fo.addr(ov[k] + 16 * tpr * g)),
                           r[k][g]);
            } else {
#pragma unroll
                for (int g = 0; g < G; g++) {
                    vst4<SMODE, decltype(st_out), decltype(st_w), false>(fo, ov[k] + 16 * tpr * g, r[k][g], nv,
                                                                          st_out, st_w);
                }
            }
        }
    }
}

// CTAs per SM: the row gather is bound by loads in flight (5 CTAs measured
// 27-41 % slower than 6 at D = 32 / 64).  8 (32 registers, the unfenced
// twin's occupancy) wherever ptxas fits the mode in 32 registers with no
// local memory; modulo (it spills at 32 for G = 1 / 2) and clamp need more
// (6; clamp with G = 4: 5, which loses nothing there, D >= 128).
#ifndef GD_GATHERR_MINB8
#define GD_GATHERR_MINB8 1
#endif
constexpr int gatherr_minb(int mode, int g) {
    return mode == kClamp ? (g == 4 ? 5 : 6) : (!GD_GATHERR_MINB8 || mode == kModulo) ? 6 : 8;
}
template <int MODE, int G, bool P2>
__global__ void __launch_bounds__(kThreads, gatherr_minb(MODE, G)) k_gatherR(const __grid_constant__ FenceDesc fd, uint64_t out,
                                                      uint64_t table, uint64_t idx, uint64_t nslots, uint32_t tpr,
                                                      uint64_t dv) {
    constexpr uint64_t ch = (uint64_t)kThreads * (4 / G);
    uint32_t nv = 0;
    const uint64_t c0 = (uint64_t)blockIdx.x * ch, s0 = c0 + threadIdx.x;
    if constexpr (hoistable(MODE)) {     // streams hoisted per CTA; table rows per slot
        const uint64_t cn = nslots > c0 ? (nslots - c0 < ch ? nslots - c0 : ch) : 0;
        const uint64_t r0 = row_of<P2>(c0, tpr, dv);                   // rows this CTA touches
        const uint64_t nr = cn ? row_of<P2>(c0 + cn - 1, tpr, dv) - r0 + 1 : 0;
        const uint64_t rb = 16ull * tpr * G;
        if (cn && range_in(fd, idx + 4 * r0, 4 * nr) && range_in(fd, out + rb * r0, rb * nr))
            gatherr_chunk<kNone, MODE, G, P2>(fd, out, table, idx, s0, nslots, tpr, dv, nv);
        else
            gatherr_chunk<MODE, MODE, G, P2>(fd, out, table, idx, s0, nslots, tpr, dv, nv);
    } else {
        gatherr_chunk<MODE, MODE, G, P2>(fd, out, table, idx, s0, nslots, tpr, dv, nv);
    }
    if constexpr (counts(MODE)) flush_violations_cta(nv, fd.viol);
}

// ---------------------------------------------------------------------------
// K4: table[sext(idx[i])] += src[i] (u32).  The read-modify-write is one
// fenced access (atomics instrumented like stores) issued as a
// no-return RED.E.ADD.
// ---------------------------------------------------------------------------
// CLAMP: every clamped RMW lands on one of the two edge words.  The thread
// adds them up (u32 addition is associative and commutative, so the final
// words are the same) and the CTA issues one atomic per edge (edge_flush).
struct EdgeSums {
    uint32_t lo = 0, hi = 0;
    bool alo = false, ahi = false;
};

template <int MODE>
__device__ __forceinline__ void fenced_red(const Fence<MODE, 4> &f4, uint64_t table, int32_t j, uint32_t v,
                                           uint32_t &nv, EdgeSums &es) {
    const uint64_t a = row_addr(table, j);
    if constexpr (MODE == kClamp) {
        if (f4.inside(a)) {
            atomicAdd(reinterpret_cast<unsigned int *>(a), v);
        } else {
            nv++;
            if (a < f4.base) {
                es.lo += v;
                es.alo = true;
            } else {
                es.hi += v;
                es.ahi = true;
            }
        }
    } else {
        if (f4.go(a, nv, 1)) atomicAdd(reinterpret_cast<unsigned int *>(f4.addr(a)), v);
    }
}

// CTA-wide sums of the clamped RMWs, one atomic per edge word.  All threads.
__device__ __forceinline__ void edge_flush(const FenceDesc &fd, const EdgeSums &es) {
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

template <int SMODE, int TMODE>
__device__ __forceinline__ void scatter_chunk(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src,
                                              uint64_t v0, uint64_t nvec, uint32_t &nv, EdgeSums &es) {
    const Fence<SMODE, 16> f16(fd);
    const Fence<TMODE, 4> f4(fd);
    uint4 j[kU];
    uint4 s[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const uint64_t v = v0 + u * kThreads;
        j[u] = make_uint4(0, 0, 0, 0);
        s[u] = make_uint4(0, 0, 0, 0);
        if (v < nvec) {
            j[u] = vld4(f16, idx + 16 * v, nv, ld_u4, ld_w);
            s[u] = vld4(f16, src + 16 * v, nv, ld_u4, ld_w);
        }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        if (v0 + u * kThreads < nvec) {
            fenced_red<TMODE>(f4, table, (int32_t)j[u].x, s[u].x, nv, es);
            fenced_red<TMODE>(f4, table, (int32_t)j[u].y, s[u].y, nv, es);
            fenced_red<TMODE>(f4, table, (int32_t)j[u].z, s[u].z, nv, es);
            fenced_red<TMODE>(f4, table, (int32_t)j[u].w, s[u].w, nv, es);
        }
    }
}

// 4 CTAs per SM in every mode (64 registers, no local memory)
template <int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_scatter(const __grid_constant__ FenceDesc fd, uint64_t table,
                                                      uint64_t idx, uint64_t src, uint64_t nvec, uint32_t tail) {
    uint32_t nv = 0;
    EdgeSums es;
    const uint64_t c0 = (uint64_t)blockIdx.x * kChunk, v0 = c0 + threadIdx.x;
    if constexpr (hoistable(MODE)) {     // streams hoisted; random RMWs fenced
        const uint64_t cn = chunk_len(nvec, c0);
        if (cn && range_in(fd, idx + 16 * c0, 16 * cn) && range_in(fd, src + 16 * c0, 16 * cn))
            scatter_chunk<kNone, MODE>(fd, table, idx, src, v0, nvec, nv, es);
        else
            scatter_chunk<MODE, MODE>(fd, table, idx, src, v0, nvec, nv, es);
    } else {
        scatter_chunk<MODE, MODE>(fd, table, idx, src, v0, nvec, nv, es);
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) {
        const Fence<MODE, 4> f4(fd);
        const uint64_t ai = idx + 16 * nvec + 4 * threadIdx.x, as = src + 16 * nvec + 4 * threadIdx.x;
        int32_t j = 0;
        uint32_t s = 0;
        if (f4.go(ai, nv, 1)) j = *reinterpret_cast<const int32_t *>(f4.addr(ai));
        if (f4.go(as, nv, 1)) s = *reinterpret_cast<const uint32_t *>(f4.addr(as));
        fenced_red<MODE>(f4, table, j, s, nv, es);
    }
    if constexpr (MODE == kClamp) edge_flush(fd, es);
    if constexpr (counts(MODE)) flush_violations(nv, fd.viol);
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
        // G: the most vectors per slot that still leaves >= 8 slots (128 B,
        // one full line) per row per warp instruction -- narrower pieces
        // multiply the L2 requests per byte (measured: D = 8 at G = 2 and
        // D = 32 at G = 4 lose 35% / 10%)
        const uint32_t vpr = D / 4;
        const uint32_t G = (vpr % 4 == 0 && vpr >= 32) ? 4 : (vpr % 2 == 0 && vpr >= 16) ? 2 : 1, tpr = vpr / G;
        const uint64_t nslots = n * tpr, per_cta = (uint64_t)kThreads * (4 / G);
        const unsigned grid = (unsigned)(nslots ? (nslots + per_cta - 1) / per_cta : 1);
        if ((tpr & (tpr - 1)) == 0) {
            const uint64_t sh = (uint64_t)__builtin_ctz(tpr);
            if (G == 4) k_gatherR<MODE, 4, true><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, sh);
            else if (G == 2) k_gatherR<MODE, 2, true><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, sh);
            else k_gatherR<MODE, 1, true><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, sh);
        } else {
            const uint64_t inv = recip64(tpr);          // tpr >= 3
            if (G == 4) k_gatherR<MODE, 4, false><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, inv);
            else if (G == 2) k_gatherR<MODE, 2, false><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, inv);
            else k_gatherR<MODE, 1, false><<<grid, kThreads, 0, s>>>(fd, out, table, idx, nslots, tpr, inv);
        }
    } else {
        const uint64_t N = n * D;                       // (n * D < 2^64: the API bounds the output bytes)
        if (N) k_gatherE<MODE><<<(unsigned)((N + kEChunk - 1) / kEChunk), kThreads, 0, s>>>(
                   fd, out, table, idx, N, D, recip64(D), (uint32_t)(kThreads / D), (uint32_t)(kThreads % D));
    }
    return cudaGetLastError();
}

template <int MODE>
cudaError_t scatter_t(const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n, cudaStream_t s) {
    // large scatters: radix-partitioned by partition slice (k_scatter.cu);
    // the direct kernel takes the rest, or the n % 4 tail
    const cudaError_t b = launch_scatter_bucketed(MODE, fd, table, idx, src, n, s);
    if (b == cudaSuccess) {
        if (n % 4 == 0) return cudaSuccess;
        const uint64_t done = n / 4 * 16;
        k_scatter<MODE><<<1, kThreads, 0, s>>>(fd, table, idx + done, src + done, 0, (uint32_t)(n % 4));
        return cudaGetLastError();
    }
    if (b != cudaErrorNotSupported) return b;
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
        case kMaskCount: return gather_t<kMaskCount>(fd, out, table, idx, n, D, s, g);
        case kClamp: return gather_t<kClamp>(fd, out, table, idx, n, D, s, g);
        default: return gather_t<kCheck>(fd, out, table, idx, n, D, s, g);
    }
}

cudaError_t launch_scatter(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src, uint64_t n,
                           cudaStream_t s, const Geom &) {
    switch (mode) {
        case kNone: return scatter_t<kNone>(fd, table, idx, src, n, s);
        case kMask: return scatter_t<kMask>(fd, table, idx, src, n, s);
        case kModulo: return scatter_t<kModulo>(fd, table, idx, src, n, s);
        case kMaskCount: return scatter_t<kMaskCount>(fd, table, idx, src, n, s);
        case kClamp: return scatter_t<kClamp>(fd, table, idx, src, n, s);
        default: return scatter_t<kCheck>(fd, table, idx, src, n, s);
    }
}

}  // namespace gd
