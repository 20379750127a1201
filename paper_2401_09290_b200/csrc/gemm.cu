// gemm.cu -- fenced bf16 GEMM C = A . B^T on the sm_100a tensor cores
// (SURVEY.md §2.7 K6, §8(a) a9).
//
// The fence of a TMA path lives in the tensor maps (there is no per-element
// address to fence once TMA moves whole tiles):
//   MASK : the operand's global address is fenced like a 16-byte access,
//          A' = (A & ((size-1) & ~15)) | base (Listing 1 lines 26-28);
//   CHECK: A' = A if A is a legal 16-byte-aligned address of the partition,
//          otherwise the operand has no rows;
//   then the row extent is clamped so the last byte of the last row lies
//   below end: rows = min(R, floor((end - A' - rowbytes) / stride) + 1).
// TMA zero-fills rows at or past that extent, so clamped rows of A / B read
// as zeros; rows of C at or past its extent are not stored.  Check mode
// counts the refused rows, (M - rowsA) + (N - rowsB) + (M - rowsC).
// Same principle as the per-access fence; sm_86 has no
// TMA, so the paper has no passage for it (reading R-TMA).
//
// Kernel (persistent, one CTA per SM, 128 x 256 output tiles in a grouped
// raster so the tiles in flight share A and B panels in L2):
//   warp 0     TMA producer: one elected thread, 4-stage mbarrier ring of
//              48 KB stages (A 128x64, B 256x64 bf16, 128-byte swizzle);
//   warp 1     MMA issuer: one thread, tcgen05.mma.cta_group::1.kind::f16
//              M=128 N=256 K=16, fp32 accumulators in TMEM, double-buffered
//              (2 x 256 columns) so the epilogue of tile i overlaps the
//              mainloop of tile i+1;
//   warp 2     TMEM allocator (512 columns);
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> bf16 -> shared-memory staging
//              -> TMA store through C's tensor map, whose extent is the
//              descriptor-fenced row count (TMA drops rows past it), then
//              release the accumulator.
// All waits are bounded: a kernel that cannot make progress sets a device
// error word and exits instead of hanging the shared context.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstring>

#include "dispatch.h"
#include "drv.h"

namespace gd {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, ACC = 2;
constexpr uint32_t A_BYTES = BM * BK * 2;          // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2;          // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t EPI_CHUNK_BYTES = 32 * 32 * 2;              // C staging chunk: 32 x 32 bf16
constexpr uint32_t EPI_BYTES = 4 * 2 * EPI_CHUNK_BYTES;        // 4 epilogue warps x double buffer
constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int THREADS = 256;
constexpr uint32_t TMEM_COLS = ACC * BN;           // 512
// raster group (m-blocks).  With forward-only K loops, groups 4 / 8 / 16 / 32
// read 1.52 / 1.10 / 1.25 / 2.27 GB per 8192^3 launch (8 best,
// profiles/r01_gemm_group_probe.txt); with K-alternating waves (krev) a group
// of 16 reads 0.92 GB and runs fastest (profiles/r01_gemm_krev_probe.txt).
// Under the 1 kW power cap sustained TFLOP/s follow the DRAM traffic.
constexpr uint32_t GROUP_M = 16;

// instruction descriptor: D f32, A/B bf16, both K-major, N=256, M=128
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ unsigned int g_gemm_timeout = 0;        // set if a bounded wait expired

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait for the phase of `bar` with parity `parity`; give up after ~2 s (a
// stalled pipeline is a bug: report it instead of hanging every tenant).
__device__ __forceinline__ bool mbar_wait(uint32_t bar, uint32_t parity) {
    uint64_t t0 = 0;
    for (uint32_t spin = 0;; spin++) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return true;
        if ((spin & 1023u) == 0) {
            const uint64_t now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 2000000000ull) break;
        }
    }
    atomicExch(&g_gemm_timeout, 1u);
    return false;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    // UMMA shared-memory descriptor, K-major, 128-byte swizzle: start >> 4,
    // LBO = 16 B (unused), SBO = 1024 B (8 rows x 128 B), version 1, layout 2.
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// ---------------------------------------------------------------------------
// Epilogue: one 32-row x 32-column chunk of the accumulator (the warp's TMEM
// lanes) -> bf16 -> shared-memory staging -> TMA store through the C tensor
// map.  The map's extent is the descriptor-fenced row count of C, so rows at
// or past it (and columns >= N) are dropped by the TMA unit itself: the C
// fence lives in the tensor map exactly like A's and B's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// chunk index c of this warp's tile: waits (lane 0) for the store that last
// used the staging buffer, writes the bf16 rows, issues the TMA store.
__device__ __forceinline__ void epi_store_chunk(const CUtensorMap *tmC, uint32_t stage_base, uint32_t chunk_no,
                                                const uint32_t (&v)[32], uint32_t lane, int col0, int row0) {
    const uint32_t buf = stage_base + (chunk_no & 1) * EPI_CHUNK_BYTES;
    if (chunk_no >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    uint32_t p[16];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
        p[e] = *reinterpret_cast<uint32_t *>(&h);
    }
    // row `lane` is 64 bytes: four 16-byte pieces, written in a lane-rotated
    // order so a warp's 16-byte stores spread over all banks (4 wavefronts)
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const uint32_t qq = (q + (lane >> 1)) & 3;
        const uint32_t a0 = qq == 0 ? p[0] : qq == 1 ? p[4] : qq == 2 ? p[8] : p[12];
        const uint32_t a1 = qq == 0 ? p[1] : qq == 1 ? p[5] : qq == 2 ? p[9] : p[13];
        const uint32_t a2 = qq == 0 ? p[2] : qq == 1 ? p[6] : qq == 2 ? p[10] : p[14];
        const uint32_t a3 = qq == 0 ? p[3] : qq == 1 ? p[7] : qq == 2 ? p[11] : p[15];
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 64 + qq * 16), "r"(a0), "r"(a1),
                     "r"(a2), "r"(a3)
                     : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmC),
                     "r"(buf), "r"(col0), "r"(row0)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}

__device__ __forceinline__ void epi_drain(uint32_t lane) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
}

// grouped raster: tiles t = 0..tm*tn-1 -> (m_blk, n_blk)
__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t tm, uint32_t tn, uint32_t group, uint32_t &mb,
                                            uint32_t &nb) {
    const uint32_t per_group = group * tn;
    const uint32_t g = t / per_group, first = g * group;
    const uint32_t gm = (tm - first < group) ? tm - first : group;
    const uint32_t r = t - g * per_group;
    mb = first + r % gm;
    nb = r / gm;
}

__global__ void __launch_bounds__(THREADS, 1)
k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
       const __grid_constant__ CUtensorMap tmC, uint32_t K, uint32_t tm, uint32_t tn, uint32_t group) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *epi = smem + STAGES * STAGE_BYTES;                    // C staging, 16 KB
    uint64_t *bars = (uint64_t *)(epi + EPI_BYTES);
    uint64_t *full = bars, *empty = bars + STAGES;
    uint64_t *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + ACC;
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * STAGES + 2 * ACC);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nkb = K / BK, ntiles = tm * tn;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < STAGES; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        for (int a = 0; a < ACC; a++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[a])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&tempty[a])));   // 4 epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        uint32_t it = 0;
        bool alive = true;
        for (uint32_t t = blockIdx.x; t < ntiles && alive; t += gridDim.x) {
            uint32_t mb, nb;
            tile_coords(t, tm, tn, group, mb, nb);
            for (uint32_t kb = 0; kb < nkb; kb++, it++) {
                const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                if (!mbar_wait(smem_u32(&empty[s]), ph ^ 1)) { alive = false; break; }
                const uint32_t fb = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE_BYTES)
                             : "memory");
                const uint32_t sa = smem_u32(smem + s * STAGE_BYTES), sb = sa + A_BYTES;
                const int kc = (int)(kb * BK);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                    ::"r"(sa), "l"(&tmA), "r"(fb), "r"(kc), "r"((int)(mb * BM))
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                    ::"r"(sb), "l"(&tmB), "r"(fb), "r"(kc), "r"((int)(nb * BN))
                    : "memory");
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        uint32_t it = 0, tl = 0;
        bool alive = true;
        for (uint32_t t = blockIdx.x; t < ntiles && alive; t += gridDim.x, tl++) {
            const uint32_t acc = tl & 1, aph = (tl >> 1) & 1;
            if (!mbar_wait(smem_u32(&tempty[acc]), aph ^ 1)) break;     // epilogue drained this accumulator
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + acc * BN;
            for (uint32_t kb = 0; kb < nkb; kb++, it++) {
                const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                if (!mbar_wait(smem_u32(&full[s]), ph)) { alive = false; break; }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sa = smem_u32(smem + s * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
                for (int k = 0; k < BK / 16; k++) {
                    const uint64_t da = sw128_desc(sa + 32 * k), db = sw128_desc(sb + 32 * k);
                    const uint32_t accum = (kb | k) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                        ::"r"(dacc), "l"(da), "l"(db), "r"(IDESC), "r"(accum)
                        : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&empty[s]))
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(smem_u32(&tfull[acc]))
                         : "memory");
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> bf16 -> smem -> TMA store ----------------
        const uint32_t wq = warp - 4;                  // TMEM lanes 32*wq .. 32*wq+31
        const uint32_t stage_base = smem_u32(epi) + wq * 2 * EPI_CHUNK_BYTES;
        uint32_t tl = 0, chunk_no = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, tl++) {
            uint32_t mb, nb;
            tile_coords(t, tm, tn, group, mb, nb);
            const uint32_t acc = tl & 1, aph = (tl >> 1) & 1;
            if (!mbar_wait(smem_u32(&tfull[acc]), aph)) break;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int row0 = (int)(mb * BM + wq * 32), n0 = (int)(nb * BN);
#pragma unroll 1
            for (int c = 0; c < BN / 32; c++) {
                uint32_t v[32];
                tmem_ld32(tmem + ((wq * 32u) << 16) + acc * BN + (uint32_t)(c * 32), v);
                if (c == BN / 32 - 1) {
                    // accumulator fully read: hand it back to the MMA warp
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc]))
                                     : "memory");
                }
                epi_store_chunk(&tmC, stage_base, chunk_no++, v, lane, n0 + c * 32, row0);
            }
        }
        epi_drain(lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// 2-SM variant: a CTA pair (cluster of 2) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 rows of A and
// its 128 rows (N half) of B, so per-SM shared-memory traffic per MMA halves
// for B -- the 1-SM kernel is shared-memory-bandwidth bound (TMA writes plus
// tensor-core operand reads of 48 KB per 512 cycles).  The leader CTA (rank
// 0) issues the MMAs; both CTAs' TMA loads complete on the leader's full
// barrier, the leader's commits multicast to both CTAs' empty / tmem-full
// barriers, and both CTAs' epilogue warps release the accumulator on the
// leader's tmem-empty barrier.  Each CTA's TMEM holds its 128 rows x 256
// fp32 columns per accumulator (2 accumulators, 512 columns).
// ---------------------------------------------------------------------------
constexpr uint32_t IDESC2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(2 * BM >> 4) << 24);
constexpr uint32_t B_HALF = BN / 2;                           // B rows staged per CTA
constexpr uint32_t STAGE2_BYTES = A_BYTES + B_HALF * BK * 2;  // 32 KB
constexpr int STAGES2 = 6;
constexpr uint32_t SMEM2_BYTES = STAGES2 * STAGE2_BYTES + EPI_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t saddr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
        const __grid_constant__ CUtensorMap tmC, uint32_t K, uint32_t tm, uint32_t tn, uint32_t group,
        uint32_t krev) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *epi = smem + STAGES2 * STAGE2_BYTES;                  // C staging, 16 KB
    uint64_t *bars = (uint64_t *)(epi + EPI_BYTES);
    uint64_t *full = bars, *empty = bars + STAGES2;
    uint64_t *tfull = bars + 2 * STAGES2, *tempty = bars + 2 * STAGES2 + ACC;
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * STAGES2 + 2 * ACC);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const uint32_t nkb = K / BK, ntiles = tm * tn;      // tm counts 256-row pair tiles

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < STAGES2; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&full[s])));    // both producers
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        for (int a = 0; a < ACC; a++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[a])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&tempty[a])));  // 2 x 4 epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        uint32_t it = 0, tl = 0;
        bool alive = true;
        for (uint32_t t = pair; t < ntiles && alive; t += npairs, tl++) {
            uint32_t mb, nb;
            tile_coords(t, tm, tn, group, mb, nb);
            const int row_a = (int)(mb * 2 * BM + rank * BM), row_b = (int)(nb * BN + rank * B_HALF);
            // krev: odd waves walk K backwards, so a wave starts on the K slices
            // the previous wave (same A panels) touched last -- still in L2
            const bool back = krev && (tl & 1);
            for (uint32_t kb = 0; kb < nkb; kb++, it++) {
                const uint32_t s = it % STAGES2, ph = (it / STAGES2) & 1;
                if (!mbar_wait(smem_u32(&empty[s]), ph ^ 1)) { alive = false; break; }
                const uint32_t fb = map_to_cta(smem_u32(&full[s]), 0);     // the leader's full barrier
                // default (.release.cta) semantics: the transaction count is all the
                // leader needs; a cluster-scope release would put a MEMBAR.GPU on
                // every stage (measured: halves tensor-pipe activity)
                asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(fb),
                             "r"(STAGE2_BYTES)
                             : "memory");
                const uint32_t sa = smem_u32(smem + s * STAGE2_BYTES), sb = sa + A_BYTES;
                const int kc = (int)((back ? nkb - 1 - kb : kb) * BK);
                asm volatile(
                    "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4}], [%2];" ::"r"(sa), "l"(&tmA), "r"(fb), "r"(kc), "r"(row_a)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4}], [%2];" ::"r"(sb), "l"(&tmB), "r"(fb), "r"(kc), "r"(row_b)
                    : "memory");
            }
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {
        // ---------------- MMA issuer (leader CTA only) ----------------
        uint32_t it = 0, tl = 0;
        bool alive = true;
        for (uint32_t t = pair; t < ntiles && alive; t += npairs, tl++) {
            const uint32_t acc = tl & 1, aph = (tl >> 1) & 1;
            if (!mbar_wait(smem_u32(&tempty[acc]), aph ^ 1)) break;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + acc * BN;
            for (uint32_t kb = 0; kb < nkb; kb++, it++) {
                const uint32_t s = it % STAGES2, ph = (it / STAGES2) & 1;
                if (!mbar_wait(smem_u32(&full[s]), ph)) { alive = false; break; }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sa = smem_u32(smem + s * STAGE2_BYTES), sb = sa + A_BYTES;
#pragma unroll
                for (int k = 0; k < BK / 16; k++) {
                    const uint64_t da = sw128_desc(sa + 32 * k), db = sw128_desc(sb + 32 * k);
                    const uint32_t accum = (kb | k) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                        ::"r"(dacc), "l"(da), "l"(db), "r"(IDESC2), "r"(accum)
                        : "memory");
                }
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                    ::"r"(smem_u32(&empty[s])), "h"((uint16_t)3)
                    : "memory");
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                ::"r"(smem_u32(&tfull[acc])), "h"((uint16_t)3)
                : "memory");
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs: own 128 rows) ----------------
        const uint32_t wq = warp - 4;
        const uint32_t stage_base = smem_u32(epi) + wq * 2 * EPI_CHUNK_BYTES;
        uint32_t tl = 0, chunk_no = 0;
        for (uint32_t t = pair; t < ntiles; t += npairs, tl++) {
            uint32_t mb, nb;
            tile_coords(t, tm, tn, group, mb, nb);
            const uint32_t acc = tl & 1, aph = (tl >> 1) & 1;
            if (!mbar_wait(smem_u32(&tfull[acc]), aph)) break;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int row0 = (int)(mb * 2 * BM + rank * BM + wq * 32);
            const int n0 = (int)(nb * BN);
#pragma unroll 1
            for (int c = 0; c < BN / 32; c++) {
                uint32_t v[32];
                tmem_ld32(tmem + ((wq * 32u) << 16) + acc * BN + (uint32_t)(c * 32), v);
                if (c == BN / 32 - 1) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        const uint32_t tb = map_to_cta(smem_u32(&tempty[acc]), 0);   // the leader's barrier
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tb)
                                     : "memory");
                    }
                }
                epi_store_chunk(&tmC, stage_base, chunk_no++, v, lane, n0 + c * 32, row0);
            }
        }
        epi_drain(lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();                 // no CTA leaves while its peer may still signal it
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

__global__ void k_add_violations(unsigned long long *viol, unsigned long long n) { atomicAdd(viol, n); }

// 2-D bf16 tensor map: inner dim = K (contiguous), outer = rows.
bool make_map(CUtensorMap *m, uint64_t addr, uint64_t K, uint64_t rows, uint64_t ld, uint32_t box_rows) {
    const cuuint64_t dims[2] = {K, rows};
    const cuuint64_t strides[1] = {ld * 2};
    const cuuint32_t box[2] = {BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = drv().TensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)addr, dims, strides, box,
                                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// C's store map: N columns x rowsC rows (the descriptor-fenced extent), boxes
// of 32 x 32 bf16, no swizzle (the staging tile is plain row-major).
bool make_map_c(CUtensorMap *m, uint64_t addr, uint64_t N, uint64_t rows, uint64_t ld) {
    const cuuint64_t dims[2] = {N, rows};
    const cuuint64_t strides[1] = {ld * 2};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = drv().TensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)addr, dims, strides, box,
                                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

// Host side of the descriptor fence (reading R-TMA).
uint64_t desc_rows(int mode, uint64_t base, uint64_t size, uint64_t p, uint64_t rows, uint64_t rowbytes,
                   uint64_t stride, uint64_t *pf) {
    *pf = p;
    if (mode == kNone) return rows;
    uint64_t f;
    if (mode == kMask || mode == kMaskCount) {
        f = (p & ((size - 1) & ~15ull)) | base;
    } else if (mode == kModulo) {
        f = base + (((p - base) % size) & ~15ull);
    } else if (mode == kClamp) {                        // largest legal 16-byte address <= p
        f = p < base ? base : (p - base > size - 16 ? base + size - 16 : p & ~15ull);
    } else {
        if (p - base > size - 16 || (p & 15)) return 0;   // not a legal 16-byte access of the partition
        f = p;
    }
    *pf = f;
    const uint64_t end = base + size;
    if (end - f < rowbytes) return 0;
    const uint64_t valid = (end - f - rowbytes) / stride + 1;
    return valid < rows ? valid : rows;
}

// Trusted all-zero row of >= 2K bytes outside every partition (allocating
// synchronises, so graph capture calls gemm_prepare first).
gd_status ensure_zero_row(gd_arena *a, uint64_t K, uint64_t *zp) {
    std::lock_guard<std::mutex> lk(a->mu);
    if (a->zero_bytes < 2ull * K) {
        // grow-only: the outgrown row stays allocated (a captured graph's
        // tensor map may still point at it) until the arena is destroyed
        void *nb = nullptr;
        cudaError_t e = cudaMalloc(&nb, 2ull * K);
        if (e == cudaSuccess) e = cudaMemset(nb, 0, 2ull * K);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            if (nb) cudaFree(nb);
            return cuda_status(e);
        }
        if (a->zero_buf) a->zero_retired.push_back(a->zero_buf);
        a->zero_buf = nb;
        a->zero_bytes = 2ull * K;
    }
    if (zp) *zp = (uint64_t)a->zero_buf;
    return GD_OK;
}

// Everything gemm_dispatch might need to do outside a stream (one-time
// function attributes, the zero row), so that it can run under capture.
gd_status gemm_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size) {
    static bool attr = [] {
        return cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) == cudaSuccess &&
               cudaFuncSetAttribute(k_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES) == cudaSuccess;
    }();
    if (!attr) return cuda_status(cudaErrorInvalidValue);
    const uint32_t M = w.u32[0], N = w.u32[1], K = w.u32[2];
    uint64_t f;
    const uint64_t rA = desc_rows(w.mode, base, size, w.ptr[1], M, 2ull * K, 2ull * w.u64[0], &f);
    const uint64_t rB = desc_rows(w.mode, base, size, w.ptr[2], N, 2ull * K, 2ull * w.u64[1], &f);
    return (rA == 0 || rB == 0) ? ensure_zero_row(a, K) : GD_OK;
}

gd_status gemm_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t s,
                        const Geom &g) {
    const uint32_t M = w.u32[0], N = w.u32[1], K = w.u32[2];
    const uint64_t lda = w.u64[0], ldb = w.u64[1], ldc = w.u64[2];
    uint64_t Af, Bf, Cf;
    uint64_t rA = desc_rows(w.mode, base, size, w.ptr[1], M, 2ull * K, 2ull * lda, &Af);
    uint64_t rB = desc_rows(w.mode, base, size, w.ptr[2], N, 2ull * K, 2ull * ldb, &Bf);
    const uint64_t rC = desc_rows(w.mode, base, size, w.ptr[0], M, 2ull * N, 2ull * ldc, &Cf);
    if (counts((int)w.mode)) {
        // counted as check mode would refuse them: rows of each operand not
        // wholly inside the partition at their unfenced address
        uint64_t t;
        const unsigned long long nv = (M - desc_rows(kCheck, base, size, w.ptr[1], M, 2ull * K, 2ull * lda, &t)) +
                                      (N - desc_rows(kCheck, base, size, w.ptr[2], N, 2ull * K, 2ull * ldb, &t)) +
                                      (M - desc_rows(kCheck, base, size, w.ptr[0], M, 2ull * N, 2ull * ldc, &t));
        if (nv) {
            k_add_violations<<<1, 1, 0, s>>>(a->d_stats + (uint64_t)w.tenant * GD_NUM_KINDS + GD_KIND_GEMM, nv);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_status(e);
        }
    }
    if (rC == 0) return GD_OK;                         // nothing may be stored
    uint64_t ldA = lda, ldB = ldb;
    if (rA == 0 || rB == 0) {
        // an operand with no rows reads as zeros: point its map at a trusted
        // zero row outside every partition
        uint64_t zp = 0;
        gd_status zs = ensure_zero_row(a, K, &zp);
        if (zs != GD_OK) return zs;
        if (rA == 0) { Af = zp; rA = 1; ldA = K; }
        if (rB == 0) { Bf = zp; rB = 1; ldB = K; }
    }
    CUtensorMap tmA, tmB, tmC;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    std::memset(&tmC, 0, sizeof(tmC));
    if (!make_map(&tmA, Af, K, rA, ldA, BM) || !make_map_c(&tmC, Cf, N, rC, ldc)) return GD_ERR_UNSUPPORTED;
    static bool attr = [] {
        return cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) == cudaSuccess &&
               cudaFuncSetAttribute(k_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES) == cudaSuccess;
    }();
    if (!attr) return cuda_status(cudaErrorInvalidValue);
    static const int force1 = [] {
        const char *e = getenv("GD_GEMM_1SM");
        return e && e[0] == '1';
    }();
    static const uint32_t group = [] {                 // raster group (m-blocks); tuning knob
        const char *e = getenv("GD_GEMM_GROUP");
        const int v = e ? atoi(e) : 0;
        return (uint32_t)(v > 0 ? v : GROUP_M);
    }();
    static const uint32_t krev = [] {                  // K-direction alternation per wave (default on)
        const char *e = getenv("GD_GEMM_KREV");
        return (uint32_t)(e ? atoi(e) : 1);
    }();
    if (rC >= 2 * BM && !force1 && g.sms >= 2) {
        // 2-SM path: B staged in N halves per CTA
        CUtensorMap tmB2;
        std::memset(&tmB2, 0, sizeof(tmB2));
        if (!make_map(&tmB2, Bf, K, rB, ldB, B_HALF)) return GD_ERR_UNSUPPORTED;
        const uint32_t tm = (uint32_t)((rC + 2 * BM - 1) / (2 * BM)), tn = (N + BN - 1) / BN;
        static const uint32_t sm_cap = [] {              // SMs a GEMM may hold (co-scheduling knob)
            const char *e = getenv("GD_GEMM_MAX_SMS");
            const int v = e ? atoi(e) : 0;
            return (uint32_t)(v >= 2 ? v : 1u << 30);
        }();
        const uint32_t sms = (uint32_t)g.sms < sm_cap ? (uint32_t)g.sms : sm_cap;
        const uint32_t ntiles = tm * tn, pairs_max = sms / 2;
        const uint32_t grid = 2 * (ntiles < pairs_max ? ntiles : pairs_max);
        k_gemm2<<<grid, THREADS, SMEM2_BYTES, s>>>(tmA, tmB2, tmC, K, tm, tn, group, krev);
        return cuda_status(cudaGetLastError());
    }
    if (!make_map(&tmB, Bf, K, rB, ldB, BN)) return GD_ERR_UNSUPPORTED;
    const uint32_t tm = (uint32_t)((rC + BM - 1) / BM), tn = (N + BN - 1) / BN;   // rC <= M
    const uint32_t ntiles = tm * tn;
    const uint32_t grid = ntiles < (uint32_t)g.sms ? ntiles : (uint32_t)g.sms;
    k_gemm<<<grid, THREADS, SMEM_BYTES, s>>>(tmA, tmB, tmC, K, tm, tn, group);
    return cuda_status(cudaGetLastError());
}

// Read-and-clear the device timeout flag (tests use it to detect a stalled pipeline).
unsigned int gemm_timeout_flag() {
    unsigned int v = 0, z = 0;
    cudaMemcpyFromSymbol(&v, g_gemm_timeout, sizeof(v));
    cudaMemcpyToSymbol(g_gemm_timeout, &z, sizeof(z));
    return v;
}

}  // namespace gd
