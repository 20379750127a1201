// k_stencil_tma.cu -- K5 v2: the fenced 5-point Jacobi sweep with both
// operands staged by TMA for sm_100a.
//
// The fence lives in the two tensor maps (reading R-TMA, oracle
// or_stencil_tma): `in` is H rows x W floats and `out` the H-1 rows x W-1
// columns that can hold interior points, each with its base fenced like a
// 16-byte access and its row count clamped so that the last byte of its last
// row lies inside the partition (desc_rows, gemm.cu).  TMA fills rows past the
// `in` extent with zeros and clips stores past the `out` extent (and past
// column W-2 / row H-2: the out map ends there), so no kernel instruction
// computes a global address at all.
//
// One CTA per tile of kBH rows x kBW output columns: one TMA load of the
// (kBH+2) x 256-float halo box, a register sliding window down one column per
// thread (3 shared loads per point), the results staged in shared memory and
// written back with one TMA store.  TMA needs every box to start 16-byte
// aligned in its innermost dimension, so tiles start at output columns
// k * kBW (kBW % 4 == 0) and the halo box 4 columns earlier; the tile holding
// column 0 (a boundary column, never written) first loads its out box through
// the same fenced map, so the store writes column 0's bytes back unchanged.
// TMA also stores whole 16-byte chunks of a row even past the map's width, so
// the out map stops at the last whole chunk before column W-1 and the at most
// three interior columns after it are stored by their threads directly, under
// the same descriptor rule (fenced base, rows below the row count).
// Six CTAs per SM (34 KB of shared memory each) keep loads, compute and
// stores of different tiles overlapped.
#include <cuda.h>

#include <cstring>

#include "dispatch.h"
#include "drv.h"

namespace gd {
namespace {

constexpr int kBW = 248;                 // output columns per tile (multiple of 4: 16-byte aligned starts)
constexpr int kBH = 16;                  // interior rows per tile (probe: 8 / 16 / 24 / 32 -> 6585 / 6878 / 6732 / 6164 GB/s)
constexpr int kInW = 256, kInH = kBH + 2;
constexpr int kThreads = 256;
constexpr uint32_t kInBytes = kInW * kInH * 4;       // 18,432
constexpr uint32_t kOutBytes = kBW * kBH * 4;        // 15,872
constexpr uint32_t kSmem = kInBytes + kOutBytes + 16 + 128;     // + 2 mbarriers + alignment slack

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ unsigned int g_stencil_tma_timeout = 0;   // set if a bounded wait expired

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait for phase 0 of `bar`; give up after ~2 s and raise the device flag
// (gd_device_flags bit 1) instead of hanging every tenant of the shared
// context on a TMA load that never completes.
__device__ __forceinline__ bool mbar_wait0(uint32_t bar) {
    uint64_t t0 = 0;
    for (uint32_t spin = 0;; spin++) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar)
            : "memory");
        if (done) return true;
        if ((spin & 1023u) == 0) {
            const uint64_t now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 2000000000ull) break;
        }
    }
    atomicExch(&g_stencil_tma_timeout, 1u);
    return false;
}

__global__ void __launch_bounds__(kThreads) k_stencil_tma(const __grid_constant__ CUtensorMap tmIn,
                                                          const __grid_constant__ CUtensorMap tmOut, float c0,
                                                          float c1, uint32_t gx, uint32_t w1, uint32_t W,
                                                          uint64_t outp, uint64_t pitch, uint64_t rout) {
    extern __shared__ __align__(128) uint8_t smem[];                  // typed shared: LDS / STS below
    float *tin = reinterpret_cast<float *>(smem);                      // [kInH][kInW]
    float *tout = reinterpret_cast<float *>(smem + kInBytes);          // [kBH][kBW]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kInBytes + kOutBytes);    // [0] in box, [1] out box
    const uint32_t bx = blockIdx.x % gx, by = blockIdx.x / gx;
    const int X = (int)bx * kBW, y0 = 1 + (int)by * kBH;              // tile: out columns X.., rows y0..
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmIn) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(kInBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(smem_u32(tin)), "l"(&tmIn), "r"(X - 4), "r"(y0 - 1), "r"(smem_u32(&bar[0]))
            : "memory");
        if (bx == 0 && w1 > 0) {                                       // column 0 must come back unchanged
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[1])),
                         "r"(kOutBytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(smem_u32(tout)), "l"(&tmOut), "r"(0), "r"(y0), "r"(smem_u32(&bar[1]))
                : "memory");
        }
    }
    __syncthreads();                                                   // barriers initialised before anyone waits
    bool ready = mbar_wait0(smem_u32(&bar[0]));
    if (bx == 0 && w1 > 0) ready = mbar_wait0(smem_u32(&bar[1])) && ready;
    // a timed-out tile computes and stores nothing (its shared memory is not
    // the data); the CTA-uniform decision keeps the barrier below reachable
    ready = __syncthreads_and(ready);
    const int c = threadIdx.x;                                         // out column X + c
    const uint32_t x = (uint32_t)X + (uint32_t)c;
    if (ready && c < kBW && x != 0) {
        // halo box column c + 4 is out column X + c
        float n = tin[c + 4], cc = tin[kInW + c + 4];
#pragma unroll 4
        for (int r = 0; r < kBH; r++) {
            const float s = tin[(r + 2) * kInW + c + 4];
            const float w = tin[(r + 1) * kInW + c + 3], e = tin[(r + 1) * kInW + c + 5];
            const float ns = __fadd_rn(n, s);
            const float we = __fadd_rn(w, e);
            const float o = __fmaf_rn(c1, __fadd_rn(ns, we), __fmul_rn(c0, cc));
            tout[r * kBW + c] = o;
            // columns w1..W-2: past the last whole 16-byte chunk of the out
            // map's rows (TMA stores whole chunks), stored directly under the
            // same descriptor rule: fenced base, rows below the row count
            if (x >= w1 && x + 2 <= W && (uint64_t)(y0 + r) < rout)
                *reinterpret_cast<float *>(outp + 4 * ((uint64_t)(y0 + r) * pitch + x)) = o;
            n = cc;
            cc = s;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");      // generic writes -> TMA reads
    __syncthreads();
    if (ready && threadIdx.x == 0 && (uint32_t)X < w1) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmOut),
                     "r"(smem_u32(tout)), "r"(X), "r"(y0)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");    // smem stays valid until read
    }
}

__global__ void k_add_count(unsigned long long *viol, unsigned long long n) { atomicAdd(viol, n); }

bool map_f32(CUtensorMap *m, uint64_t addr, uint64_t cols, uint64_t rows, uint64_t pitch_floats, uint32_t box_w,
             uint32_t box_h, bool store) {
    std::memset(m, 0, sizeof(*m));
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch_floats * 4};
    const cuuint32_t box[2] = {box_w, box_h};
    const cuuint32_t es[2] = {1, 1};
    return drv().TensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)addr, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      store ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Read-and-clear the device timeout flag of k_stencil_tma.
unsigned int stencil_tma_timeout_flag() {
    unsigned int v = 0, z = 0;
    cudaMemcpyFromSymbol(&v, g_stencil_tma_timeout, sizeof(v));
    cudaMemcpyToSymbol(g_stencil_tma_timeout, &z, sizeof(z));
    return v;
}

// Everything stencil_tma_dispatch might do outside a stream (graph capture).
gd_status stencil_tma_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size) {
    static bool attr =
        cudaFuncSetAttribute(k_stencil_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) == cudaSuccess;
    if (!attr) return cuda_status(cudaErrorInvalidValue);
    const uint64_t H = w.u32[0], W = w.u32[1], pitch = w.u64[0];
    uint64_t f;
    return desc_rows(w.mode, base, size, w.ptr[1], H, 4 * W, 4 * pitch, &f) == 0 ? ensure_zero_row(a, 2 * W)
                                                                                  : GD_OK;
}

gd_status stencil_tma_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t s,
                               const Geom &) {
    const uint64_t H = w.u32[0], W = w.u32[1], pitch = w.u64[0];
    const uint64_t out = w.ptr[0], in = w.ptr[1];
    uint64_t inf, outf;
    uint64_t rin = desc_rows(w.mode, base, size, in, H, 4 * W, 4 * pitch, &inf);
    const uint64_t rout = desc_rows(w.mode, base, size, out, H - 1, 4 * (W - 1), 4 * pitch, &outf);
    if (counts((int)w.mode)) {
        // the rows check would refuse, once per operand (oracle or_stencil_tma)
        uint64_t t;
        const unsigned long long nv = (H - desc_rows(kCheck, base, size, in, H, 4 * W, 4 * pitch, &t)) +
                                      ((H - 1) - desc_rows(kCheck, base, size, out, H - 1, 4 * (W - 1), 4 * pitch, &t));
        if (nv) {
            k_add_count<<<1, 1, 0, s>>>(a->d_stats + (uint64_t)w.tenant * GD_NUM_KINDS + GD_KIND_STENCIL, nv);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_status(e);
        }
    }
    if (rout == 0) return GD_OK;                        // nothing may be stored
    gd_status st = stencil_tma_prepare(a, w, base, size);
    if (st != GD_OK) return st;
    uint64_t in_pitch = pitch;
    if (rin == 0) {                                     // no readable row: every input reads as zero
        st = ensure_zero_row(a, 2 * W, &inf);
        if (st != GD_OK) return st;
        rin = 1;
        in_pitch = (W + 3) & ~3ull;
    }
    CUtensorMap tmIn, tmOut;
    // the out map covers whole 16-byte chunks only (TMA stores them whole):
    // columns 0..w1-1; the at most 3 interior columns past it are stored directly
    const uint64_t w1 = (W - 1) & ~3ull;
    std::memset(&tmOut, 0, sizeof(tmOut));
    if (!map_f32(&tmIn, inf, W, rin, in_pitch, kInW, kInH, false) ||
        (w1 > 0 && !map_f32(&tmOut, outf, w1, rout, pitch, kBW, kBH, true)))
        return GD_ERR_UNSUPPORTED;
    const uint64_t gx = (W - 1 + kBW - 1) / kBW, gy = (H - 2 + kBH - 1) / kBH;     // out columns 0..W-2
    if (gx * gy > 0x7FFFFFFFull) return GD_ERR_UNSUPPORTED;
    k_stencil_tma<<<(unsigned)(gx * gy), kThreads, kSmem, s>>>(tmIn, tmOut, w.f32[0], w.f32[1], (uint32_t)gx,
                                                                (uint32_t)w1, (uint32_t)W, outf, pitch, rout);
    return cuda_status(cudaGetLastError());
}

}  // namespace gd
