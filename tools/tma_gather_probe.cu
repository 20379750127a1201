// tma_gather_probe.cu -- dev probe: does a TMA tile::gather4 with a chosen L2
// promotion move fewer DRAM bytes per random 4-byte gather than LSU loads
// (which cost a 128-byte line each on B200, profiles/)?  C3 shape: 2^26
// random indices into a 2^29-word table; out[i] = table[j_i].
//
// Table viewed as a 2-D tensor of 16-byte rows (4 u32); one gather4 loads the
// 4 rows j>>2 of 4 indices.  Each CTA: 128 threads stage 1024 indices in
// shared memory, one thread issues 256 gather4 (64 B each, 128-B aligned
// slots), all wait on one mbarrier, then each thread picks word j&3 and
// stores coalesced.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/libtmagather.so tools/tma_gather_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

namespace {

constexpr int kIdx = 1024;           // indices per CTA
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(kThreads) k_tg(const __grid_constant__ CUtensorMap tm, const int32_t *idx,
                                                 uint32_t *out, uint64_t n) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *rows = sm;                                    // 256 x 128 B slots (64 B used)
    int32_t *js = reinterpret_cast<int32_t *>(sm + 256 * 128);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 256 * 128 + kIdx * 4);
    const uint64_t i0 = (uint64_t)blockIdx.x * kIdx;
    for (int t = threadIdx.x; t < kIdx; t += kThreads) js[t] = (i0 + t < n) ? __ldcs(idx + i0 + t) : 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(256 * 64)
                     : "memory");
        for (int g = 0; g < 256; g++) {
            const int32_t *q = js + 4 * g;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(rows + 128 * g)),
                "l"(&tm), "r"(0), "r"(q[0] >> 2), "r"(q[1] >> 2), "r"(q[2] >> 2), "r"(q[3] >> 2),
                "r"(smem_u32(bar))
                : "memory");
        }
    }
    // wait (phase 0)
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
    for (int t = threadIdx.x; t < kIdx; t += kThreads) {
        const int g = t >> 2, r = t & 3;
        const uint32_t w = reinterpret_cast<const uint32_t *>(rows + 128 * g + 16 * r)[js[t] & 3];
        if (i0 + t < n) __stcs(out + i0 + t, w);
    }
}

__global__ void __launch_bounds__(256) k_ld(const uint32_t *table, const int32_t *idx, uint32_t *out, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (i < n) __stcs(out + i, __ldcg(table + __ldcs(idx + i)));
}

}  // namespace

// promo: 0 none, 1 64B, 2 128B, 3 256B (CU_TENSOR_MAP_L2_PROMOTION_*)
extern "C" int tg_run(int promo, uint64_t table, uint64_t rows16, uint64_t idx, uint64_t out, uint64_t n,
                      void *stream) {
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    const cuuint64_t dims[2] = {4, rows16};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {4, 1};
    const cuuint32_t es[2] = {1, 1};
    const CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void *)table, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr[promo & 3],
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1000 + (int)r;
    const int smem = 256 * 128 + kIdx * 4 + 64;
    static bool attr = cudaFuncSetAttribute(k_tg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
    if (!attr) return 999;
    k_tg<<<(unsigned)((n + kIdx - 1) / kIdx), kThreads, smem, (cudaStream_t)stream>>>(
        tm, (const int32_t *)idx, (uint32_t *)out, n);
    return (int)cudaGetLastError();
}

extern "C" int ld_run(uint64_t table, uint64_t idx, uint64_t out, uint64_t n, void *stream) {
    k_ld<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>((const uint32_t *)table,
                                                                          (const int32_t *)idx, (uint32_t *)out, n);
    return (int)cudaGetLastError();
}
