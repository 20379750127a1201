// tma_store_probe.cu -- dev probe: which fp32 TMA store box shapes are legal.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>

__global__ void k_st(const __grid_constant__ CUtensorMap tm, int x0, int y0, int bytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 1.0f + i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                     "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(x0), "r"(y0)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

extern "C" int st_run(void *gptr, uint64_t cols, uint64_t rows, uint64_t pitch_elems, uint32_t bw, uint32_t bh,
                      int f32, int x0, int y0) {
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch_elems * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {bw, bh};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                        2, gptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1000 + (int)r;
    const int bytes = (int)(bw * bh * (f32 ? 4 : 2));
    cudaFuncSetAttribute(k_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_st<<<1, 128, bytes + 128>>>(m, x0, y0, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}
