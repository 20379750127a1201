// kernels.h -- host-side launch entry points of the fenced sm_100a kernels.
// Internal to libguardian.so (the public surface is include/guardian.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "fence_desc.h"

namespace gd {

// Geometry shared by the streaming kernels: a persistent grid of
// `sms * blocks_per_sm` CTAs (~2 K threads per SM with
// x4-unrolled 128-bit accesses keeps >6 MB in flight).
struct Geom {
    int sms;
};

cudaError_t launch_copy(int mode, const FenceDesc &fd, uint64_t dst, uint64_t src, uint64_t nbytes,
                        cudaStream_t s, const Geom &g);
cudaError_t launch_saxpy(int mode, const FenceDesc &fd, float alpha, uint64_t x, uint64_t y, uint64_t n,
                         cudaStream_t s, const Geom &g);
cudaError_t launch_gather(int mode, const FenceDesc &fd, uint64_t out, uint64_t table, uint64_t idx,
                          uint64_t n, uint32_t D, cudaStream_t s, const Geom &g);
cudaError_t launch_scatter(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src,
                           uint64_t n, cudaStream_t s, const Geom &g);
// K4 v2 (k_scatter.cu): the scatter-add of the n / 4 * 4 leading updates,
// radix-partitioned by partition slice; cudaErrorNotSupported (nothing
// issued) when it does not apply.
cudaError_t launch_scatter_bucketed(int mode, const FenceDesc &fd, uint64_t table, uint64_t idx, uint64_t src,
                                    uint64_t n, cudaStream_t s);
cudaError_t launch_stencil(int mode, const FenceDesc &fd, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                           uint64_t pitch, float c0, float c1, cudaStream_t s, const Geom &g);
cudaError_t launch_fill(uint64_t base, uint64_t offset, uint64_t nbytes, uint32_t pattern, cudaStream_t s,
                        const Geom &g);

// Host side of the TMA descriptor fence (gemm.cu): rows of `rowbytes`
// bytes, `stride` apart from p, that an operand may touch; *pf = fenced start.
uint64_t desc_rows(int mode, uint64_t base, uint64_t size, uint64_t p, uint64_t rows, uint64_t rowbytes,
                   uint64_t stride, uint64_t *pf);
unsigned int gemm_timeout_flag();
unsigned int stencil_tma_timeout_flag();

}  // namespace gd
