// dispatch.h -- the single validated launch path (api.cpp) and its users.
#pragma once
#include <cuda_runtime.h>

#include "arena.h"
#include "kernels.h"

namespace gd {
// Validate `w` (dry = true) or validate and issue it on `stream`.
// account = false skips the host launch counters (graph capture: the graph
// accounts at every replay); bytes_out / flops_out return the item's
// algorithmic work.
gd_status run_work(gd_arena *a, const gd_work &w, cudaStream_t stream, bool dry, bool account = true,
                   uint64_t *bytes_out = nullptr, uint64_t *flops_out = nullptr);
// Descriptor-fence the GEMM operands and launch the tcgen05 kernel (gemm.cu).
gd_status gemm_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t stream,
                        const Geom &g);
gd_status gemm_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size);
// K5 v2: the stencil with both operands staged by TMA (k_stencil_tma.cu).
gd_status stencil_tma_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t stream,
                               const Geom &g);
gd_status stencil_tma_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size);
// Trusted all-zero buffer of >= 2K bytes outside every partition (gemm.cu).
gd_status ensure_zero_row(gd_arena *a, uint64_t K);
gd_status cuda_status(cudaError_t e);
// Bounds-table snapshot of one partition: base, size and its generation
// (bumped at every allocation, so a freed-and-reused id is detected).
gd_status partition_snapshot(gd_arena *a, uint32_t id, uint64_t *base, uint64_t *size, uint64_t *gen);
}  // namespace gd
