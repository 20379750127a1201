// dispatch.h -- the single validated launch path (api.cpp) and its users.
#pragma once
#include <cuda_runtime.h>

#include "arena.h"
#include "kernels.h"

namespace gd {
// Validate `w` (dry = true) or validate and issue it on `stream`.
gd_status run_work(gd_arena *a, const gd_work &w, cudaStream_t stream, bool dry);
// Descriptor-fence the GEMM operands and launch the tcgen05 kernel (gemm.cu).
gd_status gemm_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t stream,
                        const Geom &g);
gd_status cuda_status(cudaError_t e);
}  // namespace gd
