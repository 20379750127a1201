// dispatch.h -- the single validated launch path (api.cpp) and its users.
#pragma once
#include <cuda_runtime.h>

#include "arena.h"
#include "kernels.h"

namespace gd {
// Mode bits of a launch: the fence mode (gd_mode) and the per-access flag.
constexpr uint32_t kModeMask = 0xFFu;
inline uint32_t base_mode(uint32_t m) { return m & kModeMask; }

// What an issued item did: its algorithmic work and whether it ran unfenced
// because its tenant was alone (native when solo).
struct LaunchOut {
    uint64_t bytes = 0, flops = 0;
    bool solo = false;
};
// Validate `w` (dry = true) or validate and issue it on `stream`.  The caller
// holds a->launch_mu shared (arena.h) from here until the work is enqueued.
// account = false skips the host launch counters (graph capture: the graph
// accounts at every replay).
gd_status run_work_locked(gd_arena *a, const gd_work &w, cudaStream_t stream, bool dry, bool account = true,
                          LaunchOut *out = nullptr);
// run_work_locked under its own shared hold of a->launch_mu.
gd_status run_work(gd_arena *a, const gd_work &w, cudaStream_t stream, bool dry);
// Descriptor-fence the GEMM operands and launch the tcgen05 kernel (gemm.cu).
gd_status gemm_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t stream,
                        const Geom &g);
gd_status gemm_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size);
// K5 v2: the stencil with both operands staged by TMA (k_stencil_tma.cu).
gd_status stencil_tma_dispatch(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size, cudaStream_t stream,
                               const Geom &g);
gd_status stencil_tma_prepare(gd_arena *a, const gd_work &w, uint64_t base, uint64_t size);
// Trusted all-zero buffer of >= 2K bytes outside every partition (gemm.cu);
// *zp = its address, read under the arena lock.  Grow-only: an outgrown row
// stays allocated until the arena is destroyed (captured graphs read it).
gd_status ensure_zero_row(gd_arena *a, uint64_t K, uint64_t *zp = nullptr);
gd_status cuda_status(cudaError_t e);
// Bounds-table snapshot of one partition: base, size and its generation
// (bumped at every allocation, so a freed-and-reused id is detected).
gd_status partition_snapshot(gd_arena *a, uint32_t id, uint64_t *base, uint64_t *size, uint64_t *gen);
}  // namespace gd
