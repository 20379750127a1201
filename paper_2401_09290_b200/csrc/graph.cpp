// graph.cpp -- captured multi-tenant steps (CUDA graphs).
//
// gd_graph_create records one round-robin issue of `items` (exactly what
// gd_launcher_run would issue) across `n_streams` tenant
// streams into a CUDA graph: a fork from an origin stream, every fenced
// kernel with its FenceDesc (the launch-time parameter augmentation of
// PAPER.md:175) baked in, a join.  gd_graph_launch replays the whole step
// with one host call.  A graph is only valid while the partitions it fences
// are the ones it captured: every replay compares their allocation
// generations and refuses (GD_ERR_UNKNOWN_PARTITION) if any was freed or
// re-allocated -- stale bounds are never used.
#include <cuda_runtime.h>

#include <mutex>
#include <shared_mutex>
#include <vector>

#include "dispatch.h"

struct gd_graph {
    gd_arena *arena = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct Use {
        uint32_t id;
        uint64_t gen;
    };
    std::vector<Use> uses;                                  // partitions fenced by the graph
    struct Cost {
        uint32_t tenant, kind;
        uint64_t bytes, flops;
    };
    std::vector<Cost> costs;                                // host accounting per replay
    bool solo = false;                                      // captured unfenced solo launches
    uint64_t epoch = 0;                                     // the arena's epoch at capture
};

namespace {

void destroy(gd_graph *g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

}  // namespace

extern "C" gd_status gd_graph_create(gd_arena *a, const gd_work *items, uint32_t n_items, uint32_t n_streams,
                                     gd_graph **out) {
    if (!a || !out || (!items && n_items) || n_streams == 0) return GD_ERR_INVALID_ARG;
    *out = nullptr;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;
    gd_graph *g = new gd_graph();
    g->arena = a;
    // partitions stay as validated until the capture is complete
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);
    {
        std::lock_guard<std::mutex> lk(a->mu);
        g->epoch = a->epoch;
    }
    for (uint32_t i = 0; i < n_items; i++) {              // validate everything first
        gd_status st = gd::run_work_locked(a, items[i], nullptr, true);
        if (st != GD_OK) {
            destroy(g);
            return st;
        }
        uint64_t base, size, gen;
        gd::partition_snapshot(a, items[i].tenant, &base, &size, &gen);
        bool seen = false;
        for (auto &u : g->uses) seen = seen || u.id == items[i].tenant;
        if (!seen) g->uses.push_back({items[i].tenant, gen});
        if (items[i].kind == GD_KIND_GEMM || (items[i].kind == GD_KIND_STENCIL && items[i].u32[2] == 1)) {
            gd_work w = items[i];
            w.mode = gd::base_mode(w.mode);
            st = w.kind == GD_KIND_GEMM ? gd::gemm_prepare(a, w, base, size) : gd::stencil_tma_prepare(a, w, base, size);
            if (st != GD_OK) {
                destroy(g);
                return st;
            }
        }
    }
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != a->device) cudaSetDevice(a->device);
    std::vector<cudaStream_t> streams(n_streams);
    cudaStream_t origin;
    cudaError_t e = cudaStreamCreateWithFlags(&origin, cudaStreamNonBlocking);
    for (uint32_t s = 0; s < n_streams && e == cudaSuccess; s++)
        e = cudaStreamCreateWithFlags(&streams[s], cudaStreamNonBlocking);
    std::vector<cudaEvent_t> evs(n_streams + 1);
    for (auto &ev : evs)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    gd_status st = GD_OK;
    if (e == cudaSuccess) e = cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        // fork: every tenant stream joins the capture through the origin
        cudaEventRecord(evs[n_streams], origin);
        for (uint32_t s = 0; s < n_streams; s++) cudaStreamWaitEvent(streams[s], evs[n_streams], 0);
        std::vector<void *> sp(n_streams);
        for (uint32_t s = 0; s < n_streams; s++) sp[s] = streams[s];
        std::vector<uint32_t> order(n_items);
        gd_schedule_round_robin(items, n_items, order.data());
        std::vector<uint32_t> rank_of(GD_MAX_TENANTS, ~0u);   // stream rank = order of first appearance
        uint32_t nt = 0;
        for (uint32_t i = 0; i < n_items; i++)
            if (rank_of[items[i].tenant] == ~0u) rank_of[items[i].tenant] = nt++;
        for (uint32_t k = 0; k < n_items && st == GD_OK; k++) {
            const gd_work &w = items[order[k]];
            const uint32_t r = rank_of[w.tenant];
            gd::LaunchOut lo;
            st = gd::run_work_locked(a, w, streams[r % n_streams], false, false, &lo);
            g->costs.push_back({w.tenant, w.kind, lo.bytes, lo.flops});
            g->solo = g->solo || lo.solo;
        }
        // join
        for (uint32_t s = 0; s < n_streams; s++) {
            cudaEventRecord(evs[s], streams[s]);
            cudaStreamWaitEvent(origin, evs[s], 0);
        }
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(origin, &graph);
        g->graph = graph;
        if (e == cudaSuccess && st == GD_OK) e = cudaGraphInstantiate(&g->exec, graph, 0);
    }
    for (auto &ev : evs) cudaEventDestroy(ev);
    for (auto &s : streams) cudaStreamDestroy(s);
    cudaStreamDestroy(origin);
    if (prev >= 0 && prev != a->device) cudaSetDevice(prev);
    if (st == GD_OK && e != cudaSuccess) st = gd::cuda_status(e);
    if (st != GD_OK) {
        destroy(g);
        return st;
    }
    *out = g;
    return GD_OK;
}

extern "C" gd_status gd_graph_launch(gd_graph *g, void *stream) {
    if (!g || !g->exec) return GD_ERR_INVALID_ARG;
    // bounds checked and the replay enqueued with partition changes held off
    std::shared_lock<std::shared_mutex> guard(g->arena->launch_mu);
    if (g->solo) {                                        // unfenced solo kernels: only while still alone
        std::lock_guard<std::mutex> lk(g->arena->mu);
        if (g->arena->epoch != g->epoch) return GD_ERR_UNKNOWN_PARTITION;
    }
    for (const auto &u : g->uses) {                       // never replay with stale bounds
        uint64_t base, size, gen;
        if (gd::partition_snapshot(g->arena, u.id, &base, &size, &gen) != GD_OK || gen != u.gen)
            return GD_ERR_UNKNOWN_PARTITION;
    }
    cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
    if (e != cudaSuccess) return gd::cuda_status(e);
    {
        std::lock_guard<std::mutex> lk(g->arena->mu);
        for (const auto &c : g->costs) {
            gd::HostCounters &hc = g->arena->host[c.tenant][c.kind];
            hc.launches++;
            hc.bytes += c.bytes;
            hc.flops += c.flops;
        }
    }
    return GD_OK;
}

extern "C" gd_status gd_graph_destroy(gd_graph *g) {
    if (!g) return GD_ERR_INVALID_ARG;
    cudaDeviceSynchronize();
    destroy(g);
    return GD_OK;
}
