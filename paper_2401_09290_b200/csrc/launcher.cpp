// launcher.cpp -- multi-tenant issue.
//
// PAPER.md:177-179 §4.2.4: one context, one stream per application, calls of
// one application in order, calls of different applications selected
// round-robin.  The hardware block scheduler then overlaps the tenants'
// kernels (spatial sharing).
#include <cuda_runtime.h>

#include <mutex>
#include <shared_mutex>
#include <vector>

#include "dispatch.h"

namespace {

// tenant rank = order of first appearance; queues keep FIFO order per tenant
void build_queues(const gd_work *items, uint32_t n, std::vector<uint32_t> &tenants,
                  std::vector<std::vector<uint32_t>> &queues, std::vector<uint32_t> &rank_of_item) {
    rank_of_item.assign(n, 0);
    for (uint32_t i = 0; i < n; i++) {
        uint32_t r = 0;
        while (r < tenants.size() && tenants[r] != items[i].tenant) r++;
        if (r == tenants.size()) {
            tenants.push_back(items[i].tenant);
            queues.emplace_back();
        }
        queues[r].push_back(i);
        rank_of_item[i] = r;
    }
}

}  // namespace

extern "C" gd_status gd_schedule_round_robin(const gd_work *items, uint32_t n_items, uint32_t *order_out) {
    if ((!items || !order_out) && n_items) return GD_ERR_INVALID_ARG;
    std::vector<uint32_t> tenants, rank;
    std::vector<std::vector<uint32_t>> queues;
    build_queues(items, n_items, tenants, queues, rank);
    std::vector<size_t> head(queues.size(), 0);
    uint32_t k = 0;
    while (k < n_items) {
        for (size_t r = 0; r < queues.size(); r++) {
            if (head[r] < queues[r].size()) order_out[k++] = queues[r][head[r]++];
        }
    }
    return GD_OK;
}

namespace {

enum Cls { kStreamCls = 0, kRandomCls = 1, kTensorCls = 2 };

int class_of(uint32_t kind) {
    if (kind == GD_KIND_GATHER || kind == GD_KIND_SCATTER) return kRandomCls;
    if (kind == GD_KIND_GEMM) return kTensorCls;
    return kStreamCls;
}

// Per-stream "latest kernel of class c" events, created for one launcher call.
struct ClassEvents {
    std::vector<cudaEvent_t> ev[3];
    std::vector<bool> live[3];
    explicit ClassEvents(uint32_t n) {
        for (int c = 0; c < 3; c++) {
            ev[c].assign(n, nullptr);
            live[c].assign(n, false);
        }
    }
    ~ClassEvents() {
        for (int c = 0; c < 3; c++)
            for (cudaEvent_t e : ev[c])
                if (e) cudaEventDestroy(e);   // released once the recorded work completes
    }
    cudaError_t record(int c, uint32_t si, cudaStream_t s) {
        if (!ev[c][si]) {
            cudaError_t e = cudaEventCreateWithFlags(&ev[c][si], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        live[c][si] = true;
        return cudaEventRecord(ev[c][si], s);
    }
    // make s wait for the latest class-c kernel of every other stream
    cudaError_t wait_all(int c, uint32_t si, cudaStream_t s) {
        for (uint32_t k = 0; k < ev[c].size(); k++) {
            if (k == si || !live[c][k]) continue;
            cudaError_t e = cudaStreamWaitEvent(s, ev[c][k], 0);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
};

}  // namespace

extern "C" gd_status gd_launcher_run_policy(gd_arena *a, const gd_work *items, uint32_t n_items,
                                            void *const *streams, uint32_t n_streams, uint32_t policy,
                                            uint32_t *order_out) {
    if (!a || ((!items) && n_items)) return GD_ERR_INVALID_ARG;
    if (n_items && (!streams || n_streams == 0)) return GD_ERR_INVALID_ARG;
    if (policy > GD_POLICY_MEMORY_LANE) return GD_ERR_INVALID_ARG;
    // Held shared from validation to the last enqueue: no partition can be
    // allocated or freed in between, so every item is issued with the bounds
    // it was validated against and a validated step is issued whole (only a
    // CUDA error can stop it part-way).
    std::shared_lock<std::shared_mutex> hold(a->launch_mu);
    for (uint32_t i = 0; i < n_items; i++) {          // nothing is issued unless everything is valid
        gd_status st = gd::run_work_locked(a, items[i], nullptr, true);
        if (st != GD_OK) return st;
    }
    std::vector<uint32_t> order(n_items), tenants, rank;
    std::vector<std::vector<uint32_t>> queues;
    build_queues(items, n_items, tenants, queues, rank);
    gd_schedule_round_robin(items, n_items, order.data());
    // (a virtual arena never launches anything: no events there)
    const bool sep = policy != GD_POLICY_ROUND_ROBIN && a->device >= 0;
    const bool lane_on = policy == GD_POLICY_MEMORY_LANE && a->device >= 0;
    ClassEvents ce(sep ? n_streams : 0);
    cudaEvent_t lane = nullptr;                        // MEMORY_LANE: the latest memory-bound kernel
    bool lane_live = false;
    struct Guard {
        cudaEvent_t &e;
        ~Guard() { if (e) cudaEventDestroy(e); }
    } guard{lane};
    if (lane_on) {
        cudaError_t e = cudaEventCreateWithFlags(&lane, cudaEventDisableTiming);
        if (e != cudaSuccess) return gd::cuda_status(e);
    }
    for (uint32_t k = 0; k < n_items; k++) {
        const uint32_t i = order[k];
        const uint32_t si = rank[i] % n_streams;
        cudaStream_t s = (cudaStream_t)streams[si];
        const int c = class_of(items[i].kind);
        cudaError_t e = cudaSuccess;
        if (sep && c != kStreamCls) e = ce.wait_all(c == kTensorCls ? kRandomCls : kTensorCls, si, s);
        if (e == cudaSuccess && lane_on && c != kTensorCls && lane_live)
            e = cudaStreamWaitEvent(s, lane, 0);
        if (e != cudaSuccess) return gd::cuda_status(e);
        gd_status st = gd::run_work_locked(a, items[i], s, false);
        if (st != GD_OK) return st;
        if (sep && c != kStreamCls) e = ce.record(c, si, s);
        if (e == cudaSuccess && lane_on && c != kTensorCls) {
            e = cudaEventRecord(lane, s);
            lane_live = true;
        }
        if (e != cudaSuccess) return gd::cuda_status(e);
        if (order_out) order_out[k] = i;
    }
    return GD_OK;
}

extern "C" gd_status gd_launcher_run(gd_arena *a, const gd_work *items, uint32_t n_items, void *const *streams,
                                     uint32_t n_streams, uint32_t *order_out) {
    return gd_launcher_run_policy(a, items, n_items, streams, n_streams, GD_POLICY_ROUND_ROBIN, order_out);
}
