// launcher.cpp -- multi-tenant issue.
//
// PAPER.md:177-179 §4.2.4: one context, one stream per application, calls of
// one application in order, calls of different applications selected
// round-robin.  The hardware block scheduler then overlaps the tenants'
// kernels (spatial sharing).
#include <cuda_runtime.h>

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

extern "C" gd_status gd_launcher_run(gd_arena *a, const gd_work *items, uint32_t n_items, void *const *streams,
                                     uint32_t n_streams, uint32_t *order_out) {
    if (!a || ((!items) && n_items)) return GD_ERR_INVALID_ARG;
    if (n_items && (!streams || n_streams == 0)) return GD_ERR_INVALID_ARG;
    for (uint32_t i = 0; i < n_items; i++) {          // nothing is issued unless everything is valid
        gd_status st = gd::run_work(a, items[i], nullptr, true);
        if (st != GD_OK) return st;
    }
    std::vector<uint32_t> order(n_items), tenants, rank;
    std::vector<std::vector<uint32_t>> queues;
    build_queues(items, n_items, tenants, queues, rank);
    gd_schedule_round_robin(items, n_items, order.data());
    for (uint32_t k = 0; k < n_items; k++) {
        const uint32_t i = order[k];
        cudaStream_t s = (cudaStream_t)streams[rank[i] % n_streams];
        gd_status st = gd::run_work(a, items[i], s, false);
        if (st != GD_OK) return st;
        if (order_out) order_out[k] = i;
    }
    return GD_OK;
}
