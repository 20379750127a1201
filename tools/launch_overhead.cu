// launch_overhead.cu -- host cost of a fenced launch through the C ABI
// (the paper's Table 5: lookup 557,
// augment 400, launch ~9000 CPU cycles).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_overhead tools/launch_overhead.cu \
//        -Iinclude -Lpaper_2401_09290_b200 -lguardian -Xlinker -rpath=$PWD/paper_2401_09290_b200
//
// Times, per call on one stream (wall clock, host side, GPU work negligible):
//   raw      : <<<>>> launch of an empty kernel with a 40-byte by-value parameter
//   gd_copy  : gd_launch_fenced_copy of 16 bytes (validation + bounds-table
//              snapshot + FenceDesc build + launch + accounting), per mode
//   check_range / memcpy checks: gd_check_range alone
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdint>

#include "guardian.h"

struct P40 {
    uint64_t a, b, c, d, e;
};
__global__ void k_empty(const __grid_constant__ P40 p) {
    if (p.a == 0x1234567 && threadIdx.x == 1000) printf("x");
}

template <typename F>
double ns_per(F f, int iters) {
    for (int i = 0; i < 1000; i++) f();
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; i++) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::nano>(t1 - t0).count() / iters;
}

int main() {
    cudaSetDevice(0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    gd_arena *a = nullptr;
    if (gd_arena_create(0, 1ull << 24, 0, &a) != GD_OK) return 1;
    gd_partition_info p;
    gd_partition_alloc(a, 1 << 22, &p);
    const int iters = 20000;
    P40 prm{1, 2, 3, 4, 5};
    double raw = ns_per([&] { k_empty<<<1, 32, 0, s>>>(prm); }, iters);
    printf("{\"raw_launch_ns\": %.1f", raw);
    const char *names[] = {"none", "mask", "check", "modulo"};
    for (int m = 0; m < 4; m++) {
        double t = ns_per([&] { gd_launch_fenced_copy(a, p.id, (gd_mode)m, p.base + 4096, p.base, 16, s); }, iters);
        printf(", \"gd_copy_%s_ns\": %.1f", names[m], t);
    }
    int ok = 0;
    double cr = ns_per([&] { gd_check_range(a, p.id, p.base + 100, 4096, &ok); }, iters);
    printf(", \"check_range_ns\": %.1f", cr);
    gd_work w[8];
    for (int i = 0; i < 8; i++) {
        w[i] = gd_work{};
        w[i].tenant = p.id;
        w[i].kind = GD_KIND_COPY;
        w[i].mode = GD_MODE_MASK;
        w[i].ptr[0] = p.base + 4096;
        w[i].ptr[1] = p.base;
        w[i].u64[0] = 16;
    }
    void *streams[1] = {s};
    double lr = ns_per([&] { gd_launcher_run(a, w, 8, streams, 1, nullptr); }, iters / 8);
    printf(", \"launcher_8_items_ns\": %.1f, \"launcher_per_item_ns\": %.1f}\n", lr, lr / 8);
    gd_arena_destroy(a);
    return 0;
}
