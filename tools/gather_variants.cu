// gather_variants.cu -- probe of random 32-bit load flavours for the fenced
// gather (dev tool).  out[i] = table[(idx[i] & keep) ...] in mask mode.
#include <cuda_runtime.h>

#include <cstdint>

template <int LD>
__device__ __forceinline__ uint32_t ldt(uint64_t a) {
    uint32_t r;
    if constexpr (LD == 0) r = __ldg(reinterpret_cast<const uint32_t *>(a));
    else if constexpr (LD == 1) r = __ldcg(reinterpret_cast<const uint32_t *>(a));
    else if constexpr (LD == 2) r = __ldcs(reinterpret_cast<const uint32_t *>(a));
    else if constexpr (LD == 3)
        asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(a));
    else if constexpr (LD == 4)
        asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(a));
    else
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(a));
    return r;
}

template <int LD, int U>
__global__ void __launch_bounds__(256) g_chunk(uint64_t base, uint64_t keep, uint64_t out, uint64_t table,
                                               uint64_t idx, uint64_t nvec) {
    const uint64_t v0 = (uint64_t)blockIdx.x * 256 * U + threadIdx.x;
    int4 j[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint64_t v = v0 + u * 256;
        j[u] = v < nvec ? __ldcs(reinterpret_cast<const int4 *>(((idx + 16 * v) & keep) | base)) : make_int4(0, 0, 0, 0);
    }
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        r[u].x = ldt<LD>(((table + (uint64_t)((int64_t)j[u].x * 4)) & keep) | base);
        r[u].y = ldt<LD>(((table + (uint64_t)((int64_t)j[u].y * 4)) & keep) | base);
        r[u].z = ldt<LD>(((table + (uint64_t)((int64_t)j[u].z * 4)) & keep) | base);
        r[u].w = ldt<LD>(((table + (uint64_t)((int64_t)j[u].w * 4)) & keep) | base);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint64_t v = v0 + u * 256;
        if (v < nvec) __stcs(reinterpret_cast<uint4 *>(((out + 16 * v) & keep) | base), r[u]);
    }
}

extern "C" int set_l2_fetch(int bytes) { return (int)cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, bytes); }
extern "C" int get_l2_fetch() {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    return (int)v;
}

template <int U>
__global__ void __launch_bounds__(256) s_chunk(uint64_t base, uint64_t keep, uint64_t table, uint64_t idx,
                                               uint64_t src, uint64_t nvec) {
    const uint64_t v0 = (uint64_t)blockIdx.x * 256 * U + threadIdx.x;
    int4 j[U];
    uint4 s[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint64_t v = v0 + u * 256;
        j[u] = v < nvec ? __ldcs(reinterpret_cast<const int4 *>(((idx + 16 * v) & keep) | base)) : make_int4(0, 0, 0, 0);
        s[u] = v < nvec ? __ldcs(reinterpret_cast<const uint4 *>(((src + 16 * v) & keep) | base)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        if (v0 + u * 256 >= nvec) continue;
        atomicAdd((unsigned *)(((table + (uint64_t)((int64_t)j[u].x * 4)) & keep) | base), s[u].x);
        atomicAdd((unsigned *)(((table + (uint64_t)((int64_t)j[u].y * 4)) & keep) | base), s[u].y);
        atomicAdd((unsigned *)(((table + (uint64_t)((int64_t)j[u].z * 4)) & keep) | base), s[u].z);
        atomicAdd((unsigned *)(((table + (uint64_t)((int64_t)j[u].w * 4)) & keep) | base), s[u].w);
    }
}

extern "C" int svariant_run(uint64_t base, uint64_t mask, uint64_t table, uint64_t idx, uint64_t src, uint64_t n,
                            void *stream) {
    const uint64_t keep = mask & ~3ull, nvec = n / 4;
    s_chunk<4><<<(unsigned)((nvec + 1023) / 1024), 256, 0, (cudaStream_t)stream>>>(base, keep, table, idx, src, nvec);
    return (int)cudaGetLastError();
}

// random reads of WB bytes (WB/16 16-byte vectors, or one 4/8-byte word) at
// WB-aligned random positions of a 2 GiB table: accesses/s vs access size
template <int WB>
__global__ void __launch_bounds__(256) r_read(uint64_t table, uint64_t idx, uint64_t n, uint64_t slots,
                                              uint32_t *sink) {
    const uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const uint32_t j = __ldcs(reinterpret_cast<const uint32_t *>(idx) + i) % (uint32_t)slots;
    const uint64_t a = table + (uint64_t)j * WB;
    uint32_t acc = 0;
    if constexpr (WB == 4) acc = __ldcg(reinterpret_cast<const uint32_t *>(a));
    else if constexpr (WB == 8) { uint2 v = __ldcg(reinterpret_cast<const uint2 *>(a)); acc = v.x ^ v.y; }
    else {
#pragma unroll
        for (int q = 0; q < WB / 16; q++) {
            uint4 v = __ldcg(reinterpret_cast<const uint4 *>(a) + q);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int rread_run(int wb, uint64_t table, uint64_t idx, uint64_t n, void *sink, void *stream) {
    const uint64_t slots = (2ull << 30) / wb;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = (unsigned)((n + 255) / 256);
    switch (wb) {
        case 4: r_read<4><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
        case 8: r_read<8><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
        case 16: r_read<16><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
        case 32: r_read<32><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
        case 64: r_read<64><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
        case 128: r_read<128><<<g, 256, 0, s>>>(table, idx, n, slots, (uint32_t *)sink); break;
    }
    return (int)cudaGetLastError();
}

extern "C" int gvariant_count() { return 9; }
extern "C" const char *gvariant_name(int v) {
    static const char *n[] = {"ldg U2", "ldcg U2", "ldcs U2", "nc.no_alloc U2", "no_alloc U2", "relaxed.gpu U2",
                              "ldcg U4", "ldcg U8", "nc.no_alloc U4"};
    return n[v];
}

extern "C" int gvariant_run(int v, uint64_t base, uint64_t mask, uint64_t out, uint64_t table, uint64_t idx,
                            uint64_t n, void *stream) {
    const uint64_t keep = mask & ~3ull, nvec = n / 4;
    cudaStream_t s = (cudaStream_t)stream;
#define G(LD, U) g_chunk<LD, U><<<(unsigned)((nvec + 256 * U - 1) / (256 * U)), 256, 0, s>>>(base, keep, out, table, idx, nvec)
    switch (v) {
        case 0: G(0, 2); break;
        case 1: G(1, 2); break;
        case 2: G(2, 2); break;
        case 3: G(3, 2); break;
        case 4: G(4, 2); break;
        case 5: G(5, 2); break;
        case 6: G(1, 4); break;
        case 7: G(1, 8); break;
        case 8: G(3, 4); break;
    }
    return (int)cudaGetLastError();
}
