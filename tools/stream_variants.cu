// stream_variants.cu -- design-space probe for the HBM-bound fenced kernels
// (dev tool, not part of libguardian.so).  Each variant is the mask-mode
// fenced copy / saxpy with a different grid and access schedule.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libvariants.so tools/stream_variants.cu
#include <cuda_runtime.h>

#include <cstdint>

struct F {
    uint64_t base, keep;
    __device__ __forceinline__ uint64_t operator()(uint64_t a) const { return (a & keep) | base; }
};

__device__ __forceinline__ uint4 ld_cs(uint64_t a) { return __ldcs(reinterpret_cast<const uint4 *>(a)); }
__device__ __forceinline__ void st_cs(uint64_t a, uint4 v) { __stcs(reinterpret_cast<uint4 *>(a), v); }
__device__ __forceinline__ uint4 ld_na(uint64_t a) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a));
    return r;
}
__device__ __forceinline__ void st_na(uint64_t a, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_def(uint64_t a) { return *reinterpret_cast<const uint4 *>(a); }
__device__ __forceinline__ void st_def(uint64_t a, uint4 v) { *reinterpret_cast<uint4 *>(a) = v; }

// V0: persistent grid-stride, interleaved unroll U (current product design)
template <int U, int LD>
__global__ void __launch_bounds__(256) v_persist(F f, uint64_t dst, uint64_t src, uint64_t nvec) {
    const uint64_t T = (uint64_t)gridDim.x * 256;
    uint64_t v = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    for (; v + (U - 1) * T < nvec; v += U * T) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint64_t a = f(src + 16 * (v + u * T));
            r[u] = LD == 0 ? ld_cs(a) : (LD == 1 ? ld_na(a) : ld_def(a));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint64_t a = f(dst + 16 * (v + u * T));
            if (LD == 0) st_cs(a, r[u]);
            else if (LD == 1) st_na(a, r[u]);
            else st_def(a, r[u]);
        }
    }
    for (; v < nvec; v += T) st_cs(f(dst + 16 * v), ld_cs(f(src + 16 * v)));
}

// V1: one-shot grid, each CTA a contiguous chunk of 256*U vectors (block-strided inside)
template <int U, int LD>
__global__ void __launch_bounds__(256) v_chunk(F f, uint64_t dst, uint64_t src, uint64_t nvec) {
    const uint64_t v0 = (uint64_t)blockIdx.x * 256 * U + threadIdx.x;
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint64_t v = v0 + u * 256;
        if (v < nvec) {
            uint64_t a = f(src + 16 * v);
            r[u] = LD == 0 ? ld_cs(a) : (LD == 1 ? ld_na(a) : ld_def(a));
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint64_t v = v0 + u * 256;
        if (v < nvec) {
            uint64_t a = f(dst + 16 * v);
            if (LD == 0) st_cs(a, r[u]);
            else if (LD == 1) st_na(a, r[u]);
            else st_def(a, r[u]);
        }
    }
}

// V2: persistent, CTA-contiguous chunks of 256*U vectors, chunk = blockIdx + k*grid
template <int U, int LD>
__global__ void __launch_bounds__(256) v_pchunk(F f, uint64_t dst, uint64_t src, uint64_t nvec) {
    const uint64_t nchunk = (nvec + 256 * U - 1) / (256 * U);
    for (uint64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const uint64_t v0 = c * 256 * U + threadIdx.x;
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t v = v0 + u * 256;
            if (v < nvec) {
                uint64_t a = f(src + 16 * v);
                r[u] = LD == 0 ? ld_cs(a) : (LD == 1 ? ld_na(a) : ld_def(a));
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t v = v0 + u * 256;
            if (v < nvec) {
                uint64_t a = f(dst + 16 * v);
                if (LD == 0) st_cs(a, r[u]);
                else if (LD == 1) st_na(a, r[u]);
                else st_def(a, r[u]);
            }
        }
    }
}

template <typename K>
static int occ(K k) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 256, 0);
    return b;
}

extern "C" int variant_count() { return 14; }

extern "C" const char *variant_name(int v) {
    static const char *n[] = {"persist U4 cs",   "persist U4 na",   "persist U4 def", "persist U8 cs",
                              "persist U8 na",   "chunk U4 cs",     "chunk U4 na",    "chunk U8 cs",
                              "chunk U8 na",     "pchunk U4 cs",    "pchunk U8 cs",   "pchunk U8 na",
                              "persist U4 cs x2grid", "pchunk U16 na"};
    return n[v];
}

extern "C" int variant_copy(int v, uint64_t base, uint64_t mask, uint64_t dst, uint64_t src, uint64_t nbytes,
                            void *stream) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    F f{base, mask & ~15ull};
    const uint64_t nvec = nbytes / 16;
    cudaStream_t s = (cudaStream_t)stream;
#define PERSIST(K, mult) K<<<sms * occ(K) * mult, 256, 0, s>>>(f, dst, src, nvec)
#define CHUNK(K, U) K<<<(unsigned)((nvec + 256 * U - 1) / (256 * U)), 256, 0, s>>>(f, dst, src, nvec)
    switch (v) {
        case 0: PERSIST((v_persist<4, 0>), 1); break;
        case 1: PERSIST((v_persist<4, 1>), 1); break;
        case 2: PERSIST((v_persist<4, 2>), 1); break;
        case 3: PERSIST((v_persist<8, 0>), 1); break;
        case 4: PERSIST((v_persist<8, 1>), 1); break;
        case 5: CHUNK((v_chunk<4, 0>), 4); break;
        case 6: CHUNK((v_chunk<4, 1>), 4); break;
        case 7: CHUNK((v_chunk<8, 0>), 8); break;
        case 8: CHUNK((v_chunk<8, 1>), 8); break;
        case 9: PERSIST((v_pchunk<4, 0>), 1); break;
        case 10: PERSIST((v_pchunk<8, 0>), 1); break;
        case 11: PERSIST((v_pchunk<8, 1>), 1); break;
        case 12: PERSIST((v_persist<4, 0>), 2); break;
        case 13: PERSIST((v_pchunk<16, 1>), 1); break;
    }
    return (int)cudaGetLastError();
}
