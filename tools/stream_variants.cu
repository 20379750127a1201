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

// TMA bulk copy (cp.async.bulk, no tensor map): each CTA moves NB buffers of
// BYTES through shared memory; one thread issues, an mbarrier collects the
// loads, bulk stores drain from shared memory.
template <int NB, int BYTES>
__global__ void __launch_bounds__(32) v_bulk(F f, uint64_t dst, uint64_t src, uint64_t nvec) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NB * BYTES);
    const uint64_t nbytes = nvec * 16, per = (uint64_t)NB * BYTES;
    const uint64_t o = (uint64_t)blockIdx.x * per;
    if (threadIdx.x != 0 || o >= nbytes) return;
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t len = nbytes - o < per ? nbytes - o : per;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"((uint32_t)len) : "memory");
    for (int b = 0; b < NB; b++) {
        const uint64_t ob = o + (uint64_t)b * BYTES;
        if (ob >= nbytes) break;
        const uint32_t sz = (uint32_t)(nbytes - ob < (uint64_t)BYTES ? nbytes - ob : BYTES);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(sm + b * BYTES)),
                     "l"(f(src + ob)), "r"(sz), "r"(bar_s)
                     : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                     bar_s)
                 : "memory");
    for (int b = 0; b < NB; b++) {
        const uint64_t ob = o + (uint64_t)b * BYTES;
        if (ob >= nbytes) break;
        const uint32_t sz = (uint32_t)(nbytes - ob < (uint64_t)BYTES ? nbytes - ob : BYTES);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(f(dst + ob)),
                     "r"((uint32_t)__cvta_generic_to_shared(sm + b * BYTES)), "r"(sz)
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int NB, int BYTES>
int bulk_launch(F f, uint64_t dst, uint64_t src, uint64_t nvec, cudaStream_t s) {
    const int smem = NB * BYTES + 16;
    cudaFuncSetAttribute(v_bulk<NB, BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const uint64_t per = (uint64_t)NB * BYTES;
    v_bulk<NB, BYTES><<<(unsigned)((nvec * 16 + per - 1) / per), 32, smem, s>>>(f, dst, src, nvec);
    return 0;
}

extern "C" int variant_count() { return 18; }

extern "C" const char *variant_name(int v) {
    static const char *n[] = {"persist U4 cs",   "persist U4 na",   "persist U4 def", "persist U8 cs",
                              "persist U8 na",   "chunk U4 cs",     "chunk U4 na",    "chunk U8 cs",
                              "chunk U8 na",     "pchunk U4 cs",    "pchunk U8 cs",   "pchunk U8 na",
                              "persist U4 cs x2grid", "pchunk U16 na", "bulk 4x16K",     "bulk 2x16K",
                              "bulk 4x8K",       "bulk 1x32K"};
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
        case 14: bulk_launch<4, 16384>(f, dst, src, nvec, s); break;
        case 15: bulk_launch<2, 16384>(f, dst, src, nvec, s); break;
        case 16: bulk_launch<4, 8192>(f, dst, src, nvec, s); break;
        case 17: bulk_launch<1, 32768>(f, dst, src, nvec, s); break;
    }
    return (int)cudaGetLastError();
}
