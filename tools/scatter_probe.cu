// scatter_probe.cu -- what limits the random scatter-add (dev probe, VERDICT r1
// item 4).  Every kernel takes 2^26 uniform random word indices (u32) and
// touches one 4-byte word per index in a table of `words` words:
//   0 read      : v = ld.global.cg [t + 4j]              (random read)
//   1 store     : st.global [t + 4j] = s                  (random write only)
//   2 red       : red.global.add.u32 (atomicAdd, no return; the product's K4)
//   3 red_ef    : red with an L2 evict_first cache-policy hint
//   4 red_el    : red with an L2 evict_last cache-policy hint
//   5 ld_st     : v = ld [t+4j]; st [t+4j] = v + s        (non-atomic RMW)
//   6 red_sorted: red at word (i * words) >> 26            (monotone: streaming)
// The table size sweeps DRAM-resident (2 GiB) to L2-resident (8-64 MiB) to
// measure the L2 atomic ceiling a bucketed (radix-partitioned) scatter would
// run at.
#include <cuda_runtime.h>

#include <cstdint>

template <int K>
__global__ void __launch_bounds__(256) probe(uint32_t *t, const uint32_t *idx, const uint32_t *src, uint64_t n,
                                             uint32_t words, uint32_t *sink) {
    const uint64_t i0 = ((uint64_t)blockIdx.x * 256 + threadIdx.x) * 4;
    if (i0 >= n) return;
    const uint4 j4 = __ldcs(reinterpret_cast<const uint4 *>(idx + i0));
    const uint4 s4 = __ldcs(reinterpret_cast<const uint4 *>(src + i0));
    const uint32_t js[4] = {j4.x % words, j4.y % words, j4.z % words, j4.w % words};
    const uint32_t ss[4] = {s4.x, s4.y, s4.z, s4.w};
    uint64_t pol = 0;
    if constexpr (K == 3) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (K == 4) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        uint32_t *a = t + js[q];
        if constexpr (K == 0) acc ^= __ldcg(a);
        else if constexpr (K == 1) __stcg(a, ss[q]);
        else if constexpr (K == 2) atomicAdd(a, ss[q]);
        else if constexpr (K == 3 || K == 4)
            asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(ss[q]), "l"(pol) : "memory");
        else if constexpr (K == 5) { const uint32_t v = __ldcg(a); __stcg(a, v + ss[q]); }
        else atomicAdd(t + (uint32_t)(((i0 + q) * (uint64_t)words) >> 26), ss[q]);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int probe_count() { return 7; }
extern "C" const char *probe_name(int k) {
    static const char *n[] = {"read", "store", "red", "red_evict_first", "red_evict_last", "ld_st", "red_sorted"};
    return n[k];
}

extern "C" int probe_run(int k, uint64_t t, uint64_t idx, uint64_t src, uint64_t n, uint32_t words, uint64_t sink,
                         void *stream) {
    const unsigned g = (unsigned)((n / 4 + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    auto T = (uint32_t *)t;
    auto I = (const uint32_t *)idx, S = (const uint32_t *)src;
    auto K = (uint32_t *)sink;
    switch (k) {
        case 0: probe<0><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 1: probe<1><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 2: probe<2><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 3: probe<3><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 4: probe<4><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 5: probe<5><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
        case 6: probe<6><<<g, 256, 0, s>>>(T, I, S, n, words, K); break;
    }
    return (int)cudaGetLastError();
}
