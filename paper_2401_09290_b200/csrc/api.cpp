// api.cpp -- the C ABI of libguardian.so (include/guardian.h).
//
// Partition manager (§4.2.1): one VMM reservation per arena,
// aligned to its own power-of-two size; buddy partitions mapped to physical
// memory in full at allocation and scrubbed (reading A15).  Parameter
// augmentation (§4.2.3): every launch builds a FenceDesc from an
// immutable snapshot of the bounds-table row and passes it by value.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <shared_mutex>

#include "arena.h"
#include "drv.h"
#include "dispatch.h"

using namespace gd;

namespace {

thread_local int g_last_cuda = 0;

gd_status cuda_fail(cudaError_t e) {
    g_last_cuda = (int)e;
    return GD_ERR_CUDA;
}
gd_status cu_fail(CUresult r) {
    g_last_cuda = (int)r;
    return GD_ERR_CUDA;
}

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
unsigned log2u(uint64_t x) {
    unsigned k = 0;
    while ((1ull << k) < x) k++;
    return k;
}

// Set the arena's device current for this thread, remembering the previous one.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (dev < 0) return;
        cudaGetDevice(&prev);
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) {
            int cur = -1;
            cudaGetDevice(&cur);
            if (cur != prev) cudaSetDevice(prev);
        }
    }
};

CUmemAllocationProp phys_prop(int device) {
    CUmemAllocationProp p;
    std::memset(&p, 0, sizeof(p));
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    return p;
}

// Map [va, va+size) to fresh physical memory (one chunk).
gd_status map_chunk(gd_arena *a, uint64_t va, uint64_t size) {
    const Drv &d = drv();
    CUmemAllocationProp p = phys_prop(a->device);
    CUmemGenericAllocationHandle h;
    CUresult r = d.MemCreate(&h, size, &p, 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY) return GD_ERR_DEVICE_OOM;
    if (r != CUDA_SUCCESS) return cu_fail(r);
    r = d.MemMap((CUdeviceptr)va, size, 0, h, 0);
    if (r != CUDA_SUCCESS) {
        d.MemRelease(h);
        return cu_fail(r);
    }
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = a->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = d.MemSetAccess((CUdeviceptr)va, size, &acc, 1);
    if (r != CUDA_SUCCESS) {
        d.MemUnmap((CUdeviceptr)va, size);
        d.MemRelease(h);
        return cu_fail(r);
    }
    Chunk c;
    c.handle = (unsigned long long)h;
    c.size = size;
    c.refs = 1;
    a->chunks[va] = c;
    return GD_OK;
}

void unmap_chunk(gd_arena *a, std::map<uint64_t, Chunk>::iterator it) {
    const Drv &d = drv();
    d.MemUnmap((CUdeviceptr)it->first, it->second.size);
    d.MemRelease((CUmemGenericAllocationHandle)it->second.handle);
    a->chunks.erase(it);
}

// Physically back a whole partition (every fenced address must be mapped: H2).
gd_status back_partition(gd_arena *a, uint64_t b, uint64_t s) {
    if (!a->vmm) return GD_OK;
    if (s >= a->gran) return map_chunk(a, b, s);
    const uint64_t g = b & ~(a->gran - 1);
    auto it = a->chunks.find(g);
    if (it != a->chunks.end()) {
        it->second.refs++;
        return GD_OK;
    }
    return map_chunk(a, g, a->gran);
}

void unback_partition(gd_arena *a, uint64_t b, uint64_t s) {
    if (!a->vmm) return;
    const uint64_t key = s >= a->gran ? b : (b & ~(a->gran - 1));
    auto it = a->chunks.find(key);
    if (it == a->chunks.end()) return;
    if (--it->second.refs == 0) unmap_chunk(a, it);
}

// Snapshot of one bounds-table row for a launch.
gd_status snapshot(gd_arena *a, uint32_t id, uint64_t *base, uint64_t *size) {
    std::lock_guard<std::mutex> lk(a->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    *base = a->parts[id].base;
    *size = a->parts[id].size;
    return GD_OK;
}

bool mul_ok(uint64_t a, uint64_t b, uint64_t *r) { return !__builtin_mul_overflow(a, b, r); }

// native-when-solo is on and exactly one partition is live
bool solo_native(gd_arena *a) {
    std::lock_guard<std::mutex> lk(a->mu);
    if (!a->native_when_solo) return false;
    uint32_t live = 0;
    for (uint32_t i = 0; i < GD_MAX_TENANTS; i++) live += a->parts[i].live ? 1u : 0u;
    return live == 1;
}

bool tenant_live(gd_arena *a, uint32_t id) {
    std::lock_guard<std::mutex> lk(a->mu);
    return id < GD_MAX_TENANTS && a->parts[id].live;
}

// The trusted device memory of an arena, one cudaMalloc outside it (SURVEY
// H9): the violation counters u64[GD_MAX_TENANTS][GD_NUM_KINDS], then a
// 256-byte all-zero block that refused check-mode loads read (FenceDesc::zero;
// nothing ever writes it).  Zeroed; synchronises.
constexpr uint64_t kStatsBytes = sizeof(unsigned long long) * GD_MAX_TENANTS * GD_NUM_KINDS;
constexpr uint64_t kZeroOff = (kStatsBytes + 255) & ~255ull, kTrustedBytes = kZeroOff + 256;

gd_status alloc_trusted(gd_arena *a) {
    void *st = nullptr;
    cudaError_t e = cudaMalloc(&st, kTrustedBytes);
    if (e != cudaSuccess) return cuda_fail(e);
    const uint64_t sp = (uint64_t)st, se = sp + kTrustedBytes;
    if (se > a->base && sp < a->base + a->size) {        // H9: never inside the arena
        cudaFree(st);
        return GD_ERR_INVALID_ARG;
    }
    e = cudaMemset(st, 0, kTrustedBytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(st);
        return cuda_fail(e);
    }
    a->d_stats = (unsigned long long *)st;
    a->d_zero = sp + kZeroOff;
    return GD_OK;
}

}  // namespace

// ===========================================================================
// Arena
// ===========================================================================

extern "C" gd_status gd_arena_create(int device, uint64_t bytes, uint32_t flags, gd_arena **out) {
    if (!out || device < 0 || flags != GD_ARENA_VMM) return GD_ERR_INVALID_ARG;
    *out = nullptr;
    if (!is_pow2(bytes) || bytes < GD_MIN_PARTITION) return GD_ERR_NOT_POW2;
    if (!drv().ok) return GD_ERR_CUDA;
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err);
    cudaFree(nullptr);                                   // make sure the primary context exists
    const Drv &d = drv();
    CUmemAllocationProp p = phys_prop(device);
    size_t gran = 0;
    CUresult r = d.MemGetAllocationGranularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    if (r != CUDA_SUCCESS) return cu_fail(r);
    const uint64_t rsize = bytes > gran ? bytes : (uint64_t)gran;
    CUdeviceptr va = 0;
    uint64_t reserve = rsize;
    r = d.MemAddressReserve(&va, rsize, rsize, 0, 0);
    if (r != CUDA_SUCCESS || (va % rsize) != 0) {        // alignment not honoured: over-reserve
        if (r == CUDA_SUCCESS) d.MemAddressFree(va, rsize);
        reserve = 2 * rsize;
        r = d.MemAddressReserve(&va, reserve, gran, 0, 0);
        if (r != CUDA_SUCCESS) return GD_ERR_DEVICE_OOM;
    }
    gd_arena *a = new gd_arena();
    a->device = device;
    a->vmm = true;
    a->reserve_va = va;
    a->reserve_size = reserve;
    a->gran = gran;
    a->base = (va + rsize - 1) & ~(rsize - 1);
    a->size = bytes;
    a->buddy.init(bytes, 12);
    cudaDeviceGetAttribute(&a->sms, cudaDevAttrMultiProcessorCount, device);
    const gd_status ts = alloc_trusted(a);
    if (ts != GD_OK) {
        d.MemAddressFree(va, reserve);
        delete a;
        return ts;
    }
    *out = a;
    return GD_OK;
}

extern "C" gd_status gd_arena_wrap(int device, uint64_t dev_ptr, uint64_t bytes, gd_arena **out) {
    if (!out) return GD_ERR_INVALID_ARG;
    *out = nullptr;
    if (!is_pow2(bytes) || bytes < GD_MIN_PARTITION) return GD_ERR_NOT_POW2;
    if (dev_ptr % bytes != 0) return GD_ERR_ALIGN;
    if (dev_ptr + bytes < dev_ptr) return GD_ERR_INVALID_ARG;
    gd_arena *a = new gd_arena();
    a->device = device < 0 ? -1 : device;
    a->vmm = false;
    a->base = dev_ptr;
    a->size = bytes;
    a->buddy.init(bytes, 12);
    if (a->device >= 0) {
        DeviceGuard dg(device);
        if (dg.err != cudaSuccess) {
            delete a;
            return cuda_fail(dg.err);
        }
        cudaDeviceGetAttribute(&a->sms, cudaDevAttrMultiProcessorCount, device);
        const gd_status ts = alloc_trusted(a);
        if (ts != GD_OK) {
            delete a;
            return ts;
        }
    }
    *out = a;
    return GD_OK;
}

extern "C" gd_status gd_arena_destroy(gd_arena *a) {
    if (!a) return GD_ERR_INVALID_ARG;
    if (a->device >= 0) {
        DeviceGuard dg(a->device);
        cudaDeviceSynchronize();
        while (!a->chunks.empty()) unmap_chunk(a, a->chunks.begin());
        if (a->vmm) drv().MemAddressFree((CUdeviceptr)a->reserve_va, a->reserve_size);
        if (a->d_stats) cudaFree(a->d_stats);
        if (a->zero_buf) cudaFree(a->zero_buf);
        for (void *z : a->zero_retired) cudaFree(z);
    }
    delete a;
    return GD_OK;
}

extern "C" gd_status gd_arena_info(const gd_arena *a, uint64_t *base, uint64_t *size, int *device) {
    if (!a) return GD_ERR_INVALID_ARG;
    if (base) *base = a->base;
    if (size) *size = a->size;
    if (device) *device = a->device;
    return GD_OK;
}

// ===========================================================================
// Partitions
// ===========================================================================

namespace {

void fill_info(uint32_t id, const Partition &p, gd_partition_info *out) {
    out->id = id;
    out->flags = p.pow2 ? GD_PART_POW2 : 0u;
    out->base = p.base;
    out->size = p.size;
    out->mask = p.size - 1;
    out->end = p.base + p.size;
}

// Carve a partition of `size` bytes (pow2: aligned to its size; exact:
// aligned to next_pow2(size), tail returned to the buddy), back it
// physically, scrub it, zero its counters.  Caller holds a->mu.
gd_status carve(gd_arena *a, uint64_t size, bool pow2, gd_partition_info *out) {
    uint32_t id = GD_MAX_TENANTS;
    for (uint32_t i = 0; i < GD_MAX_TENANTS; i++)
        if (!a->parts[i].live) {
            id = i;
            break;
        }
    if (id == GD_MAX_TENANTS) return GD_ERR_DEVICE_OOM;
    const unsigned order = log2u(size);
    uint64_t off = 0;
    const bool got = pow2 ? a->buddy.alloc(order, &off) : a->buddy.alloc_exact(size, &off);
    if (!got) return GD_ERR_DEVICE_OOM;
    auto give_back = [&] {
        if (pow2) a->buddy.free(off, order);
        else a->buddy.free_exact(off, size);
    };
    const uint64_t b = a->base + off;
    if (a->device >= 0) {
        DeviceGuard dg(a->device);
        gd_status st = back_partition(a, b, size);
        if (st != GD_OK) {
            give_back();
            return st;
        }
        // scrub (reading A15) and zero this tenant's counters.  Everything
        // already enqueued finishes first: a kernel of a tenant that ran alone
        // unfenced (native when solo) must not write the new partition after
        // its scrub.
        Geom g{a->sms};
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = launch_fill(b, 0, size, 0, 0, g);
        if (e == cudaSuccess)
            e = cudaMemset(a->d_stats + (uint64_t)id * GD_NUM_KINDS, 0, sizeof(unsigned long long) * GD_NUM_KINDS);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            unback_partition(a, b, size);
            give_back();
            return cuda_fail(e);
        }
    }
    Partition &p = a->parts[id];
    p.live = true;
    p.base = b;
    p.size = size;
    p.order = order;
    p.pow2 = pow2;
    p.gen = a->next_gen++;
    a->epoch++;
    p.sub.init(size);
    for (unsigned k = 0; k < GD_NUM_KINDS; k++) a->host[id][k] = HostCounters{};
    fill_info(id, p, out);
    return GD_OK;
}

}  // namespace

extern "C" gd_status gd_partition_alloc(gd_arena *a, uint64_t requested, gd_partition_info *out) {
    if (!a || !out || requested == 0 || requested > a->size) return GD_ERR_INVALID_ARG;
    uint64_t size = GD_MIN_PARTITION;
    while (size < requested) size <<= 1;                 // next pow2 >= max(req, 4 KiB)
    std::unique_lock<std::shared_mutex> guard(a->launch_mu);
    std::lock_guard<std::mutex> lk(a->mu);
    return carve(a, size, true, out);
}

extern "C" gd_status gd_partition_alloc_exact(gd_arena *a, uint64_t requested, gd_partition_info *out) {
    if (!a || !out || requested == 0 || requested > a->size) return GD_ERR_INVALID_ARG;
    const uint64_t g = a->vmm ? a->gran : GD_MIN_PARTITION;     // physical backing granule
    uint64_t size = (requested + g - 1) / g * g;
    if (size < GD_MIN_PARTITION) size = GD_MIN_PARTITION;
    std::unique_lock<std::shared_mutex> guard(a->launch_mu);
    std::lock_guard<std::mutex> lk(a->mu);
    return carve(a, size, (size & (size - 1)) == 0, out);
}

extern "C" gd_status gd_partition_free(gd_arena *a, uint32_t id) {
    if (!a) return GD_ERR_INVALID_ARG;
    // exclusive: no launch sits between its bounds snapshot and its enqueue
    std::unique_lock<std::shared_mutex> guard(a->launch_mu);
    std::lock_guard<std::mutex> lk(a->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    Partition &p = a->parts[id];
    if (a->device >= 0) {
        DeviceGuard dg(a->device);
        cudaDeviceSynchronize();                          // no launch may still use it
        unback_partition(a, p.base, p.size);
    }
    if (p.pow2) a->buddy.free(p.base - a->base, p.order);
    else a->buddy.free_exact(p.base - a->base, p.size);
    p.live = false;
    a->epoch++;
    return GD_OK;
}

extern "C" gd_status gd_partition_get(const gd_arena *a, uint32_t id, gd_partition_info *out) {
    if (!a || !out) return GD_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> lk(const_cast<gd_arena *>(a)->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    fill_info(id, a->parts[id], out);
    return GD_OK;
}

extern "C" gd_status gd_malloc(gd_arena *a, uint32_t id, uint64_t bytes, uint64_t *dev_addr) {
    if (!a || !dev_addr || bytes == 0) return GD_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> lk(a->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    uint64_t off = 0;
    if (!a->parts[id].sub.alloc(bytes, &off)) return GD_ERR_PARTITION_OOM;
    *dev_addr = a->parts[id].base + off;
    return GD_OK;
}

extern "C" gd_status gd_free(gd_arena *a, uint32_t id, uint64_t dev_addr) {
    if (!a) return GD_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> lk(a->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    Partition &p = a->parts[id];
    if (dev_addr < p.base || dev_addr >= p.base + p.size) return GD_ERR_UNKNOWN_ALLOC;
    if (!p.sub.free(dev_addr - p.base)) return GD_ERR_UNKNOWN_ALLOC;
    return GD_OK;
}

// ===========================================================================
// Host transfers (§4.2.2)
// ===========================================================================

namespace {
bool range_ok(uint64_t base, uint64_t size, uint64_t addr, uint64_t len) {
    const uint64_t end = base + size;
    if (len == 0) return addr >= base && addr <= end;
    if (addr < base || addr > end) return false;
    return len <= end - addr;                           // no wraparound possible
}
}  // namespace

extern "C" gd_status gd_check_range(const gd_arena *a, uint32_t id, uint64_t addr, uint64_t len, int *ok) {
    if (!a || !ok) return GD_ERR_INVALID_ARG;
    uint64_t b, s;
    gd_status st = snapshot(const_cast<gd_arena *>(a), id, &b, &s);
    if (st != GD_OK) return st;
    *ok = range_ok(b, s, addr, len) ? 1 : 0;
    return GD_OK;
}

extern "C" gd_status gd_memcpy_h2d(gd_arena *a, uint32_t id, uint64_t dst, const void *src, uint64_t n,
                                   void *stream) {
    if (!a || (!src && n)) return GD_ERR_INVALID_ARG;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);    // bounds stay valid until enqueued
    uint64_t b, s;
    gd_status st = snapshot(a, id, &b, &s);
    if (st != GD_OK) return st;
    if (!range_ok(b, s, dst, n)) return GD_ERR_OOB_RANGE;
    if (n == 0) return GD_OK;
    DeviceGuard dg(a->device);
    cudaError_t e = cudaMemcpyAsync((void *)dst, src, n, cudaMemcpyHostToDevice, (cudaStream_t)stream);
    return e == cudaSuccess ? GD_OK : cuda_fail(e);
}

extern "C" gd_status gd_memcpy_d2h(gd_arena *a, uint32_t id, void *dst, uint64_t src, uint64_t n, void *stream) {
    if (!a || (!dst && n)) return GD_ERR_INVALID_ARG;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);    // bounds stay valid until enqueued
    uint64_t b, s;
    gd_status st = snapshot(a, id, &b, &s);
    if (st != GD_OK) return st;
    if (!range_ok(b, s, src, n)) return GD_ERR_OOB_RANGE;
    if (n == 0) return GD_OK;
    DeviceGuard dg(a->device);
    cudaError_t e = cudaMemcpyAsync(dst, (const void *)src, n, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    return e == cudaSuccess ? GD_OK : cuda_fail(e);
}

extern "C" gd_status gd_memcpy_d2d(gd_arena *a, uint32_t id, uint64_t dst, uint64_t src, uint64_t n, void *stream) {
    if (!a) return GD_ERR_INVALID_ARG;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);    // bounds stay valid until enqueued
    uint64_t b, s;
    gd_status st = snapshot(a, id, &b, &s);
    if (st != GD_OK) return st;
    if (!range_ok(b, s, src, n) || !range_ok(b, s, dst, n)) return GD_ERR_OOB_RANGE;
    if (n == 0) return GD_OK;
    DeviceGuard dg(a->device);
    cudaError_t e = cudaMemcpyAsync((void *)dst, (const void *)src, n, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    return e == cudaSuccess ? GD_OK : cuda_fail(e);
}

extern "C" gd_status gd_partition_fill(gd_arena *a, uint32_t id, uint32_t pattern, uint64_t offset,
                                       uint64_t nbytes, void *stream) {
    if (!a || pattern > 1) return GD_ERR_INVALID_ARG;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);    // bounds stay valid until enqueued
    uint64_t b, s;
    gd_status st = snapshot(a, id, &b, &s);
    if (st != GD_OK) return st;
    if ((offset | nbytes) % 16) return GD_ERR_ALIGN;
    if (offset > s || nbytes > s - offset) return GD_ERR_OOB_RANGE;
    if (nbytes == 0) return GD_OK;
    DeviceGuard dg(a->device);
    Geom g{a->sms};
    cudaError_t e = launch_fill(b, offset, nbytes, pattern, (cudaStream_t)stream, g);
    return e == cudaSuccess ? GD_OK : cuda_fail(e);
}

// ===========================================================================
// Fenced launches: one validated dispatch path shared by the direct entry
// points and the multi-tenant launcher.
// ===========================================================================

namespace gd {

// Every byte an affine kernel may touch lies in [base, base + size)
// (conservative extents: a false "no" only leaves the hoisting to the kernel).
bool footprint_inside(const gd_work &w, uint64_t base, uint64_t size) {
    uint64_t n = 0;
    switch (w.kind) {
        case GD_KIND_COPY:
            return range_ok(base, size, w.ptr[0], w.u64[0]) && range_ok(base, size, w.ptr[1], w.u64[0]);
        case GD_KIND_SAXPY:
            return mul_ok(w.u64[0], 4, &n) && range_ok(base, size, w.ptr[0], n) && range_ok(base, size, w.ptr[1], n);
        case GD_KIND_STENCIL: {
            if (w.u32[2] != 0) return false;           // K5 v2: fenced through its tensor maps
            const uint64_t H = w.u32[0], W = w.u32[1], pitch = w.u64[0];
            uint64_t rows = 0;
            if (!mul_ok(H, pitch, &rows) || !mul_ok(rows + W, 4, &n)) return false;
            return range_ok(base, size, w.ptr[0], n) && range_ok(base, size, w.ptr[1], n);
        }
        default:
            return false;                              // random accesses are fenced one by one
    }
}

// Validate `w` (dry) or validate and launch it.  Structural errors are
// returned before anything is issued.
gd_status run_work_locked(gd_arena *a, const gd_work &w_in, cudaStream_t stream, bool dry, bool account,
                          LaunchOut *out) {
    if (!a) return GD_ERR_INVALID_ARG;
    gd_work w = w_in;
    if ((w.mode & ~(kModeMask | GD_FENCE_PER_ACCESS)) || base_mode(w.mode) > GD_MODE_CLAMP || w.kind >= GD_NUM_KINDS)
        return GD_ERR_INVALID_ARG;
    // GD_FENCE_PER_ACCESS: no tile-level range test (the paper's per-access
    // instrumentation; identical results); GD_CHECK_PER_ACCESS=1 forces it
    // for every launch of the process
    static const bool env_pa = [] {
        const char *e = getenv("GD_CHECK_PER_ACCESS");
        return e && e[0] == '1';
    }();
    const bool per_access = env_pa || (w.mode & GD_FENCE_PER_ACCESS);
    w.mode = base_mode(w.mode);
    uint64_t base, size;
    gd_status st = snapshot(a, w.tenant, &base, &size);
    if (st != GD_OK) return st;
    // mask fencing needs a power-of-two, size-aligned partition
    if ((w.mode == GD_MODE_MASK || w.mode == GD_MODE_MASK_COUNT) && ((size & (size - 1)) || (base & (size - 1))))
        return GD_ERR_NOT_POW2;

    uint64_t bytes = 0, flops = 0, t;
    bool empty = false;
    switch (w.kind) {
        case GD_KIND_COPY:
            if ((w.ptr[0] | w.ptr[1]) % 16) return GD_ERR_ALIGN;
            if (w.u64[0] > (1ull << 44)) return GD_ERR_INVALID_ARG;      // grid < 2^31 CTAs
            bytes = 2 * w.u64[0];
            empty = w.u64[0] == 0;
            break;
        case GD_KIND_SAXPY:
            if ((w.ptr[0] | w.ptr[1]) % 16) return GD_ERR_ALIGN;
            if (w.u64[0] > (1ull << 42)) return GD_ERR_INVALID_ARG;
            bytes = 12 * w.u64[0];
            flops = 2 * w.u64[0];
            empty = w.u64[0] == 0;
            break;
        case GD_KIND_GATHER:
            if ((w.ptr[0] | w.ptr[2]) % 16 || w.ptr[1] % 4) return GD_ERR_ALIGN;
            if (w.u32[0] == 0) return GD_ERR_INVALID_ARG;
            if (!mul_ok(w.u64[0], (uint64_t)w.u32[0], &t) || t > (1ull << 41)) return GD_ERR_INVALID_ARG;   // k_gatherE: 2^11 words per CTA
            bytes = 4 * w.u64[0] + 8 * t;
            empty = w.u64[0] == 0;
            break;
        case GD_KIND_SCATTER:
            if ((w.ptr[1] | w.ptr[2]) % 16 || w.ptr[0] % 4) return GD_ERR_ALIGN;
            if (w.u64[0] > (1ull << 42)) return GD_ERR_INVALID_ARG;
            bytes = 16 * w.u64[0];
            empty = w.u64[0] == 0;
            break;
        case GD_KIND_STENCIL: {
            const uint64_t pitch = w.u64[0], H = w.u32[0], W = w.u32[1];
            if ((w.ptr[0] | w.ptr[1]) % 16 || pitch % 4) return GD_ERR_ALIGN;
            if (pitch < W || !mul_ok(H, pitch, &t) || t > (1ull << 58)) return GD_ERR_INVALID_ARG;
            if (w.u32[2] > 1) return GD_ERR_INVALID_ARG;          // 0: K5 v1 (LSU), 1: K5 v2 (TMA)
            if (w.u32[2] == 0 && H > (1ull << 19)) return GD_ERR_UNSUPPORTED;   // v1 grid.y <= 65535
            empty = H < 3 || W < 3;
            bytes = empty ? 0 : 8 * (H - 2) * (W - 2);
            flops = empty ? 0 : 5 * (H - 2) * (W - 2);
            break;
        }
        case GD_KIND_GEMM: {
            const uint64_t M = w.u32[0], N = w.u32[1], K = w.u32[2];
            if ((w.ptr[0] | w.ptr[1] | w.ptr[2]) % 16) return GD_ERR_ALIGN;
            if (w.u64[0] < K || w.u64[1] < K || w.u64[2] < N) return GD_ERR_INVALID_ARG;
            if ((w.u64[0] | w.u64[1] | w.u64[2]) % 8) return GD_ERR_UNSUPPORTED;
            empty = M == 0 || N == 0;
            if (!empty && (K == 0 || K % 64 || N % 16)) return GD_ERR_UNSUPPORTED;
            flops = 2 * M * N * K;
            bytes = 2 * (M * K + N * K + M * N);
            break;
        }
    }
    if (dry || empty) return GD_OK;
    if (a->device < 0) return GD_ERR_UNSUPPORTED;      // virtual arena: bookkeeping only
    // PAPER.md:175 "when an application runs alone ... issues a native kernel"
    // (SPEC.md:418 --native-when-solo, off by default): validated as requested,
    // run unfenced
    // (the caller's shared hold of launch_mu keeps the partition count fixed
    // until this launch is enqueued; a later carve synchronises before it
    // scrubs, so the unfenced kernel cannot reach the new partition)
    const bool solo = w.mode != GD_MODE_NONE && solo_native(a);
    if (solo) w.mode = GD_MODE_NONE;
    // R-hoist at launch granularity: an affine kernel (copy, saxpy, stencil
    // v1) whose whole footprint lies in the partition performs exactly the
    // accesses the check predicate allows, counts none, and every modulo /
    // clamp fence of it is the identity, so the unfenced twin computes the same
    // result; the host decides it from this launch's bounds snapshot (held
    // stable by the launch guard until the enqueue).  The kernels' own
    // per-CTA test still hoists the inner tiles of a launch that crosses the
    // partition edge.  Mask mode is never hoisted, per-access launches never.
    if (!per_access && hoistable(w.mode) && footprint_inside(w, base, size)) w.mode = GD_MODE_NONE;

    FenceDesc fd;
    fd.base = base;
    fd.mask = size - 1;
    fd.mask16 = (size - 1) & ~15ull;
    fd.mask4 = (size - 1) & ~3ull;
    fd.size = size;
    fd.inv = recip64(size);
    fd.viol = a->d_stats + (uint64_t)w.tenant * GD_NUM_KINDS + w.kind;
    fd.flags = (per_access ? kNoHoist : 0u) |
               (((size & (size - 1)) == 0 && size >= (1ull << 32) && (base & (size - 1)) == 0) ? kBig : 0u);
    fd.zero = a->d_zero;
    fd.pad_ = 0;
    const Geom g{a->sms};
    DeviceGuard dg(a->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err);
    cudaError_t e = cudaSuccess;
    switch (w.kind) {
        case GD_KIND_COPY: e = launch_copy(w.mode, fd, w.ptr[0], w.ptr[1], w.u64[0], stream, g); break;
        case GD_KIND_SAXPY: e = launch_saxpy(w.mode, fd, w.f32[0], w.ptr[0], w.ptr[1], w.u64[0], stream, g); break;
        case GD_KIND_GATHER:
            e = launch_gather(w.mode, fd, w.ptr[0], w.ptr[1], w.ptr[2], w.u64[0], w.u32[0], stream, g);
            break;
        case GD_KIND_SCATTER:
            e = launch_scatter(w.mode, fd, w.ptr[0], w.ptr[1], w.ptr[2], w.u64[0], stream, g);
            break;
        case GD_KIND_STENCIL:
            if (w.u32[2] == 1) {
                st = stencil_tma_dispatch(a, w, base, size, stream, g);
                if (st != GD_OK) return st;
            } else {
                e = launch_stencil(w.mode, fd, w.ptr[0], w.ptr[1], w.u32[0], w.u32[1], w.u64[0], w.f32[0], w.f32[1],
                                   stream, g);
            }
            break;
        case GD_KIND_GEMM: {
            st = gemm_dispatch(a, w, base, size, stream, g);
            if (st != GD_OK) return st;
            break;
        }
    }
    if (e != cudaSuccess) return cuda_fail(e);
    if (out) {
        out->bytes = bytes;
        out->flops = flops;
        out->solo = solo;
    }
    if (account) {
        std::lock_guard<std::mutex> lk(a->mu);
        HostCounters &hc = a->host[w.tenant][w.kind];
        hc.launches++;
        hc.bytes += bytes;
        hc.flops += flops;
    }
    return GD_OK;
}

gd_status run_work(gd_arena *a, const gd_work &w, cudaStream_t stream, bool dry) {
    if (!a) return GD_ERR_INVALID_ARG;
    std::shared_lock<std::shared_mutex> guard(a->launch_mu);
    return run_work_locked(a, w, stream, dry);
}

gd_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GD_OK : cuda_fail(e); }

gd_status partition_snapshot(gd_arena *a, uint32_t id, uint64_t *base, uint64_t *size, uint64_t *gen) {
    std::lock_guard<std::mutex> lk(a->mu);
    if (id >= GD_MAX_TENANTS || !a->parts[id].live) return GD_ERR_UNKNOWN_PARTITION;
    *base = a->parts[id].base;
    *size = a->parts[id].size;
    *gen = a->parts[id].gen;
    return GD_OK;
}

}  // namespace gd

namespace {
gd_work mk(uint32_t id, gd_kind kind, gd_mode mode) {
    gd_work w;
    std::memset(&w, 0, sizeof(w));
    w.tenant = id;
    w.kind = kind;
    w.mode = (uint32_t)mode;
    return w;
}
}  // namespace

extern "C" gd_status gd_launch_fenced_copy(gd_arena *a, uint32_t id, gd_mode mode, uint64_t dst, uint64_t src,
                                           uint64_t nbytes, void *stream) {
    gd_work w = mk(id, GD_KIND_COPY, mode);
    w.ptr[0] = dst;
    w.ptr[1] = src;
    w.u64[0] = nbytes;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_saxpy(gd_arena *a, uint32_t id, gd_mode mode, float alpha, uint64_t x,
                                            uint64_t y, uint64_t n, void *stream) {
    gd_work w = mk(id, GD_KIND_SAXPY, mode);
    w.ptr[0] = x;
    w.ptr[1] = y;
    w.u64[0] = n;
    w.f32[0] = alpha;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_gather(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out, uint64_t table,
                                             uint64_t idx, uint64_t n, uint32_t row_elems, void *stream) {
    gd_work w = mk(id, GD_KIND_GATHER, mode);
    w.ptr[0] = out;
    w.ptr[1] = table;
    w.ptr[2] = idx;
    w.u64[0] = n;
    w.u32[0] = row_elems;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_scatter(gd_arena *a, uint32_t id, gd_mode mode, uint64_t table, uint64_t idx,
                                              uint64_t src, uint64_t n, void *stream) {
    gd_work w = mk(id, GD_KIND_SCATTER, mode);
    w.ptr[0] = table;
    w.ptr[1] = idx;
    w.ptr[2] = src;
    w.u64[0] = n;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_stencil(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out, uint64_t in,
                                              uint32_t H, uint32_t W, uint64_t pitch_elems, float c0, float c1,
                                              void *stream) {
    gd_work w = mk(id, GD_KIND_STENCIL, mode);
    w.ptr[0] = out;
    w.ptr[1] = in;
    w.u32[0] = H;
    w.u32[1] = W;
    w.u64[0] = pitch_elems;
    w.f32[0] = c0;
    w.f32[1] = c1;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_stencil_tma(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out,
                                                  uint64_t in, uint32_t H, uint32_t W, uint64_t pitch_elems, float c0,
                                                  float c1, void *stream) {
    gd_work w = mk(id, GD_KIND_STENCIL, mode);
    w.ptr[0] = out;
    w.ptr[1] = in;
    w.u32[0] = H;
    w.u32[1] = W;
    w.u32[2] = 1;
    w.u64[0] = pitch_elems;
    w.f32[0] = c0;
    w.f32[1] = c1;
    return run_work(a, w, (cudaStream_t)stream, false);
}

extern "C" gd_status gd_launch_fenced_gemm(gd_arena *a, uint32_t id, gd_mode mode, uint64_t C, uint64_t A,
                                           uint64_t B, uint32_t M, uint32_t N, uint32_t K, uint64_t lda,
                                           uint64_t ldb, uint64_t ldc, void *stream) {
    gd_work w = mk(id, GD_KIND_GEMM, mode);
    w.ptr[0] = C;
    w.ptr[1] = A;
    w.ptr[2] = B;
    w.u32[0] = M;
    w.u32[1] = N;
    w.u32[2] = K;
    w.u64[0] = lda;
    w.u64[1] = ldb;
    w.u64[2] = ldc;
    return run_work(a, w, (cudaStream_t)stream, false);
}

// ===========================================================================
// Statistics
// ===========================================================================

extern "C" gd_status gd_stats(gd_arena *a, uint32_t id, gd_stats_t *out) {
    if (!a || !out) return GD_ERR_INVALID_ARG;
    std::memset(out, 0, sizeof(*out));
    if (id != GD_ALL_TENANTS && !tenant_live(a, id)) return GD_ERR_UNKNOWN_PARTITION;
    unsigned long long dev[GD_MAX_TENANTS * GD_NUM_KINDS];
    std::memset(dev, 0, sizeof(dev));
    if (a->device >= 0) {
        DeviceGuard dg(a->device);
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = cudaMemcpy(dev, a->d_stats, sizeof(dev), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    std::lock_guard<std::mutex> lk(a->mu);
    for (uint32_t t = 0; t < GD_MAX_TENANTS; t++) {
        if (id != GD_ALL_TENANTS && t != id) continue;
        for (unsigned k = 0; k < GD_NUM_KINDS; k++) {
            const uint64_t v = dev[t * GD_NUM_KINDS + k];
            out->violations += v;
            out->violations_by_kind[k] += v;
            out->launches += a->host[t][k].launches;
            out->launches_by_kind[k] += a->host[t][k].launches;
            out->bytes += a->host[t][k].bytes;
            out->flops += a->host[t][k].flops;
        }
    }
    return GD_OK;
}

extern "C" gd_status gd_stats_reset(gd_arena *a, uint32_t id) {
    if (!a) return GD_ERR_INVALID_ARG;
    if (id != GD_ALL_TENANTS && !tenant_live(a, id)) return GD_ERR_UNKNOWN_PARTITION;
    if (a->device >= 0) {
        DeviceGuard dg(a->device);
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) {
            if (id == GD_ALL_TENANTS)
                e = cudaMemset(a->d_stats, 0, sizeof(unsigned long long) * GD_MAX_TENANTS * GD_NUM_KINDS);
            else
                e = cudaMemset(a->d_stats + (uint64_t)id * GD_NUM_KINDS, 0, sizeof(unsigned long long) * GD_NUM_KINDS);
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e);
    }
    std::lock_guard<std::mutex> lk(a->mu);
    for (uint32_t t = 0; t < GD_MAX_TENANTS; t++)
        if (id == GD_ALL_TENANTS || t == id)
            for (unsigned k = 0; k < GD_NUM_KINDS; k++) a->host[t][k] = HostCounters{};
    return GD_OK;
}

extern "C" gd_status gd_stats_device_ptr(const gd_arena *a, uint64_t *dev_ptr) {
    if (!a || !dev_ptr) return GD_ERR_INVALID_ARG;
    *dev_ptr = (uint64_t)a->d_stats;
    return GD_OK;
}

extern "C" const char *gd_status_str(gd_status s) {
    switch (s) {
        case GD_OK: return "GD_OK";
        case GD_ERR_INVALID_ARG: return "GD_ERR_INVALID_ARG";
        case GD_ERR_NOT_POW2: return "GD_ERR_NOT_POW2";
        case GD_ERR_DEVICE_OOM: return "GD_ERR_DEVICE_OOM";
        case GD_ERR_PARTITION_OOM: return "GD_ERR_PARTITION_OOM";
        case GD_ERR_UNKNOWN_PARTITION: return "GD_ERR_UNKNOWN_PARTITION";
        case GD_ERR_UNKNOWN_ALLOC: return "GD_ERR_UNKNOWN_ALLOC";
        case GD_ERR_ALIGN: return "GD_ERR_ALIGN";
        case GD_ERR_OOB_RANGE: return "GD_ERR_OOB_RANGE";
        case GD_ERR_UNSUPPORTED: return "GD_ERR_UNSUPPORTED";
        case GD_ERR_CUDA: return "GD_ERR_CUDA";
    }
    return "GD_ERR_UNKNOWN";
}

extern "C" int gd_last_cuda_error(void) { return g_last_cuda; }

extern "C" gd_status gd_arena_set_native_when_solo(gd_arena *a, int on) {
    if (!a) return GD_ERR_INVALID_ARG;
    std::unique_lock<std::shared_mutex> guard(a->launch_mu);
    std::lock_guard<std::mutex> lk(a->mu);
    a->native_when_solo = on != 0;
    a->epoch++;                                       // graphs captured under the old rule go stale
    return GD_OK;
}

extern "C" gd_status gd_device_flags(gd_arena *a, uint32_t *flags) {
    if (!a || !flags) return GD_ERR_INVALID_ARG;
    *flags = 0;
    if (a->device < 0) return GD_OK;
    DeviceGuard dg(a->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    *flags = (gemm_timeout_flag() ? 1u : 0u) | (stencil_tma_timeout_flag() ? 2u : 0u);
    return GD_OK;
}

extern "C" const char *gd_version(void) { return "guardian-b200 sm_100a (libguardian " __DATE__ ")"; }
