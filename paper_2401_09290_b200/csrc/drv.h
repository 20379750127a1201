// drv.h -- CUDA driver entry points, resolved at run time through
// cudaGetDriverEntryPoint so that libguardian.so does not link libcuda
// directly (it loads on machines without a GPU driver: the CPU test tier).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace gd {

struct Drv {
    bool ok = false;
    decltype(&::cuMemAddressReserve) MemAddressReserve = nullptr;
    decltype(&::cuMemAddressFree) MemAddressFree = nullptr;
    decltype(&::cuMemCreate) MemCreate = nullptr;
    decltype(&::cuMemRelease) MemRelease = nullptr;
    decltype(&::cuMemMap) MemMap = nullptr;
    decltype(&::cuMemUnmap) MemUnmap = nullptr;
    decltype(&::cuMemSetAccess) MemSetAccess = nullptr;
    decltype(&::cuMemGetAllocationGranularity) MemGetAllocationGranularity = nullptr;
    decltype(&::cuTensorMapEncodeTiled) TensorMapEncodeTiled = nullptr;
};

inline const Drv &drv() {
    static const Drv d = [] {
        Drv r;
        bool ok = true;
        auto get = [&ok](const char *name, void **fp) {
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, fp, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !*fp)
                ok = false;
        };
        get("cuMemAddressReserve", (void **)&r.MemAddressReserve);
        get("cuMemAddressFree", (void **)&r.MemAddressFree);
        get("cuMemCreate", (void **)&r.MemCreate);
        get("cuMemRelease", (void **)&r.MemRelease);
        get("cuMemMap", (void **)&r.MemMap);
        get("cuMemUnmap", (void **)&r.MemUnmap);
        get("cuMemSetAccess", (void **)&r.MemSetAccess);
        get("cuMemGetAllocationGranularity", (void **)&r.MemGetAllocationGranularity);
        get("cuTensorMapEncodeTiled", (void **)&r.TensorMapEncodeTiled);
        r.ok = ok;
        return r;
    }();
    return d;
}

}  // namespace gd
