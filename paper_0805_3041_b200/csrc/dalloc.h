// Device allocations of the library. Plain cudaMalloc/cudaFree, except under
// GMG_GUARD_ALLOC (debugging aid): every buffer gets its own virtual-address
// reservation with unmapped guard pages around the mapped pages, and is placed
// flush against the end (=1) or the start (=2) of its mapping, so a read or
// write past that end faults at once instead of landing on a neighbouring
// allocation.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <map>
#include <mutex>

namespace gmg_alloc {

struct Vmm {
    CUdeviceptr va;
    size_t reserve, mapped;
    CUmemGenericAllocationHandle h;
};

inline int guard_mode() {
    static const int m = [] {
        const char* e = getenv("GMG_GUARD_ALLOC");
        return e ? atoi(e) : 0;
    }();
    return m;
}

struct Drv {
    CUresult (*gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*unmap)(CUdeviceptr, size_t);
    CUresult (*release)(CUmemGenericAllocationHandle);
    CUresult (*vafree)(CUdeviceptr, size_t);
};

inline Drv& drv() {
    static Drv d = [] {
        Drv x{};
        void* h = dlopen("libcuda.so.1", RTLD_NOW);
        if (!h) abort();
        x.gran = (decltype(x.gran))dlsym(h, "cuMemGetAllocationGranularity");
        x.create = (decltype(x.create))dlsym(h, "cuMemCreate");
        x.reserve = (decltype(x.reserve))dlsym(h, "cuMemAddressReserve");
        x.map = (decltype(x.map))dlsym(h, "cuMemMap");
        x.access = (decltype(x.access))dlsym(h, "cuMemSetAccess");
        x.unmap = (decltype(x.unmap))dlsym(h, "cuMemUnmap");
        x.release = (decltype(x.release))dlsym(h, "cuMemRelease");
        x.vafree = (decltype(x.vafree))dlsym(h, "cuMemAddressFree");
        return x;
    }();
    return d;
}

inline std::map<void*, Vmm>& table() {
    static std::map<void*, Vmm> t;
    return t;
}
inline std::mutex& mtx() {
    static std::mutex m;
    return m;
}

inline cudaError_t guarded_malloc(void** out, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaFree(nullptr);  // make sure the primary context exists
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    Drv& d = drv();
    size_t g = 0;
    if (d.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    const size_t b256 = (bytes + 255) / 256 * 256;
    const size_t sz = (b256 + g - 1) / g * g + (b256 == 0 ? g : 0);
    Vmm v{};
    v.reserve = sz + 2 * g;
    v.mapped = sz;
    if (d.reserve(&v.va, v.reserve, 0, 0, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    if (d.create(&v.h, sz, &prop, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    const CUdeviceptr mb = v.va + g;
    if (d.map(mb, sz, 0, v.h, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.access(mb, sz, &acc, 1) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    void* p = reinterpret_cast<void*>(guard_mode() == 2 ? mb : mb + sz - b256);
    std::lock_guard<std::mutex> lk(mtx());
    table()[p] = v;
    *out = p;
    return cudaSuccess;
}

inline cudaError_t guarded_free(void* p) {
    std::lock_guard<std::mutex> lk(mtx());
    auto it = table().find(p);
    if (it == table().end()) return cudaFree(p);
    cudaDeviceSynchronize();
    Drv& d = drv();
    const Vmm v = it->second;
    const size_t g = (v.reserve - v.mapped) / 2;
    d.unmap(v.va + g, v.mapped);
    d.release(v.h);
    d.vafree(v.va, v.reserve);
    table().erase(it);
    return cudaSuccess;
}

}  // namespace gmg_alloc

template <class T>
inline cudaError_t dmalloc(T** p, size_t bytes) {
    if (!gmg_alloc::guard_mode()) return cudaMalloc(reinterpret_cast<void**>(p), bytes);
    return gmg_alloc::guarded_malloc(reinterpret_cast<void**>(p), bytes);
}
inline cudaError_t dfree(void* p) {
    if (!p) return cudaSuccess;
    if (!gmg_alloc::guard_mode()) return cudaFree(p);
    return gmg_alloc::guarded_free(p);
}
