// Dev tool: cost of device-memory allocation paths on this box (cudaMalloc,
// stream-ordered pool growth, VMM map) — the LEB build grows GB-sized arrays.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>

static double ms_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    const size_t GB = 1ull << 30;
    for (size_t g : {1, 4, 8}) {
        void* p;
        auto t = std::chrono::steady_clock::now();
        cudaMalloc(&p, g * GB);
        cudaDeviceSynchronize();
        double a = ms_since(t);
        t = std::chrono::steady_clock::now();
        cudaMemset(p, 0, g * GB);
        cudaDeviceSynchronize();
        double m = ms_since(t);
        t = std::chrono::steady_clock::now();
        cudaFree(p);
        double f = ms_since(t);
        std::printf("cudaMalloc %zu GB: alloc %.2f ms, first memset %.2f ms, free %.2f ms\n", g, a, m, f);
    }
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = 0;
    cudaMemPool_t pool;
    cudaMemPoolCreate(&pool, &props);
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    for (int rep = 0; rep < 2; ++rep)
        for (size_t g : {1, 4}) {
            void* p;
            auto t = std::chrono::steady_clock::now();
            cudaMallocFromPoolAsync(&p, g * GB, pool, 0);
            cudaStreamSynchronize(0);
            double a = ms_since(t);
            t = std::chrono::steady_clock::now();
            cudaMemsetAsync(p, 0, g * GB, 0);
            cudaStreamSynchronize(0);
            double m = ms_since(t);
            t = std::chrono::steady_clock::now();
            cudaFreeAsync(p, 0);
            cudaStreamSynchronize(0);
            double f = ms_since(t);
            std::printf("pool rep %d %zu GB: alloc %.2f ms, memset %.2f ms, free %.2f ms\n", rep, g, a, m, f);
        }
    cudaMemPoolTrimTo(pool, 0);
    // VMM: reserve 16 GB of VA, map 2 MB-granular chunks of 256 MB
    CUmemAllocationProp vp = {};
    vp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    vp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    vp.location.id = 0;
    size_t gran = 0;
    cuMemGetAllocationGranularity(&gran, &vp, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    CUdeviceptr va;
    cuMemAddressReserve(&va, 16 * GB, 0, 0, 0);
    CUmemAccessDesc ad = {};
    ad.location = vp.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    auto t = std::chrono::steady_clock::now();
    size_t off = 0;
    std::vector<CUmemGenericAllocationHandle> hs;
    for (int k = 0; k < 16; ++k) {
        CUmemGenericAllocationHandle h;
        const size_t chunk = 256ull << 20;
        cuMemCreate(&h, chunk, &vp, 0);
        cuMemMap(va + off, chunk, 0, h, 0);
        cuMemSetAccess(va + off, chunk, &ad, 1);
        hs.push_back(h);
        off += chunk;
    }
    std::printf("VMM: granularity %zu B, map 4 GB in 256 MB chunks %.2f ms\n", gran, ms_since(t));
    t = std::chrono::steady_clock::now();
    cudaMemset(reinterpret_cast<void*>(va), 0, off);
    cudaDeviceSynchronize();
    std::printf("VMM: first memset 4 GB %.2f ms\n", ms_since(t));
    t = std::chrono::steady_clock::now();
    CUmemGenericAllocationHandle h;
    cuMemCreate(&h, 4 * GB, &vp, 0);
    cuMemMap(va + off, 4 * GB, 0, h, 0);
    cuMemSetAccess(va + off, 4 * GB, &ad, 1);
    std::printf("VMM: map 4 GB in one chunk %.2f ms\n", ms_since(t));
    return 0;
}
