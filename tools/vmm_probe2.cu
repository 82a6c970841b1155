// Dev tool: cost of reserving / freeing device-memory-sized virtual ranges (as
// the build's growable buffers do, 25 at a time) and of mapping into them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

static double ms(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    size_t fr, tot;
    cudaMemGetInfo(&fr, &tot);
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = 0;
    CUmemAccessDesc a = {};
    a.location = p.location;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    size_t g = 0;
    cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    const size_t R = (tot + g - 1) / g * g;
    for (int rep = 0; rep < 4; ++rep) {
        CUdeviceptr va[25];
        CUmemGenericAllocationHandle h[25];
        auto t = std::chrono::steady_clock::now();
        double worst = 0;
        for (int i = 0; i < 25; ++i) {
            auto t1 = std::chrono::steady_clock::now();
            cuMemAddressReserve(&va[i], R, g, 0, 0);
            worst = std::max(worst, ms(t1));
        }
        const double tr = ms(t);
        t = std::chrono::steady_clock::now();
        double wm = 0;
        for (int i = 0; i < 25; ++i) {
            auto t1 = std::chrono::steady_clock::now();
            cuMemCreate(&h[i], 64ull << 20, &p, 0);
            cuMemMap(va[i], 64ull << 20, 0, h[i], 0);
            cuMemSetAccess(va[i], 64ull << 20, &a, 1);
            wm = std::max(wm, ms(t1));
        }
        const double tm = ms(t);
        t = std::chrono::steady_clock::now();
        for (int i = 0; i < 25; ++i) {
            cuMemUnmap(va[i], 64ull << 20);
            cuMemRelease(h[i]);
            cuMemAddressFree(va[i], R);
        }
        const double tf = ms(t);
        std::printf("rep %d: reserve 25 x %zu GB %.2f ms (worst %.2f), map 25 x 64 MB %.2f ms (worst %.2f), free %.2f ms\n",
                    rep, R >> 30, tr, worst, tm, wm, tf);
    }
    return 0;
}
