// Dev tool: per-call cost of the VMM growth path (cuMemCreate / cuMemMap /
// cuMemSetAccess) for growing chunks, idle GPU vs. GPU busy with a kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

static double ms(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
__global__ void spin(unsigned long long cycles) {
    const unsigned long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = 0;
    CUmemAccessDesc a = {};
    a.location = p.location;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int busy = 0; busy < 2; ++busy)
        for (int rep = 0; rep < 2; ++rep) {
            CUdeviceptr va;
            const size_t total = 32ull << 30;
            cuMemAddressReserve(&va, total, 0, 0, 0);
            size_t off = 0;
            CUmemGenericAllocationHandle hs[16];
            int nh = 0;
            for (size_t sz = 256ull << 20; off + sz <= total && nh < 16; sz *= 2) {
                if (busy) spin<<<148, 32>>>(2000000000ull / 10);  // ~100 ms of GPU work in flight
                auto t = std::chrono::steady_clock::now();
                cuMemCreate(&hs[nh], sz, &p, 0);
                const double tc = ms(t);
                t = std::chrono::steady_clock::now();
                cuMemMap(va + off, sz, 0, hs[nh], 0);
                const double tm = ms(t);
                t = std::chrono::steady_clock::now();
                cuMemSetAccess(va + off, sz, &a, 1);
                const double ta = ms(t);
                std::printf("busy %d rep %d size %6zu MB: create %7.2f map %6.2f access %7.2f ms\n", busy, rep,
                            sz >> 20, tc, tm, ta);
                off += sz;
                ++nh;
                cudaDeviceSynchronize();
            }
            cuMemUnmap(va, off);
            for (int i = 0; i < nh; ++i) cuMemRelease(hs[i]);
            cuMemAddressFree(va, total);
        }
    return 0;
}
