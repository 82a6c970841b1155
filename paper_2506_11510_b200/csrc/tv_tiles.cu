// Image-space sharding helpers for multi-GPU rendering: each rank renders the
// interleaved 16x16 tiles t with t % n_ranks == rank. Pack
// gathers this rank's tiles from a full-frame device buffer into a contiguous
// block of ceil(tiles / n_ranks) * 256 pixels (equal size on every rank, so one
// NCCL all-gather moves the frame); unpack scatters a gathered block back.
#include <algorithm>
#include <cstring>

#include <cuda.h>

#include "tv_trace.cuh"

namespace tvb {
namespace {

__global__ void pack_kernel(const uint64_t* __restrict__ frame, uint64_t* __restrict__ packed, int32_t w, int32_t h,
                            int32_t rank, int32_t n_ranks, int32_t ew, uint64_t slots, int unpack) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;  // packed pixel slot
    if (i >= slots) return;
    const uint32_t tiles_x = (static_cast<uint32_t>(w) + 15) / 16;
    const uint32_t tiles_y = (static_cast<uint32_t>(h) + 15) / 16;
    const uint64_t k = i >> 8, local = i & 255;
    const uint64_t t = static_cast<uint64_t>(rank) + k * static_cast<uint64_t>(n_ranks);
    if (t >= static_cast<uint64_t>(tiles_x) * tiles_y) return;
    const int px = static_cast<int>((t % tiles_x) * 16 + (local & 15));
    const int py = static_cast<int>((t / tiles_x) * 16 + (local >> 4));
    if (px >= w || py >= h) return;
    const uint64_t p = static_cast<uint64_t>(py) * w + px;
    for (int e = 0; e < ew; ++e) {
        if (unpack)
            const_cast<uint64_t*>(frame)[p * ew + e] = packed[i * ew + e];
        else
            packed[i * ew + e] = frame[p * ew + e];
    }
}

int run(const void* frame, void* packed, int32_t w, int32_t h, int32_t rank, int32_t n_ranks, int32_t ew,
        void* stream, int unpack) {
    if (!frame || !packed) return set_error(TV_ERR_ARG, "null buffer");
    if (w < 1 || h < 1 || n_ranks < 1 || rank < 0 || rank >= n_ranks || ew < 1)
        return set_error(TV_ERR_ARG, "bad tile pack arguments");
    const uint64_t words = tv_tile_pack_words(w, h, rank, n_ranks, ew);
    const uint64_t slots = words / static_cast<uint64_t>(ew);
    pack_kernel<<<static_cast<unsigned>((slots + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint64_t*>(frame), static_cast<uint64_t*>(packed), w, h, rank, n_ranks, ew, slots, unpack);
    return cuda_status(cudaGetLastError(), "tile pack");
}

}  // namespace
}  // namespace tvb

extern "C" {

uint64_t tv_tile_pack_words(int32_t width, int32_t height, int32_t rank, int32_t n_ranks, int32_t elem_words) {
    (void)rank;
    if (width < 1 || height < 1 || n_ranks < 1 || elem_words < 1) return 0;
    const uint64_t tiles = static_cast<uint64_t>((width + 15) / 16) * static_cast<uint64_t>((height + 15) / 16);
    const uint64_t per_rank = (tiles + n_ranks - 1) / n_ranks;
    return per_rank * 256 * static_cast<uint64_t>(elem_words);
}

int tv_tile_pack(const void* frame_dev, void* packed_dev, int32_t width, int32_t height, int32_t rank,
                 int32_t n_ranks, int32_t elem_words, void* stream) {
    return tvb::run(frame_dev, packed_dev, width, height, rank, n_ranks, elem_words, stream, 0);
}

int tv_tile_unpack(const void* packed_dev, void* frame_dev, int32_t width, int32_t height, int32_t rank,
                   int32_t n_ranks, int32_t elem_words, void* stream) {
    return tvb::run(frame_dev, const_cast<void*>(packed_dev), width, height, rank, n_ranks, elem_words, stream, 1);
}

int tv_ipc_export(const void* dev_ptr, uint8_t handle[64], uint64_t* offset) {
    if (!dev_ptr || !handle || !offset) return tvb::set_error(TV_ERR_ARG, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, dev_ptr);
    if (e != cudaSuccess || a.type != cudaMemoryTypeDevice)
        return tvb::set_error(TV_ERR_ARG, "ipc export: not a device pointer");
    if ((e = cudaSetDevice(a.device)) != cudaSuccess) return tvb::cuda_status(e, "cudaSetDevice");
    // the handle names the allocation containing dev_ptr: find its base
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<GetRange>(fn);
    }();
    if (!get_range) return tvb::set_error(TV_ERR_CUDA, "ipc export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return tvb::set_error(TV_ERR_CUDA, "ipc export: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return tvb::cuda_status(e, "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, 64);
    *offset = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
    return TV_OK;
}

int tv_ipc_open(const uint8_t handle[64], uint64_t offset, int device, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return tvb::set_error(TV_ERR_ARG, "null argument");
    *dev_ptr_out = nullptr;
    int rc = tvb::use_device(device);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* base = nullptr;
    rc = tvb::cuda_status(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    if (rc) return rc;
    *dev_ptr_out = static_cast<char*>(base) + offset;
    return TV_OK;
}

int tv_ipc_close(void* dev_ptr, uint64_t offset) {
    if (!dev_ptr) return TV_OK;
    return tvb::cuda_status(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset), "cudaIpcCloseMemHandle");
}

}  // extern "C"
