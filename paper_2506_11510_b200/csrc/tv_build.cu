// GPU LEB build (round-based, bit-exact with build_adaptive_grid) and the
// on-device procedural fields.
#include "tv_trace.cuh"

namespace tvb {
namespace {

// cli.cpp:317-321
__device__ double blob_density(double x, double y, double z) {
    const d3 d = sub(mk(x, y, z), mk(0.5, 0.5, 0.5));
    const double t = dmax(0.0, 1.0 - dot(d, d) / (0.45 * 0.45));
    return t * t;
}

// cli.cpp:323-346, generalised to (cells, seed)
__device__ double vnoise(double px, double py, double pz, int cells, uint64_t seed) {
    const double x = dclamp(px, 0.0, 1.0) * cells, y = dclamp(py, 0.0, 1.0) * cells, z = dclamp(pz, 0.0, 1.0) * cells;
    const int ix = min(static_cast<int>(x), cells - 1), iy = min(static_cast<int>(y), cells - 1),
              iz = min(static_cast<int>(z), cells - 1);
    const double fx = x - ix, fy = y - iy, fz = z - iz;
    double v = 0.0;
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const double w = (dx ? fx : 1.0 - fx) * (dy ? fy : 1.0 - fy) * (dz ? fz : 1.0 - fz);
                const uint64_t h = mix64(mix64(mix64(seed ^ static_cast<uint64_t>(static_cast<int64_t>(ix + dx))) ^
                                               static_cast<uint64_t>(static_cast<int64_t>(iy + dy))) ^
                                         static_cast<uint64_t>(static_cast<int64_t>(iz + dz)));
                v += w * (static_cast<double>(h >> 11) * 0x1.0p-53);
            }
    return v;
}

constexpr uint64_t kNoiseSeed = 0x5eb0a8a5c9d3f1adull;

__global__ void gen_kernel(int kind, int nx, int ny, int nz, double value, float* out) {
    const uint64_t n = static_cast<uint64_t>(nx) * ny * nz;
    for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; idx < n;
         idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx % nx), j = static_cast<int>((idx / nx) % ny),
                  k = static_cast<int>(idx / (static_cast<uint64_t>(nx) * ny));
        const double x = (i + 0.5) / nx, y = (j + 0.5) / ny, z = (k + 0.5) / nz;  // volume.hpp:44-46
        double d;
        switch (kind) {
            case 0: d = value; break;
            case 1: d = x; break;
            case 2: d = blob_density(x, y, z); break;
            case 3: d = x < 0.5 ? 1.0 : 0.0; break;
            case 4: d = vnoise(x, y, z, 8, kNoiseSeed); break;
            default: {
                double s = 0.0;
                for (int o = 0; o < 4; ++o) s += ldexp(1.0, -(o + 1)) * vnoise(x, y, z, 8 << o, kNoiseSeed + o);
                const double c = dmax(0.0, s - 0.35);
                d = c * 2.0 * blob_density(x, y, z) / 0.9375;
            }
        }
        out[idx] = static_cast<float>(d);
    }
}

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

int tv_generate_volume_dev(int32_t kind, int32_t nx, int32_t ny, int32_t nz, double value, float* out_dev,
                           int device) {
    if (!out_dev) return set_error(TV_ERR_ARG, "null output");
    if (nx < 1 || ny < 1 || nz < 1 || nx > 4096 || ny > 4096 || nz > 4096)
        return set_error(TV_ERR_CONFIG, "dims out of range [1, 4096]");
    if (kind < 0 || kind > 5) return set_error(TV_ERR_CONFIG, "unknown kind (constant|ramp|blob|step|noise|cloud)");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    gen_kernel<<<148 * 8, 256>>>(kind, nx, ny, nz, value, out_dev);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return cuda_status(e, "generate volume");
}

int tv_build_dev(const float*, const float*, const float*, int32_t, int32_t, int32_t, const tv_build_config*,
                 const tv_camera*, int, tv_grid** out, tv_build_stats*) {
    if (out) *out = nullptr;
    return set_error(TV_ERR, "tv_build_dev: GPU LEB build not available in this build");
}

int tv_build(const float*, const float*, const float*, int32_t, int32_t, int32_t, const tv_build_config*,
             const tv_camera*, int, tv_grid** out, tv_build_stats*) {
    if (out) *out = nullptr;
    return set_error(TV_ERR, "tv_build: GPU LEB build not available in this build");
}

int tv_render_regular(const float*, int32_t, int32_t, int32_t, double, const tv_camera*, const tv_render_config*, int,
                      tv_framebuffer*, tv_render_stats*) {
    return set_error(TV_ERR, "tv_render_regular: not available in this build");
}

}  // extern "C"
