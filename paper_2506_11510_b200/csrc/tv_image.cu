// Output and compare: the PFM and variance-PFM writers and the
// PFM reader (image.cpp:33-101), and cmd_compare's metrics (cli.cpp:487-531),
// with the per-pixel work on the GPU.
//
// Per pixel the writers evaluate ImageAccumulator::mean / variance_of_mean
// (image.hpp:47-69) in the same FP64 order and round to f32, so the file bytes
// equal the reference's. compare's max |a-b| and 3-sigma outlier count are
// exact; its RMSE sums the squared differences in parallel, so it agrees with
// the reference's sequential sum to a few ulp (relative 1e-12 in the tests).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tv_trace.cuh"

namespace tvb {
namespace {

int img_error(const std::string& msg) { return set_error(TV_ERR_IMAGE, msg); }

// image.hpp:47-69; out is top-down RGB f32
__global__ void pfm_pixels_kernel(const double* __restrict__ sum, const double* __restrict__ sum_sq,
                                  const uint32_t* __restrict__ counts, uint64_t n_px, int variance, float* out) {
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n_px;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t n = counts[p];
        for (int c = 0; c < 3; ++c) {
            double v = 0.0;
            if (!variance) {
                if (n) v = sum[3 * p + c] / n;
            } else if (n >= 2) {
                const double m = sum[3 * p + c] / n;
                const double var = (sum_sq[3 * p + c] - static_cast<double>(n) * m * m) / (n - 1.0);
                v = (0.0 < var ? var : 0.0) / n;  // std::max(0.0, var)
            }
            out[3 * p + c] = static_cast<float>(v);
        }
    }
}

// cli.cpp:499-528: per value d = a - b, sum d^2 and max |d|; per pixel, an
// outlier when some channel has |d| > 3 sqrt(max(0, va + vb))
__global__ void compare_kernel(const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ va,
                               const float* __restrict__ vb, uint64_t n_px, double* sq_sum, unsigned long long* max_bits,
                               unsigned long long* outliers) {
    double sq = 0.0, mx = 0.0;
    unsigned long long bad = 0;
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n_px;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        bool out = false;
        for (int c = 0; c < 3; ++c) {
            const uint64_t i = 3 * p + c;
            const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
            sq += d * d;
            mx = fmax(mx, fabs(d));
            if (va && !out) {
                const double s = static_cast<double>(va[i]) + static_cast<double>(vb[i]);
                const double sigma = sqrt(0.0 < s ? s : 0.0);
                out = fabs(d) > 3.0 * sigma;
            }
        }
        bad += out;
    }
    for (int o = 16; o; o >>= 1) {
        sq += __shfl_down_sync(0xffffffffu, sq, o);
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
        bad += __shfl_down_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sq_sum, sq);
        atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));  // mx >= 0
        atomicAdd(outliers, bad);
    }
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

#define IM_CK(x, what)                    \
    do {                                  \
        int rc_ = cuda_status((x), what); \
        if (rc_) return rc_;              \
    } while (0)

// image.cpp:35-45
int write_pfm_rows(const char* path, int w, int h, const std::vector<float>& rgb) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return img_error(std::string("cannot open for writing: ") + path);
    bool ok = std::fprintf(f, "PF\n%d %d\n-1.000000\n", w, h) > 0;
    for (int y = h - 1; ok && y >= 0; --y)  // PFM stores rows bottom to top
        ok = std::fwrite(&rgb[static_cast<size_t>(y) * w * 3], sizeof(float), static_cast<size_t>(w) * 3, f) ==
             static_cast<size_t>(w) * 3;
    ok &= std::fclose(f) == 0;
    return ok ? TV_OK : img_error(std::string("write failed: ") + path);
}

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

int tv_image_pfm_pixels(const double* sum, const double* sum_sq, const uint32_t* counts, int32_t width, int32_t height,
                        int32_t variance, int32_t on_device, int device, float* out_rgb) {
    if (!sum || !counts || !out_rgb || (variance && !sum_sq)) return set_error(TV_ERR_ARG, "null argument");
    if (width < 1 || height < 1) return set_error(TV_ERR_ARG, "bad image size");
    int rc = use_device(device);
    if (rc) return rc;
    const uint64_t n = static_cast<uint64_t>(width) * height;
    DevBuf ds, dq, dc, dout;
    const double *s = sum, *q = sum_sq;
    const uint32_t* c = counts;
    if (!on_device) {
        IM_CK(cudaMalloc(&ds.p, 3 * n * sizeof(double)), "alloc");
        IM_CK(cudaMemcpy(ds.p, sum, 3 * n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        if (variance) {
            IM_CK(cudaMalloc(&dq.p, 3 * n * sizeof(double)), "alloc");
            IM_CK(cudaMemcpy(dq.p, sum_sq, 3 * n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        }
        IM_CK(cudaMalloc(&dc.p, n * sizeof(uint32_t)), "alloc");
        IM_CK(cudaMemcpy(dc.p, counts, n * sizeof(uint32_t), cudaMemcpyHostToDevice), "H2D");
        s = static_cast<const double*>(ds.p), q = static_cast<const double*>(dq.p);
        c = static_cast<const uint32_t*>(dc.p);
    }
    IM_CK(cudaMalloc(&dout.p, 3 * n * sizeof(float)), "alloc");
    pfm_pixels_kernel<<<148 * 4, 256>>>(s, q, c, n, variance, static_cast<float*>(dout.p));
    IM_CK(cudaGetLastError(), "pfm_pixels_kernel");
    IM_CK(cudaMemcpy(out_rgb, dout.p, 3 * n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
    return TV_OK;
}

// write_pfm / write_variance_pfm (image.cpp:49-77) of an accumulator
int tv_image_write_pfm(const char* path, const tv_framebuffer* fb, int32_t width, int32_t height, int32_t variance,
                       int32_t on_device, int device) {
    if (!path || !fb) return set_error(TV_ERR_ARG, "null argument");
    std::vector<float> rgb(static_cast<size_t>(std::max(width, 0)) * std::max(height, 0) * 3);
    int rc = tv_image_pfm_pixels(fb->sum, fb->sum_sq, fb->sample_counts, width, height, variance, on_device, device,
                                 rgb.data());
    return rc ? rc : write_pfm_rows(path, width, height, rgb);
}

// write_pfm(path, FloatImage) (image.cpp:79-81)
int tv_pfm_write(const char* path, const float* rgb, int32_t width, int32_t height) {
    if (!path || !rgb || width < 1 || height < 1) return set_error(TV_ERR_ARG, "bad argument");
    std::vector<float> v(rgb, rgb + static_cast<size_t>(width) * height * 3);
    return write_pfm_rows(path, width, height, v);
}

// read_pfm (image.cpp:83-101). Call with rgb = NULL to get the size first.
int tv_pfm_read(const char* path, int32_t* width, int32_t* height, float* rgb) {
    if (!path || !width || !height) return set_error(TV_ERR_ARG, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) return img_error(std::string("cannot open: ") + path);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    // operator>> semantics: skip whitespace, read a token / number
    auto skip_ws = [&]() {
        int ch;
        while ((ch = std::fgetc(f)) != EOF && std::isspace(ch)) {
        }
        if (ch != EOF) std::ungetc(ch, f);
    };
    skip_ws();
    std::string magic;
    for (int ch; (ch = std::fgetc(f)) != EOF && !std::isspace(ch);) magic.push_back(static_cast<char>(ch));
    if (magic != "PF") return img_error(std::string("not a color PFM file: ") + path);
    int w = 0, h = 0;
    double scale = 0.0;
    if (std::fscanf(f, "%d %d %lf", &w, &h, &scale) != 3 || w < 1 || h < 1)
        return img_error(std::string("bad PFM header: ") + path);
    if (scale >= 0.0) return img_error(std::string("big-endian PFM is not supported: ") + path);
    std::fgetc(f);  // single whitespace after the scale line
    *width = w, *height = h;
    if (!rgb) return TV_OK;
    for (int y = h - 1; y >= 0; --y)
        if (std::fread(rgb + static_cast<size_t>(y) * w * 3, sizeof(float), static_cast<size_t>(w) * 3, f) !=
            static_cast<size_t>(w) * 3)
            return img_error(std::string("unexpected end of PFM data: ") + path);
    return TV_OK;
}

// cmd_compare's image metrics (cli.cpp:499-531); va / vb may both be NULL
int tv_image_compare(const float* a, const float* b, const float* va, const float* vb, uint64_t n_pixels, int device,
                     tv_compare_stats* out) {
    if (!a || !b || !out || (!va != !vb)) return set_error(TV_ERR_ARG, "null argument");
    int rc = use_device(device);
    if (rc) return rc;
    const uint64_t nv = 3 * n_pixels;
    DevBuf da, db, dva, dvb, acc;
    IM_CK(cudaMalloc(&da.p, nv * sizeof(float) + 1), "alloc");
    IM_CK(cudaMalloc(&db.p, nv * sizeof(float) + 1), "alloc");
    IM_CK(cudaMemcpy(da.p, a, nv * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    IM_CK(cudaMemcpy(db.p, b, nv * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    if (va) {
        IM_CK(cudaMalloc(&dva.p, nv * sizeof(float) + 1), "alloc");
        IM_CK(cudaMalloc(&dvb.p, nv * sizeof(float) + 1), "alloc");
        IM_CK(cudaMemcpy(dva.p, va, nv * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        IM_CK(cudaMemcpy(dvb.p, vb, nv * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    }
    IM_CK(cudaMalloc(&acc.p, 3 * sizeof(unsigned long long)), "alloc");
    IM_CK(cudaMemset(acc.p, 0, 3 * sizeof(unsigned long long)), "memset");
    auto* ap = static_cast<unsigned long long*>(acc.p);
    compare_kernel<<<148 * 4, 256>>>(static_cast<const float*>(da.p), static_cast<const float*>(db.p),
                                     static_cast<const float*>(dva.p), static_cast<const float*>(dvb.p), n_pixels,
                                     reinterpret_cast<double*>(ap), ap + 1, ap + 2);
    IM_CK(cudaGetLastError(), "compare_kernel");
    unsigned long long h[3];
    IM_CK(cudaMemcpy(h, ap, sizeof(h), cudaMemcpyDeviceToHost), "D2H");
    double sq;
    std::memcpy(&sq, &h[0], 8);
    std::memcpy(&out->max_abs_diff, &h[1], 8);
    out->rmse = nv ? std::sqrt(sq / static_cast<double>(nv)) : 0.0;
    out->outliers = h[2];
    out->outlier_fraction = va && n_pixels ? static_cast<double>(h[2]) / static_cast<double>(n_pixels) : -1.0;
    return TV_OK;
}

}  // extern "C"
