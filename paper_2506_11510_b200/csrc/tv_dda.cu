// Regular-grid comparator (config C5): RegularGrid::from_volume +
// render_reference on the GPU. The DDA marcher (regular_grid.cpp:16-118)
// drives the same integrator as the tet renderer (path_integrator.hpp:42-84),
// so both renderers consume random dimensions in lockstep. One thread traces
// one path; radiance per path goes to HBM and the shared accum_kernel adds
// samples per pixel in order, as for the tet grid.
#include <algorithm>
#include <vector>

#include "tv_trace.cuh"

namespace tvb {
namespace {

struct DdaGrid {
    const float* dens;  // extinction, already scaled (regular_grid.cpp:122-134)
    int n[3];
};

// DdaMarcher state (regular_grid.cpp:124-118): reference semantics.
struct Dda {
    d3 o, d;
    double tmax;
    int idx[3], step[3];
    double t_next[3], t_delta[3], t_cur, t_end, last_t0;
    uint64_t last_cell;
    bool escaped;

    __device__ bool start(const DdaGrid& G, d3 origin, d3 dir, double tmin_in, double tmax_in) {  // :21-51
        escaped = false;
        o = origin;
        d = dir;
        tmax = tmax_in;
        double t0, t1;
        if (!slab(o, d, dmax(0.0, tmin_in), tmax, t0, t1)) return false;
        t_end = t1;
        const d3 p = ray_at(o, d, t0 + 1e-9);
        const double pp[3] = {p.x, p.y, p.z}, oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            idx[a] = min(max(static_cast<int>(floor(pp[a] * G.n[a])), 0), G.n[a] - 1);
            if (dd[a] > 0.0) {
                step[a] = 1;
                t_next[a] = ((idx[a] + 1.0) / G.n[a] - oo[a]) / dd[a];
                t_delta[a] = 1.0 / (G.n[a] * dd[a]);
            } else if (dd[a] < 0.0) {
                step[a] = -1;
                t_next[a] = (static_cast<double>(idx[a]) / G.n[a] - oo[a]) / dd[a];
                t_delta[a] = -1.0 / (G.n[a] * dd[a]);
            } else {
                step[a] = 0;
                t_next[a] = __longlong_as_double(0x7ff0000000000000ll);
                t_delta[a] = __longlong_as_double(0x7ff0000000000000ll);
            }
        }
        t_cur = t0;
        return true;
    }

    // :53-86; returns false when the walker has escaped
    __device__ bool next(const DdaGrid& G, double& t0, double& t1, double& lambda) {
        if (escaped) return false;
        const int axis = t_next[0] <= t_next[1] ? (t_next[0] <= t_next[2] ? 0 : 2) : (t_next[1] <= t_next[2] ? 1 : 2);
        double t_exit = t_next[axis];
        t0 = t_cur;
        const uint64_t flat = (static_cast<uint64_t>(idx[2]) * G.n[1] + idx[1]) * G.n[0] + idx[0];
        lambda = static_cast<double>(G.dens[flat]);
        last_cell = flat;
        last_t0 = t_cur;
        if (t_exit >= tmax) {
            t1 = tmax;
            escaped = true;
            return true;
        }
        idx[axis] += step[axis];
        t_next[axis] += t_delta[axis];
        if (idx[axis] < 0 || idx[axis] >= G.n[axis] || t_exit >= t_end - 1e-15) {
            t_exit = t_end;
            escaped = true;
        }
        t1 = t_exit;
        t_cur = t_exit;
        return true;
    }
};

__global__ void dda_kernel(DdaGrid G, CamView C, RenderParams P, Batch B, double* rad, uint64_t* stats) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    uint64_t my_cells = 0;
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < B.n_paths; p += gridDim.x * blockDim.x) {
        // path id -> pixel and sample (tv_trace.cu path_pixel, order 0)
        const uint32_t per_unit = B.ns * 32u;
        const uint32_t unit = p / per_unit, r = p - unit * per_unit;
        uint32_t lane, s;
        if (B.order) {
            lane = r / B.ns;
            s = B.s0 + (r - lane * B.ns);
        } else {
            s = B.s0 + r / 32u;
            lane = r & 31u;
        }
        const uint32_t k = unit >> 3, sub = unit & 7u;
        const uint32_t t = static_cast<uint32_t>(B.rank) + k * static_cast<uint32_t>(B.n_ranks);
        const int px = static_cast<int>((t % B.tiles_x) * 16 + (sub & 1u) * 8 + (lane & 7u));
        const int py = static_cast<int>((t / B.tiles_x) * 16 + (sub >> 1) * 4 + (lane >> 3));
        if (px >= C.w || py >= C.h) continue;
        Rng rng;
        rng.init(P.seed, static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + px, s);
        const double jx = rng.next();
        const double jy = rng.next();
        d3 dir = primary_dir(C, px, py, jx, jy);
        const d3 env = mk(P.env[0], P.env[1], P.env[2]);
        d3 L = mk(0, 0, 0), T = mk(1, 1, 1);
        Dda m;
        d3 result;
        if (!m.start(G, mk(C.pos[0], C.pos[1], C.pos[2]), dir, 0.0, inf)) {
            result = env;
        } else {
            for (int bounce = 0;;) {  // path_integrator.hpp:48-83
                const double target = -log(1.0 - rng.next());
                double tau = 0.0;
                bool collided = false;
                double t0, t1, lambda;
                while (m.next(G, t0, t1, lambda)) {
                    ++my_cells;
                    const double seg = lambda * (t1 - t0);
                    if (lambda > 0.0 && tau + seg >= target) {
                        m.o = ray_at(m.o, m.d, m.last_t0 + (target - tau) / lambda);  // shorten: event point
                        m.escaped = false;
                        collided = true;
                        break;
                    }
                    tau += seg;
                }
                if (!collided) {
                    result = add(L, mulv(T, env));
                    break;
                }
                T = mul(T, P.default_albedo);  // cell_media: density only (mask 1)
                ++bounce;
                if (bounce >= P.max_bounces) {
                    result = L;
                    break;
                }
                bool killed = false;
                if (bounce >= 4) {
                    const double pmax = dmax(T.x, dmax(T.y, T.z));
                    if (pmax < 1e-3) {
                        if (rng.next() >= pmax) killed = true;
                        else T = divs(T, pmax);
                    }
                }
                if (killed) {
                    result = L;
                    break;
                }
                dir = sample_phase_hg(m.d, P.g, rng);
                if (!m.start(G, m.o, dir, 0.0, inf)) m.escaped = true;  // redirect (:91-96)
            }
        }
        rad[3ull * p] = result.x, rad[3ull * p + 1] = result.y, rad[3ull * p + 2] = result.z;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) my_cells += __shfl_down_sync(0xffffffffu, my_cells, off);
    if ((threadIdx.x & 31) == 0 && stats)
        atomicAdd(reinterpret_cast<unsigned long long*>(stats), static_cast<unsigned long long>(my_cells));
}

__global__ void scale_kernel(const float* in, float* out, uint64_t n, double scale) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i] * scale);  // regular_grid.cpp:129
}

}  // namespace

int validate_render_cfg(const tv_render_config* r);  // tv_capi.cu

}  // namespace tvb

using namespace tvb;

static int render_regular(const float* density, bool on_device, int32_t nx, int32_t ny, int32_t nz,
                          double density_scale, const tv_camera* camera, const tv_render_config* cfg, int device,
                          tv_framebuffer* out, tv_render_stats* stats) {
    if (!density) return set_error(TV_ERR_ARG, "density is null");
    if (nx < 1 || ny < 1 || nz < 1) return set_error(TV_ERR, "volume dimensions must be positive");
    if (density_scale < 0.0) return set_error(TV_ERR, "density scale must be non-negative");  // regular_grid.cpp:123
    int rc = validate_render_cfg(cfg);
    if (rc) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) return set_error(TV_ERR_CUDA, "no CUDA device available");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    RenderParams rp;
    rp.spp = cfg->spp;
    rp.max_bounces = cfg->max_bounces;
    rp.seed = cfg->seed;
    rp.g = cfg->hg_g;
    rp.default_albedo = cfg->default_albedo;
    rp.env[0] = cfg->environment[0], rp.env[1] = cfg->environment[1], rp.env[2] = cfg->environment[2];
    rp.emission_scale = cfg->emission_scale;

    const uint64_t nvox = static_cast<uint64_t>(nx) * ny * nz;
    const uint32_t tiles_x = (static_cast<uint32_t>(cv.w) + 15) / 16, tiles_y = (static_cast<uint32_t>(cv.h) + 15) / 16;
    const uint64_t units = static_cast<uint64_t>(tiles_x) * tiles_y * 8;
    uint64_t ns = std::max<uint64_t>(1, kMaxBatchPaths / (units * 32));
    ns = std::min<uint64_t>(ns, static_cast<uint64_t>(rp.spp));
    const uint64_t npx = static_cast<uint64_t>(cv.w) * cv.h;
    float *raw = nullptr, *dens = nullptr;
    double *rad = nullptr, *sum = nullptr, *sum_sq = nullptr;
    uint32_t* counts = nullptr;
    uint64_t* st = nullptr;
    auto cleanup = [&]() {
        cudaFree(raw), cudaFree(dens), cudaFree(rad), cudaFree(sum), cudaFree(sum_sq), cudaFree(counts), cudaFree(st);
    };
    e = on_device ? cudaSuccess : cudaMalloc(&raw, nvox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&dens, nvox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&rad, units * 32 * ns * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&sum, npx * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&sum_sq, npx * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&counts, npx * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&st, 3 * sizeof(uint64_t));
    if (e == cudaSuccess && !on_device) e = cudaMemcpy(raw, density, nvox * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(st, 0, 3 * sizeof(uint64_t));
    if (e != cudaSuccess) {
        cleanup();
        return cuda_status(e, "render_regular setup");
    }
    scale_kernel<<<148 * 8, 256>>>(on_device ? density : raw, dens, nvox, density_scale);
    DdaGrid G{dens, {nx, ny, nz}};
    RenderOut ro{sum, sum_sq, counts, st};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (uint64_t s0 = 0; s0 < static_cast<uint64_t>(rp.spp); s0 += ns) {
        Batch B{};
        B.n_units = static_cast<uint32_t>(units);
        B.s0 = static_cast<uint32_t>(s0);
        B.ns = static_cast<uint32_t>(std::min<uint64_t>(ns, rp.spp - s0));
        B.tiles_x = tiles_x;
        B.tiles_y = tiles_y;
        B.rank = 0;
        B.n_ranks = 1;
        B.n_paths = static_cast<uint32_t>(units * 32 * B.ns);
        B.first = s0 == 0 ? 1u : 0u;
        B.order = 0;
        dda_kernel<<<static_cast<unsigned>(std::min<uint64_t>((B.n_paths + 127) / 128, 148 * 64)), 128>>>(
            G, cv, rp, B, rad, st);
        accum_kernel<<<static_cast<unsigned>(std::min<uint64_t>((units * 32 + 127) / 128, 148 * 16)), 128>>>(
            B, cv, nullptr, rad, ro);
    }
    cudaEventRecord(e1);
    e = cudaGetLastError();
    uint64_t hst[3] = {0, 0, 0};
    if (e == cudaSuccess && out && out->sum) e = cudaMemcpy(out->sum, sum, npx * 3 * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && out && out->sum_sq)
        e = cudaMemcpy(out->sum_sq, sum_sq, npx * 3 * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && out && out->sample_counts)
        e = cudaMemcpy(out->sample_counts, counts, npx * sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(hst, st, sizeof(hst), cudaMemcpyDeviceToHost);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cleanup();
    if (e != cudaSuccess) return cuda_status(e, "render_regular");
    if (stats) {
        stats->cells_visited = hst[0];
        stats->paths_traced = npx * static_cast<uint64_t>(rp.spp);
        stats->degenerate_paths = 0;
        stats->seconds = ms * 1e-3;
    }
    return TV_OK;
}

extern "C" int tv_render_regular(const float* density, int32_t nx, int32_t ny, int32_t nz, double density_scale,
                                 const tv_camera* camera, const tv_render_config* cfg, int device, tv_framebuffer* out,
                                 tv_render_stats* stats) {
    return render_regular(density, false, nx, ny, nz, density_scale, camera, cfg, device, out, stats);
}

extern "C" int tv_render_regular_dev(const float* density_dev, int32_t nx, int32_t ny, int32_t nz,
                                     double density_scale, const tv_camera* camera, const tv_render_config* cfg,
                                     int device, tv_framebuffer* out, tv_render_stats* stats) {
    return render_regular(density_dev, true, nx, ny, nz, density_scale, camera, cfg, device, out, stats);
}
