// Free-flight estimators over the per-tet majorant (BASELINE north star (2),
// SURVEY.md F1 and 7): delta tracking for the render, delta and ratio tracking
// for transmittance. These are OPTIONAL modes next to the product path.
//
// The reference integrates with regular tracking (path_integrator.hpp:49-61):
// one draw per flight, tau* = -ln(1 - xi), and the exact optical depth
// lambda * dt of every crossed tet, because lambda is constant per tet. That is
// what tv_render does, bit for bit. Delta tracking samples tentative
// collisions with the per-tet majorant mu = scale * lambda (scale >= 1) and
// accepts each as real with probability lambda / mu; scale = 1 makes every
// tentative collision real (regular tracking with a fresh draw per tet).
// Ratio tracking estimates transmittance as the product of (1 - lambda / mu)
// over the tentative collisions (it has no render consumer: the reference has
// no next-event estimation). All of them draw from the path's
// RngStream (rng.hpp:19-26) in their own order, so they agree with the
// reference in distribution, not bit for bit: tests/test_gpu_tracking.py checks
// them against the regular-tracking render and the exact optical depth within
// Monte Carlo error.
//
// The traversal is the reference marcher (TetMarcher, tracer.cpp:25-127 with
// exit_face, :143-162) over the LeafRec layout, one thread per path: these
// modes are for estimator studies, not for the frame-rate path.
#include <algorithm>
#include <cmath>

#include "tv_trace.cuh"

namespace tvb {

int validate_render_cfg(const tv_render_config* r);  // tv_capi.cu

namespace {

// TetMarcher over one flight (origin o, direction dir, [seg_start, tmax)),
// calling seg(lambda, s0, s1, cell) for every crossed tet in order until it
// returns true (an event in that tet). Returns 0 when the flight escaped, 1 on
// an event, 2 when the marcher aborted (degenerate corner or the step cap).
template <class Seg>
__device__ int march_flight(const GridView& G, d3 o, d3 dir, double seg_start, double probe, double tmax,
                            uint32_t& cell, LeafRec& rec, uint32_t& steps, uint64_t& visited, Seg&& seg) {
    for (;;) {
        if (++steps > kMaxSteps) return 2;
        double t;
        int slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
        if (slot < 0) {  // one nudged retry (tracer.cpp:54-61)
            probe += kNudge;
            slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
            if (slot < 0) return 2;
        }
        const double t_exit = dmax(probe + t, seg_start);
        const double lambda = static_cast<double>(__uint_as_float(rec.w[13]));
        bool escaped;
        double s1 = t_exit;
        uint32_t next = kNoLeaf;
        if (t_exit >= tmax) {
            s1 = tmax;
            escaped = true;
        } else {
            next = nbr_leaf(sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot));
            escaped = next == kNoLeaf;
        }
        ++visited;
        if (seg(lambda, seg_start, s1)) return 1;
        if (escaped) return 0;
        rec = load_leaf(G.leaves, next);
        cell = next;
        seg_start = t_exit;
        probe = t_exit + kNudge;
    }
}

// delta tracking inside one tet: tentative collisions at rate mu = scale *
// lambda from s0; true with the event distance when one is accepted as real
__device__ __forceinline__ bool delta_segment(double lambda, double scale, double s0, double s1, Rng& rng,
                                              double& t_event) {
    if (!(lambda > 0.0)) return false;
    const double mu = scale * lambda;
    double t = s0;
    for (;;) {
        t += -log(1.0 - rng.next()) / mu;
        if (t >= s1) return false;
        if (scale == 1.0 || rng.next() * mu < lambda) {
            t_event = t;
            return true;
        }
    }
}

// trace_path (path_integrator.hpp:42-84) with delta-tracking flights; the
// event, albedo, emission, bounce cap, roulette and HG redirect are the
// reference's. The first flight honours [t_min, t_max], redirects reset it.
__device__ d3 trace_delta(const GridView& G, const RenderParams& P, double scale, d3 o, d3 dir, double t_min,
                          double tmax, Rng& rng, uint64_t& visited, bool& degenerate) {
    const d3 env = mk(P.env[0], P.env[1], P.env[2]);
    double t0, t1;
    uint32_t cell = kNone;
    if (slab(o, dir, dmax(0.0, t_min), tmax, t0, t1)) {
        d3 q = ray_at(o, dir, t0 + kNudge);
        q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
        cell = locate(G, q);
    }
    if (cell == kNone) return env;  // !m.start(primary)
    d3 radiance = mk(0, 0, 0), throughput = mk(1, 1, 1);
    LeafRec rec = load_leaf(G.leaves, cell);
    uint32_t steps = 0;
    double seg_start = t0, probe = t0 + kNudge;
    for (int bounce = 0;;) {
        double t_event = 0.0;
        const int r = march_flight(G, o, dir, seg_start, probe, tmax, cell, rec, steps, visited,
                                   [&](double lambda, double s0, double s1) {
                                       return delta_segment(lambda, scale, s0, s1, rng, t_event);
                                   });
        if (r == 2) {
            degenerate = true;
            return radiance;
        }
        if (r == 0) return add(radiance, mulv(throughput, env));
        const uint32_t mask = rec.w[12] >> 24;
        if (mask & 2u) {
            const d3 e = emission_color(static_cast<double>(__uint_as_float(rec.w[14])));
            radiance = add(radiance, mul(mulv(throughput, e), P.emission_scale));
        }
        throughput = mul(throughput, (mask & 4u) ? static_cast<double>(__uint_as_float(rec.w[15])) : P.default_albedo);
        ++bounce;
        if (bounce >= P.max_bounces) return radiance;
        if (bounce >= 4) {
            const double pm = dmax(throughput.x, dmax(throughput.y, throughput.z));
            if (pm < 1e-3) {
                if (rng.next() >= pm) return radiance;
                throughput = divs(throughput, pm);
            }
        }
        o = ray_at(o, dir, t_event);  // the event point; the redirect keeps the cell
        dir = sample_phase_hg(dir, P.g, rng);
        tmax = __longlong_as_double(0x7ff0000000000000ll);
        seg_start = 0.0;
        probe = 0.0;
    }
}

// render_image (path_integrator.hpp:87-136) with delta tracking: one thread
// per pixel, samples s = 0..spp-1 in order (ImageAccumulator::add_sample).
__global__ void render_delta_kernel(GridView G, CamView C, RenderParams P, double scale, double* sum, double* sum_sq,
                                    uint32_t* counts, unsigned long long* counters) {
    const uint64_t npx = static_cast<uint64_t>(C.w) * C.h;
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= npx) return;
    const int px = static_cast<int>(i % C.w), py = static_cast<int>(i / C.w);
    const d3 o = mk(C.pos[0], C.pos[1], C.pos[2]);
    d3 s = mk(0, 0, 0), q = mk(0, 0, 0);
    uint64_t visited = 0, deg = 0;
    for (int k = 0; k < P.spp; ++k) {
        Rng rng;
        rng.init(P.seed, i, static_cast<uint64_t>(k));
        const double jx = rng.next();
        const double jy = rng.next();
        bool d = false;
        const d3 L = trace_delta(G, P, scale, o, primary_dir(C, px, py, jx, jy), 0.0,
                                 __longlong_as_double(0x7ff0000000000000ll), rng, visited, d);
        deg += d;
        s = add(s, L);
        q = add(q, mulv(L, L));
    }
    if (sum) sum[3 * i] = s.x, sum[3 * i + 1] = s.y, sum[3 * i + 2] = s.z;
    if (sum_sq) sum_sq[3 * i] = q.x, sum_sq[3 * i + 1] = q.y, sum_sq[3 * i + 2] = q.z;
    if (counts) counts[i] = static_cast<uint32_t>(P.spp);
    atomicAdd(counters, static_cast<unsigned long long>(visited));
    if (deg) atomicAdd(counters + 1, static_cast<unsigned long long>(deg));
}

// transmittance of ray i over [t_min, t_max] (march_transmittance's range,
// tracer.cpp:176-190) by delta tracking (0 or 1) or ratio tracking (the
// product of 1 - lambda / mu over tentative collisions)
__global__ void transmittance_kernel(GridView G, const tv_ray* __restrict__ rays, uint64_t n, int mode, double scale,
                                     uint64_t seed, const uint64_t* __restrict__ pixels,
                                     const uint64_t* __restrict__ samples, double* __restrict__ out,
                                     unsigned long long* counters) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const tv_ray R = rays[i];
    const d3 o = mk(R.origin[0], R.origin[1], R.origin[2]);
    const d3 dir = mk(R.dir[0], R.dir[1], R.dir[2]);
    Rng rng;
    rng.init(seed, pixels[i], samples[i]);
    double T = 1.0;
    uint64_t visited = 0;
    bool aborted = false;
    double t0, t1;
    uint32_t cell = kNone;
    if (slab(o, dir, dmax(0.0, R.t_min), R.t_max, t0, t1)) {
        d3 q = ray_at(o, dir, t0 + kNudge);
        q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
        cell = locate(G, q);
    }
    if (cell != kNone) {
        LeafRec rec = load_leaf(G.leaves, cell);
        uint32_t steps = 0;
        const int r = march_flight(G, o, dir, t0, t0 + kNudge, R.t_max, cell, rec, steps, visited,
                                   [&](double lambda, double s0, double s1) {
                                       if (!(lambda > 0.0)) return false;
                                       if (mode == TV_TRACK_DELTA) {
                                           double te;
                                           if (delta_segment(lambda, scale, s0, s1, rng, te)) {
                                               T = 0.0;
                                               return true;  // a real collision: the ray is blocked
                                           }
                                           return false;
                                       }
                                       const double mu = scale * lambda;
                                       for (double t = s0;;) {
                                           t += -log(1.0 - rng.next()) / mu;
                                           if (t >= s1) return false;
                                           T *= 1.0 - lambda / mu;
                                           if (T == 0.0) return true;  // scale 1: the estimate is 0 from here on
                                       }
                                   });
        aborted = r == 2;
    }
    out[i] = T;
    atomicAdd(counters, static_cast<unsigned long long>(visited));
    if (aborted) atomicAdd(counters + 1, 1ull);
}

int check_tracking(int32_t tracking, double scale, bool render) {
    if (tracking != TV_TRACK_REGULAR && tracking != TV_TRACK_DELTA && tracking != TV_TRACK_RATIO)
        return set_error(TV_ERR_CONFIG, "unknown tracking mode");
    if (render && tracking == TV_TRACK_RATIO)
        return set_error(TV_ERR_CONFIG, "ratio tracking has no render estimator (no next-event estimation)");
    if (!(scale >= 1.0) || !std::isfinite(scale)) return set_error(TV_ERR_CONFIG, "majorant scale must be >= 1");
    return TV_OK;
}

struct Dev {
    void* p = nullptr;
    ~Dev() {
        if (p) cudaFree(p);
    }
};

}  // namespace
}  // namespace tvb

using namespace tvb;

#define TV_CK(x, what)                                       \
    do {                                                     \
        if (int rc_ = cuda_status((x), what)) return rc_;    \
    } while (0)

extern "C" int tv_render_tracking(const tv_grid* h, const tv_camera* camera, const tv_render_config* cfg,
                                  int32_t tracking, double majorant_scale, tv_framebuffer* out,
                                  tv_render_stats* stats) {
    if (!h) return set_error(TV_ERR_ARG, "null argument");
    int rc = check_tracking(tracking, majorant_scale, true);
    if (rc) return rc;
    if (tracking == TV_TRACK_REGULAR) return tv_render(h, camera, cfg, out, stats);
    if ((rc = validate_render_cfg(cfg))) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    RenderParams rp;
    rp.spp = cfg->spp;
    rp.max_bounces = cfg->max_bounces;
    rp.seed = cfg->seed;
    rp.g = cfg->hg_g;
    rp.default_albedo = cfg->default_albedo;
    rp.env[0] = cfg->environment[0], rp.env[1] = cfg->environment[1], rp.env[2] = cfg->environment[2];
    rp.emission_scale = cfg->emission_scale;
    const uint64_t npx = static_cast<uint64_t>(cv.w) * cv.h;
    Dev d_fb, d_ctr;
    TV_CK(cudaMalloc(&d_fb.p, npx * (6 * sizeof(double) + sizeof(uint32_t))), "alloc");
    TV_CK(cudaMalloc(&d_ctr.p, 16), "alloc");
    TV_CK(cudaMemset(d_ctr.p, 0, 16), "memset");
    double* sum = static_cast<double*>(d_fb.p);
    double* sum_sq = sum + 3 * npx;
    uint32_t* counts = reinterpret_cast<uint32_t*>(sum_sq + 3 * npx);
    cudaEvent_t e0, e1;
    TV_CK(cudaEventCreate(&e0), "event");
    TV_CK(cudaEventCreate(&e1), "event");
    cudaEventRecord(e0);
    render_delta_kernel<<<static_cast<unsigned>((npx + 127) / 128), 128>>>(
        g.view, cv, rp, majorant_scale, sum, sum_sq, counts, static_cast<unsigned long long*>(d_ctr.p));
    cudaEventRecord(e1);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    TV_CK(e, "render_delta_kernel");
    if (out && out->sum) TV_CK(cudaMemcpy(out->sum, sum, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (out && out->sum_sq)
        TV_CK(cudaMemcpy(out->sum_sq, sum_sq, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (out && out->sample_counts)
        TV_CK(cudaMemcpy(out->sample_counts, counts, npx * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H");
    unsigned long long c[2];
    TV_CK(cudaMemcpy(c, d_ctr.p, sizeof(c), cudaMemcpyDeviceToHost), "D2H");
    if (stats) {
        stats->cells_visited = c[0];
        stats->paths_traced = npx * static_cast<uint64_t>(cfg->spp);
        stats->degenerate_paths = c[1];
        stats->seconds = ms * 1e-3;
    }
    return TV_OK;
}

extern "C" int tv_transmittance_tracking(const tv_grid* h, const tv_ray* rays, uint64_t n, int32_t tracking,
                                         double majorant_scale, uint64_t seed, const uint64_t* pixels,
                                         const uint64_t* samples, double* trans_out, uint64_t stats[2]) {
    if (!h || (n && (!rays || !trans_out))) return set_error(TV_ERR_ARG, "null argument");
    int rc = check_tracking(tracking, majorant_scale, false);
    if (rc) return rc;
    if (tracking == TV_TRACK_REGULAR) return tv_march_transmittance(h, rays, n, nullptr, trans_out, stats);
    if (n && (!pixels || !samples)) return set_error(TV_ERR_ARG, "null argument");
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    const uint64_t m = n ? n : 1;
    Dev d_rays, d_pix, d_smp, d_out, d_ctr;
    TV_CK(cudaMalloc(&d_rays.p, m * sizeof(tv_ray)), "alloc");
    TV_CK(cudaMalloc(&d_pix.p, m * 8), "alloc");
    TV_CK(cudaMalloc(&d_smp.p, m * 8), "alloc");
    TV_CK(cudaMalloc(&d_out.p, m * 8), "alloc");
    TV_CK(cudaMalloc(&d_ctr.p, 16), "alloc");
    TV_CK(cudaMemset(d_ctr.p, 0, 16), "memset");
    if (n) {
        TV_CK(cudaMemcpy(d_rays.p, rays, n * sizeof(tv_ray), cudaMemcpyHostToDevice), "H2D");
        TV_CK(cudaMemcpy(d_pix.p, pixels, n * 8, cudaMemcpyHostToDevice), "H2D");
        TV_CK(cudaMemcpy(d_smp.p, samples, n * 8, cudaMemcpyHostToDevice), "H2D");
        transmittance_kernel<<<static_cast<unsigned>((n + 127) / 128), 128>>>(
            g.view, static_cast<const tv_ray*>(d_rays.p), n, tracking, majorant_scale, seed,
            static_cast<const uint64_t*>(d_pix.p), static_cast<const uint64_t*>(d_smp.p),
            static_cast<double*>(d_out.p), static_cast<unsigned long long*>(d_ctr.p));
        TV_CK(cudaGetLastError(), "transmittance_kernel");
        TV_CK(cudaMemcpy(trans_out, d_out.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
    }
    unsigned long long c[2];
    TV_CK(cudaMemcpy(c, d_ctr.p, sizeof(c), cudaMemcpyDeviceToHost), "D2H");
    if (stats) stats[0] = c[0], stats[1] = c[1];
    return TV_OK;
}
