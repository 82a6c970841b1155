// Traversal kernels: the volumetric path tracer (start / trace / accumulate),
// the deterministic segment marcher (march_segments parity entry) and batched
// locate_point.
//
// Reference semantics (paths relative to /root/reference/proj):
//   render_image  include/tetvol/path_integrator.hpp:87-136
//   trace_path    include/tetvol/path_integrator.hpp:42-84
//   TetMarcher    src/tracer.cpp:25-127, exit_face src/tracer.cpp:143-162
//
// Render pipeline per batch (this rank's pixels x a range of samples):
//   start_kernel  camera ray, slab and locate for every path — coherent work,
//                 kept out of the divergent trace loop;
//   trace_kernel  persistent warps; each lane traces one path at a time, one
//                 tet step per loop iteration. Path starts and scatter events
//                 (HG sampling, new flight tables) are deferred and run
//                 warp-batched, so the rare expensive branches are paid once
//                 for many lanes; finished lanes take new paths from the warp's
//                 claimed chunk (path regeneration with warp-level compaction).
//                 Every path's radiance goes to HBM;
//   accum_kernel  one thread per pixel adds its samples in order s = 0..spp-1,
//                 exactly the reference accumulation order
//                 (path_integrator.hpp:109-114, image.hpp:36-45), so the
//                 framebuffer is bit-comparable with the CPU reference.
#include <type_traits>

#include "tv_trace.cuh"

namespace tvb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Path id of (unit, pixel lane, sample k of the batch). order 0: the 32
// pixels of a unit for one sample are consecutive; order 1: the samples of one
// pixel are consecutive, so a warp traces many samples of few pixels.
__device__ __forceinline__ uint32_t path_id(const Batch& B, uint32_t unit, uint32_t lane, uint32_t k) {
    return unit * B.ns * 32u + (B.order ? lane * B.ns + k : k * 32u + lane);
}

__device__ __forceinline__ void path_pixel(const Batch& B, uint32_t p, int& px, int& py, uint32_t& s) {
    const uint32_t per_unit = B.ns * 32u;
    const uint32_t unit = p / per_unit, r = p - unit * per_unit;
    uint32_t lane;
    if (B.order) {
        lane = r / B.ns;
        s = B.s0 + (r - lane * B.ns);
    } else {
        s = B.s0 + r / 32u;
        lane = r & 31u;
    }
    const uint32_t k = unit >> 3, sub = unit & 7u;
    const uint32_t t = B.tile_order ? B.tile_order[k] : static_cast<uint32_t>(B.rank) + k * static_cast<uint32_t>(B.n_ranks);
    const uint32_t tx = t % B.tiles_x, ty = t / B.tiles_x;
    px = static_cast<int>(tx * 16 + (sub & 1u) * 8 + (lane & 7u));
    py = static_cast<int>(ty * 16 + (sub >> 1) * 4 + (lane >> 3));
}

enum : int { S_IDLE = 0, S_STEP = 1, S_SCATTER = 2 };

}  // namespace

// TetMarcher::start for every path of the batch (tracer.cpp:29-45), after the
// camera sample (path_integrator.hpp:110-113).
__global__ void start_kernel(GridView G, CamView C, RenderParams P, Batch B, StartRec* st, uint32_t* cells) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const d3 o = mk(C.pos[0], C.pos[1], C.pos[2]);
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < B.n_paths; p += gridDim.x * blockDim.x) {
        int px, py;
        uint32_t s;
        path_pixel(B, p, px, py, s);
        if (px >= C.w || py >= C.h) {
            cells[p] = kInvalidPixel;
            continue;
        }
        Rng rng;
        rng.init(P.seed, static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + px, s);
        const double jx = rng.next();
        const double jy = rng.next();
        const d3 dir = primary_dir(C, px, py, jx, jy);
        double t0, t1;
        uint32_t cell = kNone;
        if (slab(o, dir, 0.0, inf, t0, t1)) {
            d3 q = ray_at(o, dir, t0 + kNudge);
            q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
            cell = locate(G, q);
        } else {
            t0 = 0.0;
        }
        // the first target is drawn here, in the fully populated start kernel,
        // instead of in the trace kernel's divergent regeneration branch
        const double target = -log(1.0 - rng.next());
        st[p] = StartRec{dir.x, dir.y, dir.z, t0, rng.key, target};
        cells[p] = cell;
    }
}

#include "tv_path.inc"

// ImageAccumulator::add_sample in sample order (image.hpp:36-45); one thread
// per pixel of the batch's units.
__global__ void accum_kernel(Batch B, CamView C, const uint32_t* __restrict__ cells, const double* __restrict__ rad,
                             RenderOut O) {
    const uint32_t n_px = B.n_units * 32u;
    unsigned long long traced = 0;  // stats[1]: paths_traced (image.hpp:25)
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_px; q += gridDim.x * blockDim.x) {
        const uint32_t unit = q >> 5, lane = q & 31u;
        const uint32_t p0 = path_id(B, unit, lane, 0);
        int px, py;
        uint32_t s;
        path_pixel(B, p0, px, py, s);
        if (px >= C.w || py >= C.h) continue;
        traced += B.ns;
        const uint64_t pix = static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + px;
        double sr = 0.0, sg = 0.0, sb = 0.0, qr = 0.0, qg = 0.0, qb = 0.0;
        uint32_t n = 0;
        if (!B.first) {
            if (O.sum) sr = O.sum[3 * pix], sg = O.sum[3 * pix + 1], sb = O.sum[3 * pix + 2];
            if (O.sum_sq) qr = O.sum_sq[3 * pix], qg = O.sum_sq[3 * pix + 1], qb = O.sum_sq[3 * pix + 2];
            if (O.counts) n = O.counts[pix];
        }
        uint32_t k = 0;
        if (B.order && !(p0 & 1u)) {
            // sample-major order: the pixel's samples are consecutive paths, so two
            // samples (48 B) are three aligned 16-B loads; summation order unchanged
            const double2* r2 = reinterpret_cast<const double2*>(rad + 3ull * p0);
            for (; k + 1 < B.ns; k += 2) {
                const double2 a = r2[3 * (k >> 1)], b2 = r2[3 * (k >> 1) + 1], c2 = r2[3 * (k >> 1) + 2];
                sr += a.x, sg += a.y, sb += b2.x;
                qr += a.x * a.x, qg += a.y * a.y, qb += b2.x * b2.x;
                sr += b2.y, sg += c2.x, sb += c2.y;
                qr += b2.y * b2.y, qg += c2.x * c2.x, qb += c2.y * c2.y;
                n += 2;
            }
        }
        for (; k < B.ns; ++k) {
            const uint64_t pp = path_id(B, unit, lane, k);
            const double r = rad[3 * pp], g = rad[3 * pp + 1], b = rad[3 * pp + 2];
            sr += r, sg += g, sb += b;
            qr += r * r, qg += g * g, qb += b * b;
            ++n;
        }
        if (O.sum) O.sum[3 * pix] = sr, O.sum[3 * pix + 1] = sg, O.sum[3 * pix + 2] = sb;
        if (O.sum_sq) O.sum_sq[3 * pix] = qr, O.sum_sq[3 * pix + 1] = qg, O.sum_sq[3 * pix + 2] = qb;
        if (O.counts) O.counts[pix] = n;
    }
    // peer outputs (tv_ipc_open): publish this thread's stores before the
    // kernel ends, so a stream-ordered barrier after it covers them
    if (O.remote) __threadfence_system();
    if (O.stats) {
        for (int o = 16; o; o >>= 1) traced += __shfl_down_sync(kFull, traced, o);
        if ((threadIdx.x & 31) == 0 && traced) atomicAdd(reinterpret_cast<unsigned long long*>(O.stats + 1), traced);
    }
}

// ---------------------------------------------------------------------------
// march_segments (tracer.cpp:164-174): pass 0 counts, pass 1 writes at offsets.
__global__ void march_kernel(GridView G, const tv_ray* __restrict__ rays, uint64_t n, int pass,
                             uint64_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                             tv_segment* __restrict__ out, uint64_t cap, unsigned long long* deg) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const tv_ray R = rays[i];
    const d3 o = mk(R.origin[0], R.origin[1], R.origin[2]);
    const d3 dir = mk(R.dir[0], R.dir[1], R.dir[2]);
    const double tmax = R.t_max;
    uint64_t k = 0;
    const uint64_t base = pass ? offsets[i] : 0;
    double t0, t1;
    if (slab(o, dir, dmax(0.0, R.t_min), tmax, t0, t1)) {
        d3 q = ray_at(o, dir, t0 + kNudge);
        q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
        uint32_t cell = locate(G, q);
        if (cell != kNone) {
            double seg_start = t0, probe = t0 + kNudge;
            LeafRec rec = load_leaf(G.leaves, cell);
            for (uint32_t steps = 1;; ++steps) {
                if (steps > kMaxSteps) {
                    if (pass == 0) atomicAdd(deg, 1ull);
                    break;
                }
                double t;
                int slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
                if (slot < 0) {
                    probe += kNudge;
                    slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
                    if (slot < 0) {
                        if (pass == 0) atomicAdd(deg, 1ull);
                        break;
                    }
                }
                const double t_exit = dmax(probe + t, seg_start);
                const bool clip = t_exit >= tmax;
                const uint32_t nb = nbr_leaf(sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot));
                if (pass && base + k < cap) {
                    tv_segment sgm;
                    sgm.cell = G.leaf2tet[cell];
                    sgm.pad = 0;
                    sgm.t_enter = seg_start;
                    sgm.t_exit = clip ? tmax : t_exit;
                    out[base + k] = sgm;
                }
                ++k;
                if (clip || nb == kNoLeaf) break;
                rec = load_leaf(G.leaves, nb);
                cell = nb;
                seg_start = t_exit;
                probe = t_exit + kNudge;
            }
        }
    }
    if (pass == 0) counts[i] = k;
}

// march_transmittance (mode 0) and sample_free_path (mode 1) (tracer.cpp:176-216)
// over the same marcher as march_kernel; one thread per ray.
__global__ void medium_kernel(GridView G, const tv_ray* __restrict__ rays, uint64_t n, int mode, uint64_t seed,
                              const uint64_t* __restrict__ pixels, const uint64_t* __restrict__ samples,
                              double* __restrict__ tau_out, double* __restrict__ trans_out,
                              tv_free_path* __restrict__ fp_out, unsigned long long* counters) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const tv_ray R = rays[i];
    const d3 o = mk(R.origin[0], R.origin[1], R.origin[2]);
    const d3 dir = mk(R.dir[0], R.dir[1], R.dir[2]);
    const double tmax = R.t_max;
    double target = 0.0;
    if (mode == 1) {  // sample_free_path draws its target first (tracer.cpp:190)
        Rng rng;
        rng.init(seed, pixels[i], samples[i]);
        target = -log(1.0 - rng.next());
    }
    tv_free_path fp;
    fp.collided = 0, fp.cell = kNone, fp.distance = 0.0;
    fp.position[0] = o.x, fp.position[1] = o.y, fp.position[2] = o.z;
    double tau = 0.0;
    uint32_t visited = 0;
    bool aborted = false;
    double t0, t1;
    uint32_t cell = kNone;
    if (slab(o, dir, dmax(0.0, R.t_min), tmax, t0, t1)) {
        d3 q = ray_at(o, dir, t0 + kNudge);
        q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
        cell = locate(G, q);
    }
    if (cell != kNone) {
        double seg_start = t0, probe = t0 + kNudge, last_t1 = 0.0;
        d3 event = o;
        LeafRec rec = load_leaf(G.leaves, cell);
        for (uint32_t steps = 1;; ++steps) {
            if (steps > kMaxSteps) {
                aborted = true;
                break;
            }
            double t;
            int slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
            if (slot < 0) {
                probe += kNudge;
                slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
                if (slot < 0) {
                    aborted = true;
                    break;
                }
            }
            const double t_exit = dmax(probe + t, seg_start);
            const double s0 = seg_start, lambda = static_cast<double>(__uint_as_float(rec.w[13]));
            const uint32_t step_cell = cell;
            double s1;
            bool escaped = false;
            if (t_exit >= tmax) {  // caller-imposed range ends inside the grid
                s1 = tmax;
                escaped = true;
                event = ray_at(o, dir, tmax);
            } else {
                s1 = t_exit;
                const uint32_t nb = nbr_leaf(sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot));
                if (nb == kNoLeaf) {
                    escaped = true;
                    event = ray_at(o, dir, t_exit);
                } else {
                    rec = load_leaf(G.leaves, nb);
                    cell = nb;
                    seg_start = t_exit;
                    probe = t_exit + kNudge;
                }
            }
            ++visited;
            const double seg_tau = lambda * (s1 - s0);
            if (mode == 1 && lambda > 0.0 && tau + seg_tau >= target) {  // m.shorten (tracer.cpp:90-95)
                const double dist = (target - tau) / lambda;
                const d3 e = ray_at(o, dir, s0 + dist);
                fp.collided = 1, fp.cell = G.leaf2tet[step_cell], fp.distance = s0 + dist;
                fp.position[0] = e.x, fp.position[1] = e.y, fp.position[2] = e.z;
                break;
            }
            tau += seg_tau;
            last_t1 = s1;
            if (escaped) break;
        }
        if (mode == 1 && !fp.collided) {
            const d3 e = aborted ? ray_at(o, dir, last_t1) : event;
            fp.position[0] = e.x, fp.position[1] = e.y, fp.position[2] = e.z;
            fp.distance = last_t1;
        }
    }
    if (counters) {
        atomicAdd(counters, static_cast<unsigned long long>(visited));
        if (aborted) atomicAdd(counters + 1, 1ull);
    }
    if (mode == 0) {
        if (tau_out) tau_out[i] = tau;
        if (trans_out) trans_out[i] = exp(-tau);
    } else if (fp_out) {
        fp_out[i] = fp;
    }
}

// tetvol::trace (tracer.cpp:258-263) = trace_path (path_integrator.hpp:42-84)
// for arbitrary rays, one thread per ray, RngStream(seed, pixels[i], samples[i]).
// The first flight honours the ray's [t_min, t_max]; redirects reset it to
// [0, inf) (TetMarcher::redirect, tracer.cpp:97-105).
__global__ void trace_rays_kernel(GridView G, RenderParams P, const tv_ray* __restrict__ rays, uint64_t n,
                                  uint64_t seed, const uint64_t* __restrict__ pixels,
                                  const uint64_t* __restrict__ samples, double* __restrict__ out,
                                  unsigned long long* counters) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const tv_ray R = rays[i];
    d3 o = mk(R.origin[0], R.origin[1], R.origin[2]);
    d3 dir = mk(R.dir[0], R.dir[1], R.dir[2]);
    double tmax = R.t_max;
    Rng rng;
    rng.init(seed, pixels[i], samples[i]);
    d3 radiance = mk(0, 0, 0), throughput = mk(1, 1, 1);
    uint32_t visited = 0;
    bool degenerate = false;
    double t0, t1;
    uint32_t cell = kNone;
    if (slab(o, dir, dmax(0.0, R.t_min), tmax, t0, t1)) {
        d3 q = ray_at(o, dir, t0 + kNudge);
        q = mk(dclamp(q.x, 0.0, 1.0), dclamp(q.y, 0.0, 1.0), dclamp(q.z, 0.0, 1.0));
        cell = locate(G, q);
    }
    if (cell == kNone) {
        radiance = mk(P.env[0], P.env[1], P.env[2]);  // !m.start(primary): return environment
    } else {
        double seg_start = t0, probe = t0 + kNudge;
        LeafRec rec = load_leaf(G.leaves, cell);
        uint32_t steps = 0;
        for (int bounce = 0;;) {
            const double target = -log(1.0 - rng.next());
            double tau = 0.0;
            bool collided = false, aborted = false;
            d3 event = o;
            for (;;) {  // TetMarcher::next until escape / abort / collision
                if (++steps > kMaxSteps) {
                    aborted = true;
                    break;
                }
                double t;
                int slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
                if (slot < 0) {
                    probe += kNudge;
                    slot = exit_face(rec, ray_at(o, dir, probe), dir, t);
                    if (slot < 0) {
                        aborted = true;
                        break;
                    }
                }
                const double t_exit = dmax(probe + t, seg_start);
                const double s0 = seg_start, lambda = static_cast<double>(__uint_as_float(rec.w[13]));
                bool escaped = false;
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
                const double seg_tau = lambda * (s1 - s0);
                if (lambda > 0.0 && tau + seg_tau >= target) {  // m.shorten: stay in this cell
                    event = ray_at(o, dir, s0 + (target - tau) / lambda);
                    collided = true;
                    break;
                }
                tau += seg_tau;
                if (escaped) break;
                rec = load_leaf(G.leaves, next);
                cell = next;
                seg_start = t_exit;
                probe = t_exit + kNudge;
            }
            if (aborted) {
                degenerate = true;
                break;
            }
            if (!collided) {
                radiance = add(radiance, mulv(throughput, mk(P.env[0], P.env[1], P.env[2])));
                break;
            }
            const uint32_t mask = rec.w[12] >> 24;
            if (mask & 2u) {
                const d3 e = emission_color(static_cast<double>(__uint_as_float(rec.w[14])));
                radiance = add(radiance, mul(mulv(throughput, e), P.emission_scale));
            }
            throughput = mul(throughput, (mask & 4u) ? static_cast<double>(__uint_as_float(rec.w[15])) : P.default_albedo);
            ++bounce;
            if (bounce >= P.max_bounces) break;
            if (bounce >= 4) {
                const double pm = dmax(throughput.x, dmax(throughput.y, throughput.z));
                if (pm < 1e-3) {
                    if (rng.next() >= pm) break;
                    throughput = divs(throughput, pm);
                }
            }
            // TetMarcher::redirect: from the event point, [0, inf), same cell
            dir = sample_phase_hg(dir, P.g, rng);
            o = event;
            tmax = __longlong_as_double(0x7ff0000000000000ll);
            seg_start = 0.0;
            probe = 0.0;
        }
    }
    out[3 * i] = radiance.x, out[3 * i + 1] = radiance.y, out[3 * i + 2] = radiance.z;
    if (counters) {
        atomicAdd(counters, static_cast<unsigned long long>(visited));
        if (degenerate) atomicAdd(counters + 1, 1ull);
    }
}

__global__ void locate_kernel(GridView G, const double* __restrict__ pts, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t leaf = locate(G, mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    out[i] = leaf == kNone ? kNone : G.leaf2tet[leaf];
}

}  // namespace tvb
