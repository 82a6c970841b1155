// Traversal kernels: the volumetric path-tracing megakernel (render), the
// deterministic segment marcher (march_segments parity entry) and batched
// locate_point.
//
// Reference semantics (paths relative to /root/reference/proj):
//   render_image  include/tetvol/path_integrator.hpp:87-136
//   trace_path    include/tetvol/path_integrator.hpp:42-84
//   TetMarcher    src/tracer.cpp:25-127, exit_face src/tracer.cpp:143-162
#include "tv_trace.cuh"

namespace tvb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Work unit = one warp = an 8x4 pixel block; 8 units tile a 16x16 sharding tile.
__device__ __forceinline__ void unit_pixel(const TileSched& S, uint32_t unit, int lane, int& px, int& py) {
    const uint32_t k = unit >> 3, sub = unit & 7;
    const uint32_t t = static_cast<uint32_t>(S.rank) + k * static_cast<uint32_t>(S.n_ranks);
    const uint32_t tx = t % S.tiles_x, ty = t / S.tiles_x;
    px = static_cast<int>(tx * 16 + (sub & 1) * 8 + (lane & 7));
    py = static_cast<int>(ty * 16 + (sub >> 1) * 4 + (lane >> 3));
}

__device__ __forceinline__ d3 ray_at(d3 o, d3 d, double t) { return add(o, mul(d, t)); }

}  // namespace

// One lane owns one pixel and traces its spp samples in order s = 0..spp-1, so
// the per-pixel sums accumulate in exactly the reference order
// (path_integrator.hpp:109-114) and the framebuffer is bit-comparable. The
// outer loop advances every active lane by one event (a tet step, or a path
// start) per iteration: path regeneration keeps lanes busy without any
// cross-lane exchange.
__global__ void __launch_bounds__(kRenderThreads, kRenderMinBlocks)
    render_kernel(GridView G, CamView C, RenderParams P, TileSched S, RenderOut O) {
    const int lane = threadIdx.x & 31;
    uint64_t my_cells = 0, my_deg = 0;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const d3 cam_pos = mk(C.pos[0], C.pos[1], C.pos[2]);

    for (;;) {
        uint32_t unit = 0;
        if (lane == 0) unit = atomicAdd(S.counter, 1u);
        unit = __shfl_sync(kFull, unit, 0);
        if (unit >= S.n_units) break;
        int px, py;
        unit_pixel(S, unit, lane, px, py);
        bool active = px < C.w && py < C.h;
        const uint64_t pixel = static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + static_cast<uint64_t>(px);

        double sr = 0.0, sg = 0.0, sb = 0.0, qr = 0.0, qg = 0.0, qb = 0.0;
        uint32_t count = 0;
        int s = 0;
        bool in_path = false;

        // path state
        Rng rng;
        d3 o = cam_pos, dir = mk(0, 0, 1);
        d3 T = mk(1, 1, 1), L = mk(0, 0, 0);
        double seg_start = 0.0, probe = 0.0, tau = 0.0, target = 0.0;
        uint32_t cell = 0;
        int bounce = 0;
        uint64_t steps = 0;
        LeafRec rec;
        Verts V;

        while (__any_sync(kFull, active)) {
            if (!active) continue;
            if (!in_path) {
                if (s == P.spp) {  // pixel done: one writer per pixel, no atomics
                    if (O.sum) {
                        O.sum[3 * pixel] = sr, O.sum[3 * pixel + 1] = sg, O.sum[3 * pixel + 2] = sb;
                    }
                    if (O.sum_sq) {
                        O.sum_sq[3 * pixel] = qr, O.sum_sq[3 * pixel + 1] = qg, O.sum_sq[3 * pixel + 2] = qb;
                    }
                    if (O.counts) O.counts[pixel] = count;
                    active = false;
                    continue;
                }
                // camera sample (path_integrator.hpp:110-113)
                rng.init(P.seed, pixel, static_cast<uint64_t>(s));
                const double jx = rng.next();
                const double jy = rng.next();
                o = cam_pos;
                dir = primary_dir(C, px, py, jx, jy);
                T = mk(1, 1, 1);
                L = mk(0, 0, 0);
                bounce = 0;
                // TetMarcher::start (tracer.cpp:29-45)
                double t0, t1;
                bool hit = slab(o, dir, 0.0, inf, t0, t1);
                if (hit) {
                    d3 p = ray_at(o, dir, t0 + kNudge);
                    p = mk(dclamp(p.x, 0.0, 1.0), dclamp(p.y, 0.0, 1.0), dclamp(p.z, 0.0, 1.0));
                    cell = locate(G, p);
                    hit = cell != kNone;
                }
                if (!hit) {  // trace_path returns the environment (path_integrator.hpp:46)
                    const double cr = P.env[0], cg = P.env[1], cb = P.env[2];
                    sr += cr, sg += cg, sb += cb;
                    qr += cr * cr, qg += cg * cg, qb += cb * cb;
                    ++count;
                    ++s;
                    continue;
                }
                seg_start = t0;
                probe = t0 + kNudge;
                steps = 0;
                rec = load_leaf(G.leaves, cell);
                fetch_all(G, rec, V);
                target = -log(1.0 - rng.next());  // path_integrator.hpp:49
                tau = 0.0;
                in_path = true;
                continue;
            }

            // ---- one tet step: TetMarcher::next (tracer.cpp:47-88) ----
            bool ended = false;
            d3 result = L;
            if (++steps > kMaxSteps) {
                ++my_deg;
                ended = true;
            } else {
                double t;
                int slot = exit_face(rec.w[12], V, ray_at(o, dir, probe), dir, t);
                if (slot < 0) {
                    probe += kNudge;
                    slot = exit_face(rec.w[12], V, ray_at(o, dir, probe), dir, t);
                }
                if (slot < 0) {  // aborted: degenerate path (path_integrator.hpp:62-65)
                    ++my_deg;
                    ended = true;
                } else {
                    const double t_exit = dmax(probe + t, seg_start);
                    const double lambda = static_cast<double>(__uint_as_float(rec.w[13]));
                    ++my_cells;
                    const double seg_tau = lambda * (t_exit - seg_start);
                    if (lambda > 0.0 && tau + seg_tau >= target) {
                        // collision: shorten + media + redirect (path_integrator.hpp:56-82)
                        o = ray_at(o, dir, seg_start + (target - tau) / lambda);
                        const uint32_t mask = rec.w[12] >> 20;
                        if (mask & 2u) {
                            const d3 e = emission_color(static_cast<double>(__uint_as_float(rec.w[14])));
                            L = add(L, mul(mulv(T, e), P.emission_scale));
                        }
                        T = mul(T, (mask & 4u) ? static_cast<double>(__uint_as_float(rec.w[15])) : P.default_albedo);
                        ++bounce;
                        result = L;
                        if (bounce >= P.max_bounces) {
                            ended = true;
                        } else {
                            bool killed = false;
                            if (bounce >= 4) {
                                const double p = dmax(T.x, dmax(T.y, T.z));
                                if (p < 1e-3) {
                                    if (rng.next() >= p) killed = true;
                                    else T = divs(T, p);
                                }
                            }
                            if (killed) {
                                ended = true;
                            } else {
                                dir = sample_phase_hg(dir, P.g, rng);
                                seg_start = 0.0;
                                probe = 0.0;
                                target = -log(1.0 - rng.next());
                                tau = 0.0;
                            }
                        }
                    } else {
                        tau += seg_tau;
                        const uint32_t nb = sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot);
                        if (nb == kNone) {  // escaped: L + T * env (path_integrator.hpp:66)
                            result = add(L, mulv(T, mk(P.env[0], P.env[1], P.env[2])));
                            ended = true;
                        } else {
                            const uint32_t far_id = sel4(rec.w[8], rec.w[9], rec.w[10], rec.w[11], slot);
                            const uint4 far_q = __ldg(G.verts + far_id);
                            rec = load_leaf(G.leaves, nb);
                            carry(rec, V, far_id, far_q);
                            cell = nb;
                            seg_start = t_exit;
                            probe = t_exit + kNudge;
                        }
                    }
                }
            }
            if (ended) {  // ImageAccumulator::add_sample (image.hpp:36-45)
                sr += result.x, sg += result.y, sb += result.z;
                qr += result.x * result.x, qg += result.y * result.y, qb += result.z * result.z;
                ++count;
                ++s;
                in_path = false;
            }
        }
    }
    // per-warp reduction of the counters, one atomic per warp
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my_cells += __shfl_down_sync(kFull, my_cells, off);
        my_deg += __shfl_down_sync(kFull, my_deg, off);
    }
    if (lane == 0 && O.stats) {
        atomicAdd(reinterpret_cast<unsigned long long*>(O.stats), static_cast<unsigned long long>(my_cells));
        atomicAdd(reinterpret_cast<unsigned long long*>(O.stats + 2), static_cast<unsigned long long>(my_deg));
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
    uint64_t k = 0, base = pass ? offsets[i] : 0;
    double t0, t1;
    if (slab(o, dir, dmax(0.0, R.t_min), tmax, t0, t1)) {
        d3 p = ray_at(o, dir, t0 + kNudge);
        p = mk(dclamp(p.x, 0.0, 1.0), dclamp(p.y, 0.0, 1.0), dclamp(p.z, 0.0, 1.0));
        uint32_t cell = locate(G, p);
        if (cell != kNone) {
            double seg_start = t0, probe = t0 + kNudge;
            LeafRec rec = load_leaf(G.leaves, cell);
            Verts V;
            fetch_all(G, rec, V);
            for (uint64_t steps = 1;; ++steps) {
                if (steps > kMaxSteps) {
                    if (pass == 0) atomicAdd(deg, 1ull);
                    break;
                }
                double t;
                int slot = exit_face(rec.w[12], V, ray_at(o, dir, probe), dir, t);
                if (slot < 0) {
                    probe += kNudge;
                    slot = exit_face(rec.w[12], V, ray_at(o, dir, probe), dir, t);
                    if (slot < 0) {
                        if (pass == 0) atomicAdd(deg, 1ull);
                        break;
                    }
                }
                const double t_exit = dmax(probe + t, seg_start);
                const bool clip = t_exit >= tmax;
                const uint32_t nb = sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot);
                if (pass && base + k < cap) {
                    tv_segment sgm;
                    sgm.cell = G.leaf2tet[cell];
                    sgm.pad = 0;
                    sgm.t_enter = seg_start;
                    sgm.t_exit = clip ? tmax : t_exit;
                    out[base + k] = sgm;
                }
                ++k;
                if (clip || nb == kNone) break;
                const uint32_t far_id = sel4(rec.w[8], rec.w[9], rec.w[10], rec.w[11], slot);
                const uint4 far_q = __ldg(G.verts + far_id);
                rec = load_leaf(G.leaves, nb);
                carry(rec, V, far_id, far_q);
                cell = nb;
                seg_start = t_exit;
                probe = t_exit + kNudge;
            }
        }
    }
    if (pass == 0) counts[i] = k;
}

__global__ void locate_kernel(GridView G, const double* __restrict__ pts, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t leaf = locate(G, mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    out[i] = leaf == kNone ? kNone : G.leaf2tet[leaf];
}

}  // namespace tvb
