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
#include "tv_trace.cuh"

namespace tvb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void path_pixel(const Batch& B, uint32_t p, int& px, int& py, uint32_t& s) {
    const uint32_t per_unit = B.ns * 32u;
    const uint32_t unit = p / per_unit, r = p - unit * per_unit;
    s = B.s0 + r / 32u;
    const uint32_t lane = r & 31u;
    const uint32_t k = unit >> 3, sub = unit & 7u;
    const uint32_t t = static_cast<uint32_t>(B.rank) + k * static_cast<uint32_t>(B.n_ranks);
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
        st[p] = StartRec{dir.x, dir.y, dir.z, t0};
        cells[p] = cell;
    }
}

__global__ void __launch_bounds__(kTraceThreads, kTraceMinBlocks)
    trace_kernel(GridView G, CamView C, RenderParams P, Batch B, const StartRec* __restrict__ st,
                 const uint32_t* __restrict__ cells, double* __restrict__ rad, uint64_t* stats, uint32_t* counter) {
    __shared__ FaceTables<kTraceThreads> S;
    init_face_tables(S);
    __syncthreads();
    const int t = threadIdx.x;
    const int lane = t & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const d3 cam_pos = mk(C.pos[0], C.pos[1], C.pos[2]);
    const d3 env = mk(P.env[0], P.env[1], P.env[2]);
    uint64_t my_cells = 0, my_deg = 0;

    uint32_t chunk_next = 0, chunk_end = 0;  // warp-uniform
    bool exhausted = false;                  // warp-uniform

    int state = S_IDLE;
    uint32_t p = 0, cell = 0, steps = 0;
    int bounce = 0;
    Rng rng;
    rng.key = 0;
    rng.dim = 0;
    d3 o = cam_pos, dir = mk(0, 0, 1), T = mk(1, 1, 1), L = mk(0, 0, 0);
    double seg_start = 0.0, probe = 0.0, tau = 0.0, target = 0.0;
    LeafRec rec;

    for (;;) {
        const unsigned m_idle = __ballot_sync(kFull, state == S_IDLE);
        const unsigned m_step = __ballot_sync(kFull, state == S_STEP);
        const unsigned m_scat = __ballot_sync(kFull, state == S_SCATTER);
        const bool queue_open = !(exhausted && chunk_next >= chunk_end);
        if (!m_step && !m_scat && !queue_open) break;

        // ---- regeneration, batched: idle lanes take consecutive path ids ----
        if (m_idle && queue_open && (__popc(m_idle) >= 8 || !m_step)) {
            const uint32_t n_need = __popc(m_idle);
            const uint32_t my_rank = __popc(m_idle & lt_mask);
            uint32_t mine = kNone;
            const uint32_t avail = chunk_end - chunk_next;
            if (state == S_IDLE && my_rank < avail) mine = chunk_next + my_rank;
            const uint32_t used = min(avail, n_need);
            chunk_next += used;
            if (n_need > avail && !exhausted) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(counter, kChunk);
                base = __shfl_sync(kFull, base, 0);
                if (base >= B.n_paths) {
                    exhausted = true;
                } else {
                    chunk_next = base;
                    chunk_end = min(base + kChunk, B.n_paths);
                    const uint32_t avail2 = chunk_end - chunk_next;
                    const uint32_t r2 = my_rank - used;
                    if (state == S_IDLE && mine == kNone && r2 < avail2) mine = chunk_next + r2;
                    chunk_next += min(avail2, n_need - used);
                }
            }
            if (mine != kNone) {
                const uint32_t c = cells[mine];
                if (c == kNone) {  // ray misses the grid: trace_path returns env (path_integrator.hpp:46)
                    rad[3ull * mine] = env.x, rad[3ull * mine + 1] = env.y, rad[3ull * mine + 2] = env.z;
                } else if (c != kInvalidPixel) {
                    int px, py;
                    uint32_t s;
                    path_pixel(B, mine, px, py, s);
                    const StartRec sr = st[mine];
                    rng.init(P.seed, static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + px, s);
                    rng.dim = 2;  // the jitter draws
                    p = mine;
                    cell = c;
                    o = cam_pos;
                    dir = mk(sr.dx, sr.dy, sr.dz);
                    seg_start = sr.t0;
                    probe = sr.t0 + kNudge;
                    T = mk(1, 1, 1);
                    L = mk(0, 0, 0);
                    bounce = 0;
                    steps = 0;
                    tau = 0.0;
                    target = -log(1.0 - rng.next());  // path_integrator.hpp:49
                    rec = load_leaf(G.leaves, cell);
                    set_flight_dir(S, t, dir);
                    state = S_STEP;
                }
            }
        }

        // ---- scatter, batched: new direction + flight tables (path_integrator.hpp:82, 49) ----
        if (m_scat && (__popc(m_scat) >= 8 || !m_step)) {
            if (state == S_SCATTER) {
                dir = sample_phase_hg(dir, P.g, rng);
                seg_start = 0.0;
                probe = 0.0;
                target = -log(1.0 - rng.next());
                tau = 0.0;
                set_flight_dir(S, t, dir);
                state = S_STEP;
            }
        }

        if (state != S_STEP) continue;

        // ---- one tet step: TetMarcher::next (tracer.cpp:47-88) ----
        bool ended = false;
        d3 result = L;
        if (++steps > kMaxSteps) {
            ++my_deg;
            ended = true;
        } else {
            double tx;
            d3 pos = ray_at(o, dir, probe);
            S.pos[0][t] = pos.x, S.pos[1][t] = pos.y, S.pos[2][t] = pos.z;
            int slot = exit_face_tab(S, t, rec, tx);
            if (slot < 0) {  // degenerate corner: one nudged retry (tracer.cpp:54-61)
                probe += kNudge;
                pos = ray_at(o, dir, probe);
                S.pos[0][t] = pos.x, S.pos[1][t] = pos.y, S.pos[2][t] = pos.z;
                slot = exit_face_tab(S, t, rec, tx);
            }
            if (slot < 0) {  // aborted (path_integrator.hpp:62-65)
                ++my_deg;
                ended = true;
            } else {
                const double t_exit = dmax(probe + tx, seg_start);
                const double lambda = static_cast<double>(__uint_as_float(rec.w[13]));
                ++my_cells;
                const double seg_tau = lambda * (t_exit - seg_start);
                if (lambda > 0.0 && tau + seg_tau >= target) {
                    // collision: shorten, media, Russian roulette (path_integrator.hpp:56-81)
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
                        if (bounce >= 4) {
                            const double pmax = dmax(T.x, dmax(T.y, T.z));
                            if (pmax < 1e-3) {
                                if (rng.next() >= pmax) ended = true;
                                else T = divs(T, pmax);
                            }
                        }
                        if (!ended) state = S_SCATTER;  // redirect is deferred
                    }
                } else {
                    tau += seg_tau;
                    const uint32_t nb = sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot);
                    if (nb == kNone) {  // escaped (path_integrator.hpp:66)
                        result = add(L, mulv(T, env));
                        ended = true;
                    } else {
                        cell = nb;
                        rec = load_leaf(G.leaves, nb);
                        seg_start = t_exit;
                        probe = t_exit + kNudge;
                    }
                }
            }
        }
        if (ended) {
            rad[3ull * p] = result.x, rad[3ull * p + 1] = result.y, rad[3ull * p + 2] = result.z;
            state = S_IDLE;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my_cells += __shfl_down_sync(kFull, my_cells, off);
        my_deg += __shfl_down_sync(kFull, my_deg, off);
    }
    if (lane == 0 && stats) {
        atomicAdd(reinterpret_cast<unsigned long long*>(stats), static_cast<unsigned long long>(my_cells));
        atomicAdd(reinterpret_cast<unsigned long long*>(stats + 2), static_cast<unsigned long long>(my_deg));
    }
}

// ImageAccumulator::add_sample in sample order (image.hpp:36-45); one thread
// per pixel of the batch's units.
__global__ void accum_kernel(Batch B, CamView C, const uint32_t* __restrict__ cells, const double* __restrict__ rad,
                             RenderOut O) {
    const uint32_t n_px = B.n_units * 32u;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_px; q += gridDim.x * blockDim.x) {
        const uint32_t unit = q >> 5, lane = q & 31u;
        const uint32_t p0 = unit * B.ns * 32u + lane;
        int px, py;
        uint32_t s;
        path_pixel(B, p0, px, py, s);
        if (px >= C.w || py >= C.h) continue;
        const uint64_t pix = static_cast<uint64_t>(py) * static_cast<uint64_t>(C.w) + px;
        double sr = 0.0, sg = 0.0, sb = 0.0, qr = 0.0, qg = 0.0, qb = 0.0;
        uint32_t n = 0;
        if (!B.first) {
            if (O.sum) sr = O.sum[3 * pix], sg = O.sum[3 * pix + 1], sb = O.sum[3 * pix + 2];
            if (O.sum_sq) qr = O.sum_sq[3 * pix], qg = O.sum_sq[3 * pix + 1], qb = O.sum_sq[3 * pix + 2];
            if (O.counts) n = O.counts[pix];
        }
        for (uint32_t k = 0; k < B.ns; ++k) {
            const uint64_t pp = static_cast<uint64_t>(p0) + k * 32u;
            const double r = rad[3 * pp], g = rad[3 * pp + 1], b = rad[3 * pp + 2];
            sr += r, sg += g, sb += b;
            qr += r * r, qg += g * g, qb += b * b;
            ++n;
        }
        if (O.sum) O.sum[3 * pix] = sr, O.sum[3 * pix + 1] = sg, O.sum[3 * pix + 2] = sb;
        if (O.sum_sq) O.sum_sq[3 * pix] = qr, O.sum_sq[3 * pix + 1] = qg, O.sum_sq[3 * pix + 2] = qb;
        if (O.counts) O.counts[pix] = n;
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
                rec = load_leaf(G.leaves, nb);
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
