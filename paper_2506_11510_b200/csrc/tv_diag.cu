// Diagnostics: the memory-latency ceiling of the trace kernel on a frame
// (include/tetvol_b200_diag.h).
//
// 1. record_kernel runs every path of the frame through the integrator of
//    trace_path (path_integrator.hpp:42-84), from the same start records
//    start_kernel gives the render, and writes one 4-bit code per tet step (one
//    per MarchStep, the reference's cells_visited): the face slot the step
//    leaves by (0-3), or 4 when the flight collides and the next step re-reads
//    the same cell. Eight codes per word; each path starts on a word. Two
//    passes: count, then write at the scanned word offsets.
// 2. replay_kernel walks the render's paths again as a chain of dependent
//    64-byte LeafRec loads: each step loads the current leaf's record and takes
//    the next leaf index from that record's neighbour word named by the code,
//    exactly the render's dependence (record -> exit face -> neighbour ->
//    next record) without the geometry. Same path order, block size, per-lane
//    path regeneration from 64-path warp chunks, and shared-memory footprint
//    per block (so the same L1 size and resident warps) as the trace kernel.
//    Its steps/s is the rate of a trace kernel whose exit-face computation
//    were free.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <vector>

#include "tetvol_b200_diag.h"
#include "tv_trace.cuh"

namespace tvb {

int validate_render_cfg(const tv_render_config* r);

namespace {

constexpr unsigned kFull = 0xffffffffu;

// trace_path from a start record (the render's path p), recording or counting
// the leaf of every step
__global__ void record_kernel(GridView G, CamView C, RenderParams P, Batch B, const StartRec* __restrict__ st,
                              const uint32_t* __restrict__ cells, uint32_t* __restrict__ counts,
                              const uint64_t* __restrict__ offs, uint32_t* __restrict__ codes) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= B.n_paths) return;
    uint32_t cell = cells[p];
    uint32_t* out = offs ? codes + offs[p] : nullptr;  // word offset of this path
    uint32_t n = 0, word = 0;
    if (cell != kNone && cell != kInvalidPixel) {
        const StartRec sr = st[p];
        d3 o = mk(C.pos[0], C.pos[1], C.pos[2]);
        d3 dir = mk(sr.dx, sr.dy, sr.dz);
        double seg_start = sr.t0, probe = sr.t0 + kNudge;
        Rng rng;
        rng.key = sr.key;
        rng.dim = 3;
        double target = sr.target;
        d3 throughput = mk(1, 1, 1);
        LeafRec rec = load_leaf(G.leaves, cell);
        for (int bounce = 0;;) {
            double tau = 0.0;
            bool collided = false, aborted = false;
            d3 event = o;
            for (;;) {
                if (n + 1 > kMaxSteps) {
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
                const uint32_t next = nbr_leaf(sel4(rec.w[0], rec.w[1], rec.w[2], rec.w[3], slot));
                const double seg_tau = lambda * (t_exit - s0);
                const bool coll = lambda > 0.0 && tau + seg_tau >= target;
                if (out) {
                    word |= static_cast<uint32_t>(coll ? 4 : slot) << (4 * (n & 7));
                    if ((n & 7) == 7) out[n >> 3] = word, word = 0;
                }
                ++n;
                if (coll) {
                    event = ray_at(o, dir, s0 + (target - tau) / lambda);
                    collided = true;
                    break;
                }
                tau += seg_tau;
                if (next == kNoLeaf) break;
                rec = load_leaf(G.leaves, next);
                cell = next;
                seg_start = t_exit;
                probe = t_exit + kNudge;
            }
            if (aborted || !collided) break;
            const uint32_t mask = rec.w[12] >> 24;
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
            dir = sample_phase_hg(dir, P.g, rng);
            o = event;
            seg_start = 0.0;
            probe = 0.0;
            target = -log(1.0 - rng.next());
        }
    }
    if (out && (n & 7)) out[n >> 3] = word;
    if (!offs) counts[p] = n;
}

// dependent-gather replay of the recorded paths in render path order, with
// the trace kernel's warp schedule: idle lanes regenerate in batches
// (regen_min), lanes whose flight collided wait for a scatter batch
// (scatter_min), and the stepping lanes step until one changes state
// What-if (TMA = true): each lane fetches its record with a 64-B bulk copy
// (cp.async.bulk, the TMA unit: L2 -> shared memory, completion on a per-lane
// mbarrier) and reads it from shared memory, so the L1 / LSU data pipe sees
// only the shared-memory reads.
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load64(uint32_t dst, const void* src, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" ::"r"(mbar) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];" ::"r"(dst),
                 "l"(src), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(mbar),
        "r"(phase)
        : "memory");
}

template <int MODE>  // 0: load_leaf, 1: TMA bulk copies, 2: load_leaf_pair, 3: 32-B half records, 4: count lines
__global__ void replay_kernel(const LeafRec* __restrict__ leaves, const uint32_t* __restrict__ start,
                              const uint32_t* __restrict__ counts, const uint32_t* __restrict__ codes,
                              const uint64_t* __restrict__ offs, uint32_t n_paths, uint32_t regen_min,
                              uint32_t scatter_min, uint32_t* counter, uint32_t* sink) {
    constexpr bool TMA = MODE == 1;
    extern __shared__ uint32_t pad[];  // the render's shared-memory footprint (L1 split, blocks per SM)
    __shared__ alignas(128) uint32_t rbuf[TMA ? 128 : 1][16];
    __shared__ alignas(8) unsigned long long mbar[TMA ? 128 : 1];
    uint32_t phase = 0;
    if (TMA) {
        mbar_init(static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[threadIdx.x])), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncthreads();
    }
    enum : int { IDLE = 0, STEP = 1, WAIT = 2 };
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t chunk_next = 0, chunk_end = 0;  // warp-uniform
    bool exhausted = false;                  // warp-uniform
    int state = IDLE;
    uint32_t k = 0, n = 0;          // this lane's path: step k of n
    const uint32_t* cw = nullptr;   // its code words
    uint32_t idx = 0, word = 0, acc = 0;
    unsigned long long n_lanes = 0, n_lines = 0;  // MODE 4
    for (;;) {
        const unsigned idle = __ballot_sync(kFull, state == IDLE);
        const unsigned stepping = __ballot_sync(kFull, state == STEP);
        const unsigned waiting = __ballot_sync(kFull, state == WAIT);
        const bool open = !(exhausted && chunk_next >= chunk_end);
        if (!stepping && !waiting && !open) break;
        const uint32_t n_idle = __popc(idle);
        if (n_idle && open && (n_idle >= regen_min || !stepping)) {
            const uint32_t rank = __popc(idle & lt);
            uint32_t mine = kNone;
            const uint32_t avail = chunk_end - chunk_next;
            if (state == IDLE && rank < avail) mine = chunk_next + rank;
            const uint32_t used = min(avail, n_idle);
            chunk_next += used;
            if (n_idle > avail && !exhausted) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(counter, 64u);
                base = __shfl_sync(kFull, base, 0);
                if (base >= n_paths) {
                    exhausted = true;
                } else {
                    chunk_next = base;
                    chunk_end = min(base + 64u, n_paths);
                    const uint32_t avail2 = chunk_end - chunk_next;
                    if (state == IDLE && mine == kNone && rank - used < avail2) mine = chunk_next + (rank - used);
                    chunk_next += min(avail2, n_idle - used);
                }
            }
            if (mine != kNone) {
                k = 0;
                n = counts[mine];
                cw = codes + offs[mine];
                state = n ? STEP : IDLE;
                if (n) idx = start[mine];  // (a path without steps may start at kNone)
            }
        }
        if (waiting && (static_cast<uint32_t>(__popc(waiting)) >= scatter_min || !stepping))
            if (state == WAIT) state = k < n ? STEP : IDLE;
        const unsigned run = __ballot_sync(kFull, state == STEP);
        if (!run) continue;
        for (;;) {
            LeafRec rp;
            if (MODE == 2) {
                // a lane that is not stepping borrows its partner's index (no extra line)
                const bool st = state == STEP;
                const uint32_t pi = __shfl_xor_sync(kFull, idx, 1);
                const bool pst = __shfl_xor_sync(kFull, st ? 1u : 0u, 1) != 0;
                rp = load_leaf_pair(leaves, (!st && pst) ? pi : idx);
            }
            if (state == STEP) {
                if ((k & 7) == 0) word = cw[k >> 3];
                LeafRec r;
                if (MODE == 2) {
                    r = rp;
                } else if (MODE == 3) {
                    // what-if: a 32-B record (the first half only: the neighbour words)
                    uint32_t h[8];
                    ld256_na(leaves + idx, h);
#pragma unroll
                    for (int q = 0; q < 8; ++q) r.w[q] = h[q], r.w[8 + q] = h[q];
                } else if (TMA) {
                    const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[threadIdx.x]));
                    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&rbuf[threadIdx.x][0]));
                    bulk_load64(dst, leaves + idx, mb);
                    mbar_wait(mb, phase);
                    phase ^= 1u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(r.w[4 * q]), "=r"(r.w[4 * q + 1]), "=r"(r.w[4 * q + 2]), "=r"(r.w[4 * q + 3])
                                     : "r"(dst + 16 * q));
                } else {
                    r = load_leaf(leaves, idx);
                }
                if (MODE == 4) {  // what-if count: distinct 128-B record lines per warp load vs stepping lanes
                    const unsigned act = __activemask();
                    const unsigned peers = __match_any_sync(act, idx >> 1);
                    n_lanes += 1;
                    n_lines += (__ffs(peers) - 1) == lane ? 1u : 0u;
                }
                acc ^= r.w[5] ^ r.w[10] ^ r.w[15];
                const uint32_t code = (word >> (4 * (k & 7))) & 15u;
                ++k;
                // the next record's index comes out of this record (as in the render)
                if (code < 4) {
                    const uint32_t nx = nbr_leaf(sel4(r.w[0], r.w[1], r.w[2], r.w[3], static_cast<int>(code)));
                    if (MODE != 2 || nx != kNoLeaf) idx = nx;  // (MODE 2: idle lanes keep a valid index)
                }
                if (k >= n) state = IDLE;
                else if (code == 4) state = WAIT;  // collision: the scatter batch, then the same cell
            }
            if (__ballot_sync(kFull, state == STEP) != run) break;
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc + pad[0];  // keeps the loads alive
    if (MODE == 4) {
        atomicAdd(reinterpret_cast<unsigned long long*>(sink) + 2, n_lanes);
        atomicAdd(reinterpret_cast<unsigned long long*>(sink) + 3, n_lines);
    }
}

// words of 4-bit codes per path
__global__ void words_kernel(const uint32_t* in, uint64_t* out, uint64_t n) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = (in[i] + 7u) / 8u;
}

RenderParams params_of(const tv_render_config* r) {
    RenderParams p;
    p.spp = r->spp;
    p.max_bounces = r->max_bounces;
    p.seed = r->seed;
    p.g = r->hg_g;
    p.default_albedo = r->default_albedo;
    p.env[0] = r->environment[0], p.env[1] = r->environment[1], p.env[2] = r->environment[2];
    p.emission_scale = r->emission_scale;
    return p;
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

extern "C" int tv_diag_gather_ceiling(const tv_grid* h, const tv_camera* camera, const tv_render_config* cfg,
                                      int reps, double out[6]) {
#define CK(x, what)                                 \
    do {                                            \
        if (int rc_ = cuda_status((x), what)) return rc_; \
    } while (0)
    if (!h || !out) return set_error(TV_ERR_ARG, "null argument");
    int rc = validate_render_cfg(cfg);
    if (rc) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    const RenderParams rp = params_of(cfg);
    // one batch covering the whole frame, laid out exactly as render_frame's
    const uint32_t tiles_x = (static_cast<uint32_t>(cv.w) + 15) / 16, tiles_y = (static_cast<uint32_t>(cv.h) + 15) / 16;
    const uint64_t units = static_cast<uint64_t>(tiles_x) * tiles_y * 8;
    const uint64_t n_paths = units * 32 * static_cast<uint64_t>(rp.spp);
    if (n_paths >= (1ull << 31) || n_paths > kMaxBatchPaths)
        return set_error(TV_ERR_ARG, "diag: frame larger than one render batch");
    Batch B{};
    B.n_units = static_cast<uint32_t>(units);
    B.s0 = 0;
    B.ns = static_cast<uint32_t>(rp.spp);
    B.tiles_x = tiles_x, B.tiles_y = tiles_y;
    B.rank = 0, B.n_ranks = 1;
    B.n_paths = static_cast<uint32_t>(n_paths);
    B.first = 1;
    B.order = 1;
    B.tile_order = nullptr;
    Dev st, cells, counts, offs, seq, ctr, tmp;
    CK(cudaMalloc(&st.p, n_paths * sizeof(StartRec)), "diag alloc");
    CK(cudaMalloc(&cells.p, n_paths * 4), "diag alloc");
    CK(cudaMalloc(&counts.p, n_paths * 4), "diag alloc");
    CK(cudaMalloc(&offs.p, (n_paths + 1) * 8), "diag alloc");
    CK(cudaMalloc(&ctr.p, 256), "diag alloc");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.device);
    start_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n_paths + 255) / 256, sms * 16ull)), 256>>>(
        g.view, cv, rp, B, static_cast<StartRec*>(st.p), static_cast<uint32_t*>(cells.p));
    CK(cudaGetLastError(), "diag start");
    const unsigned rb = static_cast<unsigned>((n_paths + 127) / 128);
    record_kernel<<<rb, 128>>>(g.view, cv, rp, B, static_cast<const StartRec*>(st.p),
                               static_cast<const uint32_t*>(cells.p), static_cast<uint32_t*>(counts.p), nullptr,
                               nullptr);
    CK(cudaGetLastError(), "diag count");
    // offsets = exclusive scan of the counts (64-bit)
    CK(cudaMemset(offs.p, 0, 8), "diag");
    words_kernel<<<static_cast<unsigned>((n_paths + 255) / 256), 256>>>(static_cast<const uint32_t*>(counts.p),
                                                                        static_cast<uint64_t*>(offs.p) + 1, n_paths);
    {
        uint64_t* o1 = static_cast<uint64_t*>(offs.p) + 1;
        size_t tb = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tb, o1, o1, static_cast<int64_t>(n_paths)), "diag scan");
        CK(cudaMalloc(&tmp.p, tb), "diag alloc");
        CK(cub::DeviceScan::InclusiveSum(tmp.p, tb, o1, o1, static_cast<int64_t>(n_paths)), "diag scan");
    }
    // total steps (counts summed on the device)
    uint64_t total = 0;
    {
        Dev sum_d, tmp2;
        CK(cudaMalloc(&sum_d.p, 8), "diag alloc");
        auto in = static_cast<const uint32_t*>(counts.p);
        size_t tb = 0;
        CK(cub::DeviceReduce::Sum(nullptr, tb, in, static_cast<uint64_t*>(sum_d.p), static_cast<int64_t>(n_paths)),
           "diag sum");
        CK(cudaMalloc(&tmp2.p, tb), "diag alloc");
        CK(cub::DeviceReduce::Sum(tmp2.p, tb, in, static_cast<uint64_t*>(sum_d.p), static_cast<int64_t>(n_paths)),
           "diag sum");
        CK(cudaMemcpy(&total, sum_d.p, 8, cudaMemcpyDeviceToHost), "diag");
    }
    uint64_t words = 0;
    CK(cudaMemcpy(&words, static_cast<uint64_t*>(offs.p) + n_paths, 8, cudaMemcpyDeviceToHost), "diag");
    CK(cudaMalloc(&seq.p, std::max<uint64_t>(words, 1) * 4), "diag alloc (4 bits per tet step)");
    record_kernel<<<rb, 128>>>(g.view, cv, rp, B, static_cast<const StartRec*>(st.p),
                               static_cast<const uint32_t*>(cells.p), nullptr, static_cast<const uint64_t*>(offs.p),
                               static_cast<uint32_t*>(seq.p));
    CK(cudaGetLastError(), "diag record");
    CK(cudaDeviceSynchronize(), "diag record");
    // replay with the render's launch shape: 128 threads, its shared memory
    // per block and carveout (hence the same L1 and blocks per SM), then with
    // every warp slot of the SM filled
    size_t trace_smem = sizeof(FaceTables<kTraceThreads>) + sizeof(double) * 6 * kTraceThreads +
                        sizeof(unsigned long long) * kTraceThreads + 3 * sizeof(uint32_t) * kTraceThreads;
    // what-if knobs (dev): shared-memory footprint per block and carveout of the first replay
    if (const char* v = std::getenv("TV_DIAG_SMEM")) trace_smem = static_cast<size_t>(std::atol(v));
    const bool tma = std::getenv("TV_DIAG_TMA") && std::atoi(std::getenv("TV_DIAG_TMA")) > 0;
    const bool pair = std::getenv("TV_DIAG_PAIR") && std::atoi(std::getenv("TV_DIAG_PAIR")) > 0;
    const bool half = std::getenv("TV_DIAG_HALF") && std::atoi(std::getenv("TV_DIAG_HALF")) > 0;
    const bool count = std::getenv("TV_DIAG_COUNT") && std::atoi(std::getenv("TV_DIAG_COUNT")) > 0;
    auto rkf = tma ? replay_kernel<1>
                   : pair ? replay_kernel<2> : half ? replay_kernel<3> : count ? replay_kernel<4> : replay_kernel<0>;
    const void* rk = reinterpret_cast<const void*>(rkf);
    cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(trace_smem));
    const char* cv_env = std::getenv("TV_DIAG_CARVEOUT") ? std::getenv("TV_DIAG_CARVEOUT") : std::getenv("TV_CARVEOUT");
    cudaFuncSetAttribute(rk, cudaFuncAttributePreferredSharedMemoryCarveout, cv_env && *cv_env ? std::atoi(cv_env) : 72);
    auto env_u = [](const char* name, uint32_t d) {
        const char* v = std::getenv(name);
        return v && *v ? static_cast<uint32_t>(std::atoi(v)) : d;
    };
    const uint32_t regen_min = env_u("TV_REGEN_MIN", 5), scatter_min = env_u("TV_SCATTER_MIN", 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best[2] = {1e30, 1e30};
    int warps[2] = {0, 0};
    for (int mode = 0; mode < 2; ++mode) {
        const size_t smem = mode == 0 ? trace_smem : 0;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rk, 128, smem);
        if (const char* v = std::getenv("TV_DIAG_BLOCKS"))  // what-if: cap the resident blocks per SM
            if (mode == 0 && std::atoi(v) > 0) per_sm = std::min(per_sm, std::atoi(v));
        warps[mode] = per_sm * 4;
        const unsigned blocks = static_cast<unsigned>(sms * std::max(per_sm, 1));
        for (int r = 0; r < std::max(reps, 1); ++r) {
            CK(cudaMemset(ctr.p, 0, 256), "diag");
            cudaEventRecord(e0);
            rkf<<<blocks, 128, smem>>>(g.leaves, static_cast<const uint32_t*>(cells.p),
                                                 static_cast<const uint32_t*>(counts.p),
                                                 static_cast<const uint32_t*>(seq.p),
                                                 static_cast<const uint64_t*>(offs.p), B.n_paths, regen_min,
                                                 scatter_min, static_cast<uint32_t*>(ctr.p),
                                                 static_cast<uint32_t*>(ctr.p) + 32);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1), "diag replay");
            CK(cudaGetLastError(), "diag replay");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best[mode] = std::min(best[mode], static_cast<double>(ms));
            if (count && r == 0) {
                unsigned long long c[2];
                cudaMemcpy(c, static_cast<char*>(ctr.p) + 144, sizeof(c), cudaMemcpyDeviceToHost);
                std::fprintf(stderr, "tetvol_b200: diag replay (%s): %llu lane loads, %llu distinct record lines (%.3f)\n",
                             mode == 0 ? "trace shape" : "full occupancy", c[0], c[1],
                             c[0] ? static_cast<double>(c[1]) / c[0] : 0.0);
            }
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out[0] = total / (best[0] * 1e-3);
    out[1] = total / (best[1] * 1e-3);
    out[2] = static_cast<double>(total);
    out[3] = best[0];
    out[4] = 0.5;
    out[5] = warps[0];
    return TV_OK;
#undef CK
}
