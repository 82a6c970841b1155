// C ABI of tetvol_b200 (include/tetvol_b200.h). Host-side mirror of the
// reference API: argument validation with the reference's rules and messages,
// the pinhole camera precompute, device memory management and kernel launches.
// No exception crosses this boundary.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tv_trace.cuh"

namespace tvb {

namespace {
thread_local std::string g_err;
}

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TV_OK;
    if (e == cudaErrorMemoryAllocation)
        return set_error(TV_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    return set_error(TV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int use_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_error(TV_ERR_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) return set_error(TV_ERR_CUDA, "device index out of range");
    return cuda_status(cudaSetDevice(device), "cudaSetDevice");
}

namespace {

#define TV_CK(x, what)                                  \
    do {                                                \
        int rc_ = cuda_status((x), what);               \
        if (rc_) return rc_;                            \
    } while (0)

}  // namespace

// camera.cpp:12-45 (host; std::tan runs here, never on the device)
int host_camera(const tv_camera* c, CamView& v, d3 pn[5], double pd[5]) {
    if (!c) return set_error(TV_ERR_ARG, "camera is null");
    if (c->width < 1 || c->height < 1) return set_error(TV_ERR_CAMERA, "image dimensions must be positive");
    if (!(c->vfov_degrees > 0.0 && c->vfov_degrees < 180.0))
        return set_error(TV_ERR_CAMERA, "vfov must be in (0, 180) degrees");
    const d3 f = mk(c->forward[0], c->forward[1], c->forward[2]);
    const d3 up = mk(c->up[0], c->up[1], c->up[2]);
    if (std::sqrt(dot(f, f)) == 0.0) return set_error(TV_ERR_CAMERA, "forward vector must be nonzero");
    d3 fwd = f, upn = up;
    if (!c->basis_final) {
        fwd = normalize(f);
        const d3 upo = sub(up, mul(fwd, dot(up, fwd)));
        if (std::sqrt(dot(upo, upo)) < 1e-12)
            return set_error(TV_ERR_CAMERA, "up vector is parallel to the view direction");
        upn = normalize(upo);
    }
    const d3 right = cross(upn, fwd);
    const double kPi = 3.14159265358979323846;
    v.pos[0] = c->position[0], v.pos[1] = c->position[1], v.pos[2] = c->position[2];
    v.fwd[0] = fwd.x, v.fwd[1] = fwd.y, v.fwd[2] = fwd.z;
    v.up[0] = upn.x, v.up[1] = upn.y, v.up[2] = upn.z;
    v.right[0] = right.x, v.right[1] = right.y, v.right[2] = right.z;
    v.tan_half = std::tan(c->vfov_degrees * kPi / 360.0);
    v.aspect = static_cast<double>(c->width) / c->height;
    v.w = c->width;
    v.h = c->height;
    if (pn) {
        auto corner = [&](double u, double vv) {
            return normalize(add(add(fwd, mul(right, (2.0 * u - 1.0) * v.tan_half * v.aspect)),
                                 mul(upn, (1.0 - 2.0 * vv) * v.tan_half)));
        };
        const d3 tl = corner(0, 0), tr = corner(1, 0), bl = corner(0, 1), br = corner(1, 1);
        const d3 pos = mk(v.pos[0], v.pos[1], v.pos[2]);
        pn[0] = fwd;
        pd[0] = dot(fwd, pos) + 1e-4;
        const d3 pairs[4][2] = {{tl, bl}, {br, tr}, {tr, tl}, {bl, br}};
        for (int i = 0; i < 4; ++i) {
            d3 n = normalize(cross(pairs[i][0], pairs[i][1]));
            if (dot(n, fwd) < 0.0) n = mk(-n.x, -n.y, -n.z);
            pn[i + 1] = n;
            pd[i + 1] = dot(n, pos);
        }
    }
    return TV_OK;
}

namespace {

// RenderConfig::validate (tracer.cpp:131-141)
int validate_render(const tv_render_config* r) {
    if (!r) return set_error(TV_ERR_ARG, "render config is null");
    if (r->spp < 1) return set_error(TV_ERR_CONFIG, "spp must be at least 1");
    if (r->max_bounces < 1) return set_error(TV_ERR_CONFIG, "maxBounces must be at least 1");
    if (!(r->hg_g > -1.0 && r->hg_g < 1.0)) return set_error(TV_ERR_CONFIG, "phase anisotropy g must be in (-1, 1)");
    if (!(r->default_albedo >= 0.0 && r->default_albedo <= 1.0))
        return set_error(TV_ERR_CONFIG, "albedo must be in [0, 1]");
    if (r->environment[0] < 0.0 || r->environment[1] < 0.0 || r->environment[2] < 0.0)
        return set_error(TV_ERR_CONFIG, "environment radiance must be non-negative");
    if (r->emission_scale < 0.0) return set_error(TV_ERR_CONFIG, "emissionScale must be non-negative");
    if (!(r->exposure > 0.0)) return set_error(TV_ERR_CONFIG, "exposure must be positive");
    if (!(r->gamma > 0.0)) return set_error(TV_ERR_CONFIG, "gamma must be positive");
    return TV_OK;
}

}  // namespace

int validate_render_cfg(const tv_render_config* r) { return validate_render(r); }

namespace {

RenderParams make_params(const tv_render_config* r) {
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

// Per-device workspace reused across frames (no cudaMalloc in the per-frame
// path): the per-path buffers of a batch (start records, entry cells,
// radiance), the accumulators tv_render copies back, the queue counter, and a
// stream + events.
//
// Stream ordering. The render entry points are asynchronous on the caller's
// stream and every frame on a device shares this workspace, so frames are
// chained through `idle`: render_frame makes its stream wait for the previous
// frame's `idle` record before touching the workspace and records `idle` on
// its own stream after its last kernel. Frames issued on different streams
// (or tv_render on the workspace's own stream after an asynchronous
// tv_render_tiles) therefore run one after another on the device, never on
// the same buffers at once. Host-side buffer growth first waits for `idle`.
struct TileOrderKey {
    uint32_t k[4];
    bool operator<(const TileOrderKey& o) const { return std::lexicographical_compare(k, k + 4, o.k, o.k + 4); }
};
struct Workspace {
    std::mutex mu;
    void* paths = nullptr;
    size_t path_bytes = 0;
    void* out = nullptr;
    size_t out_bytes = 0;
    uint32_t* counter = nullptr;
    void* cold = nullptr;  // trace kernel cold path state, kColdBytes per resident thread
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t idle = nullptr;  // recorded after the last frame's last kernel
    int trace_blocks = 0, sms = 0;
    TraceFn trace = nullptr;
    int trace_threads = kTraceThreads;
    TraceFn trace_hot = nullptr;  // the same kernel on the grid's 32-B hot records (DeviceGrid::hot)
    int trace_blocks_hot = 0;
    uint32_t regen_min = 8, scatter_min = 8, order = 0;
    uint32_t tail_chunk = kChunk, tail_warps_x = 2;  // tail claims: size, and the zone in chunks per warp
    std::vector<cudaEvent_t> tev;  // per-batch kernel boundaries of the last frame (4 per batch)
    int n_timed = 0, n_launches = 0;
    // per (tiles_x, tiles_y, rank, n_ranks): that rank's tiles in processing
    // order (see tile_order_for); written once, never overwritten, so frames
    // still in flight keep reading a valid table
    struct TileTables {
        uint32_t* order = nullptr;  // this rank's tiles in processing order
        uint32_t* cost = nullptr;   // TV_TILE_ORDER=3: tet steps per list position in the last frame
    };
    std::map<TileOrderKey, TileTables> tile_orders;
    // tv_render_multi (one call at a time, g_multi_mu): the frame's accumulators
    // when this is the first grid's device, else this rank's stats words (and
    // its private frame when it cannot reach the first device)
    void* multi = nullptr;
    size_t multi_bytes = 0;
    int tile_mode = 1;
    double tile_radius = 0.8;  // outer tiles: beyond this fraction of the inscribed circle
};
Workspace g_ws[64];
std::mutex g_multi_mu;
constexpr uint32_t kSortTiles = 4096;  // TV_TILE_ORDER=3 sorts at most this many tiles per rank

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// Processing order of a rank's 16x16 tiles (the interleaved assignment t = rank
// mod n_ranks is unchanged): raster order, except that the tiles outside a
// circle around the image centre (TV_TILE_RADIUS_PCT of the inscribed circle)
// come last. Central tiles carry the long paths through the medium, so the
// persistent trace kernel's last chunks are short paths and its tail shrinks.
// Only the schedule changes: every pixel still accumulates its samples in
// order. TV_TILE_ORDER: 0 raster always, 1 (default) from 4 ranks up, 2 always,
// 3 cost-ordered from 4 ranks up, 4 cost-ordered always: the trace kernel adds
// every path's tet steps to its tile's counter, and after each frame
// tile_sort_kernel orders this rank's tiles by the last frame's cost, longest
// first (ties by tile id), for the next frame; the first frame uses the order
// of mode 2.
int tile_order_for(Workspace& w, uint32_t tiles_x, uint32_t tiles_y, int rank, int n_ranks, cudaStream_t st,
                   const uint32_t*& out, uint32_t** cost = nullptr) {
    out = nullptr;
    if (cost) *cost = nullptr;
    // measured on B200 (tools/rank_share.py, C2): the reordering shortens the
    // per-rank tail at 4 and 8 ranks (8.89 vs 9.13 ms per rank at 8) but costs
    // L2 locality on a full frame (+0.3 % at 1 and 2 ranks)
    if (w.tile_mode == 0 || ((w.tile_mode == 1 || w.tile_mode == 3) && n_ranks < 4)) return TV_OK;
    const bool by_cost = w.tile_mode >= 3;
    const TileOrderKey key{{tiles_x, tiles_y, static_cast<uint32_t>(rank), static_cast<uint32_t>(n_ranks)}};
    auto it = w.tile_orders.find(key);
    if (it != w.tile_orders.end()) {
        out = it->second.order;
        if (cost) *cost = it->second.cost;
        return TV_OK;
    }
    std::vector<uint32_t> tl;
    for (uint32_t t = static_cast<uint32_t>(rank); t < tiles_x * tiles_y; t += static_cast<uint32_t>(n_ranks))
        tl.push_back(t);
    if (tl.empty()) return TV_OK;
    const double cx = 0.5 * tiles_x, cy = 0.5 * tiles_y;
    const double rr = 0.25 * w.tile_radius * w.tile_radius * std::min(tiles_x, tiles_y) * std::min(tiles_x, tiles_y);
    auto outer = [&](uint32_t t) {
        const double dx = (t % tiles_x) + 0.5 - cx, dy = (t / tiles_x) + 0.5 - cy;
        return dx * dx + dy * dy > rr;
    };
    // raster order inside (L2 locality between neighbouring tiles), the outer
    // tiles last
    std::stable_partition(tl.begin(), tl.end(), [&](uint32_t t) { return !outer(t); });
    if (w.tile_orders.size() >= 64) {  // bounded cache: drop the tables once nothing can read them
        TV_CK(cudaEventSynchronize(w.idle), "tile order sync");
        for (auto& kv : w.tile_orders) cudaFree(kv.second.order), cudaFree(kv.second.cost);
        w.tile_orders.clear();
    }
    Workspace::TileTables tt;
    TV_CK(cudaMalloc(&tt.order, tl.size() * sizeof(uint32_t)), "tile order alloc");
    // stream-ordered upload (a pageable source is staged before the call returns)
    cudaError_t e = cudaMemcpyAsync(tt.order, tl.data(), tl.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && by_cost && tl.size() <= kSortTiles) {
        e = cudaMalloc(&tt.cost, tl.size() * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMemsetAsync(tt.cost, 0, tl.size() * sizeof(uint32_t), st);
    }
    if (e != cudaSuccess) {
        cudaFree(tt.order), cudaFree(tt.cost);
        return cuda_status(e, "tile order tables");
    }
    w.tile_orders.emplace(key, tt);
    out = tt.order;
    if (cost) *cost = tt.cost;
    return TV_OK;
}

// TV_TILE_ORDER=3: this rank's tiles by the last frame's cost (tet steps),
// descending, ties by tile id; resets the costs. One block, n <= kSortTiles.
__global__ void tile_sort_kernel(uint32_t* order, uint32_t* cost, uint32_t n) {
    __shared__ uint32_t sc[kSortTiles], st[kSortTiles];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sc[i] = cost[i], st[i] = order[i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint32_t r = 0;
        for (uint32_t j = 0; j < n; ++j) r += (sc[j] > sc[i]) || (sc[j] == sc[i] && st[j] < st[i]);
        order[r] = st[i];
        cost[i] = 0;
    }
}

int grow(void*& p, size_t& have, size_t need, cudaEvent_t idle) {
    if (have >= need) return TV_OK;
    if (idle) TV_CK(cudaEventSynchronize(idle), "workspace sync");  // frames in flight may still read p
    cudaFree(p);
    p = nullptr;
    have = 0;
    TV_CK(cudaMalloc(&p, need), "workspace alloc");
    have = need;
    return TV_OK;
}

int workspace(int device, Workspace*& out) {
    if (device < 0 || device >= 64) return set_error(TV_ERR_ARG, "device index out of range");
    Workspace& w = g_ws[device];
    if (!w.stream) {
        TV_CK(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking), "stream create");
        TV_CK(cudaEventCreate(&w.ev0), "event create");
        TV_CK(cudaEventCreate(&w.ev1), "event create");
        TV_CK(cudaEventCreateWithFlags(&w.idle, cudaEventDisableTiming), "event create");
        TV_CK(cudaEventRecord(w.idle, w.stream), "event");
        TV_CK(cudaMalloc(&w.counter, 256), "counter alloc");
        // tuning knobs (defaults are the measured best on B200)
        const int maxreg = env_int("TV_TRACE_MAXREG", 72);
        w.trace = trace_variant(maxreg, env_int("TV_TRACE_THREADS", 128), w.trace_threads);
        w.trace_hot = trace_variant(maxreg, env_int("TV_TRACE_THREADS", 128), w.trace_threads, true);
        w.regen_min = static_cast<uint32_t>(env_int("TV_REGEN_MIN", 5));
        w.scatter_min = static_cast<uint32_t>(env_int("TV_SCATTER_MIN", 2));
        w.order = static_cast<uint32_t>(env_int("TV_ORDER", 1));
        w.tail_chunk = static_cast<uint32_t>(std::min(std::max(env_int("TV_TAIL_CHUNK", 64), 1), 64));
        w.tail_warps_x = static_cast<uint32_t>(std::max(env_int("TV_TAIL_ZONE", 2), 0));
        w.tile_mode = env_int("TV_TILE_ORDER", 1);
        w.tile_radius = env_int("TV_TILE_RADIUS_PCT", 80) / 100.0;
        int per_sm = 1, per_sm_hot = 1;
        cudaFuncSetAttribute(reinterpret_cast<const void*>(w.trace), cudaFuncAttributePreferredSharedMemoryCarveout,
                             env_int("TV_CARVEOUT", 72));
        cudaFuncSetAttribute(reinterpret_cast<const void*>(w.trace_hot), cudaFuncAttributePreferredSharedMemoryCarveout,
                             env_int("TV_CARVEOUT", 72));
        cudaDeviceGetAttribute(&w.sms, cudaDevAttrMultiProcessorCount, device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(w.trace),
                                                      w.trace_threads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_hot, reinterpret_cast<const void*>(w.trace_hot),
                                                      w.trace_threads, 0);
        w.trace_blocks = w.sms * (per_sm < 1 ? 1 : per_sm);
        w.trace_blocks_hot = w.sms * (per_sm_hot < 1 ? 1 : per_sm_hot);
        if (TV_COLD_GLOBAL)
            TV_CK(cudaMalloc(&w.cold, static_cast<size_t>(w.trace_blocks) * w.trace_threads * kColdBytes),
                  "cold state alloc");
        if (env_int("TV_VERBOSE", 0))
            std::fprintf(stderr, "tetvol_b200: trace kernel maxreg=%d threads=%d, %d blocks/SM resident, %d blocks\n",
                         maxreg, w.trace_threads, per_sm, w.trace_blocks);
    }
    out = &w;
    return TV_OK;
}

// Renders this rank's tiles of one frame: per batch of samples, start ->
// trace -> accumulate (see tv_trace.cu). Asynchronous on `st`.
// Renders samples [first_sample, first_sample + spp) of this rank's pixels and
// adds them to `out` in sample order (first_sample == 0 initialises it), so
// frames that cover [0, N) leave exactly the framebuffer of one N-spp render.
int render_frame(const DeviceGrid& g, const CamView& cv, const RenderParams& rp, int rank, int n_ranks,
                 RenderOut out, Workspace& w, cudaStream_t st, uint32_t first_sample = 0) {
    const uint32_t tiles_x = (static_cast<uint32_t>(cv.w) + 15) / 16;
    const uint32_t tiles_y = (static_cast<uint32_t>(cv.h) + 15) / 16;
    const uint64_t tiles = static_cast<uint64_t>(tiles_x) * tiles_y;
    const uint64_t mine = tiles > static_cast<uint64_t>(rank) ? (tiles - rank + n_ranks - 1) / n_ranks : 0;
    const uint64_t units = mine * 8;
    w.n_timed = 0;
    w.n_launches = 0;
    if (units == 0) return TV_OK;
    // the previous frame on this device (any stream) is done with the workspace
    TV_CK(cudaStreamWaitEvent(st, w.idle, 0), "wait workspace");
    const uint32_t* tile_order = nullptr;
    uint32_t* tile_cost = nullptr;
    if (int rc = tile_order_for(w, tiles_x, tiles_y, rank, n_ranks, st, tile_order, &tile_cost)) return rc;
    uint64_t ns = std::max<uint64_t>(1, kMaxBatchPaths / (units * 32));
    ns = std::min<uint64_t>(ns, static_cast<uint64_t>(rp.spp));
    if (units * 32 * ns >= (1ull << 31)) return set_error(TV_ERR_ARG, "frame too large for one batch");
    const uint64_t max_paths = units * 32 * ns;
    const size_t need = max_paths * (sizeof(StartRec) + sizeof(uint32_t) + 3 * sizeof(double)) + 256;
    int rc = grow(w.paths, w.path_bytes, need, w.idle);
    if (rc) return rc;
    char* base = static_cast<char*>(w.paths);
    StartRec* st_rec = reinterpret_cast<StartRec*>(base);
    double* rad = reinterpret_cast<double*>(base + max_paths * sizeof(StartRec));
    uint32_t* cells = reinterpret_cast<uint32_t*>(base + max_paths * (sizeof(StartRec) + 3 * sizeof(double)));
    const uint64_t n_batches = (static_cast<uint64_t>(rp.spp) + ns - 1) / ns;
    while (w.tev.size() < 4 * n_batches) {
        cudaEvent_t e;
        TV_CK(cudaEventCreate(&e), "event create");
        w.tev.push_back(e);
    }
    for (uint64_t s0 = 0; s0 < static_cast<uint64_t>(rp.spp); s0 += ns) {
        cudaEvent_t* ev = &w.tev[4 * w.n_timed];
        ++w.n_timed;
        w.n_launches += 3;
        Batch B;
        B.n_units = static_cast<uint32_t>(units);
        B.s0 = first_sample + static_cast<uint32_t>(s0);
        B.ns = static_cast<uint32_t>(std::min<uint64_t>(ns, rp.spp - s0));
        B.tiles_x = tiles_x;
        B.tiles_y = tiles_y;
        B.rank = rank;
        B.n_ranks = n_ranks;
        B.n_paths = static_cast<uint32_t>(units * 32 * B.ns);
        B.first = s0 == 0 && first_sample == 0 ? 1u : 0u;
        B.regen_min = w.regen_min;
        B.scatter_min = w.scatter_min;
        B.order = w.order;
        B.tile_order = tile_order;
        B.tile_cost = tile_cost;
        B.cold = w.cold;
        {
            // the last tail_warps_x chunks per resident warp are claimed tail_chunk at a time
            const uint64_t zone = static_cast<uint64_t>(g.view.hot ? w.trace_blocks_hot : w.trace_blocks) *
                                  (w.trace_threads / 32) * kChunk * w.tail_warps_x;
            B.tail_chunk = w.tail_chunk;
            B.tail_from = B.n_paths > zone ? static_cast<uint32_t>(B.n_paths - zone) : 0u;
        }
        const unsigned sb = static_cast<unsigned>(std::min<uint64_t>((B.n_paths + 255) / 256, w.sms * 16ull));
        TV_CK(cudaEventRecord(ev[0], st), "event");
        start_kernel<<<sb, 256, 0, st>>>(g.view, cv, rp, B, st_rec, cells);
        TV_CK(cudaGetLastError(), "start_kernel launch");
        TV_CK(cudaMemsetAsync(w.counter, 0, sizeof(uint32_t), st), "memset counter");
        TV_CK(cudaEventRecord(ev[1], st), "event");
        if (g.view.hot)  // one 32-B load per step (HotRec); else the 64-B LeafRecs
            w.trace_hot<<<w.trace_blocks_hot, w.trace_threads, 0, st>>>(g.view, cv, rp, B, st_rec, cells, rad,
                                                                      out.stats, w.counter);
        else
            w.trace<<<w.trace_blocks, w.trace_threads, 0, st>>>(g.view, cv, rp, B, st_rec, cells, rad, out.stats,
                                                              w.counter);
        TV_CK(cudaGetLastError(), "trace_kernel launch");
        TV_CK(cudaEventRecord(ev[2], st), "event");
        const unsigned ab = static_cast<unsigned>(std::min<uint64_t>((units * 32 + 127) / 128, w.sms * 16ull));
        accum_kernel<<<ab, 128, 0, st>>>(B, cv, cells, rad, out);
        TV_CK(cudaGetLastError(), "accum_kernel launch");
        TV_CK(cudaEventRecord(ev[3], st), "event");
    }
    if (tile_cost) {  // the next frame's order, after this frame's last accumulate read the current one
        tile_sort_kernel<<<1, 1024, 0, st>>>(const_cast<uint32_t*>(tile_order), tile_cost,
                                              static_cast<uint32_t>(mine));
        TV_CK(cudaGetLastError(), "tile_sort_kernel launch");
        ++w.n_launches;
    }
    TV_CK(cudaEventRecord(w.idle, st), "event");
    return TV_OK;
}

// 1 when any output buffer lives on another device (mapped with tv_ipc_open)
int peer_outputs(int device, const void* a, const void* b, const void* c) {
    for (const void* p : {a, b, c}) {
        if (!p) continue;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (at.type == cudaMemoryTypeDevice && at.device != device) return 1;
    }
    return 0;
}

// Device time of the last frame's kernels on this device (sums over batches):
// out[0] start, out[1] trace, out[2] accumulate (ms); out[3] kernel launches.
int last_frame_timing(int device, double* out) {
    Workspace* w;
    int rc = workspace(device, w);
    if (rc) return rc;
    out[0] = out[1] = out[2] = 0.0;
    out[3] = w->n_launches;
    for (int b = 0; b < w->n_timed; ++b) {
        cudaEvent_t* ev = &w->tev[4 * b];
        TV_CK(cudaEventSynchronize(ev[3]), "timing sync");
        for (int k = 0; k < 3; ++k) {
            float ms = 0.f;
            TV_CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]), "elapsed");
            out[k] += ms;
        }
    }
    return TV_OK;
}

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

const char* tv_last_error(void) { return g_err.c_str(); }
const char* tv_version(void) { return "tetvol_b200 0.1 (sm_100a)"; }

int tv_device_count(int* out) {
    if (!out) return set_error(TV_ERR_ARG, "out is null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    *out = e == cudaSuccess ? n : 0;
    return TV_OK;
}

int tv_grid_upload(const tv_vertex* vertices, uint64_t n_vertices, const tv_tet* tets, uint64_t n_tets,
                   const uint32_t roots[24], int32_t max_level, int device, tv_grid** out) {
    if (!vertices || !tets || !roots || !out) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    if (n_tets < 24 || n_tets >= (1ull << 31)) return set_error(TV_ERR_GRID, "bad tet count");
    if (n_vertices < 8 || n_vertices > (1ull << 32)) return set_error(TV_ERR_GRID, "bad vertex count");
    if (max_level < 1 || max_level > 48) return set_error(TV_ERR_GRID, "max_level out of range");
    // Structural checks the kernels rely on (the reference's load_grid makes
    // the same range checks, builder.cpp:253-285).
    uint64_t leaves = 0;
    for (uint64_t t = 0; t < n_tets; ++t) {
        const tv_tet& tt = tets[t];
        for (int k = 0; k < 4; ++k) {
            if (tt.verts[k] >= n_vertices) return set_error(TV_ERR_GRID, "vertex id out of range");
            if (tt.neighbors[k] != TV_NO_TET && tt.neighbors[k] >= n_tets)
                return set_error(TV_ERR_GRID, "neighbor id out of range");
            if (tt.normal_ids[k] >= 18) return set_error(TV_ERR_GRID, "face normal id out of range");
        }
        const bool leaf = tt.children[0] == TV_NO_TET;
        if (!leaf && (tt.children[0] >= n_tets || tt.children[1] >= n_tets))
            return set_error(TV_ERR_GRID, "child id out of range");
        leaves += leaf;
    }
    for (int r = 0; r < 24; ++r)
        if (roots[r] >= n_tets) return set_error(TV_ERR_GRID, "root id out of range");
    int rc = use_device(device);
    if (rc) return rc;

    auto h = std::make_unique<tv_grid>();
    DeviceGrid& g = h->g;
    g.device = device;
    g.n_vertices = n_vertices;
    g.n_tets = n_tets;
    g.n_leaves = leaves;
    g.n_internal = n_tets - leaves;
    g.max_level = max_level;
    std::memcpy(g.roots, roots, sizeof(g.roots));
    std::vector<uint4> vq(n_vertices);
    for (uint64_t i = 0; i < n_vertices; ++i) vq[i] = make_uint4(vertices[i].q[0], vertices[i].q[1], vertices[i].q[2], 0);
    cudaError_t e = cudaMalloc(&g.verts, n_vertices * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMalloc(&g.tets, n_tets * sizeof(tv_tet));
    if (e != cudaSuccess) {
        free_grid(g);
        return cuda_status(e, "grid alloc");
    }
    g.bytes = n_vertices * sizeof(uint4) + n_tets * sizeof(tv_tet);
    e = cudaMemcpy(g.verts, vq.data(), n_vertices * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g.tets, tets, n_tets * sizeof(tv_tet), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        free_grid(g);
        return cuda_status(e, "grid upload");
    }
    rc = finalize_grid(g, nullptr);
    if (rc) {
        free_grid(g);
        return rc;
    }
    *out = h.release();
    return TV_OK;
}

int tv_grid_download(const tv_grid* h, tv_vertex* vertices, tv_tet* tets, uint32_t roots[24]) {
    if (!h) return set_error(TV_ERR_ARG, "grid is null");
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    if (vertices) {
        std::vector<uint4> vq(g.n_vertices);
        TV_CK(cudaMemcpy(vq.data(), g.verts, g.n_vertices * sizeof(uint4), cudaMemcpyDeviceToHost), "download");
        for (uint64_t i = 0; i < g.n_vertices; ++i) {
            vertices[i].q[0] = vq[i].x;
            vertices[i].q[1] = vq[i].y;
            vertices[i].q[2] = vq[i].z;
        }
    }
    if (tets) TV_CK(cudaMemcpy(tets, g.tets, g.n_tets * sizeof(tv_tet), cudaMemcpyDeviceToHost), "download");
    if (roots) std::memcpy(roots, g.roots, sizeof(g.roots));
    return TV_OK;
}

int tv_grid_get_info(const tv_grid* h, tv_grid_info* out) {
    if (!h || !out) return set_error(TV_ERR_ARG, "null argument");
    const DeviceGrid& g = h->g;
    out->n_vertices = g.n_vertices;
    out->n_tets = g.n_tets;
    out->n_leaves = g.n_leaves;
    out->n_internal = g.n_internal;
    out->max_level = g.max_level;
    out->max_depth = g.max_depth;
    out->device = g.device;
    out->pad = 0;
    out->device_bytes = g.bytes;
    return TV_OK;
}

void tv_grid_free(tv_grid* h) {
    if (!h) return;
    cudaSetDevice(h->g.device);
    free_grid(h->g);
    delete h;
}

int tv_render(const tv_grid* h, const tv_camera* camera, const tv_render_config* cfg, tv_framebuffer* out,
              tv_render_stats* stats) {
    if (!h) return set_error(TV_ERR_ARG, "grid is null");
    int rc = validate_render(cfg);
    if (rc) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    const uint64_t npx = static_cast<uint64_t>(cv.w) * cv.h;
    Workspace* w;
    if ((rc = workspace(g.device, w))) return rc;
    std::lock_guard<std::mutex> lk(w->mu);
    const size_t bytes = npx * (3 * sizeof(double) * 2 + sizeof(uint32_t)) + 4 * sizeof(uint64_t) + 256;
    if ((rc = grow(w->out, w->out_bytes, bytes, w->idle))) return rc;
    Workspace* s = w;
    char* base = static_cast<char*>(w->out);
    double* sum = reinterpret_cast<double*>(base);
    double* sum_sq = sum + 3 * npx;
    uint32_t* counts = reinterpret_cast<uint32_t*>(sum_sq + 3 * npx);
    uint64_t* st = reinterpret_cast<uint64_t*>(base + ((npx * 48 + npx * 4 + 63) & ~static_cast<size_t>(63)));
    RenderOut ro{sum, sum_sq, counts, st};
    TV_CK(cudaMemsetAsync(st, 0, 3 * sizeof(uint64_t), s->stream), "memset stats");
    TV_CK(cudaEventRecord(s->ev0, s->stream), "event");
    if ((rc = render_frame(g, cv, make_params(cfg), 0, 1, ro, *w, s->stream))) return rc;
    TV_CK(cudaEventRecord(s->ev1, s->stream), "event");
    if (out && out->sum)
        TV_CK(cudaMemcpyAsync(out->sum, sum, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost, s->stream), "D2H");
    if (out && out->sum_sq)
        TV_CK(cudaMemcpyAsync(out->sum_sq, sum_sq, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost, s->stream),
              "D2H");
    if (out && out->sample_counts)
        TV_CK(cudaMemcpyAsync(out->sample_counts, counts, npx * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream),
              "D2H");
    uint64_t hst[3] = {0, 0, 0};
    TV_CK(cudaMemcpyAsync(hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s->stream), "D2H");
    TV_CK(cudaStreamSynchronize(s->stream), "render");
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, s->ev0, s->ev1);
        stats->cells_visited = hst[0];
        stats->paths_traced = npx * static_cast<uint64_t>(cfg->spp);
        stats->degenerate_paths = hst[2];
        stats->seconds = ms * 1e-3;
    }
    return TV_OK;
}

int tv_render_tiles(const tv_grid* h, const tv_camera* camera, const tv_render_config* cfg, int32_t rank,
                    int32_t n_ranks, double* sum_dev, double* sum_sq_dev, uint32_t* counts_dev, uint64_t* stats_dev,
                    void* stream) {
    if (!h) return set_error(TV_ERR_ARG, "grid is null");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return set_error(TV_ERR_ARG, "bad rank / n_ranks");
    int rc = validate_render(cfg);
    if (rc) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    Workspace* w;
    if ((rc = workspace(g.device, w))) return rc;
    std::lock_guard<std::mutex> lk(w->mu);
    RenderOut ro{sum_dev, sum_sq_dev, counts_dev, stats_dev, peer_outputs(g.device, sum_dev, sum_sq_dev, counts_dev)};
    return render_frame(g, cv, make_params(cfg), rank, n_ranks, ro, *w, static_cast<cudaStream_t>(stream));
}

int tv_render_accumulate(const tv_grid* h, const tv_camera* camera, const tv_render_config* cfg,
                         int32_t first_sample, int32_t rank, int32_t n_ranks, double* sum_dev, double* sum_sq_dev,
                         uint32_t* counts_dev, uint64_t* stats_dev, void* stream) {
    if (!h) return set_error(TV_ERR_ARG, "grid is null");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return set_error(TV_ERR_ARG, "bad rank / n_ranks");
    if (first_sample < 0) return set_error(TV_ERR_ARG, "first_sample must be >= 0");
    int rc = validate_render(cfg);
    if (rc) return rc;
    if (static_cast<int64_t>(first_sample) + cfg->spp > 0xffffffffll) return set_error(TV_ERR_ARG, "sample index overflow");
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    Workspace* w;
    if ((rc = workspace(g.device, w))) return rc;
    std::lock_guard<std::mutex> lk(w->mu);
    RenderOut ro{sum_dev, sum_sq_dev, counts_dev, stats_dev, peer_outputs(g.device, sum_dev, sum_sq_dev, counts_dev)};
    return render_frame(g, cv, make_params(cfg), rank, n_ranks, ro, *w, static_cast<cudaStream_t>(stream),
                        static_cast<uint32_t>(first_sample));
}

// One process, several GPUs (SURVEY.md 8(b) tv_render_multi): rank r renders
// the interleaved 16x16 tiles t with t % n == r on grids[r]'s device, one host
// thread per rank. Where the device can reach the first grid's device directly
// (P2P over NVLink), the rank's accumulate kernel stores its pixels straight
// into the frame on that device (the gather fused into the render, as
// tv_render_tiles with peer outputs); otherwise the rank renders a private
// full frame and its tiles are merged on the host. Every pixel is rendered by
// one rank with the reference's per-pixel sample order, so the framebuffer is
// bit-identical to tv_render's for any n (two ranks on one device serialise on
// its stream and stay correct).
int tv_render_multi(const tv_grid* const* grids, int32_t n, const tv_camera* camera, const tv_render_config* cfg,
                    tv_framebuffer* out, tv_render_stats* stats) {
    if (!grids || n < 1) return set_error(TV_ERR_ARG, "need at least one grid");
    for (int r = 0; r < n; ++r)
        if (!grids[r]) return set_error(TV_ERR_ARG, "grid is null");
    int rc = validate_render(cfg);
    if (rc) return rc;
    CamView cv;
    if ((rc = host_camera(camera, cv, nullptr, nullptr))) return rc;
    const int dev0 = grids[0]->g.device;
    const uint64_t npx = static_cast<uint64_t>(cv.w) * cv.h;
    const size_t frame_bytes = npx * (6 * sizeof(double) + sizeof(uint32_t));
    const size_t stats_off = (frame_bytes + 255) & ~static_cast<size_t>(255);
    const size_t bytes = stats_off + 32 * static_cast<size_t>(n);  // + 4 stats words per rank
    const RenderParams rp = make_params(cfg);
    const uint32_t tiles_x = (static_cast<uint32_t>(cv.w) + 15) / 16, tiles_y = (static_cast<uint32_t>(cv.h) + 15) / 16;

    if ((rc = use_device(dev0))) return rc;
    Workspace* w0;
    if ((rc = workspace(dev0, w0))) return rc;
    std::lock_guard<std::mutex> lk0(g_multi_mu);  // one multi-GPU frame at a time (the multi buffers)
    if ((rc = grow(w0->multi, w0->multi_bytes, bytes, w0->idle))) return rc;
    char* f0 = static_cast<char*>(w0->multi);
    // which ranks write into dev0's frame: dev0 itself, and devices with peer access to it
    std::vector<int> direct(n, 1);
    const bool peer_ok = env_int("TV_MULTI_PEER", 1) != 0;  // 0 (tests): every rank > 0 takes the host merge
    for (int r = 0; r < n; ++r) {
        const int d = grids[r]->g.device;
        if (r > 0 && !peer_ok) {
            direct[r] = 0;
            continue;
        }
        if (d == dev0) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, d, dev0) != cudaSuccess || !ok) {
            cudaGetLastError();
            direct[r] = 0;
            continue;
        }
        if ((rc = use_device(d))) return rc;
        const cudaError_t e = cudaDeviceEnablePeerAccess(dev0, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_status(e, "peer access");
    }
    std::vector<int> rcs(n, TV_OK);
    std::vector<std::string> msgs(n);
    std::vector<std::array<uint64_t, 3>> hst(n, std::array<uint64_t, 3>{0, 0, 0});
    std::vector<std::vector<char>> priv(n);  // host copies of the private frames
    std::vector<double> ms(n, 0.0);
    auto rank_fn = [&](int r) {
        auto fail = [&](int code) {
            rcs[r] = code;
            msgs[r] = g_err;
        };
        const DeviceGrid& g = grids[r]->g;
        int c = use_device(g.device);
        if (c) return fail(c);
        Workspace* w;
        if ((c = workspace(g.device, w))) return fail(c);
        std::lock_guard<std::mutex> lk(w->mu);  // ranks sharing a device run one after the other
        // this rank's stats words: in the frame's block on dev0, else in its own device's
        uint64_t* st = reinterpret_cast<uint64_t*>(f0 + stats_off) + 4 * r;
        if (g.device != dev0) {
            if ((c = grow(w->multi, w->multi_bytes, 256, w->idle))) return fail(c);
            st = static_cast<uint64_t*>(w->multi);
        }
        // a rank that cannot write dev0's frame renders a private one (merged on the host)
        char* frame = f0;
        struct Priv {
            void* p = nullptr;
            ~Priv() { cudaFree(p); }
        } pv;
        if (!direct[r]) {
            const cudaError_t e = cudaMalloc(&pv.p, frame_bytes);
            if (e != cudaSuccess) return fail(cuda_status(e, "private frame"));
            frame = static_cast<char*>(pv.p);
        }
        double* sum = reinterpret_cast<double*>(frame);
        RenderOut ro{sum, sum + 3 * npx, reinterpret_cast<uint32_t*>(sum + 6 * npx), st,
                     g.device != dev0 && direct[r] ? 1 : 0};
        cudaStream_t sm = w->stream;
        cudaError_t e = cudaMemsetAsync(st, 0, 3 * sizeof(uint64_t), sm);
        if (e == cudaSuccess) e = cudaEventRecord(w->ev0, sm);
        if (e != cudaSuccess) return fail(cuda_status(e, "multi frame start"));
        if ((c = render_frame(g, cv, rp, r, n, ro, *w, sm))) return fail(c);
        e = cudaEventRecord(w->ev1, sm);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hst[r].data(), st, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, sm);
        if (e == cudaSuccess && !direct[r]) {
            priv[r].resize(frame_bytes);
            e = cudaMemcpyAsync(priv[r].data(), frame, frame_bytes, cudaMemcpyDeviceToHost, sm);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(sm);
        if (e != cudaSuccess) return fail(cuda_status(e, "multi frame"));
        float t = 0.f;
        cudaEventElapsedTime(&t, w->ev0, w->ev1);
        ms[r] = t;
    };
    {
        std::vector<std::thread> th;
        for (int r = 1; r < n; ++r) th.emplace_back(rank_fn, r);
        rank_fn(0);
        for (auto& t : th) t.join();
    }
    for (int r = 0; r < n; ++r)
        if (rcs[r]) return set_error(rcs[r], "rank " + std::to_string(r) + ": " + msgs[r]);
    if ((rc = use_device(dev0))) return rc;
    double* sum = reinterpret_cast<double*>(f0);
    if (out && out->sum) TV_CK(cudaMemcpy(out->sum, sum, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (out && out->sum_sq)
        TV_CK(cudaMemcpy(out->sum_sq, sum + 3 * npx, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (out && out->sample_counts)
        TV_CK(cudaMemcpy(out->sample_counts, sum + 6 * npx, npx * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H");
    // ranks without peer access: their tiles from their private frames
    for (int r = 0; r < n && out; ++r) {
        if (direct[r]) continue;
        const double* ps = reinterpret_cast<const double*>(priv[r].data());
        const uint32_t* pc = reinterpret_cast<const uint32_t*>(ps + 6 * npx);
        for (uint32_t t = static_cast<uint32_t>(r); t < tiles_x * tiles_y; t += static_cast<uint32_t>(n)) {
            const uint32_t x0 = (t % tiles_x) * 16, y0 = (t / tiles_x) * 16;
            const uint32_t x1 = std::min<uint32_t>(x0 + 16, cv.w), y1 = std::min<uint32_t>(y0 + 16, cv.h);
            for (uint32_t y = y0; y < y1; ++y) {
                const uint64_t p = static_cast<uint64_t>(y) * cv.w + x0, m = x1 - x0;
                if (out->sum) std::memcpy(out->sum + 3 * p, ps + 3 * p, 3 * m * sizeof(double));
                if (out->sum_sq) std::memcpy(out->sum_sq + 3 * p, ps + 3 * npx + 3 * p, 3 * m * sizeof(double));
                if (out->sample_counts) std::memcpy(out->sample_counts + p, pc + p, m * sizeof(uint32_t));
            }
        }
    }
    if (stats) {
        stats->cells_visited = stats->degenerate_paths = 0;
        double worst = 0.0;
        for (int r = 0; r < n; ++r) {
            stats->cells_visited += hst[r][0];
            stats->degenerate_paths += hst[r][2];
            worst = std::max(worst, ms[r]);
        }
        stats->paths_traced = npx * static_cast<uint64_t>(cfg->spp);
        stats->seconds = worst * 1e-3;  // the slowest rank's device time
    }
    return TV_OK;
}

int tv_check_camera(const tv_camera* camera) {
    CamView cv;
    return host_camera(camera, cv, nullptr, nullptr);
}

int tv_check_render_config(const tv_render_config* cfg) { return validate_render(cfg); }

int tv_last_frame_timing(int device, double out[4]) {
    if (!out) return set_error(TV_ERR_ARG, "out is null");
    int rc = use_device(device);
    if (rc) return rc;
    return last_frame_timing(device, out);
}

int tv_march_segments(const tv_grid* h, const tv_ray* rays, uint64_t n, tv_segment* out, uint64_t* offsets,
                      uint64_t cap, uint64_t* total, uint64_t* degenerate_paths) {
    if (!h || (!rays && n)) return set_error(TV_ERR_ARG, "null argument");
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    tv_ray* d_rays = nullptr;
    uint64_t *d_counts = nullptr, *d_off = nullptr;
    tv_segment* d_out = nullptr;
    unsigned long long* d_deg = nullptr;
    auto cleanup = [&]() { cudaFree(d_rays), cudaFree(d_counts), cudaFree(d_off), cudaFree(d_out), cudaFree(d_deg); };
    cudaError_t e = cudaMalloc(&d_rays, (n ? n : 1) * sizeof(tv_ray));
    if (e == cudaSuccess) e = cudaMalloc(&d_counts, (n ? n : 1) * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMalloc(&d_off, (n + 1) * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMalloc(&d_deg, sizeof(unsigned long long));
    if (e == cudaSuccess && n) e = cudaMemcpy(d_rays, rays, n * sizeof(tv_ray), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(d_deg, 0, sizeof(unsigned long long));
    const unsigned nb = static_cast<unsigned>((n + 127) / 128);
    if (e == cudaSuccess && n) {
        march_kernel<<<nb, 128>>>(g.view, d_rays, n, 0, d_counts, nullptr, nullptr, 0, d_deg);
        e = cudaGetLastError();
    }
    std::vector<uint64_t> cnt(n), off(n + 1, 0);
    if (e == cudaSuccess && n) e = cudaMemcpy(cnt.data(), d_counts, n * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + cnt[i];
    const uint64_t tot = off[n];
    const uint64_t wcap = std::min(cap, tot);
    if (e == cudaSuccess) e = cudaMemcpy(d_off, off.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && out && wcap) e = cudaMalloc(&d_out, wcap * sizeof(tv_segment));
    if (e == cudaSuccess && out && wcap && n) {
        march_kernel<<<nb, 128>>>(g.view, d_rays, n, 1, nullptr, d_off, d_out, wcap, d_deg);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && out && wcap) e = cudaMemcpy(out, d_out, wcap * sizeof(tv_segment), cudaMemcpyDeviceToHost);
    unsigned long long deg = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&deg, d_deg, sizeof(deg), cudaMemcpyDeviceToHost);
    cleanup();
    if (e != cudaSuccess) return cuda_status(e, "march_segments");
    if (offsets) std::memcpy(offsets, off.data(), (n + 1) * sizeof(uint64_t));
    if (total) *total = tot;
    if (degenerate_paths) *degenerate_paths = deg;
    return TV_OK;
}

namespace {
// shared driver of tv_march_transmittance / tv_sample_free_path
int medium(const tv_grid* h, const tv_ray* rays, uint64_t n, int mode, uint64_t seed, const uint64_t* pixels,
           const uint64_t* samples, double* tau_out, double* trans_out, tv_free_path* fp_out, uint64_t* stats) {
    if (!h || (!rays && n) || (mode == 1 && n && (!pixels || !samples))) return set_error(TV_ERR_ARG, "null argument");
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    struct Dev {
        void* p = nullptr;
        ~Dev() {
            if (p) cudaFree(p);
        }
    } d_rays, d_pix, d_smp, d_tau, d_tr, d_fp, d_ctr;
    const uint64_t m = n ? n : 1;
    TV_CK(cudaMalloc(&d_rays.p, m * sizeof(tv_ray)), "alloc");
    TV_CK(cudaMalloc(&d_ctr.p, 2 * sizeof(unsigned long long)), "alloc");
    TV_CK(cudaMemset(d_ctr.p, 0, 2 * sizeof(unsigned long long)), "memset");
    if (n) TV_CK(cudaMemcpy(d_rays.p, rays, n * sizeof(tv_ray), cudaMemcpyHostToDevice), "H2D");
    if (mode == 1) {
        TV_CK(cudaMalloc(&d_pix.p, m * 8), "alloc");
        TV_CK(cudaMalloc(&d_smp.p, m * 8), "alloc");
        TV_CK(cudaMalloc(&d_fp.p, m * sizeof(tv_free_path)), "alloc");
        if (n) TV_CK(cudaMemcpy(d_pix.p, pixels, n * 8, cudaMemcpyHostToDevice), "H2D");
        if (n) TV_CK(cudaMemcpy(d_smp.p, samples, n * 8, cudaMemcpyHostToDevice), "H2D");
    } else {
        TV_CK(cudaMalloc(&d_tau.p, m * 8), "alloc");
        TV_CK(cudaMalloc(&d_tr.p, m * 8), "alloc");
    }
    if (n) {
        medium_kernel<<<static_cast<unsigned>((n + 127) / 128), 128>>>(
            g.view, static_cast<const tv_ray*>(d_rays.p), n, mode, seed, static_cast<const uint64_t*>(d_pix.p),
            static_cast<const uint64_t*>(d_smp.p), static_cast<double*>(d_tau.p), static_cast<double*>(d_tr.p),
            static_cast<tv_free_path*>(d_fp.p), static_cast<unsigned long long*>(d_ctr.p));
        TV_CK(cudaGetLastError(), "medium_kernel");
    }
    if (n && tau_out) TV_CK(cudaMemcpy(tau_out, d_tau.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
    if (n && trans_out) TV_CK(cudaMemcpy(trans_out, d_tr.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
    if (n && fp_out) TV_CK(cudaMemcpy(fp_out, d_fp.p, n * sizeof(tv_free_path), cudaMemcpyDeviceToHost), "D2H");
    unsigned long long c[2];
    TV_CK(cudaMemcpy(c, d_ctr.p, sizeof(c), cudaMemcpyDeviceToHost), "D2H");
    if (stats) stats[0] = c[0], stats[1] = c[1];
    return TV_OK;
}
}  // namespace

int tv_trace_rays(const tv_grid* h, const tv_ray* rays, uint64_t n, const tv_render_config* cfg, uint64_t seed,
                  const uint64_t* pixels, const uint64_t* samples, double* out_rgb, uint64_t stats[2]) {
    if (!h || (n && (!rays || !pixels || !samples || !out_rgb))) return set_error(TV_ERR_ARG, "null argument");
    int rc = validate_render(cfg);
    if (rc) return rc;
    const DeviceGrid& g = h->g;
    if ((rc = use_device(g.device))) return rc;
    struct Dev {
        void* p = nullptr;
        ~Dev() {
            if (p) cudaFree(p);
        }
    } d_rays, d_pix, d_smp, d_out, d_ctr;
    const uint64_t m = n ? n : 1;
    TV_CK(cudaMalloc(&d_rays.p, m * sizeof(tv_ray)), "alloc");
    TV_CK(cudaMalloc(&d_pix.p, m * 8), "alloc");
    TV_CK(cudaMalloc(&d_smp.p, m * 8), "alloc");
    TV_CK(cudaMalloc(&d_out.p, m * 24), "alloc");
    TV_CK(cudaMalloc(&d_ctr.p, 16), "alloc");
    TV_CK(cudaMemset(d_ctr.p, 0, 16), "memset");
    if (n) {
        TV_CK(cudaMemcpy(d_rays.p, rays, n * sizeof(tv_ray), cudaMemcpyHostToDevice), "H2D");
        TV_CK(cudaMemcpy(d_pix.p, pixels, n * 8, cudaMemcpyHostToDevice), "H2D");
        TV_CK(cudaMemcpy(d_smp.p, samples, n * 8, cudaMemcpyHostToDevice), "H2D");
        trace_rays_kernel<<<static_cast<unsigned>((n + 127) / 128), 128>>>(
            g.view, make_params(cfg), static_cast<const tv_ray*>(d_rays.p), n, seed,
            static_cast<const uint64_t*>(d_pix.p), static_cast<const uint64_t*>(d_smp.p),
            static_cast<double*>(d_out.p), static_cast<unsigned long long*>(d_ctr.p));
        TV_CK(cudaGetLastError(), "trace_rays_kernel");
        TV_CK(cudaMemcpy(out_rgb, d_out.p, n * 24, cudaMemcpyDeviceToHost), "D2H");
    }
    unsigned long long c[2];
    TV_CK(cudaMemcpy(c, d_ctr.p, sizeof(c), cudaMemcpyDeviceToHost), "D2H");
    if (stats) stats[0] = c[0], stats[1] = c[1];
    return TV_OK;
}

int tv_march_transmittance(const tv_grid* h, const tv_ray* rays, uint64_t n, double* tau_out, double* trans_out,
                           uint64_t stats[2]) {
    return medium(h, rays, n, 0, 0, nullptr, nullptr, tau_out, trans_out, nullptr, stats);
}

int tv_sample_free_path(const tv_grid* h, const tv_ray* rays, uint64_t n, uint64_t seed, const uint64_t* pixels,
                        const uint64_t* samples, tv_free_path* out, uint64_t stats[2]) {
    return medium(h, rays, n, 1, seed, pixels, samples, nullptr, nullptr, out, stats);
}

int tv_locate_points(const tv_grid* h, const double* points, uint64_t n, uint32_t* out) {
    if (!h || ((!points || !out) && n)) return set_error(TV_ERR_ARG, "null argument");
    if (!n) return TV_OK;
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    double* d_p = nullptr;
    uint32_t* d_o = nullptr;
    cudaError_t e = cudaMalloc(&d_p, n * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&d_o, n * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemcpy(d_p, points, n * 3 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        locate_kernel<<<static_cast<unsigned>((n + 127) / 128), 128>>>(g.view, d_p, n, d_o);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d_o, n * sizeof(uint32_t), cudaMemcpyDeviceToHost);
    cudaFree(d_p);
    cudaFree(d_o);
    return cuda_status(e, "locate_points");
}

}  // extern "C"
