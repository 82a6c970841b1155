// Host/device declarations shared by the kernels and the C-ABI layer.
#pragma once

#include <string>

#include "tv_internal.cuh"

namespace tvb {

#ifndef TV_TRACE_THREADS
#define TV_TRACE_THREADS 128
#endif
constexpr int kTraceThreads = TV_TRACE_THREADS;
constexpr uint32_t kChunk = 64;               // paths a warp claims per queue atomic
constexpr uint32_t kInvalidPixel = 0xfffffffeu;
constexpr uint64_t kMaxBatchPaths = 1ull << 26;
constexpr uint32_t kColdBytes = 6 * 8 + 8 + 3 * 4;  // cold path state per trace thread and path slot
#ifndef TV_COLD_GLOBAL
#define TV_COLD_GLOBAL 0  // cold path state in shared memory (see tv_path.inc)
#endif

// One render batch: this rank's pixels x samples [s0, s0 + ns).
// Path index p -> unit = p / (ns * 32), s = s0 + (p / 32) % ns, lane = p % 32;
// a unit is an 8x4 pixel block, 8 units tile a 16x16 sharding tile, and tile
// t = rank + k * n_ranks (row-major tile numbering).
struct Batch {
    uint32_t n_units;
    uint32_t s0, ns;
    uint32_t tiles_x, tiles_y;
    int32_t rank, n_ranks;
    uint32_t n_paths;
    uint32_t first;  // 1 for the first batch of a frame (accumulators start at 0)
    uint32_t regen_min, scatter_min;  // warp-batching thresholds of the trace loop
    uint32_t tail_chunk;              // paths per queue claim once the queue is nearly drained (<= kChunk)
    uint32_t tail_from;               // queue position where the tail claims start
    uint32_t order;                   // path id order (see path_id in tv_trace.cu)
    const uint32_t* tile_order;       // this rank's tiles in processing order (null: t = rank + k * n_ranks)
    void* cold;                       // trace kernel: cold path state (TV_COLD_GLOBAL), kColdBytes per thread
    uint32_t* tile_cost;              // TV_TILE_ORDER=3: tet steps per tile-list position (null: off)
};

struct StartRec {  // camera ray of one path after TetMarcher::start
    double dx, dy, dz, t0;
    unsigned long long key;  // the path's RngStream key (rng.hpp:19-22)
    double target;           // first optical-depth target, -log(1 - u) at dim 3 (path_integrator.hpp:49)
};

struct RenderOut {
    double* sum;
    double* sum_sq;
    uint32_t* counts;
    uint64_t* stats;  // [cells_visited, paths_traced, degenerate_paths]
    int remote;       // outputs live on a peer GPU: fence the stores system-wide
};

__global__ void start_kernel(GridView G, CamView C, RenderParams P, Batch B, StartRec* st, uint32_t* cells);
using TraceFn = void (*)(GridView, CamView, RenderParams, Batch, const StartRec*, const uint32_t*, double*,
                         uint64_t*, uint32_t*);
// trace kernel instantiated for 4, 5, 6 or 8 resident blocks per SM
// the trace kernel for a register cap and a number of path slots per lane
TraceFn trace_variant(int maxreg, int block_threads, int& threads, bool hot = false);
__global__ void accum_kernel(Batch B, CamView C, const uint32_t* cells, const double* rad, RenderOut O);
__global__ void march_kernel(GridView G, const tv_ray* rays, uint64_t n, int pass, uint64_t* counts,
                             const uint64_t* offsets, tv_segment* out, uint64_t cap, unsigned long long* deg);
__global__ void locate_kernel(GridView G, const double* pts, uint64_t n, uint32_t* out);
__global__ void trace_rays_kernel(GridView G, RenderParams P, const tv_ray* rays, uint64_t n, uint64_t seed,
                                  const uint64_t* pixels, const uint64_t* samples, double* out,
                                  unsigned long long* counters);
__global__ void medium_kernel(GridView G, const tv_ray* rays, uint64_t n, int mode, uint64_t seed,
                              const uint64_t* pixels, const uint64_t* samples, double* tau_out, double* trans_out,
                              tv_free_path* fp_out, unsigned long long* counters);

// Device-resident grid (owned by tv_grid).
struct DeviceGrid {
    int device = 0;
    uint64_t n_vertices = 0, n_tets = 0, n_leaves = 0, n_internal = 0;
    int max_level = 48, max_depth = 0;
    uint32_t roots[24] = {};
    // reference-layout pools, kept for download / validation
    tv_tet* tets = nullptr;
    uint4* verts = nullptr;
    // traversal layout
    LeafRec* leaves = nullptr;
    NodeRec* nodes = nullptr;
    uint32_t* leaf2tet = nullptr;
    uint8_t* mask = nullptr;
    uint32_t* jump = nullptr;  // locate jump table (view.jump)
    HotRec* hot = nullptr;     // 32-B hot records (view.hot; null when the geometry does not fit them)
    GridView view{};
    uint64_t bytes = 0;
};

// Builds the traversal layout (leaves, nodes, view) from the reference pools
// already on the device (g.tets, g.verts, g.roots). Returns tv_status.
int finalize_grid(DeviceGrid& g, cudaStream_t stream);
void free_grid(DeviceGrid& g);

// thread-local error plumbing for the C ABI
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
// selects `device` (TV_ERR_CUDA when there is none)
int use_device(int device);
// camera.cpp:12-45 on the host (optional frustum planes for the build)
int host_camera(const tv_camera* c, CamView& v, d3 pn[5], double pd[5]);

}  // namespace tvb

struct tv_grid {
    tvb::DeviceGrid g;
};
