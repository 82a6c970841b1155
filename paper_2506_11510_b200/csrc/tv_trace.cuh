// Host/device declarations shared by the kernels and the C-ABI layer.
#pragma once

#include <string>

#include "tv_internal.cuh"

namespace tvb {

constexpr int kRenderThreads = 128;
constexpr int kRenderMinBlocks = 4;

struct TileSched {
    uint32_t* counter;   // device work counter (zeroed before launch)
    uint32_t n_units;    // 8 warp units per 16x16 tile of this rank
    uint32_t tiles_x;
    int32_t rank, n_ranks;
};

struct RenderOut {
    double* sum;
    double* sum_sq;
    uint32_t* counts;
    uint64_t* stats;  // [cells_visited, paths_traced, degenerate_paths]
};

__global__ void render_kernel(GridView G, CamView C, RenderParams P, TileSched S, RenderOut O);
__global__ void march_kernel(GridView G, const tv_ray* rays, uint64_t n, int pass, uint64_t* counts,
                             const uint64_t* offsets, tv_segment* out, uint64_t cap, unsigned long long* deg);
__global__ void locate_kernel(GridView G, const double* pts, uint64_t n, uint32_t* out);

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

}  // namespace tvb

struct tv_grid {
    tvb::DeviceGrid g;
};
