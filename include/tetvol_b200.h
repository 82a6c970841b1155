/* tetvol_b200 — B200-native (sm_100a) renderer and LEB builder for adaptive
 * tetrahedral grids, behind a plain C ABI.
 *
 * Drop-in boundary. Each entry point replaces one call of the reference C++
 * API (paths relative to /root/reference/proj):
 *
 *   tv_grid_upload      <- a TetGrid value as produced by TetGrid::init_roots /
 *                          build_adaptive_grid / load_grid: its pools
 *                          vertices(), tets(), roots() (tet_grid.hpp:118-122)
 *   tv_grid_download    -> TetGrid::assemble(...) input (tet_grid.hpp:110-111)
 *   tv_build            <- build_adaptive_grid(vol, cfg, camera, stats)
 *                          (builder.hpp:51-52)
 *   tv_render           <- render(grid, camera, cfg, threads) (tracer.hpp:84-85)
 *   tv_render_multi     <- render() over several GPUs from one process
 *   tv_render_tiles     <- the per-rank share of render() for multi-GPU
 *                          image-space sharding (interleaved 16x16 tiles)
 *   tv_march_segments   <- march_segments(grid, ray, stats) (tracer.hpp:49)
 *   tv_locate_points    <- TetGrid::locate_point (tet_grid.hpp:166)
 *   tv_render_regular   <- render_reference(RegularGrid::from_volume(vol, s),
 *                          camera, cfg) (regular_grid.hpp:66-67)
 *   tv_grid_save        <- save_grid(grid, path) (builder.hpp:59)
 *   tv_grid_load        <- load_grid(path) (builder.hpp:60)
 *
 * Conventions: no C++ exception crosses this boundary; every function returns
 * a tv_status (0 = TV_OK) and tv_last_error() holds a thread-local message.
 * Handles are opaque and owned by the caller (free with tv_grid_free).
 * Pointers are HOST pointers unless the name says _dev. Device work runs on
 * the grid's device; functions taking a `stream` run asynchronously on it
 * (0 = the legacy default stream) and otherwise synchronise before returning.
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point returns TV_ERR_CUDA.
 */
#ifndef TETVOL_B200_H
#define TETVOL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TV_NO_TET 0xffffffffu

typedef enum {
    TV_OK = 0,
    TV_ERR = 1,         /* runtime failure (reference: std::runtime_error)            */
    TV_ERR_CONFIG = 2,  /* ConfigError (tracer.cpp:131-141, builder.cpp:12-17)         */
    TV_ERR_CAMERA = 3,  /* CameraError (camera.cpp:15-20)                             */
    TV_ERR_GRID = 4,    /* GridError family (tet_grid.hpp:24-38)                      */
    TV_ERR_OUTSIDE = 5, /* OutsideGrid (tet_grid.hpp:33-35)                           */
    TV_ERR_CUDA = 6,    /* no device, launch or copy failure                          */
    TV_ERR_OOM = 7,     /* device allocation failed                                   */
    TV_ERR_ARG = 8,     /* null pointer / size mismatch at the ABI                    */
    TV_ERR_FORMAT = 9,  /* FormatError: malformed .tgrid (builder.cpp:184-293)          */
    TV_ERR_IO = 10,     /* IoError: cannot open / write a file                        */
    TV_ERR_VOLUME = 11, /* VolumeError / UnknownChannel (volume.hpp:13-18)            */
    TV_ERR_IMAGE = 12   /* ImageError: PFM I/O (image.cpp)                            */
} tv_status;

/* Reference Vertex (tet_grid.hpp:41-49): fixed point, position = q / 2^24. */
typedef struct {
    uint32_t q[3];
} tv_vertex;

/* Byte-identical to the reference `Tet` (tet_grid.hpp:64-75; 68 bytes), so
 * `grid.tets().data()` can be passed without conversion. */
typedef struct {
    uint32_t verts[4];
    uint32_t children[2];
    uint32_t parent;
    uint32_t neighbors[4];
    uint8_t normal_ids[4];
    uint8_t level;
    uint8_t pad0[3];
    float density, temperature, albedo; /* MediaPayload (tet_grid.hpp:53-62) */
    uint8_t mask;
    uint8_t pad1[3];
} tv_tet;

/* PinholeCamera constructor arguments (camera.hpp:18-19). The basis, tan and
 * frustum planes are derived on the host exactly as camera.cpp:12-45 does.
 * basis_final != 0 means forward/up are an already constructed camera's
 * forward() / up() (unit, orthogonal; camera.hpp:37-39): they are used as-is,
 * so a reference PinholeCamera converts without re-normalising (bit-exact). */
typedef struct {
    double position[3];
    double forward[3];
    double up[3];
    double vfov_degrees;
    int32_t width, height;
    int32_t basis_final;
    int32_t pad;
} tv_camera;

/* RenderConfig (tracer.hpp:16-28). exposure/gamma only affect 8-bit output. */
typedef struct {
    int32_t spp;
    int32_t max_bounces;
    uint64_t seed;
    double hg_g;
    double default_albedo;
    double environment[3];
    double emission_scale;
    double exposure;
    double gamma;
} tv_render_config;

/* BuildConfig (builder.hpp:21-29). */
typedef struct {
    double variation_threshold;
    int32_t max_level;
    int32_t use_camera;
    double pixel_threshold;
    double density_scale;
} tv_build_config;

/* BuildStats (builder.hpp:31-38) plus GPU round counters. */
typedef struct {
    uint64_t leaf_count;
    int32_t max_depth;
    int32_t rounds;           /* criterion rounds                       */
    double seconds;           /* device time of the build               */
    uint64_t criterion_splits;
    uint64_t propagation_splits;
    uint64_t closure_passes;  /* bisect passes summed over all rounds   */
    uint64_t voxel_visits;    /* sum over evaluated tets of owned voxels */
} tv_build_stats;

/* ImageAccumulator counters (image.hpp:23-26) plus device timing. */
typedef struct {
    uint64_t cells_visited;
    uint64_t paths_traced;
    uint64_t degenerate_paths;
    double seconds;           /* device time of the render kernel(s) */
} tv_render_stats;

/* ImageAccumulator buffers (image.hpp:21-23): sum, sum_sq = 3*W*H doubles in
 * pixel-major RGB order; sample_counts = W*H. Any pointer may be NULL to skip
 * that output. */
typedef struct {
    double* sum;
    double* sum_sq;
    uint32_t* sample_counts;
} tv_framebuffer;

/* Ray (geometry.hpp:53-60). */
typedef struct {
    double origin[3];
    double dir[3];
    double t_min, t_max;
} tv_ray;

/* RaySegment (tet_grid.hpp:82-86); cell is the reference TetId. */
typedef struct {
    uint32_t cell;
    uint32_t pad;
    double t_enter, t_exit;
} tv_segment;

typedef struct tv_grid tv_grid;
typedef struct tv_volume tv_volume;

/* cmd_compare's image metrics (cli.cpp:499-531). outlier_fraction < 0 when no
 * variance images were given (the reference reports null). */
typedef struct {
    double rmse;
    double max_abs_diff;
    double outlier_fraction;
    uint64_t outliers;
} tv_compare_stats;

typedef struct {
    uint64_t n_vertices;
    uint64_t n_tets;
    uint64_t n_leaves;
    uint64_t n_internal;
    int32_t max_level;
    int32_t max_depth;
    int32_t device;
    int32_t pad;
    uint64_t device_bytes;
} tv_grid_info;

const char* tv_last_error(void);
const char* tv_version(void);
int tv_device_count(int* out);

/* Validation alone, no device work: the PinholeCamera constructor
 * (camera.cpp:12-20), RenderConfig::validate (tracer.cpp:131-141) and
 * BuildConfig::validate (builder.cpp:12-17), with their messages. */
int tv_check_camera(const tv_camera* camera);
int tv_check_render_config(const tv_render_config* cfg);
int tv_check_build_config(const tv_build_config* cfg);

/* -- grid lifetime -------------------------------------------------------- */
int tv_grid_upload(const tv_vertex* vertices, uint64_t n_vertices, const tv_tet* tets, uint64_t n_tets,
                   const uint32_t roots[24], int32_t max_level, int device, tv_grid** out);
/* Copies the pools back (reference layout, reference TetIds). Query sizes
 * with tv_grid_get_info; any output pointer may be NULL. */
int tv_grid_download(const tv_grid* g, tv_vertex* vertices, tv_tet* tets, uint32_t roots[24]);
int tv_grid_get_info(const tv_grid* g, tv_grid_info* out);
void tv_grid_free(tv_grid* g);
/* The reference's TGRD v1 file (save_grid / load_grid, builder.cpp:184-293),
 * byte-identical to save_grid of the same pools; records are packed and
 * unpacked on the device. load applies load_grid's checks and messages
 * (TV_ERR_FORMAT) and assembles with max_level 48 as load_grid does. */
int tv_grid_save(const tv_grid* g, const char* path);
int tv_grid_load(const char* path, int device, tv_grid** out);

/* -- LEB build on the GPU --------------------------------------------------- */
/* density/temperature/albedo: nx*ny*nz floats, x fastest (volume.hpp:41-43);
 * temperature/albedo may be NULL. camera may be NULL unless use_camera. */
int tv_build(const float* density, const float* temperature, const float* albedo, int32_t nx, int32_t ny,
             int32_t nz, const tv_build_config* cfg, const tv_camera* camera, int device, tv_grid** out,
             tv_build_stats* stats);
/* Same, with the density already resident on the device (float, x fastest). */
int tv_build_dev(const float* density_dev, const float* temperature_dev, const float* albedo_dev, int32_t nx,
                 int32_t ny, int32_t nz, const tv_build_config* cfg, const tv_camera* camera, int device,
                 tv_grid** out, tv_build_stats* stats);
/* Build scratch (not in the reference, whose builder allocates on the host):
 * the device buffers a build works in stay allocated on their device after
 * the build and are reused by the next one, so warm builds do no driver
 * allocation (TV_BUILD_CACHE=0 turns this off). tv_build_trim releases them
 * (device -1: every device); tv_build_scratch_bytes reports what is held.
 * A failed build releases its device's scratch itself. */
int tv_build_trim(int device);
uint64_t tv_build_scratch_bytes(int device);
/* Procedural fields on the device (kind: 0 constant, 1 ramp, 2 blob, 3 step,
 * 4 noise, 5 cloud; cli.cpp:317-346). out_dev: nx*ny*nz f32. */
int tv_generate_volume_dev(int32_t kind, int32_t nx, int32_t ny, int32_t nz, double value, float* out_dev,
                           int device);

/* -- render ------------------------------------------------------------------ */
int tv_render(const tv_grid* g, const tv_camera* camera, const tv_render_config* cfg, tv_framebuffer* out,
              tv_render_stats* stats);
/* render() over several GPUs from one process: grids[r]
 * (normally the same grid, uploaded or built once per device) renders the
 * interleaved 16x16 tiles t with t % n == r on its device, one host thread per
 * rank. Ranks whose device has peer access to grids[0]'s device store their
 * pixels straight into the frame there (NVLink); others render a private frame
 * whose tiles are merged on the host. The framebuffer is bit-identical to
 * tv_render's for any n; stats->seconds is the slowest rank's device time.
 * Synchronous; one tv_render_multi call runs at a time. */
int tv_render_multi(const tv_grid* const* grids, int32_t n, const tv_camera* camera, const tv_render_config* cfg,
                    tv_framebuffer* out, tv_render_stats* stats);
/* Multi-GPU share: renders the interleaved 16x16 tiles t with
 * t % n_ranks == rank (tile t = row-major over ceil(W/16) x ceil(H/16)).
 * Outputs are DEVICE pointers to full-frame buffers (only this rank's pixels
 * are written) and the call is asynchronous on `stream`; stats_dev (3 u64:
 * cells_visited, paths_traced, degenerate_paths) is accumulated atomically. */
int tv_render_tiles(const tv_grid* g, const tv_camera* camera, const tv_render_config* cfg, int32_t rank,
                    int32_t n_ranks, double* sum_dev, double* sum_sq_dev, uint32_t* counts_dev, uint64_t* stats_dev,
                    void* stream);
/* Progressive accumulation: renders samples [first_sample, first_sample +
 * cfg->spp) of this rank's tiles and ADDS them to the device accumulators in
 * sample order (first_sample == 0 initialises them). Frames covering [0, N)
 * leave exactly the framebuffer of one N-spp render (bit-identical). */
int tv_render_accumulate(const tv_grid* g, const tv_camera* camera, const tv_render_config* cfg,
                         int32_t first_sample, int32_t rank, int32_t n_ranks, double* sum_dev, double* sum_sq_dev,
                         uint32_t* counts_dev, uint64_t* stats_dev, void* stream);
/* Device time (ms) of the last frame rendered on `device`, per kernel:
 * out[0] start (camera rays + locate), out[1] trace, out[2] accumulate;
 * out[3] = number of kernel launches of that frame. Synchronises on it. */
int tv_last_frame_timing(int device, double out[4]);
/* Packs this rank's tiles of a full-frame device buffer (elem_words 64-bit
 * words per pixel) into a contiguous buffer of tv_tile_pack_words() words
 * (for one NCCL all-gather), and the inverse for the gathered buffers. */
uint64_t tv_tile_pack_words(int32_t width, int32_t height, int32_t rank, int32_t n_ranks, int32_t elem_words);
int tv_tile_pack(const void* frame_dev, void* packed_dev, int32_t width, int32_t height, int32_t rank,
                 int32_t n_ranks, int32_t elem_words, void* stream);
int tv_tile_unpack(const void* packed_dev, void* frame_dev, int32_t width, int32_t height, int32_t rank,
                   int32_t n_ranks, int32_t elem_words, void* stream);
/* Direct peer writes (the gather fused into the render's accumulate step):
 * rank 0 exports its full-frame accumulators, every other rank maps them and
 * passes the mapped pointers to tv_render_tiles, whose accumulate kernel then
 * stores this rank's pixels straight into rank 0's HBM over NVLink (no pack,
 * all-gather or unpack). tv_render_tiles detects peer outputs and ends the
 * accumulate kernel with a system-scope fence, so a stream-ordered barrier
 * after it (e.g. a one-word NCCL all-reduce) publishes the pixels. The handle
 * is 64 opaque bytes (cudaIpcMemHandle_t) naming the whole allocation that
 * holds dev_ptr, and offset is dev_ptr's byte offset inside it (allocators
 * such as PyTorch's hand out sub-ranges of larger allocations). */
int tv_ipc_export(const void* dev_ptr, uint8_t handle[64], uint64_t* offset);
int tv_ipc_open(const uint8_t handle[64], uint64_t offset, int device, void** dev_ptr_out);
int tv_ipc_close(void* dev_ptr, uint64_t offset); /* dev_ptr, offset as from tv_ipc_open */

/* -- volumes in HBM (DenseVolume, volume.hpp:19-58; .dvol, volume.cpp:84-138) -- */
/* create: a zero "density" channel (volume.hpp:25); dims in [1, 4096].       */
int tv_volume_create(int32_t nx, int32_t ny, int32_t nz, int device, tv_volume** out);
int tv_volume_load(const char* path, int device, tv_volume** out); /* load_dvol */
int tv_volume_save(const tv_volume* v, const char* path);          /* save_dvol */
void tv_volume_free(tv_volume* v);
int tv_volume_get_info(const tv_volume* v, int32_t dims[3], int32_t* n_channels);
int tv_volume_channel_name(const tv_volume* v, int32_t index, char* buf, int32_t cap);
int tv_volume_channel_dev(const tv_volume* v, const char* name, float** out_dev);
int tv_volume_add_channel(tv_volume* v, const char* name);         /* zero-filled */
int tv_volume_upload(tv_volume* v, const char* name, const float* in);
int tv_volume_download(const tv_volume* v, const char* name, float* out);
/* cmd_gen on the device (cli.cpp:349-380): density of a procedural kind
 * (as tv_generate_volume_dev), temperature = clamp(density, 0, 1), constant albedo */
int tv_volume_generate(tv_volume* v, int32_t kind, double value);
int tv_volume_add_temperature(tv_volume* v);
int tv_volume_add_albedo(tv_volume* v, double albedo);
/* build_adaptive_grid(DenseVolume, ...) with the volume's density and
 * optional temperature / albedo channels (builder.cpp:164-182) */
int tv_build_volume(const tv_volume* v, const tv_build_config* cfg, const tv_camera* camera, tv_grid** out,
                    tv_build_stats* stats);

/* -- images (image.cpp:33-101) and compare (cli.cpp:487-531) ------------------ */
/* Per-pixel f32 mean (variance = 0) or variance_of_mean (variance = 1) of an
 * accumulator, top-down RGB, computed on the GPU; on_device says whether the
 * framebuffer pointers are device pointers. */
int tv_image_pfm_pixels(const double* sum, const double* sum_sq, const uint32_t* counts, int32_t width, int32_t height,
                        int32_t variance, int32_t on_device, int device, float* out_rgb);
/* write_pfm / write_variance_pfm: byte-identical files */
int tv_image_write_pfm(const char* path, const tv_framebuffer* fb, int32_t width, int32_t height, int32_t variance,
                       int32_t on_device, int device);
int tv_pfm_write(const char* path, const float* rgb, int32_t width, int32_t height);
/* read_pfm: call with rgb = NULL for the size, then with 3*W*H floats */
int tv_pfm_read(const char* path, int32_t* width, int32_t* height, float* rgb);
/* a, b (and optional va, vb): 3 * n_pixels floats each (host) */
int tv_image_compare(const float* a, const float* b, const float* va, const float* vb, uint64_t n_pixels, int device,
                     tv_compare_stats* out);

/* -- validation (TetGrid::validate, tet_grid.cpp:474-636) --------------------- */
typedef struct {
    int32_t ok;
    int32_t pad;
    uint64_t leaf_count;
    uint64_t interior_faces;
    uint64_t boundary_faces;
    char first_violation[128];
} tv_validation_report;
/* The reference's exhaustive invariant checks on the GPU, over the grid's
 * reference-layout pools; first_violation is the reference's first message. */
int tv_grid_validate(const tv_grid* g, tv_validation_report* out);
/* cmd_validate's traversal spot checks (cli.cpp:565-595): for each ray, our
 * march_segments against the brute-force traverser (tet_grid.cpp:659-698, on
 * the GPU), segments <= 1e-12 dropped; same cells and lengths within 1e-9. */
int tv_validate_rays(const tv_grid* g, const tv_ray* rays, int32_t n, int32_t* failures, int32_t* first_failed);
/* cmd_validate's n spot-check rays for a seed (cli.cpp:552-569), on the host */
int tv_validate_spot_rays(uint64_t seed, int32_t n, tv_ray* out);

/* -- parity entry points ------------------------------------------------------ */
/* Segments of n rays. offsets has n+1 entries; at most cap segments are
 * written; *total receives the full count. */
int tv_march_segments(const tv_grid* g, const tv_ray* rays, uint64_t n, tv_segment* out, uint64_t* offsets,
                      uint64_t cap, uint64_t* total, uint64_t* degenerate_paths);
/* FreePathSample (tracer.hpp:54-60); cell is the reference TetId. */
typedef struct {
    int32_t collided;
    uint32_t cell;
    double distance;
    double position[3];
} tv_free_path;

/* trace(grid, ray, cfg, rng, stats) (tracer.hpp:78-79) per ray, with
 * RngStream(seed, pixels[i], samples[i]); out_rgb: 3 doubles per ray. */
int tv_trace_rays(const tv_grid* g, const tv_ray* rays, uint64_t n, const tv_render_config* cfg, uint64_t seed,
                  const uint64_t* pixels, const uint64_t* samples, double* out_rgb, uint64_t stats[2]);
/* march_transmittance (tracer.hpp:52) per ray: tau_out = the optical depth
 * (bit-exact), trans_out = exp(-tau); either may be NULL. stats (may be NULL):
 * cells_visited, degenerate_paths. */
int tv_march_transmittance(const tv_grid* g, const tv_ray* rays, uint64_t n, double* tau_out, double* trans_out,
                           uint64_t stats[2]);
/* sample_free_path (tracer.hpp:63) per ray with RngStream(seed, pixels[i], samples[i]). */
int tv_sample_free_path(const tv_grid* g, const tv_ray* rays, uint64_t n, uint64_t seed, const uint64_t* pixels,
                        const uint64_t* samples, tv_free_path* out, uint64_t stats[2]);
/* -- free-flight estimators over the per-tet majorant (optional modes) ------------
 * The reference (and tv_render) uses regular tracking: one draw per flight and
 * the exact optical depth of every crossed tet (path_integrator.hpp:49-61).
 * Delta tracking samples tentative collisions at the per-tet majorant
 * mu = majorant_scale * density (majorant_scale >= 1) and accepts each with
 * probability density / mu; ratio tracking (transmittance only: the reference
 * has no next-event estimation) weights the ray by 1 - density / mu per
 * tentative collision. Both agree with regular tracking in distribution, not
 * bit for bit (they draw the path's RngStream in their own order). */
#define TV_TRACK_REGULAR 0
#define TV_TRACK_DELTA 1
#define TV_TRACK_RATIO 2
/* render() with the given tracking (TV_TRACK_REGULAR: exactly tv_render;
 * TV_TRACK_RATIO: TV_ERR_CONFIG). Same sample keys, camera jitter and
 * ImageAccumulator outputs as tv_render. */
int tv_render_tracking(const tv_grid* g, const tv_camera* camera, const tv_render_config* cfg, int32_t tracking,
                       double majorant_scale, tv_framebuffer* out, tv_render_stats* stats);
/* One transmittance estimate per ray over [t_min, t_max] with
 * RngStream(seed, pixels[i], samples[i]): TV_TRACK_REGULAR gives exp(-tau)
 * (march_transmittance, tracer.hpp:52; pixels / samples unused), DELTA 0 or 1,
 * RATIO the ratio-tracking weight. stats: cells_visited, degenerate_paths. */
int tv_transmittance_tracking(const tv_grid* g, const tv_ray* rays, uint64_t n, int32_t tracking,
                              double majorant_scale, uint64_t seed, const uint64_t* pixels, const uint64_t* samples,
                              double* trans_out, uint64_t stats[2]);

/* points: 3*n doubles; out: reference TetIds (TV_NO_TET when outside). */
int tv_locate_points(const tv_grid* g, const double* points, uint64_t n, uint32_t* out);

/* -- regular-grid comparator (config 5) ---------------------------------------- */
int tv_render_regular(const float* density, int32_t nx, int32_t ny, int32_t nz, double density_scale,
                      const tv_camera* camera, const tv_render_config* cfg, int device, tv_framebuffer* out,
                      tv_render_stats* stats);
/* Same, with the density already in HBM (f32, x fastest). */
int tv_render_regular_dev(const float* density_dev, int32_t nx, int32_t ny, int32_t nz, double density_scale,
                          const tv_camera* camera, const tv_render_config* cfg, int device, tv_framebuffer* out,
                          tv_render_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
