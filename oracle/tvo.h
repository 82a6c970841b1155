/* TEST INFRASTRUCTURE ONLY — the CPU oracle (C restatement) of the reference
 * `tetvol` hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product (libtetvol_b200.so) never does.
 *
 * Parity pinning: every entry point is checked against the unmodified
 * reference (oracle/_ref/libtetvol_ref.so, built from /root/reference by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/
 * (tests/test_oracle.py). Each function cites the reference file:line it
 * restates; paths are relative to /root/reference/proj.
 */
#ifndef TVO_H
#define TVO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVO_NO_TET 0xffffffffu
#define TVO_COORD_ONE (1u << 24)
#define TVO_LEVEL_CAP 48

/* status codes (mirrors ConfigError / CameraError / GridError families) */
enum { TVO_OK = 0, TVO_ERR = 1, TVO_ERR_CONFIG = 2, TVO_ERR_CAMERA = 3, TVO_ERR_GRID = 4, TVO_ERR_OUTSIDE = 5 };

/* Same byte layout as the reference `Tet` (tet_grid.hpp:64-75, 68 bytes), so
 * pools interchange with the reference by memcpy. */
typedef struct {
    uint32_t verts[4];
    uint32_t children[2];
    uint32_t parent;
    uint32_t neighbors[4];
    uint8_t normal_ids[4];
    uint8_t level;
    uint8_t pad0[3];
    float density, temperature, albedo;
    uint8_t mask;
    uint8_t pad1[3];
} tvo_tet;

typedef struct tvo_grid tvo_grid;

typedef struct {
    double pos[3], fwd[3], up[3];
    double vfov;
    int32_t width, height;
} tvo_camera_desc;

typedef struct {
    int32_t spp, max_bounces;
    uint64_t seed;
    double hg_g, default_albedo, env[3], emission_scale;
} tvo_render_cfg;

typedef struct {
    double variation_threshold;
    int32_t max_level, use_camera;
    double pixel_threshold, density_scale;
} tvo_build_cfg;

typedef struct {
    uint64_t leaf_count;
    int32_t max_depth, pad;
    double seconds;
    uint64_t criterion_splits, propagation_splits;
} tvo_build_stats;

const char* tvo_last_error(void);

/* rng.hpp:10-33 */
uint64_t tvo_mix64(uint64_t x);
void tvo_rng_draws(uint64_t seed, uint64_t pixel, uint64_t sample, int n, double* out);

/* camera.cpp:12-85 */
int tvo_primary_ray(const tvo_camera_desc* c, int px, int py, double jx, double jy, double* out6);
int tvo_camera_tet_tests(const tvo_camera_desc* c, const double* corners12, double* out2);

/* volume generators (cli.cpp:317-346 and SURVEY.md 8(d)); kind: 0 constant,
 * 1 ramp, 2 blob, 3 step, 4 noise (reference value_noise), 5 cloud */
void tvo_gen_volume(int kind, int nx, int ny, int nz, double value, float* out);
void tvo_random_cube_rays(uint64_t seed, uint64_t salt, uint64_t n, double* out);

/* grid lifetime and structure (tet_grid.cpp) */
tvo_grid* tvo_grid_init_roots(int max_level);
tvo_grid* tvo_grid_fuzzed(int steps, uint64_t seed, int max_level);
tvo_grid* tvo_grid_from_pools(const uint32_t* vq, uint64_t nv, const tvo_tet* tets, uint64_t nt,
                              const uint32_t* roots, int max_level);
void tvo_grid_free(tvo_grid* g);
void tvo_grid_counts(const tvo_grid* g, uint64_t* out4);
void tvo_grid_export(const tvo_grid* g, uint32_t* vq, tvo_tet* tets, uint32_t* roots);
int tvo_grid_refine_conforming(tvo_grid* g, uint32_t t);
void tvo_grid_fill_density(tvo_grid* g, float lambda);
int tvo_locate_point(const tvo_grid* g, const double* p, uint32_t* out);
int tvo_exit_face(const tvo_grid* g, uint32_t cell, const double* pos, const double* dir, double* t);

/* builder.cpp:83-182 */
tvo_grid* tvo_grid_build(const float* density, const float* temperature, const float* albedo, int nx, int ny,
                         int nz, const tvo_build_cfg* bc, const tvo_camera_desc* cam, tvo_build_stats* st);
void tvo_density_stats(const tvo_grid* g, const float* density, int nx, int ny, int nz, uint32_t leaf, double* out4);

/* tracer.cpp:164-267, path_integrator.hpp:42-136 */
int64_t tvo_march_segments(const tvo_grid* g, const double* rays, uint64_t n, uint32_t* cells, double* t0,
                           double* t1, uint64_t* offsets, uint64_t cap, uint64_t* stats2);
double tvo_march_transmittance(const tvo_grid* g, const double* ray8);
void tvo_sample_free_path(const tvo_grid* g, const double* ray8, uint64_t seed, uint64_t pixel, uint64_t sample,
                          double* out6);
double tvo_hg_sample_cos(double g, double xi);
void tvo_sample_phase_hg(const double* dir, double g, uint64_t seed, uint64_t pixel, uint64_t sample, double* out3);
void tvo_emission_color(double t, double* out3);
/* Renders rows y with (y % row_stride) == row_offset (stride 1 = full frame).
 * threads <= 0: all host cores. stats3: cells_visited, paths_traced, degenerate. */
int tvo_render(const tvo_grid* g, const tvo_camera_desc* c, const tvo_render_cfg* r, int threads, int row_stride,
               int row_offset, double* sum, double* sum_sq, uint32_t* counts, uint64_t* stats3, double* seconds);

/* regular_grid.cpp:16-167 */
int64_t tvo_dda_segments(const float* density, int nx, int ny, int nz, double density_scale, const double* rays,
                         uint64_t n, uint32_t* cells, double* t0, double* t1, uint64_t* offsets, uint64_t cap);
int tvo_render_regular(const float* density, int nx, int ny, int nz, double density_scale, const tvo_camera_desc* c,
                       const tvo_render_cfg* r, int threads, double* sum, double* sum_sq, uint32_t* counts,
                       uint64_t* stats3, double* seconds);

/* FNV-64 over the bit patterns of n doubles (SURVEY.md 8(c) golden hash) */
uint64_t tvo_fnv64_doubles(const double* v, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
