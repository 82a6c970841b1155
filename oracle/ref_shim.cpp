// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C-ABI shim over the UNMODIFIED reference library (`tetvol`, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Python tests,
// the golden-vector generator and bench.py's reference arm call these entry
// points through ctypes. Every function forwards to the reference API; no
// reference logic is restated here.
//
// Reference API forwarded (paths relative to /root/reference/proj):
//   TetGrid::init_roots / assemble / validate / locate_point / refine_conforming
//                                            include/tetvol/tet_grid.hpp:100-196
//   build_adaptive_grid, save_grid, load_grid include/tetvol/builder.hpp:51-61
//   march_segments / march_transmittance / exit_face / sample_free_path /
//   sample_phase_hg / hg_sample_cos / emission_color / trace / render
//                                            include/tetvol/tracer.hpp:39-85
//   PinholeCamera                             include/tetvol/camera.hpp:16-48
//   RegularGrid::from_volume / render_reference include/tetvol/regular_grid.hpp:17-67
//   DenseVolume save_dvol / load_dvol         include/tetvol/volume.hpp:19-58
//   write_pfm / write_variance_pfm / read_pfm include/tetvol/image.hpp:72-90

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "tetvol/builder.hpp"
#include "tetvol/camera.hpp"
#include "tetvol/image.hpp"
#include "tetvol/regular_grid.hpp"
#include "tetvol/rng.hpp"
#include "tetvol/tet_grid.hpp"
#include "tetvol/tracer.hpp"
#include "tetvol/volume.hpp"

using namespace tetvol;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ConfigError*>(&e)) return 2;
    if (dynamic_cast<const CameraError*>(&e)) return 3;
    if (dynamic_cast<const GridError*>(&e)) return 4;
    return 1;
}

Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }
}  // namespace

extern "C" {

struct ref_camera {
    double pos[3], fwd[3], up[3];
    double vfov;
    int32_t width, height;
};
struct ref_render_cfg {
    int32_t spp, max_bounces;
    uint64_t seed;
    double hg_g, default_albedo, env[3], emission_scale;
};
struct ref_build_cfg {
    double variation_threshold;
    int32_t max_level, use_camera;
    double pixel_threshold, density_scale;
};
struct ref_build_stats {
    uint64_t leaf_count;
    int32_t max_depth, pad;
    double seconds;
    uint64_t criterion_splits, propagation_splits;
};

static_assert(sizeof(Tet) == 68, "reference Tet layout changed");
static_assert(sizeof(Vertex) == 12, "reference Vertex layout changed");

const char* ref_last_error() { return g_err.c_str(); }

static PinholeCamera make_cam(const ref_camera* c) {
    return PinholeCamera(v3(c->pos), v3(c->fwd), v3(c->up), c->vfov, c->width, c->height);
}
static RenderConfig make_rc(const ref_render_cfg* r) {
    RenderConfig rc;
    rc.spp = r->spp;
    rc.max_bounces = r->max_bounces;
    rc.seed = r->seed;
    rc.hg_g = r->hg_g;
    rc.default_albedo = r->default_albedo;
    rc.environment = v3(r->env);
    rc.emission_scale = r->emission_scale;
    return rc;
}

void ref_grid_free(void* h) { delete static_cast<TetGrid*>(h); }

void* ref_grid_init_roots(int max_level) {
    try {
        return new TetGrid(TetGrid::init_roots(max_level));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// acceptance.cpp:63-70 / test_tet_grid.cpp:43-51 fixture
void* ref_grid_fuzzed(int steps, uint64_t seed, int max_level) {
    try {
        auto g = std::make_unique<TetGrid>(TetGrid::init_roots(max_level));
        for (int i = 0; i < steps; ++i) {
            auto leaves = g->leaf_ids();
            g->refine_conforming(leaves[mix64(seed + 0x9e3779b97f4a7c15ull * (i + 1)) % leaves.size()]);
        }
        return g.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_grid_uniform(int levels) {
    try {
        auto g = std::make_unique<TetGrid>(TetGrid::init_roots());
        refine_uniform(*g, levels);
        return g.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int ref_grid_refine_conforming(void* h, uint32_t id) {
    try {
        static_cast<TetGrid*>(h)->refine_conforming(id);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void* ref_grid_build(const float* density, const float* temperature, const float* albedo, int nx, int ny, int nz,
                     const ref_build_cfg* bc, const ref_camera* cam, ref_build_stats* out) {
    try {
        DenseVolume vol(nx, ny, nz);
        std::memcpy(vol.channel("density").data(), density, vol.voxel_count() * sizeof(float));
        if (temperature)
            std::memcpy(vol.add_channel("temperature").data(), temperature, vol.voxel_count() * sizeof(float));
        if (albedo) std::memcpy(vol.add_channel("albedo").data(), albedo, vol.voxel_count() * sizeof(float));
        BuildConfig cfg;
        cfg.variation_threshold = bc->variation_threshold;
        cfg.max_level = bc->max_level;
        cfg.use_camera = bc->use_camera != 0;
        cfg.pixel_threshold = bc->pixel_threshold;
        cfg.density_scale = bc->density_scale;
        std::unique_ptr<PinholeCamera> pc;
        if (cam) pc = std::make_unique<PinholeCamera>(make_cam(cam));
        BuildStats st;
        auto g = std::make_unique<TetGrid>(build_adaptive_grid(vol, cfg, pc.get(), &st));
        if (out) {
            out->leaf_count = st.leaf_count;
            out->max_depth = st.max_depth;
            out->seconds = st.seconds;
            out->criterion_splits = st.criterion_splits;
            out->propagation_splits = st.propagation_splits;
        }
        return g.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_grid_assemble(const uint32_t* vq, uint64_t nv, const void* tets, uint64_t nt, const uint32_t* roots,
                        int max_level) {
    try {
        std::vector<Vertex> verts(nv);
        for (uint64_t i = 0; i < nv; ++i) verts[i].q = {vq[3 * i], vq[3 * i + 1], vq[3 * i + 2]};
        std::vector<Tet> tt(nt);
        std::memcpy(tt.data(), tets, nt * sizeof(Tet));
        std::array<TetId, 24> r{};
        for (int i = 0; i < 24; ++i) r[i] = roots[i];
        return new TetGrid(TetGrid::assemble(std::move(verts), std::move(tt), r, max_level));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_grid_load(const char* path) {
    try {
        return new TetGrid(load_grid(path));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int ref_grid_save(void* h, const char* path) {
    try {
        save_grid(*static_cast<TetGrid*>(h), path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// out: n_verts, n_tets, n_leaves, max_level
void ref_grid_counts(void* h, uint64_t* out) {
    auto* g = static_cast<TetGrid*>(h);
    out[0] = g->vertex_count();
    out[1] = g->tet_count();
    out[2] = g->leaf_count();
    out[3] = static_cast<uint64_t>(g->max_level());
}

// vq: 3*nv u32; tets: nt * 68-byte reference records; roots: 24 u32
void ref_grid_export(void* h, uint32_t* vq, void* tets, uint32_t* roots) {
    auto* g = static_cast<TetGrid*>(h);
    if (vq)
        for (std::size_t i = 0; i < g->vertex_count(); ++i)
            for (int k = 0; k < 3; ++k) vq[3 * i + k] = g->vertex(static_cast<VertexId>(i)).q[k];
    if (tets) std::memcpy(tets, g->tets().data(), g->tet_count() * sizeof(Tet));
    if (roots)
        for (int i = 0; i < 24; ++i) roots[i] = g->roots()[i];
}

// DenseVolume(nx, ny, nz) + channels (names[0] must be "density"), save_dvol
int ref_dvol_save(const char* path, int nx, int ny, int nz, int n_ch, const char* const* names,
                  const float* const* data) {
    try {
        DenseVolume v(nx, ny, nz);
        for (int c = 0; c < n_ch; ++c) {
            std::vector<float>& d = c == 0 ? v.channel(names[0]) : v.add_channel(names[c]);
            std::memcpy(d.data(), data[c], d.size() * sizeof(float));
        }
        v.save_dvol(path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// load_dvol; out dims[3], n_ch; with data != NULL also copies the channels
// (names: n_ch buffers of 256 bytes, data: n_ch arrays of nx*ny*nz floats)
int ref_dvol_load(const char* path, int* dims, int* n_ch, char** names, float** data) {
    try {
        DenseVolume v = DenseVolume::load_dvol(path);
        dims[0] = v.nx(), dims[1] = v.ny(), dims[2] = v.nz();
        *n_ch = static_cast<int>(v.channel_names().size());
        if (names && data)
            for (int c = 0; c < *n_ch; ++c) {
                const std::string& n = v.channel_names()[c];
                std::strncpy(names[c], n.c_str(), 255);
                names[c][255] = 0;
                const auto& d = v.channel(n);
                std::memcpy(data[c], d.data(), d.size() * sizeof(float));
            }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_write_pfm(const char* path, int w, int h, const double* sum, const double* sum_sq, const uint32_t* counts,
                  int variance) {
    try {
        ImageAccumulator img(w, h);
        std::memcpy(img.sum.data(), sum, img.sum.size() * sizeof(double));
        std::memcpy(img.sum_sq.data(), sum_sq, img.sum_sq.size() * sizeof(double));
        std::memcpy(img.sample_counts.data(), counts, img.sample_counts.size() * sizeof(uint32_t));
        if (variance) write_variance_pfm(path, img);
        else write_pfm(path, img);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// read_pfm; rgb (3*w*h floats, top-down) may be NULL to query the size
int ref_read_pfm(const char* path, int* w, int* h, float* rgb) {
    try {
        FloatImage img = read_pfm(path);
        *w = img.width, *h = img.height;
        if (rgb) std::memcpy(rgb, img.rgb.data(), img.rgb.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// returns 1 when valid; out: leaf_count, interior_faces, boundary_faces
int ref_grid_validate(void* h, char* msg, int cap, uint64_t* out) {
    auto rep = static_cast<TetGrid*>(h)->validate();
    if (msg && cap > 0) {
        std::strncpy(msg, rep.first_violation.c_str(), static_cast<std::size_t>(cap - 1));
        msg[cap - 1] = 0;
    }
    if (out) {
        out[0] = rep.leaf_count;
        out[1] = rep.interior_faces;
        out[2] = rep.boundary_faces;
    }
    return rep.ok ? 1 : 0;
}

void ref_grid_fill_density(void* h, float lambda) {
    auto* g = static_cast<TetGrid*>(h);
    for (TetId t : g->leaf_ids()) {
        g->payload(t).density = lambda;
        g->payload(t).mask = 1;
    }
}

// payload of one tet: density, temperature, albedo, mask
void ref_grid_set_payload(void* h, uint32_t t, float density, float temperature, float albedo, uint32_t mask) {
    auto& p = static_cast<TetGrid*>(h)->payload(t);
    p.density = density;
    p.temperature = temperature;
    p.albedo = albedo;
    p.mask = static_cast<std::uint8_t>(mask);
}

int ref_locate_point(void* h, const double* p, uint32_t* out) {
    try {
        *out = static_cast<TetGrid*>(h)->locate_point(v3(p));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// returns slot or -1
int ref_exit_face(void* h, uint32_t cell, const double* pos, const double* dir, double* t) {
    auto ef = exit_face(*static_cast<TetGrid*>(h), cell, v3(pos), v3(dir));
    if (!ef) return -1;
    *t = ef->t;
    return ef->slot;
}

// rays: n x [ox oy oz dx dy dz tmin tmax]. Writes up to cap segments; offsets has
// n+1 entries. Returns the total number of segments (may exceed cap).
int64_t ref_march_segments(void* h, const double* rays, uint64_t n, uint32_t* cells, double* t0, double* t1,
                           uint64_t* offsets, uint64_t cap, uint64_t* stats) {
    auto* g = static_cast<TetGrid*>(h);
    TraceStats st;
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double* r = rays + 8 * i;
        Ray ray{v3(r), v3(r + 3), r[6], r[7]};
        auto segs = march_segments(*g, ray, &st);
        if (offsets) offsets[i] = k;
        for (auto& s : segs) {
            if (k < cap) {
                cells[k] = s.cell;
                t0[k] = s.t_enter;
                t1[k] = s.t_exit;
            }
            ++k;
        }
    }
    if (offsets) offsets[n] = k;
    if (stats) {
        stats[0] = st.cells_visited;
        stats[1] = st.degenerate_paths;
    }
    return static_cast<int64_t>(k);
}

// cmd_validate's spot-check rays (cli.cpp:552-569; sphere_dir is file-local
// there, restated here): origin on the radius-2 sphere, target in the middle half
void ref_spot_rays(uint64_t seed, int n, double* out) {
    const Vec3 center{0.5, 0.5, 0.5};
    for (int i = 0; i < n; ++i) {
        RngStream rng(seed, 0x76616c6964617465ull, static_cast<std::uint64_t>(i));
        const double u1 = rng.next(), u2 = rng.next();
        const double z = 1.0 - 2.0 * u1;
        const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        const double phi = 2.0 * 3.14159265358979323846 * u2;
        const Vec3 origin = center + Vec3{r * std::cos(phi), r * std::sin(phi), z} * 2.0;
        const double tx = 0.25 + 0.5 * rng.next(), ty = 0.25 + 0.5 * rng.next(), tz = 0.25 + 0.5 * rng.next();
        const Ray ray{origin, normalize(Vec3{tx, ty, tz} - origin)};
        double* o = out + 8 * i;
        o[0] = ray.origin.x, o[1] = ray.origin.y, o[2] = ray.origin.z;
        o[3] = ray.dir.x, o[4] = ray.dir.y, o[5] = ray.dir.z, o[6] = ray.t_min, o[7] = ray.t_max;
    }
}

// the spot-check loop itself (cli.cpp:569-595) with the reference's
// march_segments and BruteForceTraverser
void ref_spot_checks(void* h, int n, uint64_t seed, int* failures, int* first) {
    const TetGrid& grid = *static_cast<TetGrid*>(h);
    BruteForceTraverser oracle(grid);
    std::vector<double> rays(8 * static_cast<size_t>(n));
    ref_spot_rays(seed, n, rays.data());
    *failures = 0, *first = -1;
    auto keep = [](const std::vector<RaySegment>& in) {
        std::vector<RaySegment> o;
        for (const auto& s : in)
            if (s.t_exit - s.t_enter > 1e-12) o.push_back(s);
        return o;
    };
    for (int i = 0; i < n; ++i) {
        const double* r = &rays[8 * static_cast<size_t>(i)];
        Ray ray{v3(r), v3(r + 3), r[6], r[7]};
        auto got = keep(march_segments(grid, ray));
        auto want = keep(oracle.segments(ray));
        bool ok = got.size() == want.size();
        for (std::size_t k = 0; ok && k < got.size(); ++k)
            ok = got[k].cell == want[k].cell &&
                 std::fabs((got[k].t_exit - got[k].t_enter) - (want[k].t_exit - want[k].t_enter)) <= 1e-9;
        if (!ok) {
            ++*failures;
            if (*first < 0) *first = i;
        }
    }
}

// tetvol::trace of one ray with RngStream(seed, pixel, sample); stats: cells, degenerate
void ref_trace_ray(void* h, const double* r, const ref_render_cfg* c, uint64_t seed, uint64_t pixel, uint64_t sample,
                   double* out, uint64_t* stats) {
    Ray ray{v3(r), v3(r + 3), r[6], r[7]};
    RngStream rng(seed, pixel, sample);
    TraceStats st;
    const Vec3 L = trace(*static_cast<TetGrid*>(h), ray, make_rc(c), rng, &st);
    out[0] = L.x, out[1] = L.y, out[2] = L.z;
    stats[0] += st.cells_visited;
    stats[1] += st.degenerate_paths;
}

double ref_march_transmittance(void* h, const double* r) {
    Ray ray{v3(r), v3(r + 3), r[6], r[7]};
    return march_transmittance(*static_cast<TetGrid*>(h), ray);
}

// out: collided, px, py, pz, cell, distance
void ref_sample_free_path(void* h, const double* r, uint64_t seed, uint64_t pixel, uint64_t sample, double* out) {
    Ray ray{v3(r), v3(r + 3), r[6], r[7]};
    RngStream rng(seed, pixel, sample);
    auto fp = sample_free_path(*static_cast<TetGrid*>(h), ray, rng);
    out[0] = fp.collided;
    out[1] = fp.position.x;
    out[2] = fp.position.y;
    out[3] = fp.position.z;
    out[4] = fp.cell;
    out[5] = fp.distance;
}

void ref_rng_draws(uint64_t seed, uint64_t pixel, uint64_t sample, int n, double* out) {
    RngStream rng(seed, pixel, sample);
    for (int i = 0; i < n; ++i) out[i] = rng.next();
}

uint64_t ref_mix64(uint64_t x) { return mix64(x); }

double ref_hg_sample_cos(double g, double xi) { return hg_sample_cos(g, xi); }

void ref_sample_phase_hg(const double* dir, double g, uint64_t seed, uint64_t pixel, uint64_t sample, double* out) {
    RngStream rng(seed, pixel, sample);
    Vec3 w = sample_phase_hg(v3(dir), g, rng);
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
}

void ref_emission_color(double t, double* out) {
    Vec3 c = emission_color(t);
    out[0] = c.x;
    out[1] = c.y;
    out[2] = c.z;
}

int ref_primary_ray(const ref_camera* c, int px, int py, double jx, double jy, double* out) {
    try {
        Ray r = make_cam(c).primary_ray(px, py, jx, jy);
        out[0] = r.origin.x, out[1] = r.origin.y, out[2] = r.origin.z;
        out[3] = r.dir.x, out[4] = r.dir.y, out[5] = r.dir.z;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// corners: 12 doubles; out[0] = outside_frustum, out[1] = projected size
int ref_camera_tet_tests(const ref_camera* c, const double* corners, double* out) {
    try {
        PinholeCamera cam = make_cam(c);
        std::array<Vec3, 4> cs{v3(corners), v3(corners + 3), v3(corners + 6), v3(corners + 9)};
        out[0] = cam.tet_outside_frustum(cs) ? 1.0 : 0.0;
        out[1] = cam.projected_size_pixels(cs);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Radiance of one camera sample through the reference integrator (trace()).
void ref_trace_sample(void* h, const ref_camera* c, const ref_render_cfg* r, int px, int py, int s, double* out,
                      uint64_t* cells) {
    PinholeCamera cam = make_cam(c);
    RenderConfig rc = make_rc(r);
    RngStream rng(rc.seed, static_cast<uint64_t>(py) * cam.width() + px, static_cast<uint64_t>(s));
    const double jx = rng.next();
    const double jy = rng.next();
    TraceStats st;
    Vec3 L = trace(*static_cast<TetGrid*>(h), cam.primary_ray(px, py, jx, jy), rc, rng, &st);
    out[0] = L.x, out[1] = L.y, out[2] = L.z;
    if (cells) *cells = st.cells_visited;
}

// Full-frame render through tetvol::render. Buffers are optional (nullptr skips
// the copy). stats: cells_visited, paths_traced, degenerate_paths.
int ref_render(void* h, const ref_camera* c, const ref_render_cfg* r, int threads, double* sum, double* sum_sq,
               uint32_t* counts, uint64_t* stats, double* seconds) {
    try {
        ImageAccumulator acc = render(*static_cast<TetGrid*>(h), make_cam(c), make_rc(r), threads);
        if (sum) std::memcpy(sum, acc.sum.data(), acc.sum.size() * sizeof(double));
        if (sum_sq) std::memcpy(sum_sq, acc.sum_sq.data(), acc.sum_sq.size() * sizeof(double));
        if (counts) std::memcpy(counts, acc.sample_counts.data(), acc.sample_counts.size() * sizeof(uint32_t));
        if (stats) {
            stats[0] = acc.cells_visited;
            stats[1] = acc.paths_traced;
            stats[2] = acc.degenerate_paths;
        }
        if (seconds) *seconds = acc.seconds;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Regular-grid comparator (config 5): RegularGrid::from_volume + render_reference.
int ref_render_regular(const float* density, int nx, int ny, int nz, double density_scale, const ref_camera* c,
                       const ref_render_cfg* r, int threads, double* sum, double* sum_sq, uint32_t* counts,
                       uint64_t* stats, double* seconds) {
    try {
        DenseVolume vol(nx, ny, nz);
        std::memcpy(vol.channel("density").data(), density, vol.voxel_count() * sizeof(float));
        RegularGrid rg = RegularGrid::from_volume(vol, density_scale);
        ImageAccumulator acc = render_reference(rg, make_cam(c), make_rc(r), threads);
        if (sum) std::memcpy(sum, acc.sum.data(), acc.sum.size() * sizeof(double));
        if (sum_sq) std::memcpy(sum_sq, acc.sum_sq.data(), acc.sum_sq.size() * sizeof(double));
        if (counts) std::memcpy(counts, acc.sample_counts.data(), acc.sample_counts.size() * sizeof(uint32_t));
        if (stats) {
            stats[0] = acc.cells_visited;
            stats[1] = acc.paths_traced;
            stats[2] = acc.degenerate_paths;
        }
        if (seconds) *seconds = acc.seconds;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// DDA segments through a regular grid (regular_grid.hpp:58).
int64_t ref_dda_segments(const float* density, int nx, int ny, int nz, double density_scale, const double* rays,
                         uint64_t n, uint32_t* cells, double* t0, double* t1, uint64_t* offsets, uint64_t cap) {
    DenseVolume vol(nx, ny, nz);
    std::memcpy(vol.channel("density").data(), density, vol.voxel_count() * sizeof(float));
    RegularGrid rg = RegularGrid::from_volume(vol, density_scale);
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double* r = rays + 8 * i;
        Ray ray{v3(r), v3(r + 3), r[6], r[7]};
        auto segs = dda_march(rg, ray);
        if (offsets) offsets[i] = k;
        for (auto& s : segs) {
            if (k < cap) {
                cells[k] = s.cell;
                t0[k] = s.t_enter;
                t1[k] = s.t_exit;
            }
            ++k;
        }
    }
    if (offsets) offsets[n] = k;
    return static_cast<int64_t>(k);
}

// density_stats_in_tet (ownership form, builder.hpp:44-45): min, max, mean, count
void ref_density_stats(void* h, const float* density, int nx, int ny, int nz, uint32_t leaf, double* out) {
    DenseVolume vol(nx, ny, nz);
    std::memcpy(vol.channel("density").data(), density, vol.voxel_count() * sizeof(float));
    DensityStats s = density_stats_in_tet(vol, *static_cast<TetGrid*>(h), leaf);
    out[0] = s.min;
    out[1] = s.max;
    out[2] = s.mean;
    out[3] = static_cast<double>(s.count);
}

}  // extern "C"

extern "C" {
// acceptance.cpp:49-61 random_cube_ray, computed with the reference's own types
void ref_random_cube_rays(uint64_t seed, uint64_t salt, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        RngStream rng(seed, salt, i);
        double u1 = rng.next(), u2 = rng.next();
        double z = 1.0 - 2.0 * u1;
        double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        double phi = 2.0 * 3.14159265358979323846 * u2;
        Vec3 origin = Vec3{0.5, 0.5, 0.5} + Vec3{r * std::cos(phi), r * std::sin(phi), z} * 2.0;
        double a = rng.next(), b = rng.next(), c = rng.next();
        Vec3 target{0.25 + 0.5 * a, 0.25 + 0.5 * b, 0.25 + 0.5 * c};
        Vec3 d = normalize(target - origin);
        double* w = out + 8 * i;
        w[0] = origin.x, w[1] = origin.y, w[2] = origin.z, w[3] = d.x, w[4] = d.y, w[5] = d.z, w[6] = 0.0;
        w[7] = std::numeric_limits<double>::infinity();
    }
}
}
