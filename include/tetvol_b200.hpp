// tetvol_b200.hpp — header-only C++ shim with the reference `tetvol` API
// shape over the C ABI (tetvol_b200.h).
//
// A caller of the reference library switches the hot path by including this
// header next to the reference headers and calling tetvol::b200::render /
// build_adaptive_grid / march_segments instead of tetvol::render /
// build_adaptive_grid / march_segments (tracer.hpp:49,84-85,
// builder.hpp:51-52). Arguments, return types, counters and exception types
// are the reference's own; status codes from the C ABI are rethrown as
// ConfigError / CameraError / GridError / OutsideGrid / std::runtime_error.
// The `threads` argument of render is accepted and ignored (the GPU is
// selected by `device`).
#pragma once

#include <array>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tetvol_b200.h"
#include "tetvol/builder.hpp"
#include "tetvol/camera.hpp"
#include "tetvol/image.hpp"
#include "tetvol/tet_grid.hpp"
#include "tetvol/tracer.hpp"
#include "tetvol/volume.hpp"

namespace tetvol::b200 {

static_assert(sizeof(tv_tet) == sizeof(Tet), "tv_tet must mirror tetvol::Tet byte for byte");
static_assert(sizeof(tv_vertex) == sizeof(Vertex), "tv_vertex must mirror tetvol::Vertex");

inline void check(int rc) {
    if (rc == TV_OK) return;
    const std::string msg = tv_last_error();
    switch (rc) {
        case TV_ERR_CONFIG: throw ConfigError(msg);
        case TV_ERR_CAMERA: throw CameraError(msg);
        case TV_ERR_GRID: throw GridError(msg);
        case TV_ERR_OUTSIDE: throw OutsideGrid(msg);
        case TV_ERR_FORMAT: throw FormatError(msg);
        case TV_ERR_IO: throw IoError(msg);
        default: throw std::runtime_error("tetvol_b200: " + msg);
    }
}

// A constructed PinholeCamera, converted without re-normalising its basis.
inline tv_camera to_c(const PinholeCamera& c) {
    tv_camera o{};
    const Vec3 p = c.position(), f = c.forward(), u = c.up();
    o.position[0] = p.x, o.position[1] = p.y, o.position[2] = p.z;
    o.forward[0] = f.x, o.forward[1] = f.y, o.forward[2] = f.z;
    o.up[0] = u.x, o.up[1] = u.y, o.up[2] = u.z;
    o.vfov_degrees = c.vfov_degrees();
    o.width = c.width();
    o.height = c.height();
    o.basis_final = 1;
    return o;
}

inline tv_render_config to_c(const RenderConfig& r) {
    tv_render_config o{};
    o.spp = r.spp;
    o.max_bounces = r.max_bounces;
    o.seed = r.seed;
    o.hg_g = r.hg_g;
    o.default_albedo = r.default_albedo;
    o.environment[0] = r.environment.x, o.environment[1] = r.environment.y, o.environment[2] = r.environment.z;
    o.emission_scale = r.emission_scale;
    o.exposure = r.exposure;
    o.gamma = r.gamma;
    return o;
}

inline tv_build_config to_c(const BuildConfig& b) {
    tv_build_config o{};
    o.variation_threshold = b.variation_threshold;
    o.max_level = b.max_level;
    o.use_camera = b.use_camera ? 1 : 0;
    o.pixel_threshold = b.pixel_threshold;
    o.density_scale = b.density_scale;
    return o;
}

// A TetGrid resident in one GPU's HBM. Move-only; frees on destruction.
class DeviceGrid {
public:
    explicit DeviceGrid(const TetGrid& g, int device = 0) {
        std::array<uint32_t, 24> roots{};
        for (int i = 0; i < 24; ++i) roots[i] = g.roots()[i];
        check(tv_grid_upload(reinterpret_cast<const tv_vertex*>(g.vertices().data()), g.vertex_count(),
                             reinterpret_cast<const tv_tet*>(g.tets().data()), g.tet_count(), roots.data(),
                             g.max_level(), device, &h_));
    }
    explicit DeviceGrid(tv_grid* h) : h_(h) {}
    DeviceGrid(DeviceGrid&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceGrid& operator=(DeviceGrid&& o) noexcept {
        if (this != &o) {
            tv_grid_free(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    DeviceGrid(const DeviceGrid&) = delete;
    DeviceGrid& operator=(const DeviceGrid&) = delete;
    ~DeviceGrid() { tv_grid_free(h_); }

    const tv_grid* handle() const { return h_; }
    tv_grid_info info() const {
        tv_grid_info i{};
        check(tv_grid_get_info(h_, &i));
        return i;
    }
    // Back to a reference TetGrid (TetGrid::assemble; validate() applies).
    TetGrid download() const {
        const tv_grid_info i = info();
        std::vector<Vertex> v(i.n_vertices);
        std::vector<Tet> t(i.n_tets);
        std::array<uint32_t, 24> r{};
        check(tv_grid_download(h_, reinterpret_cast<tv_vertex*>(v.data()), reinterpret_cast<tv_tet*>(t.data()),
                               r.data()));
        std::array<TetId, 24> roots{};
        for (int k = 0; k < 24; ++k) roots[k] = r[k];
        return TetGrid::assemble(std::move(v), std::move(t), roots, i.max_level);
    }

private:
    tv_grid* h_ = nullptr;
};

// builder.hpp:59-60 — the reference's TGRD v1 file, packed / unpacked on the device
inline void save_grid(const DeviceGrid& grid, const std::string& path) { check(tv_grid_save(grid.handle(), path.c_str())); }
inline DeviceGrid load_grid_device(const std::string& path, int device = 0) {
    tv_grid* h = nullptr;
    check(tv_grid_load(path.c_str(), device, &h));
    return DeviceGrid(h);
}

// tracer.hpp:84-85
inline ImageAccumulator render(const DeviceGrid& grid, const PinholeCamera& camera, const RenderConfig& cfg,
                               int /*threads*/ = 0) {
    ImageAccumulator acc(camera.width(), camera.height());
    tv_framebuffer fb{acc.sum.data(), acc.sum_sq.data(), acc.sample_counts.data()};
    tv_render_stats st{};
    const tv_camera c = to_c(camera);
    const tv_render_config r = to_c(cfg);
    check(tv_render(grid.handle(), &c, &r, &fb, &st));
    acc.cells_visited = st.cells_visited;
    acc.paths_traced = st.paths_traced;
    acc.degenerate_paths = st.degenerate_paths;
    acc.seconds = st.seconds;
    return acc;
}

// render() over several GPUs from one process: one DeviceGrid per device
// (the same grid uploaded or built on each); the same ImageAccumulator bit for bit.
inline ImageAccumulator render_multi(const std::vector<const DeviceGrid*>& grids, const PinholeCamera& camera,
                                     const RenderConfig& cfg) {
    ImageAccumulator acc(camera.width(), camera.height());
    tv_framebuffer fb{acc.sum.data(), acc.sum_sq.data(), acc.sample_counts.data()};
    tv_render_stats st{};
    const tv_camera c = to_c(camera);
    const tv_render_config r = to_c(cfg);
    std::vector<const tv_grid*> hs;
    for (const DeviceGrid* g : grids) hs.push_back(g->handle());
    check(tv_render_multi(hs.data(), static_cast<int32_t>(hs.size()), &c, &r, &fb, &st));
    acc.cells_visited = st.cells_visited;
    acc.paths_traced = st.paths_traced;
    acc.degenerate_paths = st.degenerate_paths;
    acc.seconds = st.seconds;
    return acc;
}

// Drop-in overload on a host TetGrid (uploads once per call).
inline ImageAccumulator render(const TetGrid& grid, const PinholeCamera& camera, const RenderConfig& cfg,
                               int threads = 0, int device = 0) {
    return render(DeviceGrid(grid, device), camera, cfg, threads);
}

// builder.hpp:51-52 on the GPU; the grid stays in HBM (download() for a TetGrid).
inline DeviceGrid build_adaptive_grid(const DenseVolume& vol, const BuildConfig& cfg,
                                      const PinholeCamera* camera = nullptr, BuildStats* stats = nullptr,
                                      int device = 0) {
    const tv_build_config b = to_c(cfg);
    tv_camera c{};
    if (camera) c = to_c(*camera);
    tv_grid* h = nullptr;
    tv_build_stats st{};
    const float* temp = vol.has_channel("temperature") ? vol.channel("temperature").data() : nullptr;
    const float* alb = vol.has_channel("albedo") ? vol.channel("albedo").data() : nullptr;
    check(tv_build(vol.channel("density").data(), temp, alb, vol.nx(), vol.ny(), vol.nz(), &b,
                   camera ? &c : nullptr, device, &h, &st));
    if (stats) {
        stats->leaf_count = st.leaf_count;
        stats->max_depth = st.max_depth;
        stats->seconds = st.seconds;
        stats->criterion_splits = st.criterion_splits;
        stats->propagation_splits = st.propagation_splits;
    }
    return DeviceGrid(h);
}

// tracer.hpp:49, batched over many rays.
inline std::vector<std::vector<RaySegment>> march_segments(const DeviceGrid& grid, const std::vector<Ray>& rays,
                                                           TraceStats* stats = nullptr) {
    std::vector<tv_ray> rr(rays.size());
    for (size_t i = 0; i < rays.size(); ++i) {
        const Ray& r = rays[i];
        rr[i] = tv_ray{{r.origin.x, r.origin.y, r.origin.z}, {r.dir.x, r.dir.y, r.dir.z}, r.t_min, r.t_max};
    }
    std::vector<uint64_t> off(rays.size() + 1);
    uint64_t total = 0, deg = 0;
    check(tv_march_segments(grid.handle(), rr.data(), rr.size(), nullptr, off.data(), 0, &total, &deg));
    std::vector<tv_segment> seg(total);
    check(tv_march_segments(grid.handle(), rr.data(), rr.size(), seg.data(), off.data(), total, &total, &deg));
    std::vector<std::vector<RaySegment>> out(rays.size());
    for (size_t i = 0; i < rays.size(); ++i)
        for (uint64_t k = off[i]; k < off[i + 1]; ++k) out[i].push_back(RaySegment{seg[k].cell, seg[k].t_enter, seg[k].t_exit});
    if (stats) {
        stats->cells_visited += total;
        stats->degenerate_paths += deg;
    }
    return out;
}

inline std::vector<tv_ray> to_c(const std::vector<Ray>& rays) {
    std::vector<tv_ray> rr(rays.size());
    for (size_t i = 0; i < rays.size(); ++i) {
        const Ray& r = rays[i];
        rr[i] = tv_ray{{r.origin.x, r.origin.y, r.origin.z}, {r.dir.x, r.dir.y, r.dir.z}, r.t_min, r.t_max};
    }
    return rr;
}

// march_transmittance (tracer.hpp:52), batched
inline std::vector<double> march_transmittance(const DeviceGrid& grid, const std::vector<Ray>& rays,
                                               TraceStats* stats = nullptr) {
    const auto rr = to_c(rays);
    std::vector<double> out(rays.size());
    uint64_t st[2] = {0, 0};
    check(tv_march_transmittance(grid.handle(), rr.data(), rr.size(), nullptr, out.data(), st));
    if (stats) stats->cells_visited += st[0], stats->degenerate_paths += st[1];
    return out;
}

// trace / sample_free_path (tracer.hpp:63, 78-79), batched; ray i uses RngStream(seed, pixels[i], samples[i])
inline std::vector<Vec3> trace(const DeviceGrid& grid, const std::vector<Ray>& rays, const RenderConfig& cfg,
                               uint64_t seed, const std::vector<uint64_t>& pixels,
                               const std::vector<uint64_t>& samples, TraceStats* stats = nullptr) {
    const auto rr = to_c(rays);
    const tv_render_config rc = to_c(cfg);
    std::vector<double> rgb(3 * rays.size());
    uint64_t st[2] = {0, 0};
    check(tv_trace_rays(grid.handle(), rr.data(), rr.size(), &rc, seed, pixels.data(), samples.data(), rgb.data(), st));
    if (stats) stats->cells_visited += st[0], stats->degenerate_paths += st[1];
    std::vector<Vec3> out(rays.size());
    for (size_t i = 0; i < rays.size(); ++i) out[i] = Vec3{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return out;
}

inline std::vector<FreePathSample> sample_free_path(const DeviceGrid& grid, const std::vector<Ray>& rays,
                                                    uint64_t seed, const std::vector<uint64_t>& pixels,
                                                    const std::vector<uint64_t>& samples,
                                                    TraceStats* stats = nullptr) {
    const auto rr = to_c(rays);
    std::vector<tv_free_path> fp(rays.size());
    uint64_t st[2] = {0, 0};
    check(tv_sample_free_path(grid.handle(), rr.data(), rr.size(), seed, pixels.data(), samples.data(), fp.data(), st));
    if (stats) stats->cells_visited += st[0], stats->degenerate_paths += st[1];
    std::vector<FreePathSample> out(rays.size());
    for (size_t i = 0; i < rays.size(); ++i) {
        out[i].collided = fp[i].collided != 0;
        out[i].position = Vec3{fp[i].position[0], fp[i].position[1], fp[i].position[2]};
        out[i].cell = fp[i].cell;
        out[i].distance = fp[i].distance;
    }
    return out;
}
}  // namespace tetvol::b200
