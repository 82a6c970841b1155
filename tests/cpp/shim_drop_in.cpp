// Drop-in check of include/tetvol_b200.hpp against the UNMODIFIED reference
// library (linked from oracle/_ref): the same TetGrid / PinholeCamera /
// RenderConfig / BuildConfig values go through tetvol:: (CPU) and
// tetvol::b200:: (GPU), and the results must be bit-identical.
// Built by tests/cpp/Makefile; run by tests/test_gpu_shim.py on a GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tetvol_b200.hpp"

using namespace tetvol;

static DenseVolume blob(int n) {
    DenseVolume v(n, n, n);
    auto& d = v.channel("density");
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                Vec3 p = v.voxel_center(i, j, k) - Vec3{0.5, 0.5, 0.5};
                double t = std::max(0.0, 1.0 - length_sq(p) / (0.45 * 0.45));
                d[v.index(i, j, k)] = static_cast<float>(t * t);
            }
    return v;
}

// field-wise (padding bytes are unspecified)
static bool same_tets(const TetGrid& a, const TetGrid& b) {
    if (a.tet_count() != b.tet_count() || a.vertex_count() != b.vertex_count()) return false;
    for (size_t v = 0; v < a.vertex_count(); ++v)
        for (int k = 0; k < 3; ++k)
            if (a.vertices()[v].q[k] != b.vertices()[v].q[k]) return false;
    for (size_t t = 0; t < a.tet_count(); ++t) {
        const Tet &x = a.tets()[t], &y = b.tets()[t];
        for (int k = 0; k < 4; ++k)
            if (x.verts[k] != y.verts[k] || x.neighbors[k] != y.neighbors[k] || x.normal_ids[k] != y.normal_ids[k])
                return false;
        if (x.children[0] != y.children[0] || x.children[1] != y.children[1] || x.parent != y.parent ||
            x.level != y.level || x.payload.mask != y.payload.mask ||
            std::memcmp(&x.payload.density, &y.payload.density, 4) ||
            std::memcmp(&x.payload.temperature, &y.payload.temperature, 4) ||
            std::memcmp(&x.payload.albedo, &y.payload.albedo, 4))
            return false;
    }
    for (int r = 0; r < 24; ++r)
        if (a.roots()[r] != b.roots()[r]) return false;
    return true;
}

static std::vector<std::array<uint32_t, 12>> leaf_set(const TetGrid& g) {
    std::vector<std::array<uint32_t, 12>> out;
    for (TetId t : g.leaf_ids()) {
        std::array<std::array<uint32_t, 3>, 4> c;
        for (int k = 0; k < 4; ++k) c[k] = g.vertex(g.tet(t).verts[k]).q;
        std::sort(c.begin(), c.end());
        std::array<uint32_t, 12> key;
        for (int k = 0; k < 4; ++k)
            for (int a = 0; a < 3; ++a) key[3 * k + a] = c[k][a];
        out.push_back(key);
    }
    std::sort(out.begin(), out.end());
    return out;
}

#define REQUIRE(x)                                                       \
    do {                                                                 \
        if (!(x)) {                                                      \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #x); \
            return 1;                                                    \
        }                                                                \
    } while (0)

int main() {
    DenseVolume vol = blob(48);
    BuildConfig bc;
    bc.variation_threshold = 0.15;
    bc.max_level = 11;
    bc.density_scale = 8.0;
    TetGrid ref = build_adaptive_grid(vol, bc);
    PinholeCamera cam({0.5, 0.5, -2}, {0, 0.05, 1}, {0, 1, 0}, 40, 96, 80);
    RenderConfig rc;
    rc.spp = 4;
    rc.max_bounces = 16;
    rc.seed = 5;
    rc.hg_g = 0.2;

    // render(): reference CPU vs GPU on the same uploaded grid
    ImageAccumulator a = render(ref, cam, rc, 0);
    b200::DeviceGrid dg(ref);
    ImageAccumulator b = b200::render(dg, cam, rc);
    REQUIRE(a.cells_visited == b.cells_visited);
    REQUIRE(a.degenerate_paths == b.degenerate_paths);
    REQUIRE(std::memcmp(a.sum.data(), b.sum.data(), a.sum.size() * sizeof(double)) == 0);
    REQUIRE(std::memcmp(a.sum_sq.data(), b.sum_sq.data(), a.sum_sq.size() * sizeof(double)) == 0);
    REQUIRE(a.sample_counts == b.sample_counts);

    // render_multi(): three ranks (all on device 0 here) give the same accumulator
    b200::DeviceGrid dg2(ref);
    ImageAccumulator m = b200::render_multi({&dg, &dg2, &dg}, cam, rc);
    REQUIRE(m.cells_visited == a.cells_visited);
    REQUIRE(std::memcmp(a.sum.data(), m.sum.data(), a.sum.size() * sizeof(double)) == 0);
    REQUIRE(std::memcmp(a.sum_sq.data(), m.sum_sq.data(), a.sum_sq.size() * sizeof(double)) == 0);
    REQUIRE(a.sample_counts == m.sample_counts);

    // build_adaptive_grid(): GPU build, downloaded, passes validate(), same leaves
    BuildStats st;
    b200::DeviceGrid built = b200::build_adaptive_grid(vol, bc, nullptr, &st);
    TetGrid back = built.download();
    REQUIRE(back.validate().ok);
    REQUIRE(back.leaf_count() == ref.leaf_count());
    REQUIRE(leaf_set(back) == leaf_set(ref));

    // march_segments(): batched on the GPU vs per ray on the CPU
    std::vector<Ray> rays;
    for (int i = 0; i < 500; ++i) {
        RngStream r(3, 7, i);
        Vec3 o{r.next() * 3 - 1, r.next() * 3 - 1, -1.5};
        Vec3 t{0.2 + 0.6 * r.next(), 0.2 + 0.6 * r.next(), 0.2 + 0.6 * r.next()};
        rays.push_back(Ray{o, normalize(t - o)});
    }
    auto segs = b200::march_segments(dg, rays);
    for (size_t i = 0; i < rays.size(); ++i) {
        auto want = march_segments(ref, rays[i]);
        REQUIRE(want.size() == segs[i].size());
        for (size_t k = 0; k < want.size(); ++k) {
            REQUIRE(want[k].cell == segs[i][k].cell);
            REQUIRE(want[k].t_enter == segs[i][k].t_enter);
            REQUIRE(want[k].t_exit == segs[i][k].t_exit);
        }
    }

    // .tgrid: our device-packed file loads in the reference with the same pools,
    // and the reference's file loads on the device with the same pools
    {
        const std::string p1 = "/tmp/shim_drop_in_a.tgrid", p2 = "/tmp/shim_drop_in_b.tgrid";
        b200::save_grid(dg, p1);
        TetGrid back = load_grid(p1);
        REQUIRE(back.tet_count() == ref.tet_count() && back.vertex_count() == ref.vertex_count());
        REQUIRE(same_tets(back, ref));
        save_grid(ref, p2);
        TetGrid dev_back = b200::load_grid_device(p2).download();
        REQUIRE(same_tets(dev_back, ref));
        try {
            b200::load_grid_device("/tmp/shim_drop_in_missing.tgrid");
            REQUIRE(false);
        } catch (const IoError&) {
        }
        std::remove(p1.c_str());
        std::remove(p2.c_str());
    }

    // trace / transmittance / free path agree with the reference entry points
    {
        std::vector<Ray> rr(rays.begin(), rays.begin() + 100);
        std::vector<uint64_t> px(rr.size()), sm(rr.size());
        for (size_t i = 0; i < rr.size(); ++i) px[i] = 5 * i + 1, sm[i] = i % 3;
        RenderConfig tc;
        tc.max_bounces = 12;
        auto L = b200::trace(dg, rr, tc, 9, px, sm);
        auto T = b200::march_transmittance(dg, rr);
        auto F = b200::sample_free_path(dg, rr, 9, px, sm);
        for (size_t i = 0; i < rr.size(); ++i) {
            RngStream r1(9, px[i], sm[i]), r2(9, px[i], sm[i]);
            const Vec3 want = trace(ref, rr[i], tc, r1);
            REQUIRE(std::memcmp(&want, &L[i], sizeof(Vec3)) == 0);
            REQUIRE(std::fabs(T[i] - march_transmittance(ref, rr[i])) <= 4e-16 * std::fabs(T[i]) + 1e-300);
            const FreePathSample f = sample_free_path(ref, rr[i], r2);
            REQUIRE(f.collided == F[i].collided && f.distance == F[i].distance && f.cell == F[i].cell);
        }
    }

    // exceptions map back to the reference types
    try {
        RenderConfig bad;
        bad.spp = 0;
        b200::render(dg, cam, bad);
        REQUIRE(false);
    } catch (const ConfigError&) {
    }
    std::printf("shim ok: %zu leaves, %llu cells, framebuffer bit-identical\n", ref.leaf_count(),
                static_cast<unsigned long long>(b.cells_visited));
    return 0;
}
