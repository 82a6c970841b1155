"""Optional free-flight estimators (csrc/tv_tracking.cu): delta and ratio
tracking over the per-tet majorant. They are not bit-comparable with the
reference, which uses regular tracking (path_integrator.hpp:49-61; SURVEY.md
F1), so they are checked in distribution against the reference itself: the
exact optical depth of the oracle's marcher (transmittance) and the oracle's
regular-tracking render (per-pixel z-scores within Monte Carlo error, the
acceptance-9 style criterion of acceptance.cpp:372-407).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tv():
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tv


def _media_grid(tv, steps=300, seed=0x61):
    g = O.fuzzed(O.c_oracle(), steps, seed)
    p = g.pools()
    rng = np.random.default_rng(seed)
    lm = p.leaf_mask
    p.tets["density"][lm] = np.where(rng.random(lm.sum()) < 0.3, 0.0, rng.random(lm.sum()) * 6).astype(np.float32)
    p.tets["mask"][lm] = 1
    return O.from_pools(O.c_oracle(), p), tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)


def _vacuum(tv):
    vp = O.init_roots(O.c_oracle()).pools()
    return tv.TetGrid.upload(vp.vq, vp.tets.view(tv.TET_DTYPE), vp.roots, 48)


@pytest.mark.parametrize("mode,scale", [(1, 1.0), (1, 3.0), (2, 1.0), (2, 2.0)])
def test_transmittance_estimators_unbiased(tv, mode, scale):
    """Mean of N estimates per ray against exp(-tau) of the exact optical depth
    (the oracle marcher's segments): per-ray z-scores within 5.5 sigma, and
    their average within 5 / sqrt(rays)."""
    rg, dg = _media_grid(tv)
    rays = O.random_cube_rays(21, 0x747261636b, 200)
    rays[::4, 7] = rays[::4, 6] + 0.3  # finite t_max
    _, tr_exact, _, _ = tv.march_transmittance(dg, rays)
    n = 2048
    rep = np.repeat(rays, n, axis=0)
    samples = np.tile(np.arange(n, dtype=np.uint64), len(rays))
    pixels = np.repeat(np.arange(len(rays), dtype=np.uint64), n)
    est, cells, deg = tv.transmittance_tracking(dg, rep, mode, scale, 5, pixels, samples)
    assert deg == 0 and cells > 0
    est = est.reshape(len(rays), n)
    assert np.all((est >= 0.0) & (est <= 1.0))
    if mode == 1:
        assert np.all((est == 0.0) | (est == 1.0))  # delta tracking: blocked or not
    mean = est.mean(axis=1)
    var = np.maximum(est.var(axis=1, ddof=1), tr_exact * (1 - tr_exact) / 4) / n  # floor: rays with T near 0 / 1
    z = (mean - tr_exact) / np.sqrt(np.maximum(var, 1e-30))
    z[(tr_exact == 1.0) & (mean == 1.0)] = 0.0
    assert np.max(np.abs(z)) < 5.5, (np.argmax(np.abs(z)), mean[np.argmax(np.abs(z))])
    assert abs(z.mean()) < 5.0 / np.sqrt(len(rays))


def test_regular_mode_is_the_reference_path(tv):
    rg, dg = _media_grid(tv)
    rays = O.random_cube_rays(3, 0x726567, 300)
    _, tr, _, _ = tv.march_transmittance(dg, rays)
    est, _, _ = tv.transmittance_tracking(dg, rays, tv.TRACK_REGULAR)
    assert np.array_equal(est.view(np.uint64), tr.view(np.uint64))
    cam = tv.PinholeCamera((0.4, 0.5, -1.6), (0, 0, 1), (0, 1, 0), 45, 40, 30)
    rc = tv.RenderConfig(spp=4, max_bounces=8, seed=2)
    a = tv.render(dg, cam, rc)
    b = tv.render_tracking(dg, cam, rc, tv.TRACK_REGULAR)
    assert np.array_equal(a.sum.view(np.uint64), b.sum.view(np.uint64)) and a.cells_visited == b.cells_visited


def test_vacuum_exact(tv):
    vac = _vacuum(tv)
    rays = O.random_cube_rays(4, 0x766163, 64)
    for mode in (1, 2):
        est, _, _ = tv.transmittance_tracking(vac, rays, mode, 1.5, 1, 0, np.arange(64, dtype=np.uint64))
        assert np.all(est == 1.0)
    b = tv.render_tracking(vac, tv.PinholeCamera(width=24, height=16), tv.RenderConfig(spp=3, environment=(0.25, 0.5, 2.0)))
    m = b.mean()
    assert np.all(m[..., 0] == 0.25) and np.all(m[..., 1] == 0.5) and np.all(m[..., 2] == 2.0)
    assert b.paths_traced == 24 * 16 * 3 and np.all(b.sample_counts == 3)


@pytest.mark.parametrize("scale", [1.0, 2.5])
def test_delta_render_matches_reference_in_distribution(tv, scale):
    """Delta-tracking render against the oracle's regular-tracking render of the
    C1 grid (multi-bounce, 64 spp): per-pixel z of the mean difference."""
    vol = O.gen_volume("blob", 64)
    g, _ = O.build(O.c_oracle(), vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
    p = g.pools()
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    w, h, spp = 64, 48, 64
    kw = dict(spp=spp, max_bounces=64, seed=11, hg_g=0.3)
    a = g.render(O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, w, h), O.render_cfg(**kw), 0)
    b = tv.render_tracking(dg, tv.PinholeCamera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, w, h),
                           tv.RenderConfig(**kw), tv.TRACK_DELTA, scale)
    assert b.degenerate_paths == 0 and b.paths_traced == w * h * spp
    ma, mb = a["sum"] / spp, b.sum / spp
    va = np.maximum(a["sum_sq"] / spp - ma * ma, 0) / spp
    vb = np.maximum(b.sum_sq / spp - mb * mb, 0) / spp
    se = np.sqrt(va + vb)
    live = se > 0
    assert np.array_equal(ma[~live], mb[~live])  # noise-free pixels (rays missing the medium) agree exactly
    z = (mb[live] - ma[live]) / se[live]
    assert np.mean(np.abs(z) > 3.0) < 0.015, np.mean(np.abs(z) > 3.0)
    # the image means agree within their Monte Carlo error
    assert abs(mb.mean() - ma.mean()) < 4 * np.sqrt((va + vb).sum()) / ma.size
    # at scale 1 a tentative collision is real: steps per path match regular tracking's (same tets crossed
    # in distribution); null collisions never add steps
    assert 0.9 < b.cells_visited / a["cells_visited"] < 1.1


def test_tracking_errors(tv):
    vac = _vacuum(tv)
    cam, rc = tv.PinholeCamera(width=8, height=8), tv.RenderConfig(spp=1)
    with pytest.raises(tv.ConfigError, match="ratio tracking"):
        tv.render_tracking(vac, cam, rc, tv.TRACK_RATIO)
    with pytest.raises(tv.ConfigError, match="majorant"):
        tv.render_tracking(vac, cam, rc, tv.TRACK_DELTA, 0.5)
    with pytest.raises(tv.ConfigError, match="majorant"):
        tv.transmittance_tracking(vac, O.random_cube_rays(1, 1, 4), tv.TRACK_RATIO, float("inf"))
    with pytest.raises(tv.ConfigError, match="unknown"):
        tv.transmittance_tracking(vac, O.random_cube_rays(1, 1, 4), 7)
    with pytest.raises(tv.ConfigError):
        tv.render_tracking(vac, cam, tv.RenderConfig(spp=0), tv.TRACK_DELTA)


def test_delta_render_emission_albedo_in_distribution(tv):
    """Delta tracking with per-cell albedo and temperature emission (mask bits 2,
    4) on a fuzzed grid, against the oracle's regular-tracking render."""
    C = O.c_oracle()
    g = O.fuzzed(C, 300, 0x77)
    p = g.pools()
    rng = np.random.default_rng(5)
    leaf = p.leaf_mask
    p.tets["density"][leaf] = rng.random(leaf.sum()).astype(np.float32) * 6
    p.tets["temperature"][leaf] = rng.random(leaf.sum()).astype(np.float32) * 1.2
    p.tets["albedo"][leaf] = rng.random(leaf.sum()).astype(np.float32)
    p.tets["mask"][leaf] = 7
    g2 = O.from_pools(C, p)
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    w, h, spp = 48, 36, 128
    kw = dict(spp=spp, max_bounces=16, seed=3, emission_scale=2.0, hg_g=-0.4)
    cam = ((0.2, 0.7, -1.5), (0.1, -0.1, 1), (0, 1, 0), 50, w, h)
    a = g2.render(O.camera(*cam), O.render_cfg(**kw), 0)
    b = tv.render_tracking(dg, tv.PinholeCamera(*cam), tv.RenderConfig(**kw), tv.TRACK_DELTA, 2.0)
    ma, mb = a["sum"] / spp, b.sum / spp
    va = np.maximum(a["sum_sq"] / spp - ma * ma, 0) / spp
    vb = np.maximum(b.sum_sq / spp - mb * mb, 0) / spp
    se = np.sqrt(va + vb)
    live = se > 0
    assert np.array_equal(ma[~live], mb[~live])
    z = (mb[live] - ma[live]) / se[live]
    assert np.mean(np.abs(z) > 3.0) < 0.015, np.mean(np.abs(z) > 3.0)
    assert abs(mb.mean() - ma.mean()) < 4 * np.sqrt((va + vb).sum()) / ma.size
