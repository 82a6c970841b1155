"""Edge cases of the hot path against the reference / oracle, bit for bit:
uniform LEB refinement KATs (test_tet_grid.cpp:169-184, acceptance 2), a 1x1
image, a camera inside the cube, rays grazing faces / edges / vertices, rays
that miss, max_bounces 1, and a vacuum grid with an environment colour.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ref = O.ref_oracle()


@pytest.fixture(scope="module")
def tv():
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tv


def upload(tv, p):
    return tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)


@pytest.mark.parametrize("levels,leaves", [(3, 192), (6, 1536)])
def test_uniform_refinement_kat(tv, levels, leaves):
    """threshold 0 on a ramp refines every leaf to max_level: 24 * 2^L leaves,
    the reference's refine_uniform leaf set (test_tet_grid.cpp:169-184)."""
    from test_gpu_build import canonical

    vol = O.gen_volume("ramp", 64)  # every level-L tet owns voxels with different values
    dg, st = tv.build_adaptive_grid(vol, tv.BuildConfig(0.0, levels, False, 1.0, 1.0))
    assert st.leaf_count == leaves and st.max_depth == levels
    v, t, _ = dg.download()
    if ref is not None:
        p = O.Grid(ref, ref.fn("grid_uniform")(levels)).pools()
        a = canonical(p.vq, p.tets)[:, :12]
        b = canonical(v, t.view(O.TET_DTYPE))[:, :12]
        assert np.array_equal(a, b)


@pytest.fixture(scope="module")
def media(tv):
    g = O.fuzzed(O.c_oracle(), 300, 0x77)
    p = g.pools()
    rng = np.random.default_rng(7)
    lm = p.leaf_mask
    p.tets["density"][lm] = (rng.random(lm.sum()) * 4).astype(np.float32)
    p.tets["mask"][lm] = 1
    return O.from_pools(O.c_oracle(), p), upload(tv, p)


def _same_render(tv, og, dg, cam_args, **rc):
    cam = tv.PinholeCamera(*cam_args)
    trc = dict(rc)
    if "env" in trc:
        trc["environment"] = trc.pop("env")
    mine = tv.render(dg, cam, tv.RenderConfig(**trc))
    want = og.render(O.camera(*cam_args), O.render_cfg(**rc), 0)
    assert mine.cells_visited == want["cells_visited"]
    assert np.array_equal(mine.sum.view(np.uint64), want["sum"].view(np.uint64))
    assert np.array_equal(mine.sum_sq.view(np.uint64), want["sum_sq"].view(np.uint64))
    return mine


def test_one_pixel_image(tv, media):
    og, dg = media
    _same_render(tv, og, dg, ((0.5, 0.5, -1.5), (0, 0, 1), (0, 1, 0), 30, 1, 1), spp=40, max_bounces=16, seed=2)


def test_camera_inside_the_cube(tv, media):
    og, dg = media
    _same_render(tv, og, dg, ((0.4, 0.55, 0.5), (0.3, -0.2, 1), (0, 1, 0), 70, 33, 17), spp=3, max_bounces=16, seed=5)


def test_single_bounce_and_environment(tv, media):
    og, dg = media
    _same_render(tv, og, dg, ((0.5, 0.5, -1.5), (0, 0, 1), (0, 1, 0), 45, 24, 20), spp=2, max_bounces=1, seed=1,
                 env=(0.25, 0.5, 2.0), default_albedo=0.3)


def test_camera_looking_away_misses_everything(tv, media):
    og, dg = media
    img = _same_render(tv, og, dg, ((0.5, 0.5, -1.5), (0, 0, -1), (0, 1, 0), 40, 16, 16), spp=2, max_bounces=8,
                       seed=0)
    assert img.cells_visited == 0 and np.all(img.sum == 2.0)


def test_grazing_rays(tv, media):
    """rays along cube faces, edges, through grid vertices and along LEB planes"""
    og, dg = media
    rays = []
    for a in [0.0, 0.25, 0.5, 0.75, 1.0]:
        for b in [0.0, 0.125, 0.5, 1.0]:
            rays.append([a, b, -1, 0, 0, 1, 0, np.inf])       # along z through (a, b)
            rays.append([-1, a, b, 1, 0, 0, 0, np.inf])       # along x
            rays.append([a, -1, b, 0, 1, 0, 0, np.inf])       # along y
            d = np.array([1.0, 1.0, 1.0]) / np.sqrt(3.0)
            rays.append([a - 1, b - 1, -1, *d, 0, np.inf])    # diagonal through lattice points
    rays = np.array(rays)
    seg, off, deg = tv.march_segments(dg, rays)
    cells, t0, t1, off_r, st = og.march_segments(rays)
    assert np.array_equal(off, off_r)
    assert np.array_equal(seg["cell"], cells)
    assert np.array_equal(seg["t_enter"].view(np.uint64), t0.view(np.uint64))
    assert np.array_equal(seg["t_exit"].view(np.uint64), t1.view(np.uint64))
    assert deg == int(st[1])
