"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar: traversal cell ids and segment endpoints are
bit-exact against the reference TetMarcher on the reference's own grid
(uploaded with TetIds preserved); single-scatter radiance matches the oracle
framebuffer bit-for-bit (tolerance stated below is the fallback bar), and the
counters (cells_visited, degenerate_paths) are exact.
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


def upload(tv, g: O.Grid):
    p = g.pools()
    return tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)


@pytest.fixture(scope="module")
def c1(tv):
    """blob 64^3, thr 0.15, max_level 12, density_scale 8."""
    vol = O.gen_volume("blob", 64)
    g, st = O.build(O.c_oracle(), vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
    return vol, g, upload(tv, g)


def test_upload_roundtrip(tv, c1):
    _, g, dg = c1
    p = g.pools()
    v, t, r = dg.download()
    assert np.array_equal(v, p.vq)
    assert t.tobytes() == p.tets.tobytes()
    assert np.array_equal(r, p.roots)
    info = dg.info()
    assert info["n_leaves"] == 51020 and info["n_tets"] == 102016 and info["max_depth"] == 12


def _segments_equal(tv, g, dg, rays):
    cells, t0, t1, off, stats = g.march_segments(rays)
    seg, off_d, deg = tv.march_segments(dg, rays)
    assert np.array_equal(off_d, off), "per-ray segment counts differ"
    assert np.array_equal(seg["cell"], cells), "visited-tet sequence differs"
    # bit-exact endpoints
    assert np.array_equal(seg["t_enter"].view(np.uint64), t0.view(np.uint64))
    assert np.array_equal(seg["t_exit"].view(np.uint64), t1.view(np.uint64))
    assert deg == stats[1]
    return len(cells)


def test_march_segments_fuzzed_acceptance5(tv):
    """acceptance.cpp:215-246 rays on fuzzed_grid(400, 0x52), bit-exact."""
    g = O.fuzzed(O.c_oracle(), 400, 0x52)
    dg = upload(tv, g)
    rays = O.random_cube_rays(5, 0x7472617665727365, 10000)
    n = _segments_equal(tv, g, dg, rays)
    assert n > 100000


def test_march_segments_c1_primary_rays(tv, c1):
    """All 262,144 C1 primary rays (jitter from RngStream(0, y*256+x, s)): 5,097,636 segments."""
    _, g, dg = c1
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 256, 256)
    C = O.c_oracle()
    rays = np.zeros((256 * 256 * 4, 8))
    out = np.zeros(6)
    import ctypes

    k = 0
    draws = np.zeros(2)
    for y in range(256):
        for x in range(256):
            for s in range(4):
                C.fn("rng_draws")(0, y * 256 + x, s, 2, draws.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
                C.fn("primary_ray")(ctypes.byref(cam), x, y, draws[0], draws[1],
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
                rays[k, :6] = out
                rays[k, 6] = 0.0
                rays[k, 7] = np.inf
                k += 1
    n = _segments_equal(tv, g, dg, rays)
    assert n == 5097636


def test_march_segments_finite_tmax(tv, c1):
    """t_max inside the cube clips the last segment (tracer.cpp:71-76)."""
    _, g, dg = c1
    rays = O.random_cube_rays(11, 0x1234, 2000)
    rays[:, 7] = 2.0
    _segments_equal(tv, g, dg, rays)


def test_locate_points(tv, c1):
    _, g, dg = c1
    rng = np.random.default_rng(3)
    pts = rng.random((20000, 3))
    # include faces, edges and exact vertices (ties resolve towards child A)
    pts[:2000] = np.round(pts[:2000] * 64) / 64
    pts[2000:2050] = 0.5
    pts[2050:2100] = rng.integers(0, 3, (50, 3)) * 0.5
    got = tv.locate_points(dg, pts)
    want = np.array([g.locate(p) for p in pts], dtype=np.uint32)
    assert np.array_equal(got, want)


def test_locate_points_on_jump_table_boundaries(tv, c1):
    """locate starts at the jump table's node (GridView::jump, 128^3 cubes) or
    at the guessed root: points on the cube boundaries of that table (i / 128),
    on the leaves' own vertices, just off them (+-1 ulp, +-1e-12), and on the
    faces of the unit cube land in the reference's leaf."""
    _, g, dg = c1
    rng = np.random.default_rng(11)
    n = 6000
    pts = np.round(rng.random((n, 3)) * 128) / 128  # jump-table cube corners / edges / faces
    pts[:1000, 0] = rng.random(1000)
    verts = np.asarray(g.pools().vq, dtype=np.float64) / 2.0 ** 24
    vi = rng.integers(0, len(verts), 2000)
    pts[1000:3000] = verts[vi]
    pts[3000:4000] = np.nextafter(pts[3000:4000], 2.0)
    pts[4000:5000] = np.nextafter(pts[4000:5000], -1.0)
    pts[5000:6000] = np.clip(pts[5000:6000] + rng.choice([-1e-12, 1e-12], (1000, 3)), 0.0, 1.0)
    pts = np.clip(pts, 0.0, 1.0)
    # points on the faces of the unit cube, where every camera ray enters (locate's
    # root fast path accepts the root's outer face at violation 0)
    face = rng.random((4000, 3))
    ax = rng.integers(0, 3, 4000)
    face[np.arange(4000), ax] = rng.integers(0, 2, 4000).astype(np.float64)
    face[:500] = np.round(face[:500] * 64) / 64  # cube-face points on pyramid and triangle edges
    pts = np.concatenate([pts, face])
    got = tv.locate_points(dg, pts)
    want = np.array([g.locate(p) for p in pts], dtype=np.uint32)
    assert np.array_equal(got, want)


def _render_both(tv, g, dg, cam_kw, rc_kw):
    cam = O.camera(**cam_kw)
    rc = O.render_cfg(**rc_kw)
    a = g.render(cam, rc, 0)
    b = tv.render(dg, tv.PinholeCamera(cam_kw["pos"], cam_kw["fwd"], cam_kw["up"], cam_kw["vfov"], cam_kw["width"],
                                       cam_kw["height"]), tv.RenderConfig(**{k: v for k, v in rc_kw.items()}))
    return a, b


def test_render_c1_single_scatter_bit_exact(tv, c1):
    """C1 (256^2, 4 spp, max_bounces 2): golden FNV 5dd59ba4fb717d7f, cells 4,612,915."""
    _, g, dg = c1
    a, b = _render_both(tv, g, dg, dict(pos=(0.5, 0.5, -2), fwd=(0, 0, 1), up=(0, 1, 0), vfov=40, width=256, height=256),
                        dict(spp=4, max_bounces=2, seed=0))
    assert b.cells_visited == a["cells_visited"] == 4612915
    assert b.degenerate_paths == a["degenerate_paths"] == 0
    assert np.array_equal(b.sample_counts, a["counts"])
    # fallback bar (north star): per-pixel relative error <= 1e-3 (absolute where the mean is 0)
    ma, mb = a["sum"] / 4, b.sum / 4
    rel = np.abs(mb - ma) / np.maximum(np.abs(ma), 1e-300)
    assert np.all((rel <= 1e-3) | ((ma == 0) & (np.abs(mb) <= 1e-3)))
    # the real bar: bit-identical framebuffer
    assert O.fnv64(b.sum) == 0x5DD59BA4FB717D7F
    assert np.array_equal(b.sum.view(np.uint64), a["sum"].view(np.uint64))
    assert np.array_equal(b.sum_sq.view(np.uint64), a["sum_sq"].view(np.uint64))


def test_render_c1_multibounce(tv, c1):
    """C1 grid, max_bounces 64 (Russian roulette + HG redirects), 8 spp, g = 0.3."""
    _, g, dg = c1
    a, b = _render_both(tv, g, dg, dict(pos=(0.5, 0.5, -2), fwd=(0, 0, 1), up=(0, 1, 0), vfov=40, width=128, height=96),
                        dict(spp=8, max_bounces=64, seed=7, hg_g=0.3))
    assert b.cells_visited == a["cells_visited"]
    assert np.array_equal(b.sum.view(np.uint64), a["sum"].view(np.uint64))


def test_render_emission_and_albedo(tv):
    """Temperature emission LUT and per-cell albedo (mask bits 2, 4) on a fuzzed grid."""
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
    a, b = _render_both(tv, g2, dg, dict(pos=(0.2, 0.7, -1.5), fwd=(0.1, -0.1, 1), up=(0, 1, 0), vfov=50, width=64,
                                         height=48),
                        dict(spp=16, max_bounces=16, seed=3, emission_scale=2.0, hg_g=-0.4))
    assert b.cells_visited == a["cells_visited"]
    assert np.array_equal(b.sum.view(np.uint64), a["sum"].view(np.uint64))


def test_render_vacuum_is_environment(tv):
    """test_tracer.cpp:304-317: vacuum returns the environment exactly."""
    C = O.c_oracle()
    g = O.init_roots(C)
    g.fill_density(0.0)
    dg = upload(tv, g)
    b = tv.render(dg, tv.PinholeCamera(width=32, height=24), tv.RenderConfig(spp=3, environment=(0.25, 0.5, 2.0)))
    m = b.mean()
    assert np.all(m[..., 0] == 0.25) and np.all(m[..., 1] == 0.5) and np.all(m[..., 2] == 2.0)


def test_render_odd_sizes_and_ranks(tv, c1):
    """Frame not a multiple of the 16x16 tile; the union of rank shares equals the full frame."""
    import torch

    _, g, dg = c1
    cam = tv.PinholeCamera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 75, 41)
    rc = tv.RenderConfig(spp=2, max_bounces=8, seed=1)
    full = tv.render(dg, cam, rc)
    acc = torch.zeros(75 * 41 * 3, dtype=torch.float64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    for r in range(3):
        part = torch.zeros_like(acc)
        tv.render_tiles(dg, cam, rc, r, 3, part.data_ptr(), None, None, stats.data_ptr(), 0)
        torch.cuda.synchronize()
        acc += part
    assert np.array_equal(acc.cpu().numpy().view(np.uint64), full.sum.view(np.uint64))
    assert int(stats[0]) == full.cells_visited


def test_config_errors_mirror_reference(tv, c1):
    _, _, dg = c1
    with pytest.raises(tv.ConfigError, match="spp must be at least 1"):
        tv.render(dg, tv.PinholeCamera(), tv.RenderConfig(spp=0))
    with pytest.raises(tv.ConfigError, match="phase anisotropy"):
        tv.render(dg, tv.PinholeCamera(), tv.RenderConfig(hg_g=1.0))
    with pytest.raises(tv.CameraError, match="vfov"):
        tv.render(dg, tv.PinholeCamera(vfov_degrees=180.0), tv.RenderConfig())
    with pytest.raises(tv.CameraError, match="parallel"):
        tv.render(dg, tv.PinholeCamera(forward=(0, 1, 0), up=(0, 1, 0)), tv.RenderConfig())


def test_multi_batch_frame_matches_progressive_frames(tv, c1):
    """A frame larger than one sample batch (2^26 paths) is rendered in several
    batches; their ordered accumulation must equal rendering the same samples as
    progressive single-batch frames (tv_render_accumulate), bit for bit."""
    import torch

    _, _, dg = c1
    w, h, spp = 512, 512, 300  # 78.6M paths -> 2 batches of the trace kernel
    cam = tv.PinholeCamera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, w, h)
    rc = tv.RenderConfig(spp=spp, max_bounces=2, seed=3)
    full = tv.render(dg, cam, rc)
    s = torch.zeros(3 * w * h, dtype=torch.float64, device="cuda")
    q = torch.zeros_like(s)
    c = torch.zeros(w * h, dtype=torch.int32, device="cuda")
    first = 0
    for part in (100, 100, 100):
        tv.render_accumulate(dg, cam, tv.RenderConfig(spp=part, max_bounces=2, seed=3), first, s.data_ptr(),
                             q.data_ptr(), c.data_ptr(), None)
        first += part
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy().view(np.uint64), full.sum.view(np.uint64))
    assert np.array_equal(q.cpu().numpy().view(np.uint64), full.sum_sq.view(np.uint64))
    assert np.all(c.cpu().numpy() == spp) and full.paths_traced == w * h * spp


def _media_grid(tv, steps=300, seed=0x61):
    g = O.fuzzed(O.c_oracle(), steps, seed)
    p = g.pools()
    rng = np.random.default_rng(seed)
    lm = p.leaf_mask
    p.tets["density"][lm] = np.where(rng.random(lm.sum()) < 0.3, 0.0, rng.random(lm.sum()) * 6).astype(np.float32)
    p.tets["mask"][lm] = 1
    ref_g = O.from_pools(O.ref_oracle() or O.c_oracle(), p)
    return p, ref_g, tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)


def test_march_transmittance(tv):
    """tracer.cpp:176-187: the optical depth bit-exact (sequential sum over the
    reference's segments), exp(-tau) within 2 ulp of the reference's std::exp."""
    p, rg, dg = _media_grid(tv)
    rays = O.random_cube_rays(7, 0x7472616e73, 3000)
    rays[::3, 7] = rays[::3, 6] + 0.4  # finite t_max: clipped final segments
    tau, tr, cells, deg = tv.march_transmittance(dg, rays)
    cells_ref, t0, t1, off, _ = rg.march_segments(rays)
    lam = p.tets["density"].astype(np.float64)
    for i in range(len(rays)):
        want = 0.0
        for k in range(int(off[i]), int(off[i + 1])):
            want += lam[cells_ref[k]] * (t1[k] - t0[k])
        assert tau[i] == want, i
        ref_t = rg.chk.fn("march_transmittance")(rg.h, rays[i].ctypes.data_as(O._D))
        assert abs(tr[i] - ref_t) <= 2 * np.spacing(ref_t), i
    assert cells == len(cells_ref) and deg == 0
    vp = O.init_roots(O.c_oracle()).pools()
    vac = tv.TetGrid.upload(vp.vq, vp.tets.view(tv.TET_DTYPE), vp.roots, 48)
    _, tr0, _, _ = tv.march_transmittance(vac, rays[:50])
    assert np.all(tr0 == 1.0)  # vacuum is exactly 1 (test_tracer.cpp:149-164)


def test_sample_free_path(tv):
    """tracer.cpp:189-216 against the reference, record for record."""
    p, rg, dg = _media_grid(tv, 250, 0x62)
    rays = O.random_cube_rays(9, 0x66726565, 2000)
    rays[1::4, 7] = rays[1::4, 6] + 0.3
    pix = np.arange(len(rays), dtype=np.uint64) * 7 + 3
    smp = np.arange(len(rays), dtype=np.uint64) % 5
    got = tv.sample_free_path(dg, rays, 11, pix, smp)
    n_coll = 0
    for i in range(len(rays)):
        out = np.zeros(6)
        rg.chk.fn("sample_free_path")(rg.h, rays[i].ctypes.data_as(O._D), 11, int(pix[i]), int(smp[i]),
                                      out.ctypes.data_as(O._D))
        assert bool(got["collided"][i]) == bool(out[0]), i
        assert np.array_equal(got["position"][i], out[1:4]), i
        assert got["distance"][i] == out[5], i
        if out[0]:
            n_coll += 1
            assert got["cell"][i] == int(out[4]), i
    assert 100 < n_coll < len(rays)


def test_trace_rays_matches_reference_trace(tv):
    """tetvol::trace (tracer.cpp:258-263) for arbitrary rays, incl. finite t_max
    and rays starting inside the cube, with emission and albedo channels."""
    ref = O.ref_oracle()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    g = O.fuzzed(O.c_oracle(), 300, 0x71)
    p = g.pools()
    rng = np.random.default_rng(71)
    lm = p.leaf_mask
    n = int(lm.sum())
    p.tets["density"][lm] = (rng.random(n) * 5).astype(np.float32)
    p.tets["temperature"][lm] = rng.random(n).astype(np.float32)
    p.tets["albedo"][lm] = rng.random(n).astype(np.float32)
    p.tets["mask"][lm] = np.where(rng.random(n) < 0.5, 7, 1).astype(np.uint8)
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    rg = O.from_pools(ref, p)
    rays = O.random_cube_rays(4, 0x7472616365, 1500)
    rays[::5, 7] = rays[::5, 6] + 0.35
    rays[1::7, 0:3] = rng.random((len(rays[1::7]), 3))  # origins inside the cube
    cfg = dict(spp=1, max_bounces=24, seed=0, hg_g=0.4, default_albedo=0.7, env=(1.0, 0.5, 0.25),
               emission_scale=2.0)
    rc = tv.RenderConfig(max_bounces=24, hg_g=0.4, default_albedo=0.7, environment=(1.0, 0.5, 0.25),
                         emission_scale=2.0)
    pix = np.arange(len(rays), dtype=np.uint64) * 3 + 1
    smp = np.arange(len(rays), dtype=np.uint64) % 7
    got, cells, deg = tv.trace(dg, rays, rc, 5, pix, smp)
    orc = O.render_cfg(**cfg)
    st = np.zeros(2, np.uint64)
    for i in range(len(rays)):
        out = np.zeros(3)
        ref.fn("trace_ray")(rg.h, rays[i].ctypes.data_as(O._D), O.C.byref(orc), 5, int(pix[i]), int(smp[i]),
                            out.ctypes.data_as(O._D), st.ctypes.data_as(O._U64))
        assert np.array_equal(got[i].view(np.uint64), out.view(np.uint64)), (i, got[i], out)
    assert cells == int(st[0]) and deg == int(st[1])
