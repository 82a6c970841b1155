"""Pins the CPU oracle (C restatement, oracle/tvo.c) to the reference.

Two anchors:
  * tests/golden/golden.json — known-answer values produced by the unmodified
    reference (tests/golden/make_golden.py); these run everywhere;
  * oracle/_ref — the reference library itself, when it was built here; the
    randomized cross-checks below compare the restatement against it directly.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
_D = C.POINTER(C.c_double)


def h(*arrays) -> str:
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


def bits(x: float) -> str:
    return np.float64(x).view(np.uint64).item().to_bytes(8, "big").hex()


@pytest.fixture(scope="module")
def chk():
    return O.c_oracle()


@pytest.fixture(scope="module")
def c1(chk):
    vol = O.gen_volume("blob", 64)
    g, st = O.build(chk, vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
    return vol, g, st


def test_rng_kat(chk):
    assert [bits(x) for x in O.rng_draws(chk, 7, 123, 9, 16)] == GOLD["rng_7_123_9"]
    for k, v in GOLD["mix64"].items():
        assert chk.fn("mix64")(int(k)) == v


def test_tracer_kats(chk):
    for k, v in GOLD["hg_sample_cos"].items():
        g, xi = map(float, k.split("_"))
        assert bits(chk.fn("hg_sample_cos")(g, xi)) == v
    e = np.zeros(3)
    for k, v in GOLD["emission_color"].items():
        chk.fn("emission_color")(float(k), e.ctypes.data_as(_D))
        assert [bits(x) for x in e] == v
    d = np.array([np.frombuffer(bytes.fromhex(b)[::-1], np.float64)[0] for b in GOLD["phase_dir"]])
    w = np.zeros(3)
    for k, v in GOLD["sample_phase_hg"].items():
        g, i = k.split("_")
        chk.fn("sample_phase_hg")(d.ctypes.data_as(_D), float(g), 8, 0x697369, int(i), w.ctypes.data_as(_D))
        assert [bits(x) for x in w] == v


def test_hg_inversion_matches_numeric_cdf(chk):
    """acceptance.cpp:354-366: xi = 0.5 inversion within 1e-6 of a numeric CDF inversion."""
    g = 0.9
    cdf = lambda c: (1 - g * g) / (2 * g) * (1.0 / np.sqrt(1 + g * g - 2 * g * c) - 1.0 / (1 + g))
    lo, hi = -1.0, 1.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if cdf(mid) < 0.5:
            lo = mid
        else:
            hi = mid
    assert abs(chk.fn("hg_sample_cos")(0.9, 0.5) - 0.5 * (lo + hi)) <= 1e-6


def test_camera_kat(chk):
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 256, 256)
    out = np.zeros(6)
    for k, v in GOLD["primary_ray"].items():
        x, y, jx, jy = k.split("_")
        chk.fn("primary_ray")(C.byref(cam), int(x), int(y), float(jx), float(jy), out.ctypes.data_as(_D))
        assert [bits(x) for x in out] == v


def test_camera_errors(chk):
    out = np.zeros(6)
    bad = O.camera(vfov=0.0)
    assert chk.fn("primary_ray")(C.byref(bad), 0, 0, 0.0, 0.0, out.ctypes.data_as(_D)) == 3
    assert "vfov" in chk.err()
    bad = O.camera(fwd=(0, 1, 0), up=(0, 1, 0))
    assert chk.fn("primary_ray")(C.byref(bad), 0, 0, 0.0, 0.0, out.ctypes.data_as(_D)) == 3
    assert "parallel" in chk.err()


def test_init_roots_and_fuzz(chk):
    g = O.init_roots(chk)
    p = g.pools()
    assert g.counts() == GOLD["init_roots"]["counts"]
    assert h(p.vq, p.tets, p.roots) == GOLD["init_roots"]["sha"]
    assert g.counts()["n_verts"] == 15 and g.counts()["n_leaves"] == 24
    f = O.fuzzed(chk, 400, 0x52)
    pf = f.pools()
    assert f.counts() == GOLD["fuzzed_400_0x52"]["counts"]
    assert h(pf.vq, pf.tets, pf.roots) == GOLD["fuzzed_400_0x52"]["sha"]


def test_acceptance5_segments(chk):
    f = O.fuzzed(chk, 400, 0x52)
    rays = O.random_cube_rays(5, 0x7472617665727365, 10000)
    assert h(rays) == GOLD["acceptance5_rays_sha"]
    cells, t0, t1, off, st = f.march_segments(rays)
    a5 = GOLD["acceptance5_segments"]
    assert len(cells) == a5["total"] and int(st[1]) == a5["degenerate"]
    assert h(cells, t0, t1, off) == a5["sha"]


def test_volumes(chk):
    assert h(O.gen_volume("blob", 64)) == GOLD["blob64_sha"]
    assert h(O.gen_volume("cloud", 64)) == GOLD["cloud64_sha"]
    assert h(O.gen_volume("noise", 32)) == GOLD["noise32_sha"]


def test_c1_build(c1):
    _, g, st = c1
    p = g.pools()
    gold = GOLD["c1_grid"]
    assert g.counts() == gold["counts"]
    assert {k: v for k, v in st.items() if k != "seconds"} == gold["stats"]
    assert h(p.vq, p.tets, p.roots) == gold["sha"]
    assert bits(float(p.tets["density"][p.leaf_mask].astype(np.float64).sum())) == gold["sum_leaf_density"]


def test_c1_render_golden(chk, c1):
    _, g, _ = c1
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 256, 256)
    img = g.render(cam, O.render_cfg(spp=4, max_bounces=2, seed=0), 0)
    gold = GOLD["c1_render"]
    assert img["cells_visited"] == gold["cells_visited"] == 4612915
    assert hex(O.fnv64(img["sum"])) == gold["fnv_sum"] == "0x5dd59ba4fb717d7f"
    assert hex(O.fnv64(img["sum_sq"])) == gold["fnv_sum_sq"]
    # thread-count invariance (test_tracer.cpp:356-372)
    img1 = g.render(cam, O.render_cfg(spp=4, max_bounces=2, seed=0), 1)
    assert np.array_equal(img1["sum"].view(np.uint64), img["sum"].view(np.uint64))


def test_c1_locate_golden(c1):
    _, g, _ = c1
    rng = np.random.default_rng(3)
    pts = rng.random((5000, 3))
    pts[:1000] = np.round(pts[:1000] * 64) / 64
    assert h(np.array([g.locate(q) for q in pts], np.uint32)) == GOLD["c1_locate_sha"]


def test_camera_build_golden(chk):
    cam11 = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 16, 128, 128)
    g, st = O.build(chk, O.gen_volume("blob", 32), O.build_cfg(0.15, 9, True, 0.5, 1.0), cam11)
    p = g.pools()
    gold = GOLD["acc11_camera_build"]
    assert g.counts() == gold["counts"] and st["criterion_splits"] == gold["criterion_splits"]
    assert h(p.vq, p.tets, p.roots) == gold["sha"]


def test_cloud64_camera_build_golden(chk):
    camc = O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
    g, st = O.build(chk, O.gen_volume("cloud", 64), O.build_cfg(0.15, 18, True, 1.0, 16.0), camc)
    p = g.pools()
    gold = GOLD["cloud64_camera_build"]
    assert g.counts() == gold["counts"]
    assert h(p.vq, p.tets, p.roots) == gold["sha"]


# ---------------------------------------------------------------- vs _ref ---
ref = O.ref_oracle()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
def test_random_fuzz_grids_vs_reference(chk):
    for seed in [1, 2, 3]:
        a = O.fuzzed(chk, 150, seed, 30)
        b = O.fuzzed(ref, 150, seed, 30)
        assert a.pools().tets.tobytes() == b.pools().tets.tobytes()
        rays = O.random_cube_rays(seed, 99, 500)
        x = a.march_segments(rays)
        y = b.march_segments(rays)
        for u, v in zip(x, y):
            assert np.array_equal(u, v)


@needs_ref
def test_exit_face_and_free_path_vs_reference(chk):
    a = O.fuzzed(chk, 60, 9)
    b = O.fuzzed(ref, 60, 9)
    rng = np.random.default_rng(0)
    p = a.pools()
    leaves = np.nonzero(p.leaf_mask)[0]
    for i in range(500):
        cell = int(leaves[rng.integers(len(leaves))])
        q = p.vq[p.tets["verts"][cell]].astype(np.float64) / 2**24
        w = rng.random(4)
        w /= w.sum()
        pos = (w[:, None] * q).sum(0)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        assert a.exit_face(cell, pos, d) == b.exit_face(cell, pos, d)
    a.fill_density(2.0)
    b.fill_density(2.0)
    r = np.zeros(6)
    s = np.zeros(6)
    rays = O.random_cube_rays(4, 5, 300)
    for i in range(300):
        chk.fn("sample_free_path")(a.h, rays[i].ctypes.data_as(_D), 7, 1, i, r.ctypes.data_as(_D))
        ref.fn("sample_free_path")(b.h, rays[i].ctypes.data_as(_D), 7, 1, i, s.ctypes.data_as(_D))
        assert np.array_equal(r.view(np.uint64), s.view(np.uint64))
        assert chk.fn("march_transmittance")(a.h, rays[i].ctypes.data_as(_D)) == ref.fn("march_transmittance")(
            b.h, rays[i].ctypes.data_as(_D))


@needs_ref
def test_multibounce_render_with_media_vs_reference(chk):
    """Emission + albedo + HG anisotropy + Russian roulette through both integrators."""
    a = O.fuzzed(chk, 200, 0x77)
    p = a.pools()
    rng = np.random.default_rng(5)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 6
    p.tets["temperature"][lm] = rng.random(lm.sum()).astype(np.float32) * 1.2
    p.tets["albedo"][lm] = rng.random(lm.sum()).astype(np.float32)
    p.tets["mask"][lm] = 7
    ga, gb = O.from_pools(chk, p), O.from_pools(ref, p)
    cam = O.camera((0.2, 0.7, -1.5), (0.1, -0.1, 1), (0, 1, 0), 50, 48, 32)
    rc = O.render_cfg(spp=16, max_bounces=16, seed=3, emission_scale=2.0, hg_g=-0.4)
    x, y = ga.render(cam, rc, 0), gb.render(cam, rc, 0)
    assert x["cells_visited"] == y["cells_visited"]
    assert np.array_equal(x["sum"].view(np.uint64), y["sum"].view(np.uint64))
    assert np.array_equal(x["sum_sq"].view(np.uint64), y["sum_sq"].view(np.uint64))


@needs_ref
def test_step_and_noise_builds_vs_reference(chk):
    for kind, n, thr, ml, sc in [("step", 16, 0.5, 6, 1.0), ("noise", 24, 0.2, 10, 3.0), ("ramp", 12, 0.05, 8, 1.0)]:
        vol = O.gen_volume(kind, n)
        ga, sa = O.build(chk, vol, O.build_cfg(thr, ml, False, 1.0, sc))
        gb, sb = O.build(ref, vol, O.build_cfg(thr, ml, False, 1.0, sc))
        assert ga.pools().tets.tobytes() == gb.pools().tets.tobytes()
        assert sa["criterion_splits"] == sb["criterion_splits"]


@needs_ref
def test_regular_grid_vs_reference(chk):
    vol = O.gen_volume("cloud", 24)
    rays = O.random_cube_rays(3, 17, 400)
    out = []
    for lib in (chk, ref):
        off = np.zeros(401, np.uint64)
        F = C.POINTER(C.c_float)
        tot = lib.fn("dda_segments")(vol.ctypes.data_as(F), 24, 24, 24, 4.0, rays.ctypes.data_as(_D), 400, None, None,
                                     None, off.ctypes.data_as(C.POINTER(C.c_uint64)), 0)
        cells = np.zeros(tot, np.uint32)
        t0 = np.zeros(tot)
        t1 = np.zeros(tot)
        lib.fn("dda_segments")(vol.ctypes.data_as(F), 24, 24, 24, 4.0, rays.ctypes.data_as(_D), 400,
                               cells.ctypes.data_as(C.POINTER(C.c_uint32)), t0.ctypes.data_as(_D),
                               t1.ctypes.data_as(_D), off.ctypes.data_as(C.POINTER(C.c_uint64)), tot)
        out.append((cells, t0, t1, off))
    for u, v in zip(*out):
        assert np.array_equal(u, v)


def test_tgrid_restatement_golden(c1):
    """oracle/tgrid.py restates save_grid; pinned to the reference's C1 file bytes."""
    from oracle.tgrid import tgrid_bytes

    p = c1[1].pools()
    raw = tgrid_bytes(p.vq, p.tets, p.roots)
    assert len(raw) == GOLD["c1_tgrid"]["bytes"]
    assert hashlib.sha256(raw).hexdigest() == GOLD["c1_tgrid"]["sha256"]


@needs_ref
def test_tgrid_restatement_matches_reference(tmp_path):
    from oracle.tgrid import tgrid_bytes

    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 16, 128, 128)
    vol = O.gen_volume("blob", 24)
    temp = (vol * 0.7).astype(np.float32)
    alb = np.full_like(vol, 0.5)
    for g in [O.fuzzed(ref, 200, 5), O.build(ref, vol, O.build_cfg(0.15, 9, True, 0.5, 1.0), cam, temp, alb)[0]]:
        fn = str(tmp_path / "g.tgrid")
        assert ref.fn("grid_save")(g.h, fn.encode()) == 0
        p = g.pools()
        assert tgrid_bytes(p.vq, p.tets, p.roots) == open(fn, "rb").read()


@needs_ref
def test_pfm_restatement_matches_reference(tmp_path):
    from oracle.images import mean_f32, pfm_bytes, variance_f32

    rng = np.random.default_rng(4)
    w, h = 7, 5
    cnt = rng.integers(0, 4, w * h).astype(np.uint32)
    s = rng.random(3 * w * h) * cnt.repeat(3)
    q = s * s / np.maximum(cnt, 1).repeat(3) + rng.random(3 * w * h) * 0.1
    for variance in (0, 1):
        fn = str(tmp_path / f"r{variance}.pfm")
        assert ref.fn("write_pfm")(fn.encode(), w, h, s.ctypes.data_as(_D), q.ctypes.data_as(_D),
                                   cnt.ctypes.data_as(C.POINTER(C.c_uint32)), variance) == 0
        px = variance_f32(s, q, cnt) if variance else mean_f32(s, cnt)
        raw = open(fn, "rb").read()
        assert pfm_bytes(px, w, h) == raw
        W, H = C.c_int(), C.c_int()
        back = np.zeros(3 * w * h, np.float32)
        assert ref.fn("read_pfm")(fn.encode(), C.byref(W), C.byref(H), back.ctypes.data_as(C.POINTER(C.c_float))) == 0
        assert (W.value, H.value) == (w, h) and np.array_equal(back, px.ravel())


@needs_ref
def test_dvol_restatement_matches_reference(tmp_path):
    from oracle.images import dvol_bytes

    dims = (5, 4, 3)
    rng = np.random.default_rng(2)
    chans = {"density": rng.random((3, 4, 5), dtype=np.float32), "temperature": rng.random((3, 4, 5), dtype=np.float32),
             "albedo": np.full((3, 4, 5), 0.25, np.float32)}
    fn = str(tmp_path / "v.dvol")
    names = (C.c_char_p * 3)(*[k.encode() for k in chans])
    F = C.POINTER(C.c_float)
    data = (F * 3)(*[v.ctypes.data_as(F) for v in chans.values()])
    assert ref.fn("dvol_save")(fn.encode(), *dims, 3, names, data) == 0
    assert dvol_bytes(dims, chans) == open(fn, "rb").read()


@pytest.mark.skipif(O.ref_pad_oracle() is None or ref is None, reason="oracle/_ref/pad not built")
def test_padded_reference_build_renders_identically():
    """oracle/_ref/pad (alignas(64) TraceStats) only changes the
    counter layout: the multi-threaded render is bit-identical to the shipped one."""
    vol = O.gen_volume("cloud", 32)
    cam = O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 48, 40)
    outs = []
    for chk in (ref, O.ref_pad_oracle()):
        g, _ = O.build(chk, vol, O.build_cfg(0.15, 24, True, 1.0, 16.0), cam)
        outs.append(g.render(cam, O.render_cfg(spp=2, max_bounces=16), 4))
    a, b = outs
    assert a["cells_visited"] == b["cells_visited"]
    for k in ("sum", "sum_sq", "counts"):
        if k in a:
            assert np.array_equal(a[k], b[k])
