"""N2 / N3: device volumes (.dvol, cmd_gen), PFM output, compare metrics and
progressive accumulation, against the compiled reference and the restatements
in oracle/images.py.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from oracle.images import compare, dvol_bytes, mean_f32, pfm_bytes, variance_f32

pytestmark = pytest.mark.gpu
ref = O.ref_oracle()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built")
F = C.POINTER(C.c_float)


@pytest.fixture(scope="module")
def tv():
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tv


# ------------------------------------------------------------------ volumes ---
def test_generate_matches_host_generators(tv):
    for kind in ["constant", "ramp", "blob", "step", "noise", "cloud"]:
        v = tv.DenseVolume.generate(kind, (20, 20, 20), value=0.75, with_temperature=True, albedo=0.3)
        host = O.gen_volume(kind, 20, 0.75)
        d = v.channel("density")
        assert np.array_equal(d.view(np.uint32), host.view(np.uint32)), kind
        assert v.channel_names() == ["density", "temperature", "albedo"]
        assert np.array_equal(v.channel("temperature"), np.clip(host, np.float32(0), np.float32(1)))
        assert np.all(v.channel("albedo") == np.float32(0.3))


def test_dvol_save_is_byte_identical(tv, tmp_path):
    v = tv.DenseVolume.generate("cloud", (12, 10, 8), with_temperature=True, albedo=0.5)
    fn = tmp_path / "v.dvol"
    v.save(fn)
    chans = {n: v.channel(n) for n in v.channel_names()}
    assert fn.read_bytes() == dvol_bytes((12, 10, 8), chans)
    if ref is not None:
        fr = tmp_path / "r.dvol"
        names = (C.c_char_p * 3)(*[k.encode() for k in chans])
        data = (F * 3)(*[a.ctypes.data_as(F) for a in chans.values()])
        assert ref.fn("dvol_save")(str(fr).encode(), 12, 10, 8, 3, names, data) == 0
        assert fr.read_bytes() == fn.read_bytes()


def test_dvol_load_roundtrip_and_build(tv, tmp_path):
    host = O.gen_volume("blob", 24)
    temp = (host * 0.5).astype(np.float32)
    fn = tmp_path / "b.dvol"
    fn.write_bytes(dvol_bytes((24, 24, 24), {"density": host, "temperature": temp}))
    v = tv.DenseVolume.load(fn)
    assert v.dims == (24, 24, 24) and v.channel_names() == ["density", "temperature"]
    assert np.array_equal(v.channel("density"), host) and np.array_equal(v.channel("temperature"), temp)
    bc = tv.BuildConfig(0.15, 10, False, 1.0, 4.0)
    g1, s1 = tv.build_adaptive_grid_volume(v, bc)
    g2, s2 = tv.build_adaptive_grid(host, bc, temperature=temp)
    assert s1.leaf_count == s2.leaf_count
    _, t1, _ = g1.download()
    _, t2, _ = g2.download()
    assert t1.tobytes() == t2.tobytes()


def _bad_dvols(raw: bytes):
    hdr = lambda k, v: raw[:4 + 4 * k] + int(v).to_bytes(4, "little") + raw[8 + 4 * k:]  # noqa: E731
    yield "magic", b"DVOX" + raw[4:]
    yield "version", hdr(0, 3)
    yield "dims", hdr(1, 0)
    yield "dims big", hdr(3, 4097)
    yield "channels", hdr(4, 0)
    yield "channels big", hdr(4, 17)
    yield "empty name", raw[:24] + b"\x00" + raw[25:]
    dup = bytearray(raw)
    at = 24 + 1 + len("density") + 1
    dup[at:at + 7] = b"density"
    yield "duplicate", bytes(dup[:at + 7]) + raw[at + 7:] if raw[at - 1] == 7 else None
    yield "truncated names", raw[:27]
    yield "truncated data", raw[:-5]
    yield "empty", b""


@needs_ref
def test_dvol_load_errors_match_reference(tv, tmp_path):
    a = O.gen_volume("ramp", 6)
    raw = dvol_bytes((6, 6, 6), {"density": a, "albedo": a * 0})  # 'albedo' is 6 letters: no dup case
    raw2 = dvol_bytes((6, 6, 6), {"density": a, "Density": a})
    cases = list(_bad_dvols(raw)) + [("duplicate", raw2[:25 + 7 + 1] + b"density" + raw2[25 + 7 + 1 + 7:])]
    for name, bad in cases:
        if bad is None:
            continue
        fn = tmp_path / "bad.dvol"
        fn.write_bytes(bad)
        dims, nch = (C.c_int * 3)(), C.c_int()
        assert ref.fn("dvol_load")(str(fn).encode(), dims, C.byref(nch), None, None) != 0, name
        want = ref.err()
        with pytest.raises(tv.VolumeError) as e:
            tv.DenseVolume.load(fn)
        assert str(e.value) == want, (name, str(e.value), want)


def test_volume_errors(tv):
    v = tv.DenseVolume.create(4, 4, 4)
    with pytest.raises(tv.VolumeError, match="unknown channel: albedo"):
        v.channel("albedo")
    v.add_channel("albedo")
    with pytest.raises(tv.VolumeError, match="channel already exists: albedo"):
        v.add_channel("albedo")
    with pytest.raises(tv.ConfigError, match="dims out of range"):
        tv.DenseVolume.create(0, 4, 4)
    with pytest.raises(tv.ConfigError):
        tv.DenseVolume.generate("blob", (4, 4, 4), albedo=1.5)


# ------------------------------------------------------------------- images ---
@pytest.fixture(scope="module")
def scene(tv):
    g, _ = O.build(O.c_oracle(), O.gen_volume("blob", 32), O.build_cfg(0.15, 10, False, 1.0, 8.0))
    p = g.pools()
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    cam = tv.PinholeCamera((0.5, 0.5, -1.5), (0, 0, 1), (0, 1, 0), 40, 48, 40)
    return dg, cam


@needs_ref
def test_pfm_writers_byte_identical(tv, scene, tmp_path):
    dg, cam = scene
    img = tv.render(dg, cam, tv.RenderConfig(spp=5, max_bounces=16, seed=2))
    img.sample_counts[:7] = [0, 1, 0, 1, 2, 0, 1]  # exercise n = 0 / 1 / 2
    for variance in (False, True):
        fn = tmp_path / f"m{int(variance)}.pfm"
        (tv.write_variance_pfm if variance else tv.write_pfm)(fn, img)
        fr = tmp_path / f"r{int(variance)}.pfm"
        assert ref.fn("write_pfm")(str(fr).encode(), img.width, img.height, img.sum.ctypes.data_as(O._D),
                                   img.sum_sq.ctypes.data_as(O._D), img.sample_counts.ctypes.data_as(O._U32),
                                   int(variance)) == 0
        assert fn.read_bytes() == fr.read_bytes()
        px = variance_f32(img.sum, img.sum_sq, img.sample_counts) if variance else mean_f32(img.sum,
                                                                                             img.sample_counts)
        assert fn.read_bytes() == pfm_bytes(px, img.width, img.height)
        back = tv.read_pfm(fn)
        assert (back.width, back.height) == (img.width, img.height)
        assert np.array_equal(back.rgb.reshape(-1, 3), px)
    fi = tv.read_pfm(tmp_path / "m0.pfm")
    tv.write_pfm(tmp_path / "copy.pfm", fi)
    assert (tmp_path / "copy.pfm").read_bytes() == (tmp_path / "m0.pfm").read_bytes()


@needs_ref
def test_read_pfm_errors_match_reference(tv, tmp_path):
    good = pfm_bytes(np.ones((6, 3), np.float32), 3, 2)
    cases = {"magic": b"Pf" + good[2:], "header": b"PF\n3\n", "zero": b"PF\n0 2\n-1.0\n", "bigendian": b"PF\n3 2\n1.0\n",
             "short": good[:-4], "empty": b""}
    for name, raw in cases.items():
        fn = tmp_path / f"{name}.pfm"
        fn.write_bytes(raw)
        w, h = C.c_int(), C.c_int()
        assert ref.fn("read_pfm")(str(fn).encode(), C.byref(w), C.byref(h), None if name != "short" else
                                  (C.c_float * 6)()) != 0, name
        want = ref.err()
        with pytest.raises(tv.ImageError) as e:
            tv.read_pfm(fn)
        assert str(e.value) == want, (name, str(e.value), want)


def test_compare_metrics(tv, scene, tmp_path):
    dg, cam = scene
    a = tv.render(dg, cam, tv.RenderConfig(spp=8, max_bounces=16, seed=1))
    b = tv.render(dg, cam, tv.RenderConfig(spp=8, max_bounces=16, seed=2))
    files = {}
    for k, img in (("a", a), ("b", b)):
        tv.write_pfm(tmp_path / f"{k}.pfm", img)
        tv.write_variance_pfm(tmp_path / f"v{k}.pfm", img)
        files[k] = tv.read_pfm(tmp_path / f"{k}.pfm")
        files["v" + k] = tv.read_pfm(tmp_path / f"v{k}.pfm")
    got = tv.compare_images(files["a"], files["b"], files["va"], files["vb"])
    want = compare(files["a"].rgb, files["b"].rgb, files["va"].rgb, files["vb"].rgb)
    assert got["maxAbsDiff"] == want["maxAbsDiff"]
    assert got["outliers"] == want["outliers"] and got["outlierFraction"] == want["outlierFraction"]
    assert got["rmse"] == pytest.approx(want["rmse"], rel=1e-12)  # parallel vs sequential sum of squares
    same = tv.compare_images(files["a"], files["a"])
    assert same["rmse"] == 0.0 and same["maxAbsDiff"] == 0.0 and same["outlierFraction"] is None
    with pytest.raises(tv.FormatError, match="image dimensions differ"):
        tv.compare_images(files["a"], tv.FloatImage(1, 1, np.zeros((1, 1, 3), np.float32)))
    with pytest.raises(tv.ConfigError, match="must be given together"):
        tv.compare_images(files["a"], files["b"], files["va"], None)


def test_progressive_accumulation_is_bit_identical(tv, scene):
    import torch

    dg, cam = scene
    n = cam.width * cam.height
    s = torch.zeros(3 * n, dtype=torch.float64, device="cuda")
    q = torch.zeros(3 * n, dtype=torch.float64, device="cuda")
    c = torch.zeros(n, dtype=torch.int32, device="cuda")
    st = torch.zeros(3, dtype=torch.int64, device="cuda")
    first = 0
    for spp in [3, 1, 4, 2]:  # frames covering samples [0, 10)
        tv.render_accumulate(dg, cam, tv.RenderConfig(spp=spp, max_bounces=16, seed=9), first, s.data_ptr(),
                             q.data_ptr(), c.data_ptr(), st.data_ptr())
        first += spp
    torch.cuda.synchronize()
    full = tv.render(dg, cam, tv.RenderConfig(spp=10, max_bounces=16, seed=9))
    assert np.array_equal(s.cpu().numpy().view(np.uint64), full.sum.view(np.uint64))
    assert np.array_equal(q.cpu().numpy().view(np.uint64), full.sum_sq.view(np.uint64))
    assert np.all(c.cpu().numpy() == 10)
    assert int(st[0]) == full.cells_visited and int(st[1]) == full.paths_traced
