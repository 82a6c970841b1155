"""N1: .tgrid I/O on the device (tv_grid_save / tv_grid_load) against the
reference's save_grid / load_grid (builder.cpp:184-293).

  * save of uploaded reference pools is byte-identical to save_grid (golden
    SHA-256 of the C1 file, and the numpy restatement oracle/tgrid.py);
  * a GPU-built grid saved by us loads in the reference, passes validate(),
    and the reference renders it bit-identically to our renderer;
  * load of a reference-written file reproduces its pools; every malformed-file
    case fails with the reference's own FormatError message.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from oracle.tgrid import TET_RECORD, tgrid_bytes

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
ref = O.ref_oracle()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built")
FIELDS = ["verts", "children", "parent", "neighbors", "normal_ids", "level", "density", "temperature", "albedo", "mask"]


@pytest.fixture(scope="module")
def tv():
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tv


@pytest.fixture(scope="module")
def c1():
    g, _ = O.build(O.c_oracle(), O.gen_volume("blob", 64), O.build_cfg(0.15, 12, False, 1.0, 8.0))
    return g.pools()


def upload(tv, p):
    return tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)


def test_save_is_byte_identical_to_save_grid(tv, c1, tmp_path):
    fn = tmp_path / "c1.tgrid"
    upload(tv, c1).save(fn)
    raw = fn.read_bytes()
    assert len(raw) == GOLD["c1_tgrid"]["bytes"]
    assert hashlib.sha256(raw).hexdigest() == GOLD["c1_tgrid"]["sha256"]
    assert raw == tgrid_bytes(c1.vq, c1.tets, c1.roots)


def test_gpu_build_roundtrips_through_reference(tv, tmp_path):
    vol = O.gen_volume("cloud", 32)
    cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 96, 80)
    dg, _ = tv.build_adaptive_grid(vol, tv.BuildConfig(0.15, 15, True, 1.0, 16.0), cam)
    fn = tmp_path / "gpu.tgrid"
    dg.save(fn)
    v, t, r = dg.download()
    assert fn.read_bytes() == tgrid_bytes(v, t.view(O.TET_DTYPE), r)
    rc = tv.RenderConfig(spp=3, max_bounces=16, seed=5)
    mine = tv.render(dg, cam, rc)
    if ref is None:
        return
    h = ref.fn("grid_load")(str(fn).encode())
    rg = O.Grid(ref, h)
    msg = O.C.create_string_buffer(256)
    out = np.zeros(3, np.uint64)
    assert ref.fn("grid_validate")(rg.h, msg, 256, out.ctypes.data_as(O._U64)) == 1, msg.value.decode()
    img = rg.render(O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 96, 80), O.render_cfg(3, 16, 5), 0)
    assert img["cells_visited"] == mine.cells_visited
    assert np.array_equal(img["sum"].view(np.uint64), mine.sum.view(np.uint64))


@needs_ref
def test_load_reference_file(tv, tmp_path):
    g = O.fuzzed(ref, 300, 7)
    rng = np.random.default_rng(1)
    p0 = g.pools()
    for t in np.nonzero(p0.leaf_mask)[0][:200]:
        ref.fn("grid_set_payload")(g.h, int(t), float(rng.random() * 4), float(rng.random()), 0.25, 7)
    fn = tmp_path / "ref.tgrid"
    assert ref.fn("grid_save")(g.h, str(fn).encode()) == 0
    p = g.pools()
    dg = tv.load_grid(fn)
    info = dg.info()
    assert info["max_level"] == 48 and info["n_leaves"] == int(p.leaf_mask.sum())
    v, t, r = dg.download()
    t = t.view(O.TET_DTYPE)
    assert np.array_equal(v, p.vq) and np.array_equal(r, p.roots)
    for k in FIELDS:
        assert np.array_equal(t[k], p.tets[k]), k
    # and it renders like the same pools uploaded directly
    cam = tv.PinholeCamera((0.5, 0.5, -1.5), (0, 0, 1), (0, 1, 0), 45, 40, 40)
    rc = tv.RenderConfig(spp=2, max_bounces=8, seed=1)
    a, b = tv.render(dg, cam, rc), tv.render(upload(tv, p), cam, rc)
    assert np.array_equal(a.sum.view(np.uint64), b.sum.view(np.uint64))


def _corrupt(raw: bytes, nv: int, nt: int):
    """Malformed variants of a valid file, each hitting one load_grid check."""
    hdr = 16
    tets_at = hdr + nv * 12 + 8
    roots_at = tets_at + nt * 90
    rec = lambda i: tets_at + i * 90  # noqa: E731
    off = {n: TET_RECORD.fields[n][1] for n in TET_RECORD.names}
    b = bytearray

    def put(buf, at, val, n):
        buf[at:at + n] = int(val).to_bytes(n, "little")
        return bytes(buf)

    yield "magic", b"TGRX" + raw[4:]
    yield "version", put(b(raw), 4, 2, 4)
    yield "vertex count", put(b(raw), 8, 7, 8)
    yield "coordinate", put(b(raw), hdr + 5 * 12 + 4, (1 << 24) + 1, 4)
    yield "tet count", put(b(raw), hdr + nv * 12, 23, 8)
    yield "vertex id", put(b(raw), rec(30) + off["verts"], nv, 4)
    yield "tet id", put(b(raw), rec(31) + off["parent"], 1 << 40, 8)
    yield "normal id", put(b(raw), rec(32) + off["normal_ids"] + 2, 18, 1)
    yield "child id", put(b(raw), rec(33) + off["children"], nt + 5, 8)
    yield "parent id", put(b(raw), rec(34) + off["parent"], nt, 8)
    yield "neighbor id", put(b(raw), rec(35) + off["neighbors"] + 8, nt + 1, 8)
    two = put(b(raw), rec(40) + off["normal_ids"], 30, 1)  # later record: vertex id wins (record 20)
    yield "first record wins", put(b(two), rec(20) + off["verts"] + 4, nv + 3, 4)
    yield "root id", put(b(raw), roots_at + 8 * 3, nt, 8)
    yield "root sentinel", put(b(raw), roots_at + 8 * 5, (1 << 64) - 1, 8)
    yield "truncated tets", raw[:rec(50) + 17]
    yield "truncated verts", raw[:hdr + 4 * 12 + 3]
    yield "truncated roots", raw[:roots_at + 8 * 10]
    yield "empty", b""


@needs_ref
def test_load_errors_match_reference(tv, tmp_path):
    g = O.fuzzed(ref, 120, 3)
    fn = tmp_path / "ok.tgrid"
    assert ref.fn("grid_save")(g.h, str(fn).encode()) == 0
    raw = fn.read_bytes()
    c = g.counts()
    for name, bad in _corrupt(raw, c["n_verts"], c["n_tets"]):
        path = tmp_path / f"bad_{name.replace(' ', '_')}.tgrid"
        path.write_bytes(bad)
        assert not ref.fn("grid_load")(str(path).encode()), name
        want = ref.err()
        with pytest.raises(tv.FormatError) as e:
            tv.load_grid(path)
        got = str(e.value)
        assert got == want, (name, got, want)


def test_io_errors(tv, c1, tmp_path):
    with pytest.raises(tv.IoError, match="cannot open for writing"):
        upload(tv, c1).save(tmp_path / "no" / "such" / "dir.tgrid")
    with pytest.raises(tv.IoError, match="cannot open"):
        tv.load_grid(tmp_path / "missing.tgrid")
