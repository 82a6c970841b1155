"""TetGrid::validate on the GPU (tv_grid_validate) against the reference's own
validate() on the same pools: ok flag, first violation message, leaf and face
counts — on valid grids and on pools corrupted one invariant at a time. Plus
cmd_validate's traversal spot checks against the reference's loop.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ref = O.ref_oracle()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def tv():
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tv


def ref_report(p):
    g = O.from_pools(ref, p)
    msg = C.create_string_buffer(256)
    out = np.zeros(3, np.uint64)
    ok = ref.fn("grid_validate")(g.h, msg, 256, out.ctypes.data_as(O._U64))
    return dict(ok=bool(ok), firstViolation=msg.value.decode() or None, leafCount=int(out[0]),
                interiorFaces=int(out[1]), boundaryFaces=int(out[2]))


def mine(tv, p):
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    r = dg.validate()
    return {k: (int(v) if isinstance(v, (np.integer,)) else v) for k, v in r.items()}


@needs_ref
def test_valid_grids(tv):
    grids = [O.fuzzed(O.c_oracle(), 300, 11).pools(), O.init_roots(O.c_oracle()).pools(),
             O.build(O.c_oracle(), O.gen_volume("blob", 48), O.build_cfg(0.15, 12, False, 1.0, 8.0))[0].pools()]
    for p in grids:
        r = mine(tv, p)
        assert r == ref_report(p) and r["ok"]


def _corruptions(p):
    """(name, pools) with one invariant broken; every case must still pass the upload range checks."""
    leaf = np.nonzero(p.leaf_mask)[0]
    internal = np.nonzero(~p.leaf_mask)[0]
    rng = np.random.default_rng(0)

    def cp():
        return O.Pools(p.vq.copy(), p.tets.copy(), p.roots.copy(), p.max_level)

    q = cp()
    q.tets["normal_ids"][leaf[5], 1] ^= 1
    yield "normal flipped", q
    q = cp()
    t = leaf[17]
    nb = q.tets["neighbors"][t]
    s = int(np.nonzero(nb != O.NO_TET)[0][0])
    q.tets["neighbors"][t, s] = leaf[3] if nb[s] != leaf[3] else leaf[4]
    yield "neighbor not reciprocal", q
    q = cp()
    deep = internal[q.tets["level"][internal] > 0]
    q.tets["level"][deep[2]] = 60
    yield "level cap", q
    q = cp()
    q.tets["mask"][internal[4]] = 1
    yield "internal payload", q
    q = cp()
    c = q.tets["children"][internal[6], 0]
    q.tets["parent"][c] = internal[7]
    yield "child parent", q
    q = cp()
    c = q.tets["children"][internal[8], 1]
    q.tets["level"][c] += 1
    yield "child level", q
    q = cp()
    v = q.tets["verts"][leaf[9], 0]
    q.vq[v, 0] += 1
    yield "vertex moved", q
    q = cp()
    q.vq[q.tets["verts"][leaf[11], 2]] = q.vq[q.tets["verts"][leaf[11], 3]]
    yield "duplicate vertex", q
    q = cp()
    q.roots[3] = internal[-1] if q.tets["level"][internal[-1]] else leaf[-1]
    yield "root table", q
    q = cp()
    t = leaf[20]
    q.tets["verts"][t, [0, 1]] = q.tets["verts"][t, [1, 0]]
    yield "orientation", q
    q = cp()
    t = leaf[25]
    b = int(np.nonzero(q.tets["neighbors"][t] == O.NO_TET)[0][0]) if np.any(q.tets["neighbors"][t] == O.NO_TET) else 0
    q.tets["neighbors"][t, b] = leaf[26]
    yield "boundary link", q
    q = cp()
    t = leaf[int(rng.integers(len(leaf)))]
    q.tets["normal_ids"][t] = (q.tets["normal_ids"][t] + 2) % 18
    yield "normals shuffled", q


@needs_ref
def test_corrupted_pools_match_reference(tv):
    p = O.fuzzed(O.c_oracle(), 400, 5).pools()
    seen = set()
    for name, q in _corruptions(p):
        want = ref_report(q)
        got = mine(tv, q)
        assert got == want, (name, got, want)
        assert not got["ok"], name
        seen.add(got["firstViolation"])
    assert len(seen) >= 8, seen  # the cases reach distinct checks


@needs_ref
def test_gpu_build_validates(tv):
    vol = O.gen_volume("cloud", 40)
    cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 128, 128)
    dg, _ = tv.build_adaptive_grid(vol, tv.BuildConfig(0.15, 16, True, 1.0, 16.0), cam)
    r = dg.validate()
    v, t, roots = dg.download()
    assert r == ref_report(O.Pools(v, t.view(O.TET_DTYPE), roots, 48)) and r["ok"]


@needs_ref
def test_spot_checks_match_reference(tv):
    for steps, seed in [(200, 1), (500, 4)]:
        p = O.fuzzed(O.c_oracle(), steps, seed).pools()
        dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
        got = dg.spot_check(60, seed)
        f, first = C.c_int(), C.c_int()
        g = O.from_pools(ref, p)
        ref.fn("spot_checks")(g.h, 60, seed, C.byref(f), C.byref(first))
        assert got == (f.value, first.value)
        assert got == (0, -1)
