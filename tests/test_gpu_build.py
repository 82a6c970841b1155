"""GPU LEB build parity: tv_build against build_adaptive_grid (builder.cpp:118-182).

Tet and vertex ids are allocation-order artefacts, so parity is
on the canonical leaf set: every leaf as its sorted four fixed-point corners,
plus the f32 bit patterns of its payload and its mask — bit-exact. The
downloaded GPU grid must also pass the reference's own TetGrid::validate()
(conformity, reciprocal neighbour links, canonical normals, exact volume), and
render bit-identically to the oracle-built grid.
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


def canonical(vq, tets):
    leaf = tets["children"][:, 0] == O.NO_TET
    t = tets[leaf]
    corners = vq[t["verts"]]  # (L, 4, 3)
    order = np.lexsort((corners[:, :, 2], corners[:, :, 1], corners[:, :, 0]), axis=1)
    corners = np.take_along_axis(corners, order[:, :, None], axis=1).reshape(len(t), 12)
    pay = np.stack([t["density"].view(np.uint32), t["temperature"].view(np.uint32), t["albedo"].view(np.uint32),
                    t["mask"].astype(np.uint32), t["level"].astype(np.uint32)], axis=1)
    rows = np.concatenate([corners.astype(np.uint64), pay.astype(np.uint64)], axis=1)
    idx = np.lexsort(rows.T[::-1])
    return rows[idx]


def gpu_build(tv, vol, bc, cam=None, temperature=None, albedo=None):
    tb = tv.BuildConfig(bc.variation_threshold, bc.max_level, bool(bc.use_camera), bc.pixel_threshold,
                        bc.density_scale)
    tcam = None
    if cam is not None:
        tcam = tv.PinholeCamera(tuple(cam.pos), tuple(cam.fwd), tuple(cam.up), cam.vfov, cam.width, cam.height)
    return tv.build_adaptive_grid(vol, tb, tcam, temperature=temperature, albedo=albedo)


def check_same(tv, vol, bc, cam=None, temperature=None, albedo=None, validate=True):
    og, ost = O.build(O.c_oracle(), vol, bc, cam, temperature, albedo)
    dg, dst = gpu_build(tv, vol, bc, cam, temperature, albedo)
    v, t, r = dg.download()
    p = og.pools()
    assert dst.leaf_count == ost["leaf_count"]
    assert dst.max_depth == ost["max_depth"]
    assert len(t) == len(p.tets) and len(v) == len(p.vq)
    a, b = canonical(p.vq, p.tets), canonical(v, t.view(O.TET_DTYPE))
    assert np.array_equal(a, b), "canonical leaf set / payload bits differ"
    # total bisections are order independent; the criterion/propagation split is reported
    assert dst.criterion_splits + dst.propagation_splits == ost["criterion_splits"] + ost["propagation_splits"]
    ref = O.ref_oracle()
    if validate and ref is not None:
        pools = O.Pools(v, t.view(O.TET_DTYPE), r, 48)
        rg = O.from_pools(ref, pools)
        msg = O.C.create_string_buffer(256)
        out = np.zeros(3, np.uint64)
        ok = ref.fn("grid_validate")(rg.h, msg, 256, out.ctypes.data_as(O._U64))
        assert ok == 1, msg.value.decode()
    return og, ost, dg, dst


def test_build_c1_blob(tv):
    vol = O.gen_volume("blob", 64)
    og, ost, dg, dst = check_same(tv, vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
    assert dst.leaf_count == 51020
    # the GPU-built grid renders bit-identically (golden C1 hash)
    img = tv.render(dg, tv.PinholeCamera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 256, 256),
                    tv.RenderConfig(spp=4, max_bounces=2, seed=0))
    assert img.cells_visited == 4612915
    assert O.fnv64(img.sum) == 0x5DD59BA4FB717D7F


def test_build_constant_stays_at_roots(tv):
    """test_builder.cpp:53-72"""
    vol = O.gen_volume("constant", 8, 1.0)
    _, _, dg, dst = check_same(tv, vol, O.build_cfg(0.1, 10, False, 1.0, 2.5))
    assert dst.leaf_count == 24 and dst.max_depth == 0 and dst.criterion_splits == 0
    _, t, _ = dg.download()
    assert np.all(t["density"] == np.float32(2.5)) and np.all(t["mask"] == 1)


def test_build_step_noise_ramp(tv):
    for kind, n, thr, ml, sc in [("step", 16, 0.5, 6, 1.0), ("noise", 24, 0.2, 10, 3.0), ("ramp", 12, 0.05, 8, 1.0),
                                 ("step", 33, 0.3, 15, 4.0)]:
        check_same(tv, O.gen_volume(kind, n), O.build_cfg(thr, ml, False, 1.0, sc))


def test_build_camera_criterion_acceptance11(tv):
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 16, 128, 128)
    _, _, _, dst = check_same(tv, O.gen_volume("blob", 32), O.build_cfg(0.15, 9, True, 0.5, 1.0), cam)
    assert dst.leaf_count == 7528


def test_build_cloud64_camera(tv):
    """cloud64 + camera -> 361,510 leaves."""
    cam = O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
    _, _, _, dst = check_same(tv, O.gen_volume("cloud", 64), O.build_cfg(0.15, 18, True, 1.0, 16.0), cam)
    assert dst.leaf_count == 361510


def test_build_with_temperature_and_albedo(tv):
    vol = O.gen_volume("noise", 20)
    temp = np.clip(vol, 0, 1).astype(np.float32)
    alb = (0.3 + 0.5 * O.gen_volume("ramp", 20)).astype(np.float32)
    check_same(tv, vol, O.build_cfg(0.1, 9, False, 1.0, 5.0), None, temp, alb)


def test_build_nonuniform_dims(tv):
    vol = np.ascontiguousarray(O.gen_volume("cloud", 48)[:, 5:37, 3:43])  # (48, 32, 40)
    check_same(tv, vol, O.build_cfg(0.3, 14, False, 1.0, 8.0))
    # dims below and across the 8^3 brick size: only partial bricks on two axes
    vol = np.ascontiguousarray(O.gen_volume("noise", 21)[:5, :7, :])  # (5, 7, 21)
    check_same(tv, vol, O.build_cfg(0.1, 12, False, 1.0, 4.0))
    vol = np.ascontiguousarray(O.gen_volume("blob", 40)[:, :, :33])  # (40, 40, 33)
    check_same(tv, vol, O.build_cfg(0.2, 12, False, 1.0, 8.0))


def test_build_config_errors(tv):
    vol = O.gen_volume("blob", 8)
    with pytest.raises(tv.ConfigError, match="variationThreshold"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(variation_threshold=-1.0))
    with pytest.raises(tv.ConfigError, match="maxLevel"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(max_level=49))
    with pytest.raises(tv.ConfigError, match="useCamera"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(use_camera=True))


def test_build_leaves_the_default_mempool_alone(tv):
    """Build scratch is the library's own (VMM mappings kept for the next
    build): the device's default pool keeps its release threshold,
    and two builds of the same field give identical grids (determinism)."""
    from cuda.bindings import runtime as rt

    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    assert err == rt.cudaError_t.cudaSuccess
    attr = rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold
    err, before = rt.cudaMemPoolGetAttribute(pool, attr)
    vol = O.gen_volume("cloud", 48)
    bc = tv.BuildConfig(0.3, 12, False, 1.0, 8.0)
    g1, s1 = tv.build_adaptive_grid(vol, bc)
    g2, s2 = tv.build_adaptive_grid(vol, bc)
    err, after = rt.cudaMemPoolGetAttribute(pool, attr)
    assert int(after) == int(before)
    v1, t1, r1 = g1.download()
    v2, t2, r2 = g2.download()
    assert s1.leaf_count == s2.leaf_count
    assert np.array_equal(v1, v2) and np.array_equal(t1.view(np.uint8), t2.view(np.uint8))


def test_build_from_misaligned_device_volume(tv):
    """tv_build_dev reads the volume as float4; a channel pointer that is not
    16-byte aligned is copied first and builds the same grid."""
    import torch

    vol = O.gen_volume("cloud", 40)
    flat = torch.from_numpy(np.ascontiguousarray(vol).reshape(-1)).cuda()
    shifted = torch.zeros(flat.numel() + 1, dtype=torch.float32, device="cuda")
    shifted[1:] = flat
    bc = tv.BuildConfig(0.3, 12, False, 1.0, 8.0)
    g1, s1 = tv.build_adaptive_grid_dev(flat.data_ptr(), (40, 40, 40), bc)
    g2, s2 = tv.build_adaptive_grid_dev(shifted[1:].data_ptr(), (40, 40, 40), bc)
    assert shifted[1:].data_ptr() % 16 != 0
    v1, t1, _ = g1.download()
    v2, t2, _ = g2.download()
    assert s1.leaf_count == s2.leaf_count
    assert np.array_equal(v1, v2) and np.array_equal(t1.view(np.uint8), t2.view(np.uint8))


def test_build_scratch_allocators_agree(tv, tmp_path):
    """Build scratch is VMM-backed and kept per device between builds
    (tv_build_trim releases it). A buffer grows by mapping more physical memory
    behind its pointer; one that outgrows its virtual range moves its handles
    to a larger range without a copy. Each subprocess first builds a different
    field (leaving stale scratch behind), then the cloud64 + camera grid:
    default; TV_BUILD_VMM_TIGHT=1 (granule steps, exactly-sized ranges: every
    growth is a move); TV_BUILD_NO_VMM=1 (cudaMalloc + copy); TV_BUILD_CACHE=0
    (fresh scratch per build); TV_BUILD_POISON=1 (every byte a build has not
    written reads 0x5A); TV_VOX_BRICKS=0 (per-voxel ownership sweeps instead
    of 8^3 bricks); TV_HANG_PROBE=0 (every closure pass scans all tet ids for
    hanging edges) and TV_HANG_PROBE_COST=1 with TV_HANG_CHECK=1 (nearly every
    pass finds them by probes around the new midpoints, and the build fails if
    a full scan marks anything more). All give the same grid, byte for byte."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import oracle as O, paper_2506_11510_b200 as tv; "
            "tv.build_adaptive_grid(O.gen_volume('noise', 80), tv.BuildConfig(0.05, 14, False, 1.0, 3.0)); "
            "held = tv.build_scratch_bytes(0); "
            "cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024); "
            "g, s = tv.build_adaptive_grid(O.gen_volume('cloud', 64), tv.BuildConfig(0.15, 18, True, 1.0, 16.0), cam); "
            "v, t, r = g.download(); np.savez(sys.argv[1], v=v, t=t.view(np.uint8), n=s.leaf_count, held=held)" % root)
    out = {}
    for name, env in [("vmm", {}), ("tight", {"TV_BUILD_VMM_TIGHT": "1"}), ("malloc", {"TV_BUILD_NO_VMM": "1"}),
                      ("nocache", {"TV_BUILD_CACHE": "0"}), ("poison", {"TV_BUILD_POISON": "1"}),
                      ("poison_tight", {"TV_BUILD_POISON": "1", "TV_BUILD_VMM_TIGHT": "1"}),
                      ("no_bricks", {"TV_VOX_BRICKS": "0"}), ("scan_hanging", {"TV_HANG_PROBE": "0"}),
                      ("probe_hanging", {"TV_HANG_PROBE_COST": "1", "TV_HANG_CHECK": "1"})]:
        f = str(tmp_path / f"{name}.npz")
        e = dict(os.environ, **env)
        subprocess.run([sys.executable, "-c", code, f], check=True, env=e, timeout=300)
        out[name] = np.load(f)
    assert int(out["vmm"]["n"]) == 361510
    assert int(out["vmm"]["held"]) > 0 and int(out["nocache"]["held"]) == 0
    for name in out:
        assert np.array_equal(out[name]["v"], out["vmm"]["v"]), name
        assert np.array_equal(out[name]["t"], out["vmm"]["t"]), name


def test_build_trim_releases_scratch(tv):
    vol = O.gen_volume("cloud", 40)
    bc = tv.BuildConfig(0.3, 12, False, 1.0, 8.0)
    g1, s1 = tv.build_adaptive_grid(vol, bc)
    assert tv.build_scratch_bytes(0) > 0
    tv.build_trim(0)
    assert tv.build_scratch_bytes(0) == 0
    g2, s2 = tv.build_adaptive_grid(vol, bc)
    v1, t1, _ = g1.download()
    v2, t2, _ = g2.download()
    assert np.array_equal(v1, v2) and np.array_equal(t1.view(np.uint8), t2.view(np.uint8))
    tv.build_trim()


def test_build_bricks_match_per_voxel_sweep_cloud256(tv):
    """At 256^3 most 8^3 bricks stay uniform through the early rounds and
    descend whole: the grid (pools and stats) must equal the per-voxel
    ownership sweep's (TV_VOX_BRICKS=0) byte for byte. The CPU oracle is too
    slow at this size; test_build_cloud64_camera and the others pin the
    per-voxel sweep to it."""
    import hashlib
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib, torch; sys.path.insert(0, %r); import paper_2506_11510_b200 as tv; "
            "n = 256; vol = torch.empty(n ** 3, dtype=torch.float32, device='cuda'); "
            "tv.generate_volume_dev('cloud', n, vol.data_ptr()); "
            "cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024); "
            "g, s = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(1.0, 24, True, 1.0, 16.0), cam); "
            "v, t, r = g.download(); h = hashlib.sha256(v.tobytes() + t.tobytes() + r.tobytes()).hexdigest(); "
            "print(h, s.leaf_count, s.rounds, s.criterion_splits, s.propagation_splits)" % root)
    outs = []
    for env in ({}, {"TV_VOX_BRICKS": "0"}, {"TV_HANG_PROBE": "0"}, {"TV_HANG_PROBE_COST": "2", "TV_HANG_CHECK": "1"}):
        p = subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, **env), timeout=300,
                           capture_output=True, text=True)
        outs.append(p.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] == outs[2] == outs[3]
    assert int(outs[0].split()[1]) == 3840746


def test_build_probe_hanging_test_matches_scan_on_other_fields(tv):
    """The probe hanging test (csrc/tv_build.cu, hanging_probe_kernel) forced on
    every closure pass, with TV_HANG_CHECK=1 (the build fails if the full scan
    marks anything more), on fields other than the cloud: value noise without a
    camera and a step field; the grid equals the default build's byte for byte."""
    import hashlib
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r); import oracle as O, paper_2506_11510_b200 as tv; "
            "out = []\n"
            "for kind, n, thr, ml in (('noise', 96, 0.05, 16), ('step', 64, 0.1, 14), ('ramp', 48, 0.02, 15)):\n"
            "    g, s = tv.build_adaptive_grid(O.gen_volume(kind, n), tv.BuildConfig(thr, ml, False, 1.0, 4.0))\n"
            "    v, t, r = g.download(); out.append(hashlib.sha256(v.tobytes() + t.tobytes()).hexdigest()[:16] + ':' + str(s.leaf_count))\n"
            "print(' '.join(out))" % root)
    outs = []
    for env in ({"TV_HANG_PROBE": "0"}, {"TV_HANG_PROBE_COST": "1", "TV_HANG_CHECK": "1"}, {}):
        p = subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, **env), timeout=300,
                           capture_output=True, text=True)
        outs.append(p.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] == outs[2], outs
