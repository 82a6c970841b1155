"""N4: the tetvol_b200 command-line tool (cli.cpp's subcommands over the C ABI):
the JSON reports (schema 1, the reference's keys), the files it writes, and
the exit codes (0 ok, 1 failure, 2 usage / config error), end to end on the GPU.
"""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from oracle.images import compare, dvol_bytes

pytestmark = pytest.mark.gpu
ref = O.ref_oracle()
CLI = os.path.join(os.path.dirname(__file__), "..", "paper_2506_11510_b200", "_lib", "tetvol_b200")


def run(*args, rc=0):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert p.returncode == rc, (args, p.returncode, p.stdout, p.stderr)
    return (json.loads(p.stdout) if rc == 0 and p.stdout.strip() else None), p


@pytest.fixture(scope="module")
def work(tmp_path_factory):
    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    return tmp_path_factory.mktemp("cli")


def test_gen_build_validate_stats(work):
    vol = work / "b.dvol"
    j, _ = run("gen", "--kind", "blob", "--dims", "32", "--out", vol, "--with-temperature", "--with-albedo", "0.6")
    assert j == {"schema": 1, "command": "gen", "kind": "blob", "dims": [32, 32, 32],
                 "channels": ["density", "temperature", "albedo"], "out": str(vol)}
    host = O.gen_volume("blob", 32)
    want = dvol_bytes((32, 32, 32), {"density": host, "temperature": np.clip(host, np.float32(0), np.float32(1)),
                                     "albedo": np.full_like(host, np.float32(0.6))})
    assert vol.read_bytes() == want

    grid = work / "b.tgrid"
    j, _ = run("build", "--volume", vol, "--out", grid, "--threshold", "0.15", "--max-level", "12",
               "--density-scale", "8")
    assert set(j) == {"schema", "command", "leafCount", "maxDepthReached", "buildSeconds", "criterionSplits",
                      "propagationSplits", "tetCount", "vertexCount", "out"}
    og, st = O.build(O.c_oracle(), host, O.build_cfg(0.15, 12, False, 1.0, 8.0),
                     temperature=np.clip(host, np.float32(0), np.float32(1)), albedo=np.full_like(host, np.float32(0.6)))
    assert j["leafCount"] == st["leaf_count"] and j["tetCount"] == og.counts()["n_tets"]

    j, p = run("validate", "--grid", grid, "--rays", "40", "--seed", "3")
    assert j["ok"] is True and j["firstViolation"] is None and j["rayChecks"] == 40 and j["rayFailures"] == 0
    assert "grid OK" in p.stderr
    if ref is not None:
        rg = O.Grid(ref, ref.fn("grid_load")(str(grid).encode()))
        msg = C.create_string_buffer(256)
        out = np.zeros(3, np.uint64)
        assert ref.fn("grid_validate")(rg.h, msg, 256, out.ctypes.data_as(O._U64)) == 1
        assert [j["leafCount"], j["interiorFaces"], j["boundaryFaces"]] == out.tolist()

    j, _ = run("stats", "--grid", grid)
    pools = O.Grid(ref, ref.fn("grid_load")(str(grid).encode())).pools() if ref is not None else og.pools()
    lm = pools.leaf_mask
    d = pools.tets["density"][lm].astype(np.float64)
    lev = pools.tets["level"][lm]
    assert j["leafCount"] == int(lm.sum()) and j["maxLeafLevel"] == int(lev.max())
    assert j["leavesPerLevel"] == np.bincount(lev).tolist()
    assert j["density"] == {"min": d.min(), "max": d.max(), "mean": np.cumsum(d)[-1] / len(d)}

    j, _ = run("stats", "--volume", vol)
    assert j["kind"] == "volume" and j["dims"] == [32, 32, 32]
    ch = j["channels"][0]
    dd = host.ravel().astype(np.float64)
    assert ch == {"name": "density", "min": dd.min(), "max": dd.max(), "mean": np.cumsum(dd)[-1] / dd.size}


def test_render_compare(work):
    vol = work / "c.dvol"
    run("gen", "--kind", "cloud", "--dims", "24", "--out", vol)
    grid = work / "c.tgrid"
    cam = ["--position", "0.5,0.5,-1.2", "--forward", "0,0,1", "--vfov", "40", "--width", "40", "--height", "32"]
    cfg = work / "r.ini"
    cfg.write_text("[render]\nspp = 6\nmax_bounces = 16  # comment\nseed = 4\n[build]\ndensity_scale = 16\n")
    run("build", "--volume", vol, "--out", grid, "--threshold", "0.15", "--max-level", "14", "--config", cfg)
    out = {}
    for mode in ("tet", "reference"):
        src = ["--grid", grid] if mode == "tet" else ["--volume", vol, "--reference"]
        j, _ = run("render", *src, *cam, "--config", cfg, "--pfm", work / f"{mode}.pfm", "--var-pfm",
                   work / f"{mode}_v.pfm", "--ppm", work / f"{mode}.ppm", "--stats-out", work / f"{mode}.json")
        assert j["mode"] == mode and j["spp"] == 6 and j["seed"] == 4 and j["paths"] == 40 * 32 * 6
        assert json.loads((work / f"{mode}.json").read_text()) == j
        assert (work / f"{mode}.ppm").read_bytes().startswith(b"P6\n40 32\n255\n")
        assert len((work / f"{mode}.ppm").read_bytes()) == len(b"P6\n40 32\n255\n") + 40 * 32 * 3
        out[mode] = j
    assert out["reference"]["cellCount"] == 24 ** 3
    if ref is not None:  # the tet render's PFM equals the reference renderer on the same file
        rg = O.Grid(ref, ref.fn("grid_load")(str(grid).encode()))
        img = rg.render(O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 40, 32), O.render_cfg(6, 16, 4), 0)
        fn = work / "ref.pfm"
        assert ref.fn("write_pfm")(str(fn).encode(), 40, 32, img["sum"].ctypes.data_as(O._D),
                                   img["sum_sq"].ctypes.data_as(O._D), img["counts"].ctypes.data_as(O._U32), 0) == 0
        assert fn.read_bytes() == (work / "tet.pfm").read_bytes()
        assert out["tet"]["cellsVisited"] == img["cells_visited"]

    j, _ = run("compare", "--image-a", work / "tet.pfm", "--image-b", work / "reference.pfm", "--stats-a",
               work / "tet.json", "--stats-b", work / "reference.json", "--var-a", work / "tet_v.pfm", "--var-b",
               work / "reference_v.pfm")
    import paper_2506_11510_b200 as tv

    a, b = tv.read_pfm(work / "tet.pfm"), tv.read_pfm(work / "reference.pfm")
    va, vb = tv.read_pfm(work / "tet_v.pfm"), tv.read_pfm(work / "reference_v.pfm")
    want = compare(a.rgb, b.rgb, va.rgb, vb.rgb)
    assert j["maxAbsDiff"] == want["maxAbsDiff"] and j["outlierFraction"] == want["outlierFraction"]
    assert j["rmse"] == pytest.approx(want["rmse"], rel=1e-12)
    ta, tb = out["tet"], out["reference"]
    assert j["speedup"] == tb["seconds"] / ta["seconds"]
    assert j["cellCountRatio"] == tb["cellCount"] / ta["cellCount"]
    assert j["cellsVisitedRatio"] == pytest.approx((tb["cellsVisited"] / tb["paths"]) /
                                                   (ta["cellsVisited"] / ta["paths"]), rel=1e-15)
    j, _ = run("compare", "--image-a", work / "tet.pfm", "--image-b", work / "tet.pfm", "--stats-a",
               work / "tet.json", "--stats-b", work / "tet.json")
    assert j["rmse"] == 0.0 and j["outlierFraction"] is None and j["speedup"] == 1.0


def test_exit_codes(work):
    run(rc=2)
    run("nope", rc=2)
    run("gen", "--out", work / "x.dvol", rc=2)                          # --kind is required
    run("gen", "--kind", "blob", "--out", work / "x.dvol", "--bogus", rc=2)
    run("gen", "--kind", "torus", "--out", work / "x.dvol", rc=2)        # ConfigError
    run("gen", "--kind", "blob", "--dims", "0", "--out", work / "x.dvol", rc=2)
    run("gen", "--kind", "blob", "--dims", "4", "--out", work / "x.dvol", "--with-albedo", "2", rc=2)
    run("render", "--grid", work / "missing.tgrid", rc=1)                # IoError
    run("render", "--grid", "a", "--volume", "b", rc=2)                  # excludes
    run("render", "--reference", rc=2)                                  # needs --volume
    run("render", rc=2)                                                 # needs --grid or --volume
    run("stats", rc=2)
    bad = work / "bad.tgrid"
    bad.write_bytes(b"TGRX")
    _, p = run("validate", "--grid", bad, rc=1)
    assert "not a TGRD file" in p.stderr
    vol = work / "e.dvol"
    run("gen", "--kind", "constant", "--dims", "8", "--out", vol)
    _, p = run("render", "--volume", vol, "--spp", "0", rc=2)
    assert "spp must be at least 1" in p.stderr
    _, p = run("render", "--volume", vol, "--forward", "0,0,1", "--look-at", "1,1,1", rc=2)
    assert "look_at or forward" in p.stderr
    cfg = work / "bad.ini"
    cfg.write_text("[camera]\nzoom = 2\n")
    _, p = run("build", "--volume", vol, "--out", work / "e.tgrid", "--config", cfg, rc=2)
    assert "unknown key 'camera.zoom'" in p.stderr
    p = subprocess.run([CLI, "gen", "--help"], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and "--kind" in p.stdout
