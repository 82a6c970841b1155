"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libtetvol_ref.so, compiled
from /root/reference/proj/src by `make -f oracle/Makefile ref`) on the
known-answer workloads of SURVEY.md 8(c) and the reference's own tests, and
records bit patterns / hashes. tests/test_oracle.py then pins the C
restatement (oracle/liboracle.so) to these values without needing the
reference, and the GPU tests pin the CUDA path to the oracle.

    python tests/golden/make_golden.py
"""
import ctypes as C
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

_D = C.POINTER(C.c_double)


def h(*arrays) -> str:
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


def bits(x: float) -> str:
    return np.float64(x).view(np.uint64).item().to_bytes(8, "big").hex()


def c1_rays(chk, W=256, H=256, spp=4):
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, W, H)
    out = np.zeros(6)
    d = np.zeros(2)
    rays = np.zeros((W * H * spp, 8))
    k = 0
    for y in range(H):
        for x in range(W):
            for s in range(spp):
                chk.fn("rng_draws")(0, y * W + x, s, 2, d.ctypes.data_as(_D))
                chk.fn("primary_ray")(C.byref(cam), x, y, d[0], d[1], out.ctypes.data_as(_D))
                rays[k, :6] = out
                rays[k, 7] = np.inf
                k += 1
    return rays


def main():
    R = O.ref_oracle()
    if R is None:
        sys.exit("oracle/_ref/libtetvol_ref.so missing: run `make -f oracle/Makefile ref` (needs /root/reference)")
    gold = {"generator": "tests/golden/make_golden.py", "source": "reference tetvol compiled from /root/reference"}

    # rng.hpp KAT (test_tracer.cpp:53-70 uses RngStream(7, 123, 9))
    gold["rng_7_123_9"] = [bits(x) for x in O.rng_draws(R, 7, 123, 9, 16)]
    gold["mix64"] = {str(x): R.fn("mix64")(x) for x in [0, 1, 2, 12345, 0xDEADBEEF, 2**63]}

    # tracer.cpp KATs
    gold["hg_sample_cos"] = {f"{g}_{xi}": bits(R.fn("hg_sample_cos")(g, xi))
                             for g in [0.0, 0.3, 0.6, 0.9, -0.5] for xi in [0.0, 0.1, 0.5, 0.9, 0.999]}
    e = np.zeros(3)
    em = {}
    for t in [-1.0, 0.0, 0.05, 0.2, 0.5, 0.77, 0.999, 1.0, 3.0]:
        R.fn("emission_color")(t, e.ctypes.data_as(_D))
        em[str(t)] = [bits(x) for x in e]
    gold["emission_color"] = em
    w = np.zeros(3)
    dirn = np.array([0.3, -0.8, 0.52])
    dirn = dirn / np.sqrt((dirn[0] * dirn[0] + dirn[1] * dirn[1]) + dirn[2] * dirn[2])
    ph = {}
    for g in [0.0, 0.3, 0.9, -0.5]:
        for i in range(4):
            R.fn("sample_phase_hg")(dirn.ctypes.data_as(_D), g, 8, 0x697369, i, w.ctypes.data_as(_D))
            ph[f"{g}_{i}"] = [bits(x) for x in w]
    gold["phase_dir"] = [bits(x) for x in dirn]
    gold["sample_phase_hg"] = ph

    # camera.cpp KATs
    cam = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 256, 256)
    out = np.zeros(6)
    pr = {}
    for (x, y, jx, jy) in [(0, 0, 0.0, 0.0), (17, 200, 0.25, 0.75), (255, 255, 0.999, 0.5)]:
        R.fn("primary_ray")(C.byref(cam), x, y, jx, jy, out.ctypes.data_as(_D))
        pr[f"{x}_{y}_{jx}_{jy}"] = [bits(v) for v in out]
    gold["primary_ray"] = pr

    # tet_grid: roots, fuzzed grids
    g0 = O.init_roots(R)
    p0 = g0.pools()
    gold["init_roots"] = {"counts": g0.counts(), "sha": h(p0.vq, p0.tets, p0.roots)}
    fz = O.fuzzed(R, 400, 0x52)
    pf = fz.pools()
    gold["fuzzed_400_0x52"] = {"counts": fz.counts(), "sha": h(pf.vq, pf.tets, pf.roots)}
    rays = O.random_cube_rays(5, 0x7472617665727365, 10000, R)
    gold["acceptance5_rays_sha"] = h(rays)
    cells, t0, t1, off, st = fz.march_segments(rays)
    gold["acceptance5_segments"] = {"total": int(len(cells)), "sha": h(cells, t0, t1, off),
                                    "degenerate": int(st[1])}

    # C1
    vol = O.gen_volume("blob", 64)
    gold["blob64_sha"] = h(vol)
    gold["cloud64_sha"] = h(O.gen_volume("cloud", 64))
    gold["noise32_sha"] = h(O.gen_volume("noise", 32))
    g, st = O.build(R, vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
    p = g.pools()
    lm = p.leaf_mask
    gold["c1_grid"] = {"counts": g.counts(), "stats": {k: v for k, v in st.items() if k != "seconds"},
                       "sha": h(p.vq, p.tets, p.roots),
                       "sum_leaf_density": bits(float(p.tets["density"][lm].astype(np.float64).sum()))}
    with tempfile.TemporaryDirectory() as td:  # save_grid bytes (builder.cpp:210-235)
        fn = os.path.join(td, "c1.tgrid")
        assert R.fn("grid_save")(g.h, fn.encode()) == 0, R.err()
        raw = open(fn, "rb").read()
    gold["c1_tgrid"] = {"bytes": len(raw), "sha256": hashlib.sha256(raw).hexdigest()}
    rc = O.render_cfg(spp=4, max_bounces=2, seed=0)
    img = g.render(cam, rc, 0)
    gold["c1_render"] = {"cells_visited": img["cells_visited"], "degenerate_paths": img["degenerate_paths"],
                         "fnv_sum": hex(O.fnv64(img["sum"])), "fnv_sum_sq": hex(O.fnv64(img["sum_sq"])),
                         "sum_total": bits(float(img["sum"].sum()))}
    rc64 = O.render_cfg(spp=64, max_bounces=64, seed=0)
    img64 = g.render(cam, rc64, 0)
    gold["c1_multibounce_64spp"] = {"cells_visited": img64["cells_visited"], "fnv_sum": hex(O.fnv64(img64["sum"]))}
    crays = c1_rays(R)
    cc, ct0, ct1, coff, _ = g.march_segments(crays)
    gold["c1_primary_segments"] = {"total": int(len(cc)), "sha": h(cc, ct0, ct1, coff)}
    rng = np.random.default_rng(3)
    pts = rng.random((5000, 3))
    pts[:1000] = np.round(pts[:1000] * 64) / 64
    gold["c1_locate_sha"] = h(np.array([g.locate(q) for q in pts], np.uint32))

    # camera-criterion build (acceptance 11 shape: blob 32, vfov 16, 128^2, pixel_threshold 0.5)
    cam11 = O.camera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 16, 128, 128)
    g11, st11 = O.build(R, O.gen_volume("blob", 32), O.build_cfg(0.15, 9, True, 0.5, 1.0), cam11)
    p11 = g11.pools()
    gold["acc11_camera_build"] = {"counts": g11.counts(), "sha": h(p11.vq, p11.tets, p11.roots),
                                  "criterion_splits": st11["criterion_splits"]}
    # cloud 64 with the C2 camera (SURVEY.md 8(d) field) — build parity target
    camc = O.camera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
    gc, stc = O.build(R, O.gen_volume("cloud", 64), O.build_cfg(0.15, 18, True, 1.0, 16.0), camc)
    pc = gc.pools()
    gold["cloud64_camera_build"] = {"counts": gc.counts(), "sha": h(pc.vq, pc.tets, pc.roots),
                                    "criterion_splits": stc["criterion_splits"],
                                    "propagation_splits": stc["propagation_splits"], "max_depth": stc["max_depth"]}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
