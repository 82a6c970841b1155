"""SURVEY.md 8(d) "CPU timing": the reference's own CPU renderer and builder,
timed with its own clocks (ImageAccumulator::seconds, path_integrator.hpp:91,134),
beside the GPU path on the same inputs. One JSON object per row.

    python tools/cpu_report.py render [c1 c2 c3 c5]   # on the GPU box: all host cores
    python tools/cpu_report.py build [256 512]         # single-threaded reference build (C4 extrapolation)

render rows time both reference builds: "shipped" (oracle/_ref) and "padded"
(oracle/_ref/pad, alignas(64) TraceStats). C1 and C2 run at their
full spp; C3 and C5 at 32 spp (the GPU rows in r01_configs.jsonl are 32 spp too;
1024 spp is 32x that, cost being linear in spp). The C2/C3 tet grids come from
the GPU build, whose leaf set tests/test_gpu_build.py proves identical to the
reference builder's; the reference assembles its own TetGrid from them.

Test/measurement tooling: this is one of the places allowed to call oracle/.
"""
import json
import os
import platform
import resource
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import oracle as O

CAM2 = ((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
CAM1 = ((0.5, 0.5, -2.0), (0, 0, 1), (0, 1, 0), 40, 256, 256)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def row(**kw):
    kw.setdefault("host", {"cpu": cpu_model(), "nproc": os.cpu_count()})
    print(json.dumps(kw), flush=True)


def time_both(pools, cam, rc, label, gpu_ms=None, **extra):
    for name, chk in (("shipped", O.ref_oracle()), ("padded", O.ref_pad_oracle())):
        if chk is None:
            continue
        g = O.from_pools(chk, pools)
        out = g.render(O.camera(*cam), rc, 0)
        s = out["seconds"]
        paths = cam[4] * cam[5] * rc.spp
        r = dict(config=label, build=name, threads=os.cpu_count(), spp=rc.spp, seconds=s,
                 samples_per_s=paths / s, tet_steps_per_s=out["cells_visited"] / s,
                 cells_per_path=out["cells_visited"] / paths, **extra)
        if gpu_ms is not None:
            r["gpu_ms"] = gpu_ms
            r["gpu_speedup"] = s * 1e3 / gpu_ms
        row(**r)
        del g


def gpu_grid(n, thr, ml, cam):
    import torch

    import paper_2506_11510_b200 as tv

    vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    tv.generate_volume_dev("cloud", n, vol.data_ptr())
    pc = tv.PinholeCamera(cam[0], cam[1], cam[2], cam[3], cam[4], cam[5])
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(thr, ml, True, 1.0, 16.0), pc)
    torch.cuda.synchronize()
    return tv, g, vol, pc


def gpu_ms(tv, g, pc, spp, frames=2):
    rc = tv.RenderConfig(spp=spp, max_bounces=64, seed=0)
    return min(tv.render(g, pc, rc).seconds for _ in range(frames)) * 1e3


def render_rows(which):
    if "c1" in which:
        vol = O.gen_volume("blob", 64)
        g, _ = O.build(O.ref_oracle(), vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
        p = g.pools()
        ms = None
        try:
            import paper_2506_11510_b200 as tv

            if tv.device_count() > 0:
                dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
                rc = tv.RenderConfig(spp=4, max_bounces=2, seed=0)
                ms = min(tv.render(dg, tv.PinholeCamera(*CAM1), rc).seconds for _ in range(3)) * 1e3
        except OSError:  # no CUDA library here: CPU rows only
            pass
        time_both(p, CAM1, O.render_cfg(spp=4, max_bounces=2), "C1 (blob 64^3, 256^2 x 4 spp, 2 bounces)",
                  gpu_ms=ms)
    for key, n, thr, ml, spp in (("c2", 256, 0.15, 24, 32), ("c3", 512, 0.15, 27, 32)):
        if key not in which:
            continue
        tv, g, vol, pc = gpu_grid(n, thr, ml, CAM2)
        ms = gpu_ms(tv, g, pc, spp)
        v, t, r = g.download()
        pools = O.Pools(v, t.view(O.TET_DTYPE), r, ml)
        g.close()
        del vol
        time_both(pools, CAM2, O.render_cfg(spp=spp, max_bounces=64), f"{key.upper()} (cloud {n}^3, thr {thr}, "
                  f"1024^2 x {spp} spp)", gpu_ms=ms, leaves=int(pools.leaf_mask.sum()))
    if "c5" in which:
        import torch

        import paper_2506_11510_b200 as tv

        n = 512
        dvol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
        tv.generate_volume_dev("cloud", n, dvol.data_ptr())
        pc = tv.PinholeCamera(*CAM2)
        reg = tv.render_reference_dev(dvol.data_ptr(), (n, n, n), 16.0, pc, tv.RenderConfig(spp=32, max_bounces=64,
                                                                                              seed=0))
        host = dvol.cpu().numpy()
        del dvol
        rc = O.render_cfg(spp=32, max_bounces=64)
        for name, chk in (("shipped", O.ref_oracle()), ("padded", O.ref_pad_oracle())):
            if chk is None:
                continue
            sm, sq = np.zeros(1024 * 1024 * 3), np.zeros(1024 * 1024 * 3)
            cnt = np.zeros(1024 * 1024, np.uint32)
            st = np.zeros(3, np.uint64)
            sec = O.C.c_double()
            rc_ = chk.fn("render_regular")(O._ptr(host, O._F), n, n, n, 16.0, O.C.byref(O.camera(*CAM2)),
                                           O.C.byref(rc), 0, O._ptr(sm, O._D), O._ptr(sq, O._D),
                                           O._ptr(cnt, O._U32), O._ptr(st, O._U64), O.C.byref(sec))
            assert rc_ == 0, chk.err()
            paths = 1024 * 1024 * 32
            row(config="C5 regular grid (cloud 512^3, 1024^2 x 32 spp)", build=name, threads=os.cpu_count(),
                seconds=sec.value, samples_per_s=paths / sec.value, cells_per_path=int(st[0]) / paths,
                gpu_ms=reg.seconds * 1e3, gpu_speedup=sec.value / reg.seconds)


def build_rows(sizes):
    """single-threaded reference builder (builder.cpp:118-162), C4 settings
    (no camera, threshold 2.0, max_level 3*log2(n))."""
    for n in sizes:
        vol = O.gen_volume("cloud", n)
        ml = 3 * int(np.log2(n))
        t = time.time()
        g, _ = O.build(O.ref_oracle(), vol, O.build_cfg(2.0, ml, False, 1.0, 16.0))
        s = time.time() - t
        leaves = int(g.pools().leaf_mask.sum())
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024
        row(config=f"C4 CPU build (cloud {n}^3, no camera, thr 2.0, max_level {ml})", build="shipped",
            threads=1, seconds=s, leaves=leaves, leaves_per_s=leaves / s, peak_rss_bytes=rss,
            rss_bytes_per_leaf=rss / leaves)
        del g


if __name__ == "__main__":
    mode, rest = sys.argv[1], sys.argv[2:]
    if mode == "render":
        render_rows(rest or ["c1", "c2", "c3", "c5"])
    else:
        build_rows([int(x) for x in rest] or [256, 512])
