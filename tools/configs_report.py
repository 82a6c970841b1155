"""Measure the BASELINE configs beyond the bench line (C2 threshold sweep, C3/C5
at 512^3, C4 build at 1024^3) on one B200; prints one JSON object per row.

    python tools/configs_report.py [rows...]   rows: c2 c3 c5 c4 (default: all)
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2506_11510_b200 as tv

CAM = dict(position=(0.5, 0.5, -1.2), forward=(0.0, 0.0, 1.0), up=(0.0, 1.0, 0.0), vfov_degrees=40.0, width=1024,
           height=1024)


def field(n):
    vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    tv.generate_volume_dev("cloud", n, vol.data_ptr())
    return vol


def build(vol, n, thr, ml, camera=True):
    """two builds: the first of a size grows the build scratch (VMM mappings,
    kept per device between builds), the second reuses it; returns the second
    grid, its stats, and the first build's device seconds"""
    cam = tv.PinholeCamera(**CAM) if camera else None
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(thr, ml, camera, 1.0, 16.0), cam)
    torch.cuda.synchronize()
    first = st.seconds
    g.close()
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(thr, ml, camera, 1.0, 16.0), cam)
    torch.cuda.synchronize()
    return g, st, first


def render(g, spp=32, frames=2):
    cam = tv.PinholeCamera(**CAM)
    rc = tv.RenderConfig(spp=spp, max_bounces=64, seed=0)
    best = None
    for _ in range(frames):
        img = tv.render(g, cam, rc)
        if best is None or img.seconds < best.seconds:
            best = img
    return best


def row(**kw):
    print(json.dumps(kw), flush=True)


def c2():
    vol = field(256)
    for thr in [0.15, 1.0, 2.0, 4.0]:
        g, st, first = build(vol, 256, thr, 24)
        img = render(g)
        i = g.info()
        row(config="C2", field="cloud 256^3 + camera", threshold=thr, max_level=24, leaves=i["n_leaves"],
            tets=i["n_tets"], build_s=st.seconds, build_s_first=first, rounds=st.rounds, ms_per_frame=img.seconds * 1e3,
            samples_per_s=img.paths_traced / img.seconds, cells_per_path=img.cells_visited / img.paths_traced,
            tet_steps_per_s=img.cells_visited / img.seconds)
        g.close()


def c3_c5():
    vol = field(512)
    res = {}
    for thr in [0.15, 2.0, 4.0]:  # 4.0: the paper-like operating point (a few M leaves from 512^3)
        g, st, first = build(vol, 512, thr, 27)
        img = render(g)
        i = g.info()
        res[thr] = img
        row(config="C3 (1 GPU, 32 spp)", field="cloud 512^3 + camera", threshold=thr, max_level=27,
            leaves=i["n_leaves"], tets=i["n_tets"], build_s=st.seconds, build_s_first=first, ms_per_frame_32spp=img.seconds * 1e3,
            ms_per_frame_1024spp_extrapolated=img.seconds * 1e3 * 32, cells_per_path=img.cells_visited / img.paths_traced,
            tet_steps_per_s=img.cells_visited / img.seconds)
        g.close()
    cam = tv.PinholeCamera(**CAM)
    rc = tv.RenderConfig(spp=32, max_bounces=64, seed=0)
    reg = tv.render_reference_dev(vol.data_ptr(), (512, 512, 512), 16.0, cam, rc)
    for thr, img in res.items():
        row(config="C5", field="cloud 512^3", regular_ms=reg.seconds * 1e3,
            regular_cells_per_path=reg.cells_visited / reg.paths_traced, tet_threshold=thr,
            tet_ms=img.seconds * 1e3, tet_cells_per_path=img.cells_visited / img.paths_traced,
            speedup_tet_vs_regular=reg.seconds / img.seconds)


def c4():
    vol = field(1024)
    for thr in [2.0, 1.75, 1.5]:  # leaves ~50M +- 10 %
        g, st, first = build(vol, 1024, thr, 30, camera=False)
        i = g.info()
        row(config="C4", field="cloud 1024^3 (no camera)", threshold=thr, max_level=30, leaves=i["n_leaves"],
            tets=i["n_tets"], build_s_device=st.seconds, build_s_device_first=first, rounds=st.rounds,
            closure_passes=st.closure_passes, leaves_per_s=i["n_leaves"] / st.seconds,
            voxel_visits=st.voxel_visits, voxel_visits_per_s=st.voxel_visits / st.seconds, max_depth=st.max_depth)
        g.close()



def warmup():
    """one small build + render first, so no row pays the process's first-use costs"""
    vol = field(64)
    g, _, _ = build(vol, 64, 0.15, 18)
    render(g, spp=1, frames=1)
    g.close()




def c3_shares():
    """C3 as the BASELINE names it (1024 spp, sharded over 2/4/8 GPUs): the
    slowest rank's share of the frame, rendered on this one GPU (rank 0 and
    rank N-1), at the BASELINE threshold 0.15 and the paper-like 4.0."""
    vol = field(512)
    cam = tv.PinholeCamera(**CAM)
    rc = tv.RenderConfig(spp=1024, max_bounces=64, seed=0)
    s = torch.zeros(1024 * 1024 * 3, dtype=torch.float64, device="cuda")
    q = torch.zeros_like(s)
    c = torch.zeros(1024 * 1024, dtype=torch.int32, device="cuda")
    st = torch.zeros(3, dtype=torch.int64, device="cuda")
    for thr in [0.15, 4.0]:
        g, _, _ = build(vol, 512, thr, 27)
        for nr in (8, 4, 2):
            worst = 0.0
            cells = 0
            for r in ([0, nr - 1]):
                st.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                tv.render_tiles(g, cam, rc, r, nr, s.data_ptr(), q.data_ptr(), c.data_ptr(), st.data_ptr(), 0)
                e1.record()
                torch.cuda.synchronize()
                worst = max(worst, e0.elapsed_time(e1))
                cells = max(cells, int(st[0]))
            row(config=f"C3 share (1024 spp, {nr} ranks)", field="cloud 512^3 + camera", threshold=thr,
                leaves=g.info()["n_leaves"], slowest_rank_ms=worst,
                frame_ms_at_n_gpus_render_only=worst, samples_per_s_whole_job=1024 * 1024 * 1024 / (worst * 1e-3),
                rank_tet_steps=cells)
        g.close()


if __name__ == "__main__":
    rows = sys.argv[1:] or ["c2", "c3", "c4"]  # also: c3shares
    warmup()
    if "c2" in rows:
        c2()
    if "c3" in rows or "c5" in rows:
        c3_c5()
    if "c4" in rows:
        c4()
    if "c3shares" in rows:
        c3_shares()
