"""The latency-ceiling diagnostic (include/tetvol_b200_diag.h): its recording
pass must reproduce the render's tet-step count exactly (same path order, RNG
streams and integrator), and both replays must run."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_gather_ceiling_records_the_render_step_stream():
    import paper_2506_11510_b200 as tv

    vol = O.gen_volume("cloud", 48)
    cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 96, 64)
    grid, _ = tv.build_adaptive_grid(vol, tv.BuildConfig(0.3, 14, True, 1.0, 16.0), cam)
    rc = tv.RenderConfig(spp=4, max_bounces=16, seed=3)
    img = tv.render(grid, cam, rc)
    d = tv.diag_gather_ceiling(grid, cam, rc, reps=1)
    assert d["steps"] == img.cells_visited
    assert d["steps_per_s"] > 0 and d["steps_per_s_full_occupancy"] > 0
    assert d["warps_per_sm"] >= 4
    assert np.isfinite(d["replay_ms"]) and d["replay_ms"] > 0
