"""Dev tool: the trace kernel's memory-latency ceiling on the bench frame (C2),
next to the render itself (include/tetvol_b200_diag.h)."""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2506_11510_b200 as tv
from bench import BUILD, CAM, GRID_N, SPP

vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", GRID_N, vol.data_ptr())
cam = tv.PinholeCamera(**CAM)
grid, _ = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD), cam)
del vol
rc = tv.RenderConfig(spp=SPP, max_bounces=64, seed=0)
img = None
for _ in range(3):
    img = tv.render(grid, cam, rc)
t = tv.last_frame_timing(0)
d = tv.diag_gather_ceiling(grid, cam, rc, reps=3)
out = {"render_ms": img.seconds * 1e3, "trace_ms": t["trace_ms"], "cells_visited": img.cells_visited,
       "trace_steps_per_s": img.cells_visited / (t["trace_ms"] * 1e-3), **d}
out["frac_of_ceiling"] = out["trace_steps_per_s"] / d["steps_per_s"]
out["workload"] = "bench.py C2 frame"
print(json.dumps(out), flush=True)
if len(sys.argv) > 1:  # e.g. profiles/trace_kernel_ceiling.json (bench.py reports it in roofline.latency_ceiling)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
assert d["steps"] == img.cells_visited, "recorded steps differ from the render's cells_visited"
