"""Dev tool: the north-star frame (1024^2 x 32 spp, max_bounces 64) on GPU-built
grids of the procedural cloud at several (variation threshold, pixel threshold)
operating points: leaves, steps per path and device ms per frame (one JSON row each)."""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2506_11510_b200 as tv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ml = 3 * (n.bit_length() - 1)
points = [tuple(float(x) for x in p.split(":")) for p in (sys.argv[2:] or ["4:1", "4:2", "2:2", "2:4", "8:1", "1:4"])]
vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", n, vol.data_ptr())
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
rc = tv.RenderConfig(spp=32, max_bounces=64, seed=0)
for thr, pix in points:
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(thr, ml, True, pix, 16.0), cam)
    best = None
    for _ in range(4):
        img = tv.render(g, cam, rc)
        best = img if best is None or img.seconds < best.seconds else best
    print(json.dumps({"grid": f"cloud {n}^3", "threshold": thr, "pixel_threshold": pix, "max_level": ml,
                      "leaves": st.leaf_count, "ms_per_frame": best.seconds * 1e3,
                      "steps_per_path": best.cells_visited / best.paths_traced,
                      "g_steps_per_s": best.cells_visited / best.seconds / 1e9,
                      "samples_per_s": best.paths_traced / best.seconds}), flush=True)
    del g
