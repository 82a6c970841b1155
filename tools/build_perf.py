"""Dev tool: GPU LEB build of a procedural cloud + camera criterion, then render timing."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2506_11510_b200 as tv
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
ml = int(sys.argv[3]) if len(sys.argv) > 3 else 21
spp = int(sys.argv[4]) if len(sys.argv) > 4 else 32
vol = torch.empty(n * n * n, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", n, vol.data_ptr())
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
bc = tv.BuildConfig(thr, ml, True, 1.0, 16.0)
for i in range(2):
    t = time.time()
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), bc, cam)
    torch.cuda.synchronize()
    print(f"build cloud{n} thr={thr}: wall {time.time()-t:.3f}s {st}", flush=True)
print(g.info(), flush=True)
rc = tv.RenderConfig(spp=spp, max_bounces=64, seed=0)
for i in range(3):
    img = tv.render(g, cam, rc)
    print(f"render 1024^2 x {spp}: dev {img.seconds*1e3:.2f} ms cells/path {img.cells_visited/img.paths_traced:.2f} "
          f"{img.cells_visited/img.seconds/1e9:.2f} G steps/s {img.paths_traced/img.seconds/1e6:.1f} M samples/s deg {img.degenerate_paths}", flush=True)
