"""Dev tool for ncu: build the C2 grid, then render one frame at a reduced spp."""
import sys
sys.path.insert(0, ".")
import paper_2506_11510_b200 as tv
import torch

spp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", n, vol.data_ptr())
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(0.15, 24, True, 1.0, 16.0), cam)
img = tv.render(g, cam, tv.RenderConfig(spp=spp, max_bounces=64, seed=0))
print(st.leaf_count, img.cells_visited, img.seconds * 1e3, "ms")
