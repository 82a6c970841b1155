"""Dev tool: per-rank frame time of the C2 frame for n_ranks = 1, 2, 4, 8 on one
GPU (rank 0's interleaved tiles), i.e. the render side of the scaling run
without the NCCL gather; prints ms and the implied strong-scaling efficiency."""
import sys

sys.path.insert(0, ".")
import torch

import paper_2506_11510_b200 as tv

n = 256
vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", n, vol.data_ptr())
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024)
grid, _ = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(0.15, 24, True, 1.0, 16.0), cam)
rc = tv.RenderConfig(spp=32, max_bounces=64, seed=0)
s = torch.zeros(1024 * 1024 * 3, dtype=torch.float64, device="cuda")
q = torch.zeros_like(s)
c = torch.zeros(1024 * 1024, dtype=torch.int32, device="cuda")
st = torch.zeros(3, dtype=torch.int64, device="cuda")
base = None
for nr in (1, 2, 4, 8):
    times = []
    for r in ([0, nr - 1] if nr > 1 else [0]):
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tv.render_tiles(grid, cam, rc, r, nr, s.data_ptr(), q.data_ptr(), c.data_ptr(), st.data_ptr(), 0)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
    ms = max(times)
    base = base or ms
    print(f"n_ranks {nr}: max rank frame {ms:.2f} ms, efficiency {base / (nr * ms):.3f}", flush=True)
