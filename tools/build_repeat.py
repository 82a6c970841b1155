"""Dev tool: repeat the GPU LEB build of one field and print each build's device / wall time."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2506_11510_b200 as tv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ml = int(sys.argv[3]) if len(sys.argv) > 3 else 24
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, 1024, 1024) if n <= 512 else None
vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
tv.generate_volume_dev("cloud", n, vol.data_ptr())
for r in range(reps):
    t = time.time()
    g, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(thr, ml, cam is not None, 1.0, 16.0), cam)
    torch.cuda.synchronize()
    print(f"rep {r}: device {st.seconds:.3f} s wall {time.time() - t:.3f} s leaves {st.leaf_count} rounds {st.rounds}",
          flush=True)
    g.close()
