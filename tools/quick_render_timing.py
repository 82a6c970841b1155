"""Dev tool: per-kernel frame timing (start / trace / accumulate) of the bench
frame, with and without the locate jump table (TV_JUMP_RES is read at grid
finalize, so each setting builds its grid in a fresh process)."""
import json
import os
import subprocess
import sys

CODE = ("import sys, json; sys.path.insert(0, '.'); import torch; import paper_2506_11510_b200 as tv;"
        "from bench import BUILD, CAM, GRID_N, SPP;"
        "vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device='cuda');"
        "tv.generate_volume_dev('cloud', GRID_N, vol.data_ptr()); cam = tv.PinholeCamera(**CAM);"
        "g, _ = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD), cam);"
        "rc = tv.RenderConfig(spp=SPP, max_bounces=64, seed=0)\n"
        "best = None\n"
        "for _ in range(4):\n"
        "    img = tv.render(g, cam, rc); t = tv.last_frame_timing(0)\n"
        "    if best is None or img.seconds < best[0]: best = (img.seconds, t)\n"
        "print(json.dumps({'frame_ms': best[0] * 1e3, **best[1]}))")
for res in sys.argv[1:] or ["0", "128"]:
    r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, TV_JUMP_RES=res), capture_output=True,
                       text=True, timeout=600)
    print(json.dumps({"TV_JUMP_RES": res, "result": (r.stdout.strip().splitlines() or [r.stderr[-400:]])[-1]}),
          flush=True)
