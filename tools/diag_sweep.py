"""Dev tool: the latency-ceiling replay (tv_diag_gather_ceiling) on the C2 frame
under what-if L1 / occupancy settings: TV_DIAG_SMEM (shared bytes per block) and
TV_DIAG_CARVEOUT, one process per setting (the carveout is per process)."""
import json
import os
import subprocess
import sys

CFGS = [(27136, 72), (27136, 100), (8704, 72), (8704, 40), (8704, 25), (16384, 60), (0, 0), (0, 25)]
for smem, cv in CFGS:
    env = dict(os.environ, TV_DIAG_SMEM=str(smem), TV_DIAG_CARVEOUT=str(cv))
    code = ("import sys, json; sys.path.insert(0, '.'); import torch; import paper_2506_11510_b200 as tv;"
            "from bench import BUILD, CAM, GRID_N, SPP;"
            "vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device='cuda');"
            "tv.generate_volume_dev('cloud', GRID_N, vol.data_ptr()); cam = tv.PinholeCamera(**CAM);"
            "g, _ = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD), cam);"
            "d = tv.diag_gather_ceiling(g, cam, tv.RenderConfig(spp=SPP, max_bounces=64, seed=0), 2);"
            "print(json.dumps(d))")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(json.dumps({"smem": smem, "carveout": cv, "result": line}), flush=True)
