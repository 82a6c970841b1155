"""Dev tool: the latency-ceiling replay (tv_diag_gather_ceiling) on the C2 frame
under what-if L1 / occupancy settings: TV_DIAG_SMEM (shared bytes per block),
TV_DIAG_CARVEOUT and TV_DIAG_BLOCKS (resident blocks per SM), one process per
setting. Arguments: smem_carveout_blocks triples (default: the built-in list)."""
import json
import os
import subprocess
import sys

CFGS = [(27136, 72, 7), (18432, 50, 6), (18432, 60, 7), (9216, 25, 6), (9216, 30, 7), (9216, 20, 5), (9216, 35, 8),
        (0, 0, 6), (0, 0, 5), (0, 0, 4), (0, 0, 8)]
if len(sys.argv) > 1:
    CFGS = [tuple(int(x) for x in c.split("_")) for c in sys.argv[1:]]
for smem, cv, blocks in CFGS:
    env = dict(os.environ, TV_DIAG_SMEM=str(smem), TV_DIAG_CARVEOUT=str(cv), TV_DIAG_BLOCKS=str(blocks))
    code = ("import sys, json; sys.path.insert(0, '.'); import torch; import paper_2506_11510_b200 as tv;"
            "from bench import BUILD, CAM, GRID_N, SPP;"
            "vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device='cuda');"
            "tv.generate_volume_dev('cloud', GRID_N, vol.data_ptr()); cam = tv.PinholeCamera(**CAM);"
            "g, _ = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD), cam);"
            "d = tv.diag_gather_ceiling(g, cam, tv.RenderConfig(spp=SPP, max_bounces=64, seed=0), 2);"
            "print(json.dumps(d))")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(json.dumps({"smem": smem, "carveout": cv, "blocks": blocks, "result": line}), flush=True)
