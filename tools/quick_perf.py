"""Quick device timing of the render kernel on an oracle-built grid (dev tool)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle as O
import paper_2506_11510_b200 as tv

kind = sys.argv[1] if len(sys.argv) > 1 else "blob"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.15
ml = int(sys.argv[4]) if len(sys.argv) > 4 else 12
scale = float(sys.argv[5]) if len(sys.argv) > 5 else 8.0
res = int(sys.argv[6]) if len(sys.argv) > 6 else 1024
spp = int(sys.argv[7]) if len(sys.argv) > 7 else 32
mb = int(sys.argv[8]) if len(sys.argv) > 8 else 64
vol = O.gen_volume(kind, n)
t = time.time()
g, st = O.build(O.c_oracle(), vol, O.build_cfg(thr, ml, False, 1.0, scale))
print("oracle build", time.time() - t, st, flush=True)
p = g.pools()
dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
print(dg.info(), flush=True)
cam = tv.PinholeCamera((0.5, 0.5, -1.2), (0, 0, 1), (0, 1, 0), 40, res, res)
rc = tv.RenderConfig(spp=spp, max_bounces=mb, seed=0)
for i in range(4):
    t = time.time()
    img = tv.render(dg, cam, rc)
    wall = time.time() - t
    print(f"render {res}^2 x {spp} spp mb={mb}: dev {img.seconds*1e3:.2f} ms wall {wall*1e3:.1f} ms "
          f"cells {img.cells_visited} ({img.cells_visited/img.paths_traced:.2f}/path) "
          f"{img.cells_visited/img.seconds/1e9:.2f} G steps/s {img.paths_traced/img.seconds/1e6:.1f} M samples/s "
          f"deg {img.degenerate_paths}", flush=True)
