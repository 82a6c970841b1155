"""Helper for tests/test_gpu_variants.py (run as a subprocess so that the
TV_* environment knobs are read by a fresh library workspace): renders the C1
grid with multiple bounces, HG scattering, emission and albedo, and prints
the FNV-1a hash of the framebuffer's sum bits and the cell count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_2506_11510_b200 as tv

vol = O.gen_volume("blob", 64)
g, _ = O.build(O.c_oracle(), vol, O.build_cfg(0.15, 12, False, 1.0, 8.0))
p = g.pools()
rng = np.random.default_rng(11)
leaf = p.leaf_mask
p.tets["temperature"][leaf] = (rng.random(leaf.sum()) * 1.2).astype(np.float32)
p.tets["albedo"][leaf] = rng.random(leaf.sum()).astype(np.float32)
p.tets["mask"][leaf] = 7
dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
cam = tv.PinholeCamera((0.5, 0.5, -2), (0, 0, 1), (0, 1, 0), 40, 160, 120)
rc = tv.RenderConfig(spp=16, max_bounces=64, seed=3, hg_g=0.4)
img = tv.render(dg, cam, rc)
img2 = tv.render(dg, cam, rc)  # a second frame: schedules that adapt between frames (TV_TILE_ORDER=4)
assert O.fnv64(img2.sum) == O.fnv64(img.sum) and img2.cells_visited == img.cells_visited
print(f"{O.fnv64(img.sum):016x} {O.fnv64(img.sum_sq):016x} {img.cells_visited}")
