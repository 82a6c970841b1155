"""Dev tool: per-round times of the brick / voxel-sweep kernels in an ncu launch list."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = {}
for r in rows[1:]:
    x = float(r[vi].replace(",", ""))
    x = x / 1e6 if r[ui].startswith("n") else (x / 1e3 if r[ui].startswith("u") else x)
    for k in ["brick_voxels", "brick_descend", "brick_init", "vox_stats", "hanging"]:
        if k in r[ki]:
            d.setdefault(k, []).append(round(x, 2))
for k, l in d.items():
    print(k, round(sum(l), 1), l if k in ("brick_voxels", "vox_stats") else "")
