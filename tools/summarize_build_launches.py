"""Dev tool: per-kernel totals of an ncu launch list (gpu__time_duration.sum) of
tools/build_repeat.py (one build), plus the per-round voxel-sweep times.

    python tools/summarize_build_launches.py launches.csv "title" > profiles/<name>.csv
"""
import collections
import csv
import re
import sys


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    sweeps = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui].startswith("n") else (v / 1e3 if r[ui].startswith("u") else v)
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"^void ", "", name)
        name = re.sub(r"tvb::<unnamed>::", "", name)
        name = re.sub(r"^cub::(\w+)<.*", r"\1", name)
        if name == "gen_kernel":  # the procedural field, not the build
            continue
        agg[name][0] += 1
        agg[name][1] += v
        if name.startswith("vox_stats_kernel"):
            sweeps.append(v)
    tot = sum(v for _, v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none) of {title};")
    print("# cold-cache and serialised: compare shares, not absolutes.")
    print(f"# build kernels total {tot:.1f} ms over {sum(c for c, _ in agg.values())} launches")
    print("kernel,launches,total_ms,share")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k},{c},{v:.3f},{v / tot:.4f}")
    print("# voxel sweep per round (ms): " + " ".join(f"{x:.2f}" for x in sweeps))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
