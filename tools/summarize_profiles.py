"""Dev tool: turn the gpurun_out/ ncu outputs of tools/profile_round.sh into the
committed summaries under profiles/ (rNN prefix = build round)."""
import collections
import csv
import json
import subprocess
import sys

RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = "gpurun_out/"


def launches():
    rows = list(csv.reader(open(G + "launches.csv")))
    hdr = None
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr and len(r) > 5 and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
            k = r[hdr["Kernel Name"]].replace("<unnamed>::", "").split("(")[0].replace("void ", "")
            k = k.split("<")[0].split("::")[-1]
            agg[k] += float(r[hdr["Metric Value"]].replace(",", "")) / 1e6
            cnt[k] += 1
    render = ["start_kernel", "trace_kernel_t", "accum_kernel"]
    frame = sum(agg[k] for k in render)
    out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none) of tools/prof_render.py 32:",
           "# the C2 GPU LEB build, then one 1024x1024 x 32 spp frame; cold-cache and serialised,",
           f"# so compare shares, not absolutes. Frame kernels total {frame:.2f} ms.",
           "kernel,launches,total_ms,share"]
    for k in render:
        out.append(f"{k},{cnt[k]},{agg[k]:.3f},{agg[k] / frame:.4f} of frame")
    build = [k for k in agg if k not in render]
    out.append(f"# build kernels: {sum(agg[k] for k in build):.2f} ms over {sum(cnt[k] for k in build)} launches")
    for k in sorted(build, key=lambda k: -agg[k])[:14]:
        out.append(f"{k},{cnt[k]},{agg[k]:.3f},build")
    open(f"profiles/{RND}_launches_c2.csv", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def dram(steps):
    rows = [r for r in csv.reader(open(G + "trace_dram.csv")) if r]
    h0 = next(i for i, r in enumerate(rows) if r[0] == "ID")
    hdr = {h: i for i, h in enumerate(rows[h0])}
    m = {r[hdr["Metric Name"]]: float(r[hdr["Metric Value"]].replace(",", "")) for r in rows[h0 + 1:] if len(r) > 5}
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    out = {"kernel": "trace_kernel_t<72, 1, 128>", "config": "C2 1024x1024 x 32 spp (bench.py workload)",
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "tet_steps_per_launch": steps, "dram_bytes_per_step": (rd + wr) / steps,
           "l2_bytes_per_step": m["lts__t_sectors.sum"] * 32 / steps,
           "l1_global_bytes_per_step": m["l1tex__t_sectors.sum"] * 32 / steps,
           "l1_hit_pct": m["l1tex__t_sector_hit_rate.pct"], "l2_hit_pct": m["lts__t_sector_hit_rate.pct"],
           "duration_ms_under_ncu": m["gpu__time_duration.sum"] / 1e6, "round": RND}
    json.dump(out, open("profiles/trace_kernel_dram.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


def full():
    raw = subprocess.run(["ncu", "-i", G + "prof_trace.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    d = {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__t_sector_hit_rate.pct",
            "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__sass_average_branch_targets_threads_uniform.pct"]
    out = [f"# ncu --set full of trace_kernel (tools/prof_render.py 4: C2 grid, 1024^2 x 4 spp), {RND}",
           "metric,value,unit"]
    for k in keys:
        if k in d:
            out.append(f"{k},{d[k][0]},{d[k][1]}")
    st = [h for h in rows[0] if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(float(d[h][0].replace(",", "") or 0) for h in st)
    out.append("# warp stall sampling shares")
    for h in sorted(st, key=lambda h: -float(d[h][0].replace(",", "") or 0))[:10]:
        v = float(d[h][0].replace(",", "") or 0)
        out.append(f"stall_{h.replace('smsp__pcsamp_warps_issue_stalled_', '')},{v / tot:.4f},share")
    open(f"profiles/{RND}_trace_kernel_ncu_full.csv", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    launches()
    dram(int(sys.argv[2]) if len(sys.argv) > 2 else 6601802105)
    full()
