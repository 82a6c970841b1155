"""Dev tool: key metrics and stall shares of an ncu report (`--set full`).

    python tools/ncu_key.py report.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__sass_average_branch_targets_threads_uniform.pct"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {a: (c, b) for a, b, c in zip(h, u, v)}
    for k in KEYS:
        if k in d:
            print(f"{k},{d[k][0]},{d[k][1]}")
    st = [x for x in h if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")]
    tot = sum(float(d[x][0].replace(",", "") or 0) for x in st) or 1.0
    for x in sorted(st, key=lambda x: -float(d[x][0].replace(",", "") or 0))[:8]:
        print(f"stall_{x.replace('smsp__pcsamp_warps_issue_stalled_', '')},{float(d[x][0].replace(',', '')) / tot:.3f},share")


if __name__ == "__main__":
    main(sys.argv[1])
