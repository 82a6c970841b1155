"""Benchmark: BASELINE.json metric on config C2.

Workload (one "step" = one frame): procedural cloud 256^3 -> LEB tet grid built
on the GPU with the camera criterion (threshold 0.15, max_level 24,
density_scale 16, pixel_threshold 1) -> 1024x1024 render at 32 spp,
max_bounces 64, camera (0.5, 0.5, -1.2) looking +z, vfov 40. The grid (12.1M
leaves, 3.3 GB in HBM) is resident before timing; it is larger than L2, which
is how this benchmark satisfies the L2 rule (no flush between steps).

With --gpus N (torchrun, one rank per GPU) every rank holds a replica of the
grid and renders the interleaved 16x16 tiles t with t % N == rank of the SAME
frame (strong scaling). Frame assembly is inside the timed step: by default
(--gather-mode p2p) every rank's accumulate kernel stores its pixels straight
into rank 0's frame buffers over NVLink (CUDA IPC mappings) and a one-word
NCCL all-reduce on the render stream is the completion barrier; with
--gather-mode nccl (also the automatic fallback when peer mappings fail) the
tiles are packed, all-gathered over NCCL and unpacked on every rank.

--impl reference times the reference's own CPU renderer (oracle/_ref, compiled
from /root/reference) on this box's host cores on a bounded sample of the same
workload (the first CPU_SPP samples of every pixel of the same frame).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_IMG = H_IMG = 1024
SPP = 32
GRID_N = 256
BUILD = dict(variation_threshold=0.15, max_level=24, use_camera=True, pixel_threshold=1.0, density_scale=16.0)
CAM = dict(position=(0.5, 0.5, -1.2), forward=(0.0, 0.0, 1.0), up=(0.0, 1.0, 0.0), vfov_degrees=40.0, width=W_IMG,
           height=H_IMG)
# algorithmic bytes per tet step. The shipped layout reads
# exactly one 64-B LeafRec per step (two 256-bit loads), the same figure.
BYTES_PER_STEP = 64
WORKLOAD = ("C2: procedural cloud 256^3 -> GPU LEB grid (camera criterion, threshold 0.15, max_level 24, "
            "density_scale 16, pixel_threshold 1) -> 1024x1024 x 32 spp, max_bounces 64")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.window = None  # (t0, t1) host monotonic bounds of the timed region

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # started ahead of the timed region; wait until it is sampling
            t_end = time.monotonic() + 5.0
            while not self.rows and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts + [time.monotonic()])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        if self.window is not None:  # only the samples taken inside the timed region
            rows = [r for r in rows if self.window[0] <= r[7] <= self.window[1]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


CPU_SPP = 8  # cpu_baseline sample: ~10 s of host work on 16 cores
REF_SPP = 4  # --impl reference: samples per pixel per timed step


def cpu_render_sample(v, t, r, max_level, threads=0, padded=False):
    """The reference renderer (oracle/_ref) on the same grid and frame, spp = CPU_SPP.
    padded=True uses oracle/_ref/pad (alignas(64) TraceStats); None if absent."""
    import oracle as O

    if padded:
        chk, kind = O.ref_pad_oracle(), "reference"
        if chk is None:
            return None, kind, 0
    else:
        chk = O.ref_oracle()
        kind = "reference"
    if chk is None:
        chk, kind = O.c_oracle(), "port"
    g = O.from_pools(chk, O.Pools(v, t.view(O.TET_DTYPE), r, max_level))
    cam = O.camera(CAM["position"], CAM["forward"], CAM["up"], CAM["vfov_degrees"], W_IMG, H_IMG)
    rc = O.render_cfg(spp=CPU_SPP, max_bounces=64, seed=0)
    out = g.render(cam, rc, threads)
    cores = threads if threads > 0 else os.cpu_count()
    return out, kind, cores


def run_reference(args, rank, world):
    """--impl reference: the reference CPU renderer on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import paper_2506_11510_b200 as tv  # grid construction only (reference arm)
    import torch

    torch.cuda.set_device(0)
    vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device="cuda")
    tv.generate_volume_dev("cloud", GRID_N, vol.data_ptr())
    grid, bst = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD),
                                           tv.PinholeCamera(**CAM))
    v, t, r = grid.download()
    grid.close()
    del vol
    import oracle as O

    chk = O.ref_oracle()
    kind = "reference" if chk is not None else "port"
    chk = chk or O.c_oracle()
    t0 = time.time()
    g = O.from_pools(chk, O.Pools(v, t.view(O.TET_DTYPE), r, BUILD["max_level"]))
    assemble_s = time.time() - t0
    cam = O.camera(CAM["position"], CAM["forward"], CAM["up"], CAM["vfov_degrees"], W_IMG, H_IMG)
    rc = O.render_cfg(spp=REF_SPP, max_bounces=64, seed=0)
    for _ in range(args.warmup):
        g.render(cam, rc, 0)
    secs, cells = [], 0
    for _ in range(args.steps):
        out = g.render(cam, rc, 0)
        secs.append(out["seconds"])
        cells = out["cells_visited"]
    per = float(np.mean(secs))
    samples = W_IMG * H_IMG * REF_SPP
    value = samples / per
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": "samples/s", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"spp={REF_SPP} of the same frame (first samples of every pixel)",
                   "leaves": int((t["children"][:, 0] == 0xFFFFFFFF).sum())},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                         "sample": f"1024x1024 x {REF_SPP} spp of the C2 frame, all host threads (render(..., threads=0))"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tet_steps_per_s": cells / per, "cells_per_path": cells / samples,
        "grid_assemble_s": assemble_s, "cpu_model": _cpu_model(),
    }
    print(json.dumps(line), flush=True)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", action="store_true", help="use the multi-GPU tile gather path even on one rank")
    ap.add_argument("--gather-mode", default="p2p", choices=["nccl", "p2p"],
                    help="multi-GPU frame assembly: NCCL all-gather of packed tiles, or direct peer writes of every "
                         "rank's pixels into rank 0's accumulators (CUDA IPC) with a one-word all-reduce barrier")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2506_11510_b200 as tv
    from paper_2506_11510_b200 import sharding

    torch.cuda.set_device(local)
    multi = world > 1 or args.gather  # --gather exercises the NCCL tile path even on one rank
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local

    # ---- grid: generated and built in HBM (not timed) ----
    vol = torch.empty(GRID_N ** 3, dtype=torch.float32, device="cuda")
    tv.generate_volume_dev("cloud", GRID_N, vol.data_ptr(), device=dev)
    cam = tv.PinholeCamera(**CAM)
    grid, bst = tv.build_adaptive_grid_dev(vol.data_ptr(), (GRID_N,) * 3, tv.BuildConfig(**BUILD), cam, device=dev)
    del vol
    info = grid.info()
    rc = tv.RenderConfig(spp=SPP, max_bounces=64, seed=0)

    npx = W_IMG * H_IMG
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    sum_ = torch.zeros(npx * 3, dtype=torch.float64, device="cuda")
    sum_sq = torch.zeros(npx * 3, dtype=torch.float64, device="cuda")
    counts = torch.zeros(npx, dtype=torch.int32, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    words = tv.tile_pack_words(W_IMG, H_IMG, rank, world, 3)
    packed = torch.zeros(words, dtype=torch.float64, device="cuda")
    gathered = torch.zeros(words * world, dtype=torch.float64, device="cuda")
    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    p2p = multi and args.gather_mode == "p2p"
    out_ptrs = (sum_.data_ptr(), sum_sq.data_ptr(), counts.data_ptr())
    gather_note = None
    if p2p:  # every rank's accumulate kernel writes into rank 0's frame over NVLink
        try:
            peer = sharding.PeerFrame(W_IMG, H_IMG, rank, dev)
            ok = torch.ones(1, device="cuda")
        except Exception as e:  # e.g. no peer access between these GPUs: the NCCL gather instead
            peer, ok, gather_note = None, torch.zeros(1, device="cuda"), f"p2p unavailable ({e!r}); NCCL all-gather"
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if float(ok[0]) == 0.0:
            if peer is not None:
                peer.close()
            p2p, args.gather_mode = False, "nccl"
            gather_note = gather_note or "p2p unavailable on some rank; NCCL all-gather"
        else:
            out_ptrs = peer.ptrs
            if rank == 0:
                sum_ = peer.local[0]
            fence = torch.zeros(1, dtype=torch.float32, device="cuda")

    def step(i, timed=False):
        if timed:
            k_start[i].record(stream)
        tv.render_tiles(grid, cam, rc, rank, world, out_ptrs[0], out_ptrs[1], out_ptrs[2], stats.data_ptr(), sh)
        if timed:
            k_end[i].record(stream)
        if p2p:
            with torch.cuda.stream(stream):  # completion barrier: every rank's pixels have landed
                dist.all_reduce(fence)
        elif multi:
            tv.tile_pack(sum_.data_ptr(), packed.data_ptr(), W_IMG, H_IMG, rank, world, 3, sh)
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(gathered, packed)
            for r in range(world):
                tv.tile_unpack(gathered[r * words:(r + 1) * words].data_ptr(), sum_.data_ptr(), W_IMG, H_IMG, r,
                               world, 3, sh)

    clk = ClockSampler(dev).__enter__()  # sampling (every 100 ms) from before the warm-up
    for i in range(args.warmup):
        step(i)
    stream.synchronize()
    stats.zero_()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    h0 = time.monotonic()
    t0.record(stream)
    for i in range(args.steps):
        step(i, timed=True)
    t1.record(stream)
    stream.synchronize()
    clk.window = (h0, time.monotonic())
    time.sleep(0.15)  # let the sample covering the region's end arrive
    clk.__exit__(None, None, None)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    kern_ms = float(np.mean([k_start[i].elapsed_time(k_end[i]) for i in range(args.steps)]))
    # per-kernel device time of the last timed frame (CUDA events recorded by the
    # library on `stream` around start / trace / accumulate)
    timing = tv.last_frame_timing(dev)
    trace_ms = timing["trace_ms"]
    st = stats.cpu().numpy()
    cells_rank = int(st[0]) // args.steps
    if multi:
        red = torch.tensor([ms, kern_ms, float(cells_rank)], dtype=torch.float64, device="cuda")
        mx = red.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = red.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, kern_ms_max = float(mx[0]), float(mx[1])
        cells_frame = int(tot[2])
    else:
        kern_ms_max = kern_ms
        cells_frame = cells_rank
    samples = npx * SPP
    value = samples / (ms * 1e-3)

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not multi:
        hs = torch.empty(npx * 3, dtype=torch.float64, pin_memory=True).numpy()
        hq = torch.empty(npx * 3, dtype=torch.float64, pin_memory=True).numpy()
        hc = torch.empty(npx, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        tv.render_into(grid, cam, rc, hs, hq, hc)
        t_e = time.perf_counter()
        for _ in range(args.steps):
            tv.render_into(grid, cam, rc, hs, hq, hc)
        e2e_s = (time.perf_counter() - t_e) / args.steps
        e2e = {"value": samples / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": 96 + 88,
               "d2h_bytes_per_step": npx * (24 + 24 + 4) + 24, "ms_per_step": e2e_s * 1e3,
               "path": "tv_render (C ABI): kernel params H2D, sum/sum_sq/sample_counts D2H into pinned host memory"}
    else:
        host = torch.empty(npx * 3, dtype=torch.float64, pin_memory=True)
        for i in range(2):
            step(0)
        stream.synchronize()
        dist.barrier()
        t_e = time.perf_counter()
        for i in range(args.steps):
            step(0)
            if rank == 0:
                with torch.cuda.stream(stream):
                    host.copy_(sum_, non_blocking=True)
            stream.synchronize()
        e2e_s = (time.perf_counter() - t_e) / args.steps
        e2 = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(e2, op=dist.ReduceOp.MAX)
        e2e_s = float(e2[0])
        e2e = {"value": samples / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": 96 + 88,
               "d2h_bytes_per_step": npx * 24, "ms_per_step": e2e_s * 1e3,
               "path": ("tv_render_tiles writing rank 0's frame over NVLink (P2P) + one-word all-reduce barrier"
                        if p2p else "tv_render_tiles + NCCL all-gather of packed tiles") +
                       " + D2H of the frame sums on rank 0"}

    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    achieved = cells_rank * BYTES_PER_STEP / (trace_ms * 1e-3) / 1e9
    traffic, dram, l2 = None, None, None
    prof = os.path.join(ROOT, "profiles", "trace_kernel_dram.json")
    kern_s = trace_ms * 1e-3
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            # ncu DRAM / L2 bytes per tet step at the bench config (one --set full
            # capture, profiles/), scaled to this rank's launch
            traffic = pj["dram_bytes_per_step"] * cells_rank
            dram = {"bytes_per_step": pj["dram_bytes_per_step"], "achieved": traffic / kern_s / 1e9,
                    "frac": traffic / kern_s / 1e9 / hbm, "source": f"ncu, {pj.get('round', '?')}"}
            if pj.get("l2_bytes_per_step"):
                l2b = pj["l2_bytes_per_step"] * cells_rank
                l2 = {"bytes_per_step": pj["l2_bytes_per_step"], "achieved": l2b / kern_s / 1e9,
                      "hit_pct": pj.get("l2_hit_pct"), "source": f"ncu lts__t_bytes, {pj.get('round', '?')}"}
        except Exception:
            traffic = None
    # the measured latency ceiling of this frame (tools/diag_ceiling.py: the
    # frame's recorded tet-step stream replayed as dependent record loads with
    # the trace kernel's launch shape and schedule, no geometry)
    ceiling = None
    cprof = os.path.join(ROOT, "profiles", "trace_kernel_ceiling.json")
    if os.path.exists(cprof):
        try:
            cj = json.load(open(cprof))
            if world == 1 and int(cj["steps"]) == cells_rank:  # the same frame
                steps_s = cells_rank / (trace_ms * 1e-3)
                ceiling = {"steps_per_s": cj["steps_per_s"], "replay_ms": cj["replay_ms"],
                           "frac": steps_s / cj["steps_per_s"], "warps_per_sm": cj["warps_per_sm"],
                           "source": "tools/diag_ceiling.py (profiles/trace_kernel_ceiling.json)"}
        except Exception:
            ceiling = None
    # `achieved` / `frac` follow the contract: ALGORITHMIC bytes (64 per tet
    # step) over the kernel's time, against the HBM copy peak.
    # Most of those bytes are served by L2 (rays of one pixel and neighbouring
    # pixels reuse records), so frac near or above 1 is request throughput, not
    # a DRAM bound: `dram` is what HBM actually moved. The kernel is bound by
    # the latency of its one dependent record load per step (the measured
    # ceiling) and by instruction issue.
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": "trace_kernel", "kernel_ms": trace_ms,
                "frame_kernels_ms": {"start": timing["start_ms"], "trace": trace_ms, "accumulate": timing["accum_ms"]},
                "bytes_per_step": BYTES_PER_STEP, "tet_steps_per_launch": cells_rank,
                "algorithmic_bytes_per_launch": cells_rank * BYTES_PER_STEP,
                "achieved_is": "algorithmic request bytes (served mostly from L2), not DRAM traffic",
                "dram": dram, "l2": l2, "latency_ceiling": ceiling,
                "limiter": ("dependent record-load stream (latency ceiling, DESIGN.md 4)"
                            if ceiling and ceiling["frac"] > 0.95 else
                            "instruction issue under the dependent record-load latency (DESIGN.md 4)"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback 6650 GB/s"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, t, r = grid.download()
            out, kind, cores = cpu_render_sample(v, t, r, BUILD["max_level"])
            cpu = {"value": npx * CPU_SPP / out["seconds"], "unit": "samples/s", "cores": cores, "kind": kind,
                   "sample": f"1024x1024 x {CPU_SPP} spp of the same C2 frame (first samples per pixel), threads=all",
                   "seconds": out["seconds"], "tet_steps_per_s": out["cells_visited"] / out["seconds"]}
            # the shipped build false-shares its per-thread counters;
            # the same sources with alignas(64) TraceStats are the fair CPU figure.
            po, _, _ = cpu_render_sample(v, t, r, BUILD["max_level"], padded=True)
            if po is not None:
                cpu["padded"] = {
                    "value": npx * CPU_SPP / po["seconds"], "unit": "samples/s", "cores": cores,
                    "seconds": po["seconds"], "tet_steps_per_s": po["cells_visited"] / po["seconds"],
                    "build": "oracle/_ref/pad: reference sources with struct alignas(64) TraceStats"}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "failed", "error": repr(e)}

    if rank == 0:
        line = {
            "metric": "samples/s", "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (procedural cloud field, GPU-built LEB grid)",
            "config": {"workload": WORKLOAD, "leaves": info["n_leaves"], "tets": info["n_tets"],
                       "grid_bytes": info["device_bytes"], "max_depth": info["max_depth"],
                       "l2": "inputs larger than L2 (3.3 GB grid), no flush", "parallelism": f"image tiles x{world}",
                       "build_s_device": bst.seconds},
            "tet_steps_per_s": cells_frame / (ms * 1e-3), "cells_per_path": cells_frame / samples,
            "ms_per_frame": ms, "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": (timing["launches"] + (0 if p2p else (1 + world if multi else 0))) * args.steps,
            "gather_mode": args.gather_mode if multi else None, "gather_note": gather_note,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        if p2p:
            peer.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
