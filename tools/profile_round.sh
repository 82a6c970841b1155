#!/bin/bash
# GPU session for the profiles/ evidence: plain bench line, the trace kernel's
# DRAM / L2 traffic at the bench config, the per-launch list of one frame, and
# one ncu --set full capture (4 spp) of the trace kernel.
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_p.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_p.log
python tools/prof_render.py 32 > gpurun_out/plain32.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors.sum,l1tex__t_sectors.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:trace_kernel -c 1 --csv --log-file gpurun_out/trace_dram.csv python tools/prof_render.py 32 > gpurun_out/ncu_dram.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_render.py 32 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_render.py 4 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -c 1 -o gpurun_out/prof_trace python tools/prof_render.py 4 > gpurun_out/ncu_full.log 2>&1
