#!/bin/bash
# Dev tool: one ncu --set full capture of trace_kernel (C2 grid, 4 spp) after a
# clean run of the same command; the report lands in gpurun_out/prof_trace.ncu-rep.
python tools/prof_render.py 4 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -c 1 -f -o gpurun_out/prof_trace \
    python tools/prof_render.py 4 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
