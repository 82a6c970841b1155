#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none -k regex:start_kernel -c 1 -o gpurun_out/prof_start python tools/prof_render.py 32 > gpurun_out/g17_ncu.log 2>&1
