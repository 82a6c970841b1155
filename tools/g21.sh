#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none -k regex:vox_stats -s 22 -c 1 -o gpurun_out/prof_vox python tools/build_repeat.py 1024 2.0 30 1 > gpurun_out/g21_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:vox_stats -s 1 -c 1 -o gpurun_out/prof_vox1 python tools/build_repeat.py 1024 2.0 30 1 > gpurun_out/g21_ncu1.log 2>&1
