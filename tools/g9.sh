#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python tools/diag_sweep.py > gpurun_out/g9_diag_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/prof_replay python tools/diag_ceiling.py > gpurun_out/g9_ncu_replay.log 2>&1
