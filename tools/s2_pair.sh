#!/bin/bash
# Dev tool: latency-ceiling replay with per-lane vs lane-pair record loads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/diag_ceiling.py > gpurun_out/s2_base.log 2>&1
TV_DIAG_PAIR=1 timeout 600 python tools/diag_ceiling.py > gpurun_out/s2_pair.log 2>&1
VARIANTS="base pair" bash tools/variants.sh
