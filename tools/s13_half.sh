#!/bin/bash
# Dev tool: latency-ceiling replay with 64-B records vs a hypothetical 32-B record (one 256-bit load per step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TV_DIAG_HALF=1 timeout 600 python tools/diag_ceiling.py > gpurun_out/s13_half.log 2>&1
timeout 600 python tools/diag_ceiling.py > gpurun_out/s13_base.log 2>&1
