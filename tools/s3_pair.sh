#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TV_DIAG_PAIR=1 timeout 600 python tools/diag_ceiling.py > gpurun_out/s3_pair.log 2>&1
