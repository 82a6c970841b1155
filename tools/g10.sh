#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python tools/diag_sweep.py > gpurun_out/g10_diag_sweep.log 2>&1
