#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/diag_sweep.py 27136_72_7 > gpurun_out/g27_base.log 2>&1
TV_DIAG_TMA=1 timeout 900 python tools/diag_sweep.py 18432_72_7 27136_72_6 0_0_8 > gpurun_out/g27_tma.log 2>&1
