#!/bin/bash
# Dev tool: 32-B hot records: parity tests and C2 frame timing with / without them
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_c2_parity.py -x > gpurun_out/s17_parity.log 2>&1; echo "rc=$?" >> gpurun_out/s17_parity.log
timeout 300 python tools/build_perf.py 256 0.15 24 32 > gpurun_out/s17_hot.log 2>&1
TV_HOT=0 timeout 300 python tools/build_perf.py 256 0.15 24 32 > gpurun_out/s17_leaf.log 2>&1
