#!/bin/bash
# Dev tool: probe hanging test with one prober per new midpoint: build tests, C4 check, cost sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_build.py -x > gpurun_out/s12_build_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s12_build_tests.log
TV_HANG_CHECK=1 TV_HANG_PROBE_COST=1 timeout 300 python tools/build_repeat.py 1024 1.75 30 2 > gpurun_out/s12_c4_check1.log 2>&1; echo "rc=$?" >> gpurun_out/s12_c4_check1.log
for c in 64 16 8 4 2; do
TV_HANG_PROBE_COST=$c timeout 300 python tools/build_repeat.py 1024 1.75 30 4 > gpurun_out/s12_c4_cost$c.log 2>&1
done
