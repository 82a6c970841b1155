#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -m gpu tests/test_gpu_variants.py tests/test_gpu_multigpu.py -x > gpurun_out/g29_tests.log 2>&1
for m in 1 3 1 3; do
  echo "== TV_TILE_ORDER=$m" >> gpurun_out/g29_tail.log
  TV_TILE_ORDER=$m timeout 600 python tools/rank_share.py >> gpurun_out/g29_tail.log 2>&1
done
