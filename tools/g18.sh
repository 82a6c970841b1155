#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in "64 2" "8 2" "16 2" "8 4" "32 4" "64 2"; do
  set -- $cfg
  echo "== TV_TAIL_CHUNK=$1 TV_TAIL_ZONE=$2" >> gpurun_out/g18_tail.log
  TV_TAIL_CHUNK=$1 TV_TAIL_ZONE=$2 timeout 600 python tools/rank_share.py >> gpurun_out/g18_tail.log 2>&1
done
