#!/bin/bash
# Dev tool: sweep trace-kernel tuning knobs on the C2 workload (one process per config).
out=gpurun_out/sweep.log
: > $out
for cfg in ${SWEEP:-"4 4 4 50" "5 4 4 60" "4 2 2 50" "5 2 2 60" "4 1 1 50" "5 1 4 60" "4 4 1 50"}; do
  set -- $(echo $cfg | tr '_' ' ')
  echo "minb=$1 regen=$2 scatter=$3 carveout=$4" >> $out
  TV_TRACE_MINB=$1 TV_REGEN_MIN=$2 TV_SCATTER_MIN=$3 TV_CARVEOUT=$4 timeout 120 python tools/build_perf.py 256 0.15 24 32 2>&1 | grep render | tail -1 >> $out
done
