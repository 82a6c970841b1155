#!/bin/bash
# Dev tool: sweep trace-kernel tuning knobs on the C2 workload (one process per config).
# SWEEP entries: maxreg_regen_scatter_carveout_threads_order
out=gpurun_out/sweep.log
: > $out
for cfg in ${SWEEP:-"72_5_2_72_128_1"}; do
  set -- $(echo $cfg | tr '_' ' ')
  echo "maxreg=$1 regen=$2 scatter=$3 carveout=$4 threads=${5:-128} order=${6:-1}" >> $out
  TV_VERBOSE=1 TV_TRACE_MAXREG=$1 TV_REGEN_MIN=$2 TV_SCATTER_MIN=$3 TV_CARVEOUT=$4 TV_TRACE_THREADS=${5:-128} TV_ORDER=${6:-1} timeout 120 python tools/build_perf.py ${GRIDN:-256} ${THR:-0.15} 24 32 2>&1 | grep -E "render|tetvol_b200:" | tail -2 >> $out
done
