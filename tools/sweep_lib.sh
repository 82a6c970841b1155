#!/bin/bash
# Dev tool: like sweep.sh, over kernel-variant libraries: SWEEP entries are
# lib_maxreg_carveout (lib = name under _lib/var/, or base).
out=gpurun_out/sweep_lib.log
: > $out
for cfg in $SWEEP; do
  set -- $(echo $cfg | tr '_' ' ')
  lib=paper_2506_11510_b200/_lib/var/$1/libtetvol_b200.so
  [ $1 = base ] && lib=paper_2506_11510_b200/_lib/libtetvol_b200.so
  echo "lib=$1 maxreg=$2 carveout=$3" >> $out
  TETVOL_B200_LIB=$PWD/$lib TV_VERBOSE=1 TV_TRACE_MAXREG=$2 TV_CARVEOUT=$3 timeout 120 python tools/build_perf.py ${GRIDN:-256} ${THR:-0.15} 24 32 2>&1 | grep -E "render|tetvol_b200: trace" | tail -2 >> $out
done
