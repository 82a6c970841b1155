#!/bin/bash
# Dev tool: time kernel variants built with `make OUT=_lib/var/<name> VARIANT=...`
# on the C2 workload, and check each one's C1 framebuffer bits.
out=gpurun_out/variants.log
: > $out
for n in ${VARIANTS:-base}; do
  lib=paper_2506_11510_b200/_lib/var/$n/libtetvol_b200.so
  [ $n = base ] && lib=paper_2506_11510_b200/_lib/libtetvol_b200.so
  echo "== $n" >> $out
  TETVOL_B200_LIB=$PWD/$lib timeout 300 python -m pytest -q -m gpu tests/test_gpu_parity.py -k "render_c1 or emission" 2>&1 | tail -1 >> $out
  TETVOL_B200_LIB=$PWD/$lib timeout 200 python tools/build_perf.py ${GRIDN:-256} ${THR:-0.15} 24 32 2>&1 | grep -E "render" | tail -2 >> $out
done
