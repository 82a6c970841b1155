#!/bin/bash
# Dev tool: one GPU session of round 2 — GPU tests of the changed paths, C4 / C2 build timings, the
# latency-ceiling diagnostic, the bench line and the C4 build launch list (outputs under gpurun_out/).
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -m gpu tests/test_gpu_build.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_c2_parity.py tests/test_gpu_multigpu.py tests/test_gpu_edge.py -x > gpurun_out/r02_tests.log 2>&1
TV_VERBOSE=3 timeout 300 python tools/build_repeat.py 1024 2.0 30 3 > gpurun_out/r02_c4_v3.log 2>&1
timeout 300 python tools/build_repeat.py 256 0.15 24 3 > gpurun_out/r02_c2b.log 2>&1
timeout 600 python tools/diag_ceiling.py > gpurun_out/r02_diag.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python tools/build_repeat.py 1024 2.0 30 1 > gpurun_out/r02_c4_ncu.log 2>&1
