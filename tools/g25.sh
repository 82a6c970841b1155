#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -m gpu tests/test_gpu_build.py tests/test_gpu_diag.py -x > gpurun_out/g25_tests.log 2>&1
timeout 300 python tools/build_repeat.py 1024 2.0 30 4 > gpurun_out/g25_c4.log 2>&1
timeout 300 python tools/build_repeat.py 256 0.15 24 4 > gpurun_out/g25_c2b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g25_c4_launches.csv python tools/build_repeat.py 1024 2.0 30 1 > gpurun_out/g25_c4_ncu.log 2>&1
