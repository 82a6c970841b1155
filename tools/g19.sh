#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_edge.py tests/test_gpu_c2_parity.py tests/test_gpu_build.py tests/test_gpu_multigpu.py -x > gpurun_out/g19_tests.log 2>&1
timeout 600 python tools/quick_render_timing.py 0 32 128 > gpurun_out/g19_timing.log 2>&1
