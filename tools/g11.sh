#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_variants.py -x > gpurun_out/g11_tests.log 2>&1
SWEEP="cs_72_72 base_80_50 base_80_45 base_80_55 base_80_40 base_72_60 base_72_57 base_72_65 cs_72_72" bash tools/sweep_lib.sh; cp gpurun_out/sweep_lib.log gpurun_out/g11_sweep.log
