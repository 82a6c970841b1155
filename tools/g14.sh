#!/bin/bash
cd $GRAFT_REPO_ROOT
TETVOL_B200_LIB=$PWD/paper_2506_11510_b200/_lib/var/yo/libtetvol_b200.so timeout 600 python -m pytest -q -m gpu tests/test_gpu_parity.py -x > gpurun_out/g14_tests_yo.log 2>&1
SWEEP="base_72_72 yo_72_72 yo_72_58 yo_72_62 yo_72_66 yo_80_50 yo_80_55 yo_72_50 base_72_72" bash tools/sweep_lib.sh; cp gpurun_out/sweep_lib.log gpurun_out/g14_sweep.log
