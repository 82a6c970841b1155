#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python tools/diag_ceiling.py profiles/trace_kernel_ceiling.json > gpurun_out/g20_diag.log 2>&1
cp profiles/trace_kernel_ceiling.json gpurun_out/trace_kernel_ceiling.json
timeout 900 python bench.py > gpurun_out/g20_bench.log 2>&1
