#!/bin/bash
# Dev tool: final validation of this session (GPU tests, smoke, bench, reference arm)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/s19_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s19_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s19_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s19_smoke.log
timeout 900 python bench.py > gpurun_out/s19_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s19_ref.log 2>&1
