#!/bin/bash
# Dev tool: the round-2 validation session (all GPU tests, smoke, bench, reference arm, profiles/ capture, C4 configs).
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/g28_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g28_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g28_ref.log 2>&1
bash tools/profile_round.sh
timeout 1500 python tools/configs_report.py c4 > gpurun_out/g28_c4.jsonl 2>&1
