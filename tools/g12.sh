#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/g12_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g12_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g12_bench.log 2>&1
timeout 900 python bench.py --gather --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g12_bench_gather1.log 2>&1
timeout 1500 python tools/configs_report.py > gpurun_out/g12_configs.jsonl 2>gpurun_out/g12_configs.err
