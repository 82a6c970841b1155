#!/bin/bash
# Dev tool: the round-2 validation session (all GPU tests, smoke, bench, reference arm, profiles/ capture,
# latency ceiling, configs, C4 build launch list).
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/fin4_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin4_smoke.log
timeout 600 python tools/diag_ceiling.py gpurun_out/fin4_ceiling.json > gpurun_out/fin4_diag.log 2>&1
cp gpurun_out/fin4_ceiling.json profiles/trace_kernel_ceiling.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/fin4_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin4_ref.log 2>&1
bash tools/profile_round.sh
timeout 2400 python tools/configs_report.py c2 c3 c5 c4 > gpurun_out/fin4_configs.jsonl 2> gpurun_out/fin4_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin4_c4_launches.csv python tools/build_repeat.py 1024 1.75 30 1 > gpurun_out/fin4_c4_ncu.log 2>&1
