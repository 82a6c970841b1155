#!/bin/bash
# One GPU session: full GPU test suite, smoke, bench (with clocks), launch list and
# an ncu --set full capture of the trace kernel. Outputs under gpurun_out/.
set -o pipefail
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python tools/prof_render.py 32 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_render.py 32 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_render.py 4 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -c 1 -o gpurun_out/prof_trace python tools/prof_render.py 4 > gpurun_out/ncu_full.log 2>&1
