#!/bin/bash
# GPU check of the whole suite (no -x: report every failure), smoke and the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/check_tests.log 2>&1
echo "rc=$?" >> gpurun_out/check_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
