#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shaping.py tests/test_gpu_prefill.py -q -x > gpurun_out/shaping_tests.log 2>&1
echo "rc=$?" >> gpurun_out/shaping_tests.log
timeout 300 python scripts/bench_prefill.py > gpurun_out/prefill_bench2.log 2>&1
