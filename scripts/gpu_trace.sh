#!/bin/bash
# GQA decode timeline + prefill issuer-reorder check
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/profile_decode.py --iters 20 --config 70b --layers 4 --trace gpurun_out/gqa_trace.json > gpurun_out/trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_decode.py -q -x > gpurun_out/trace_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/trace_tests.log
timeout 600 python scripts/bench_prefill.py > gpurun_out/prefill_bench.log 2>&1
