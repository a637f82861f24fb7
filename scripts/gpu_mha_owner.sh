#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x > gpurun_out/owner_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/owner_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/owner_bench.log 2>&1
timeout 600 python scripts/bench_configs.py --only 13b > gpurun_out/owner_configs.log 2>&1
CFG=7b bash scripts/gpu_trace2.sh
