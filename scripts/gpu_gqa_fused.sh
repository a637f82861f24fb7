#!/bin/bash
# GQA fused append + in-kernel merge + early prefetch: tests, timeline, configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py -q -x -k "gqa or early or graph or w1" > gpurun_out/gqaf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gqaf_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k 70b >> gpurun_out/gqaf_tests.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/gqaf_tests.log
timeout 300 python scripts/profile_decode.py --iters 20 --config 70b --layers 4 --trace gpurun_out/gqa_trace2.json > gpurun_out/gqaf_trace.log 2>&1
timeout 600 python scripts/bench_configs.py --only 70b > gpurun_out/gqaf_configs.log 2>&1
timeout 600 python scripts/trace_engine.py > gpurun_out/engine_trace.log 2>&1
