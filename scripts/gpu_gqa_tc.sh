#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export BATON_GQA_VARIANT=${VAR:-20}
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py -q -x -k "gqa or early" > gpurun_out/gqa_tc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gqa_tc_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k 70b >> gpurun_out/gqa_tc_tests.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/gqa_tc_tests.log
timeout 300 python scripts/bench_configs.py --only 70b --steps 30 > gpurun_out/gqa_tc_configs.log 2>&1
timeout 300 python scripts/profile_decode.py --iters 50 --layers 1 --config 70b > gpurun_out/gqa_tc_l2.log 2>&1
timeout 300 python scripts/trace_gqa_tc.py > gpurun_out/gqa_tc_trace.log 2>&1
