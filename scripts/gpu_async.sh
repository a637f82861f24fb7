#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "async or w1" > gpurun_out/async_tests.log 2>&1
echo "rc=$?" >> gpurun_out/async_tests.log
timeout 1500 python scripts/policy_compare.py --dataset d2 --batches 2,4,6,8,10 > gpurun_out/ablation_d2.log 2>&1
timeout 1500 python scripts/policy_compare.py --dataset d1 --batches 4,8 --no-shape > gpurun_out/ablation_d1.log 2>&1
