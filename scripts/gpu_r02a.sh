#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_policies.py tests/test_gpu_handoff.py tests/test_gpu_bench_multirank.py "tests/test_gpu_engine.py::test_random_stream_replay_hybrid_store" "tests/test_gpu_engine.py::test_w1_replay" "tests/test_gpu_engine.py::test_random_stream_replay_host_stash" -q -x > gpurun_out/r02a_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02a_tests.log
timeout 900 python bench.py --config 13b > gpurun_out/bench_13b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_13b.log
timeout 900 python bench.py --config stress --no-full-run --no-cpu-baseline > gpurun_out/bench_stress.log 2>&1; echo "rc=$?" >> gpurun_out/bench_stress.log
timeout 900 python scripts/bench_hybrid.py > gpurun_out/hybrid.log 2>&1; echo "rc=$?" >> gpurun_out/hybrid.log
timeout 1200 python scripts/policy_traces.py --dataset d2 --out gpurun_out/r02_traces > gpurun_out/traces_d2.log 2>&1; echo "rc=$?" >> gpurun_out/traces_d2.log
