#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_engine.py::test_gqa_graph_step_deferred_merge_equals_eager_and_oracle tests/test_gpu_fullsize.py::test_70b_gqa_shard_full_size tests/test_gpu_decode.py -q -x > gpurun_out/r02/gqa2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gqa2_tests.log
for rep in 1 2; do
timeout 900 python bench.py --config 70b --steps 100 --warmup 10 --windows 3 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/r02/bench_70b_g1_$rep.log 2>&1
done
