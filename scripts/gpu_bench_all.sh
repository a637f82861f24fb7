#!/bin/bash
# every bench.py config on one GPU + the 2-rank-on-one-GPU bench tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 7b 13b 70b stress; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_$c.log
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_bench_multirank.py -q > gpurun_out/bench_mr.log 2>&1
echo "rc=$?" >> gpurun_out/bench_mr.log
