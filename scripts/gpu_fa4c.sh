#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > gpurun_out/fa4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/fa4_tests.log
timeout 300 python scripts/bench_prefill.py > gpurun_out/fa4_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:prefill_fa4 -c 1 -o gpurun_out/fa4_70b_c python scripts/bench_prefill.py --only 70b:3400 --iters 1 > gpurun_out/fa4_ncu.log 2>&1
