#!/bin/bash
# FA4-layout prefill: parity tests, then a8 TFLOP/s (FA4 vs the round-1 kernel, experiment build)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > gpurun_out/fa4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/fa4_tests.log
timeout 300 python scripts/bench_prefill.py > gpurun_out/fa4_bench.log 2>&1
python -m paper_2410_18701_b200.build --experiments > /dev/null 2>&1
BATON_PF_KERNEL=1 timeout 300 python scripts/bench_prefill.py > gpurun_out/fa4_bench_old.log 2>&1
timeout 300 python scripts/bench_prefill.py > gpurun_out/fa4_bench2.log 2>&1
python -m paper_2410_18701_b200.build > /dev/null 2>&1
ncu --set full --clock-control none -k regex:prefill_fa4 -c 1 -o gpurun_out/fa4_70b python scripts/bench_prefill.py --only 70b:3400 --iters 1 > gpurun_out/fa4_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_handoff.py -q -x > gpurun_out/handoff_tests.log 2>&1; echo "rc=$?" >> gpurun_out/handoff_tests.log
timeout 900 python bench.py --config 13b --no-cpu-baseline > gpurun_out/bench_13b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_13b.log
timeout 900 python scripts/bench_hybrid.py > gpurun_out/hybrid2.log 2>&1; echo "rc=$?" >> gpurun_out/hybrid2.log
bash scripts/ab_gqa_r02.sh
