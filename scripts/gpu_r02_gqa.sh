#!/bin/bash
# the deferred GQA merge + device completion flags: parity, then the 70b bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_bench_multirank.py tests/test_gpu_handoff.py -q -x -k "not stress_shard_full_size" > gpurun_out/r02/gqa_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gqa_tests.log
timeout 900 python bench.py --config 70b --no-cpu-baseline > gpurun_out/r02/bench_70b_defer.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc -s 200 -c 1 -o gpurun_out/r02/gqa_defer_full python bench.py --config 70b --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/r02/ncu_gqa_defer_run.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_70b.csv python bench.py --config 70b --steps 3 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > /dev/null 2>&1
