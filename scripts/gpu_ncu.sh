#!/bin/bash
# ncu --set full of the default kernels inside their configs (one launch each)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc -s 40 -c 1 -o gpurun_out/gqa_tc_full -f python scripts/bench_configs.py --only 70b --steps 4 --warmup 3 > gpurun_out/ncu_gqa_tc.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 40 -c 1 -o gpurun_out/mha_full -f python scripts/bench_configs.py --only 7b --steps 4 --warmup 3 > gpurun_out/ncu_mha.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_70b.csv python scripts/bench_configs.py --only 70b --steps 2 --warmup 3 > /dev/null 2>&1
