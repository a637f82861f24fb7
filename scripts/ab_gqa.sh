#!/bin/bash
# A/B of GQA decode variants in the engine path (70B shard), alternating runs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# the sweep variants and timelines exist in experiment builds only
python -m paper_2410_18701_b200.build --experiments > /dev/null
: > gpurun_out/ab_gqa.log
for rep in 1 2 3; do
  for v in ${VARIANTS:-0 20}; do
    echo "variant $v" >> gpurun_out/ab_gqa.log
    BATON_GQA_VARIANT=$v timeout 300 python scripts/bench_configs.py --only 70b --steps 40 >> gpurun_out/ab_gqa.log 2>&1
  done
done
