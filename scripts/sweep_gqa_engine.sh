#!/bin/bash
# GQA pipeline variants in the engine path (70B shard, decode-step graphs) + parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# the sweep variants and timelines exist in experiment builds only
python -m paper_2410_18701_b200.build --experiments > /dev/null
: > gpurun_out/sweep_gqa_engine.log
for v in ${VARIANTS:-0 6 7 8}; do
  echo "variant $v" >> gpurun_out/sweep_gqa_engine.log
  BATON_GQA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py -q -x -k "gqa or early" 2>&1 | tail -1 >> gpurun_out/sweep_gqa_engine.log
  BATON_GQA_VARIANT=$v timeout 300 python scripts/bench_configs.py --only 70b --steps 30 >> gpurun_out/sweep_gqa_engine.log 2>&1
done
