#!/bin/bash
# GQA decode with the layer's K/V resident in L2 (consumer-bound): timing + ncu source profile
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# the sweep variants and timelines exist in experiment builds only
python -m paper_2410_18701_b200.build --experiments > /dev/null
for v in 0 10; do
  BATON_GQA_VARIANT=$v timeout 300 python scripts/profile_decode.py --iters 50 --layers 1 --config 70b > gpurun_out/gqa_l2_v$v.log 2>&1
done
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:decode_gqa -s 3 -c 1 -o gpurun_out/gqa_l2 -f python scripts/profile_decode.py --iters 2 --layers 1 --config 70b > gpurun_out/ncu_gqa_l2.log 2>&1
