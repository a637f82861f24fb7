#!/bin/bash
# A/B of the prefill lazy-rescale threshold (BATON_PF_RESCALE_T: 0 = rescale whenever
# the row max moves, 8 = default) on the configs' prompt shapes, graph-timed; then
# one ncu --set full capture of the 70B-shaped prefill (3400 tokens, 64q/8kv).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_prefill.log
for rep in 1 2; do
  for t in 0 8; do
    echo "rescale_t $t" >> gpurun_out/ab_prefill.log
    BATON_PF_RESCALE_T=$t timeout 300 python scripts/bench_prefill.py --iters 50 >> gpurun_out/ab_prefill.log 2>&1
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o gpurun_out/prefill_full -f python scripts/bench_prefill.py --iters 2 --only 70b:3400 > gpurun_out/ncu_prefill.log 2>&1
