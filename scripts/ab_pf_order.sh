#!/bin/bash
# Prefill varlen item order (BATON_PF_ORDER: 0 prompt-major, 1 global heaviest first)
# x softmax split (BATON_PF_SPLIT 1|2): parity of the varlen tests under the new order,
# graph-timed A/B on the configs' shapes, and ncu DRAM bytes of the 7b 64-prompt mix.
cd "$(dirname "$0")/.."
O=gpurun_out/pfo
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for sp in 1; do
    for od in 0 1; do
      echo "order $od split $sp" >> $O/ab.log
      BATON_PF_ORDER=$od BATON_PF_SPLIT=$sp timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
    done
  done
done
for od in 0 1; do
  BATON_PF_ORDER=$od timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:prefill_attention -s 4 -c 1 --csv python scripts/bench_prefill.py --iters 2 --only 7b-mix64 > $O/ncu_order$od.csv 2>&1
done
