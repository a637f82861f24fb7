#!/bin/bash
# Prefill varlen L2 panels (BATON_PF_PANEL_MB; 0 = one panel = global heaviest first)
# and prompt-major order (BATON_PF_ORDER=2): parity, then graph-timed A/B on the batches.
cd "$(dirname "$0")/.."
O=gpurun_out/pfp2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for mb in 0 32 48 64 96; do
    echo "panel $mb" >> $O/ab.log
    BATON_PF_PANEL_MB=$mb timeout 300 python scripts/bench_prefill.py --iters 20 --batches-only >> $O/ab.log 2>&1
  done
  echo "panel -1" >> $O/ab.log
  BATON_PF_ORDER=2 timeout 300 python scripts/bench_prefill.py --iters 20 --batches-only >> $O/ab.log 2>&1
done
