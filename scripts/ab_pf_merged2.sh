#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/pfm2
mkdir -p $O
BATON_PF_MERGED=1 BATON_PF_LOCK=1 timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  echo "cfg 2cta" >> $O/ab.log
  BATON_PF_MERGED=0 timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  for lk in 0 1; do
    echo "cfg merged_lock$lk" >> $O/ab.log
    BATON_PF_MERGED=1 BATON_PF_LOCK=$lk timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
