#!/bin/bash
# prefill: one CTA per SM with two pipelines taking turns at the SFU (BATON_PF_MERGED=1)
# vs two CTAs per SM (0): parity of the prefill paths with MERGED, then graph-timed A/B
cd "$(dirname "$0")/.."
O=gpurun_out/pfm
mkdir -p $O
BATON_PF_MERGED=1 timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in 0 1; do
    echo "merged $v" >> $O/ab.log
    BATON_PF_MERGED=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
