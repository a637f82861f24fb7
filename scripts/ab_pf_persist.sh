#!/bin/bash
# Persistent prefill: parity tests of every a8 path, then an A/B of the launch shape
# (BATON_PF_PERSIST=1: two CTAs per SM walk the items; 0: one CTA per item, round 1)
# on the configs' prompt shapes and the bench's 64-prompt mixes, graph-timed.
cd "$(dirname "$0")/.."
O=gpurun_out/pfp
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in 0 1; do
    echo "persist $v" >> $O/ab.log
    BATON_PF_PERSIST=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
