#!/bin/bash
# Prefill warp-uniform skips (dead 32-key chunks above the diagonal, warps past the
# prompt): parity of every a8 path, then an A/B (BATON_PF_SKIP=0/1), graph-timed.
cd "$(dirname "$0")/.."
O=gpurun_out/pfk
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in 0 1; do
    echo "skip $v" >> $O/ab.log
    BATON_PF_SKIP=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
