#!/bin/bash
# Prefill softmax threads per query row: BATON_PF_SPLIT=2 (8 softmax warps, two threads
# per row) parity tests, then an A/B against SPLIT=1 on the configs' prompt shapes.
cd "$(dirname "$0")/.."
O=gpurun_out/pfs
mkdir -p $O
BATON_PF_SPLIT=2 timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in 1 2; do
    echo "split $v" >> $O/ab.log
    BATON_PF_SPLIT=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
BATON_PF_SPLIT=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o $O/pf2_70b -f python scripts/bench_prefill.py --iters 2 --only 70b:3400 > $O/ncu_pf2_70b.log 2>&1
