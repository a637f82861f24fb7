#!/bin/bash
# A/B of the deferred split-K merge on the MHA decode step (7b, 13b) in an experiment
# build: BATON_DEFER_MERGE=0 (in-layer merges) vs 1 (merge in the next layer's launch);
# parity of the product path first
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_decode.py tests/test_gpu_fullsize.py -q -x -k "not stress_shard" > gpurun_out/r02/defer_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02/defer_tests.log
python -m paper_2410_18701_b200.build --experiments > /dev/null 2>&1
: > gpurun_out/r02/ab_defer.log
for rep in 1 2; do
  for cfg in 7b 13b; do
    for v in 0 1; do
      BATON_DEFER_MERGE=$v timeout 900 python bench.py --config $cfg --steps 100 --warmup 10 --windows 3 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/ab_tmp.log 2>&1
      python -c "
import json
for l in open('gpurun_out/ab_tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'cfg': '$cfg', 'defer': $v, 'rep': $rep, 'value': d['value'], 'frac': d['roofline']['frac'], 'windows': [(w['t0'], round(w['value']), round(w['attn_frac'],3)) for w in d['windows']]}))
" >> gpurun_out/r02/ab_defer.log
    done
  done
done
python -m paper_2410_18701_b200.build > /dev/null 2>&1
