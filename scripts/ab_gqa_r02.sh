#!/bin/bash
# GQA decode (70b config) A/B in an experiment build: 20 = tcgen05 + combine (default),
# 22 = no combine at all (wrong outputs; the combine hop's cost), 23 = published tickets +
# a combine that merges under the attention tail.  Parity of 23 first.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2410_18701_b200.build --experiments > /dev/null 2>&1
BATON_GQA_VARIANT=23 timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fullsize.py -q -x -k "gqa or 70b or Hq or engine" > gpurun_out/ab_gqa23_tests.log 2>&1
echo "rc=$?" >> gpurun_out/ab_gqa23_tests.log
: > gpurun_out/ab_gqa_r02.log
for rep in 1 2; do
  for v in 20 22 23; do
    BATON_GQA_VARIANT=$v timeout 600 python bench.py --config 70b --steps 100 --warmup 10 --windows 3 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/ab_tmp.log 2>&1
    python -c "
import json,sys
for l in open('gpurun_out/ab_tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'variant': $v, 'rep': $rep, 'value': d['value'], 'frac': d['roofline']['frac'], 'windows': [(w['t0'], round(w['value']), round(w['attn_frac'],3)) for w in d['windows']]}))
" >> gpurun_out/ab_gqa_r02.log
  done
done
python -m paper_2410_18701_b200.build > /dev/null 2>&1
