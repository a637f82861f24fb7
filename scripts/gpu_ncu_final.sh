#!/bin/bash
# ncu --set full of the prefill (70B prompt, 7B 64-prompt mix) and of one GQA decode
# launch inside the 70b bench, after the elect.sync issuers
cd "$(dirname "$0")/.."
O=gpurun_out/ncuf
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o $O/pf_70b -f python scripts/bench_prefill.py --iters 2 --only 70b:3400 > $O/ncu_pf_70b.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o $O/pf_mix64 -f python scripts/bench_prefill.py --iters 2 --only 7b-mix64 > $O/ncu_pf_mix.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc -s 200 -c 1 \
  -o $O/gqa_full -f python bench.py --config 70b --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > $O/ncu_gqa.log 2>&1
