#!/bin/bash
# round-2 late: bench lines of every config on the current HEAD (persistent prefill),
# and ncu --set full of the prefill kernel on the 7b 64-prompt mix and the 70B prompt
cd "$(dirname "$0")/.."
O=gpurun_out/r02l
mkdir -p $O
timeout 900 python bench.py > $O/bench_7b.log 2>&1
for c in 13b stress; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o $O/pf_mix64 -f python scripts/bench_prefill.py --iters 2 --only 7b-mix64 > $O/ncu_pf_mix.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 4 -c 1 \
  -o $O/pf_70b -f python scripts/bench_prefill.py --iters 2 --only 70b:3400 > $O/ncu_pf_70b.log 2>&1
