#!/bin/bash
# round-2 closing evidence after the elect.sync issuers: smoke, the four bench lines,
# the GPU suite, the launch list of the default bench command, the GQA chain trace
cd "$(dirname "$0")/.."
O=gpurun_out/r02z
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
for c in 70b 13b stress; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > $O/ncu_launch_run.log 2>&1
OUT=$O/trg bash scripts/gpu_trace_gqa_r02.sh
