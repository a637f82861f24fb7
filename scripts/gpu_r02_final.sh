#!/bin/bash
# round-2 evidence: the whole GPU suite, smoke, the default bench line (+ reference arm),
# the ncu launch list of the bench command and one --set full capture of the top kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/r02/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 200 -c 1 -o gpurun_out/r02/mha_full python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/r02/ncu_full_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc -s 200 -c 1 -o gpurun_out/r02/gqa_full python bench.py --config 70b --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/r02/ncu_gqa_run.log 2>&1
for c in 13b 70b stress; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02/bench_$c.log 2>&1
done
