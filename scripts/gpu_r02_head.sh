#!/bin/bash
# round-2 evidence on the current HEAD: GPU suite, smoke, default bench line + reference arm,
# the launch list of the bench command, one --set full capture of the MHA decode, the 70b line
cd "$(dirname "$0")/.."
O=gpurun_out/r02h
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > $O/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 200 -c 1 -o $O/mha_full python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > $O/ncu_full_run.log 2>&1
timeout 900 python bench.py --config 70b --no-cpu-baseline > $O/bench_70b.log 2>&1
