#!/bin/bash
# round-2 closing evidence on HEAD: GPU suite, smoke, the default bench line (+ reference
# arm), the 70b line, and the launch list of the bench command
cd "$(dirname "$0")/.."
O=${OUT:-gpurun_out/r02f}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py --config 70b --no-cpu-baseline > $O/bench_70b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --windows 1 --no-e2e --no-cpu-baseline --no-full-run > $O/ncu_launch_run.log 2>&1
