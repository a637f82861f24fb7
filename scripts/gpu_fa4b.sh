#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > gpurun_out/fa4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/fa4_tests.log
timeout 300 python scripts/bench_prefill.py > gpurun_out/fa4_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:prefill_fa4 -c 1 -o gpurun_out/fa4_70b_b python scripts/bench_prefill.py --only 70b:3400 --iters 1 > gpurun_out/fa4_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_handoff.py "tests/test_gpu_engine.py::test_random_stream_replay_hybrid_store" -q -x > gpurun_out/handoff_tests.log 2>&1; echo "rc=$?" >> gpurun_out/handoff_tests.log
timeout 900 python scripts/bench_hybrid.py --workloads priority > gpurun_out/hybrid3.log 2>&1; echo "rc=$?" >> gpurun_out/hybrid3.log
python -m paper_2410_18701_b200.build --experiments > /dev/null 2>&1
for v in 20 21; do
  BATON_GQA_VARIANT=$v timeout 600 python bench.py --config 70b --steps 100 --warmup 10 --windows 3 --no-e2e --no-cpu-baseline --no-full-run > gpurun_out/ab_tmp.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'variant': $v, 'value': d['value'], 'frac': d['roofline']['frac'], 'windows': [(w['t0'], round(w['value']), round(w['attn_frac'],3)) for w in d['windows']]}))
" >> gpurun_out/ab_gqa_r02b.log
done
python -m paper_2410_18701_b200.build > /dev/null 2>&1
