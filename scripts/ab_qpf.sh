#!/bin/bash
# (the prefetch code was reverted after this A/B: profiles/r01_l2_prefetch_ab.md; the env vars are no-ops now)
# A/B of the pre-wait L2 prefetch of q rows (BATON_QPF) and the e2e pass of bench.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_qpf.log
for rep in 1 2; do
  for f in 0 1; do
    echo "gqa qpf $f" >> gpurun_out/ab_qpf.log
    BATON_QPF=$f timeout 300 python scripts/bench_configs.py --only 70b --steps 40 >> gpurun_out/ab_qpf.log 2>&1
    echo "mha qpf $f" >> gpurun_out/ab_qpf.log
    BATON_QPF=$f timeout 400 python bench.py --no-cpu-baseline 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'value': d['value'], 'frac': d['roofline']['frac'], 'e2e': d['e2e']['value']}))" \
      >> gpurun_out/ab_qpf.log 2>&1
  done
done
