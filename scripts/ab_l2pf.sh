#!/bin/bash
# (the prefetch code was reverted after this A/B: profiles/r01_l2_prefetch_ab.md; the env vars are no-ops now)
# A/B of the pre-wait L2 prefetch of statically assigned items (decode kernels),
# alternating runs: GQA (70B shard, BATON_GQA_L2PF = static items per CTA) and
# MHA (bench.py 7B, BATON_MHA_L2PF = "static items,prefetching CTAs").
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_l2pf.log
if [ -n "$PARITY" ]; then
  BATON_GQA_L2PF=3 BATON_MHA_L2PF=2,740 timeout 900 python -m pytest tests -m gpu -q -x \
    -k "decode or engine or fullsize or gqa" > gpurun_out/ab_l2pf_parity.log 2>&1
  echo "parity rc=$?" >> gpurun_out/ab_l2pf_parity.log
fi
for rep in 1 2; do
  for n in ${GQA_NS:-1 2 3 4}; do
    echo "gqa nstatic $n" >> gpurun_out/ab_l2pf.log
    BATON_GQA_L2PF=$n timeout 300 python scripts/bench_configs.py --only 70b --steps 40 >> gpurun_out/ab_l2pf.log 2>&1
  done
  for m in ${MHA_NS:-1,0 2,148 2,370 2,740}; do
    echo "mha $m" >> gpurun_out/ab_l2pf.log
    BATON_MHA_L2PF=$m timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'value': d['value'], 'frac': d['roofline']['frac'], 'e2e': d['e2e']['value']}))" \
      >> gpurun_out/ab_l2pf.log 2>&1
  done
done
