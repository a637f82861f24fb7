#!/bin/bash
# GQA decode chain between two consecutive layers of the decode-step graph (70B shard,
# deferred split-K merge): experiment build, globaltimer trace, product build restored
cd "$(dirname "$0")/.."
O=${OUT:-gpurun_out/trg}
mkdir -p $O
python -m paper_2410_18701_b200.build --experiments > $O/build.log 2>&1
for rep in 1 2 3; do
  BATON_GQA_VARIANT=20 timeout 600 python scripts/trace_engine.py --config 70b --out $O/trace_$rep.json > $O/trace_$rep.log 2>&1
done
python -m paper_2410_18701_b200.build > $O/build_product.log 2>&1
