#!/bin/bash
# clock64 per-tile timeline of the prefill kernel (experiment build), product build restored
cd "$(dirname "$0")/.."
O=${OUT:-gpurun_out/trpf}
mkdir -p $O
python -m paper_2410_18701_b200.build --experiments > $O/build.log 2>&1
for sh in 70b:3400 7b:1800; do
  for rep in 1 2; do
    timeout 300 python scripts/trace_prefill.py --shape $sh --out $O/trace_${sh/:/_}_$rep.json >> $O/trace.log 2>&1
  done
done
python -m paper_2410_18701_b200.build > $O/build_product.log 2>&1
