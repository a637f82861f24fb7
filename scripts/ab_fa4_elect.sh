#!/bin/bash
# FA4-layout prefill (experiment) with the converged-warp MMA issuer vs the product kernel:
# parity of the prefill tests with BATON_PF_KERNEL=2, then graph-timed A/B
cd "$(dirname "$0")/.."
O=gpurun_out/fa4e
mkdir -p $O
python -m paper_2410_18701_b200.build --experiments > $O/build.log 2>&1
BATON_PF_KERNEL=2 timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py -q -x -k "not shape_step" > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in 1 2; do
    echo "kernel $v" >> $O/ab.log
    BATON_PF_KERNEL=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
python -m paper_2410_18701_b200.build > $O/build_product.log 2>&1
