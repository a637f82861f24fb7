#!/bin/bash
# Prefill MMA issuer: whole warp + elect.sync (new) vs a single lane == 0 thread (old,
# build/ab_old/).  Parity of every a8 path on the new build, then alternating builds
# graph-timed, then the clock64 trace of the new one (experiment build).
cd "$(dirname "$0")/.."
O=gpurun_out/pfe
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {   # use old|new
  if [ "$1" = old ]; then cp build/ab_old/prefill_attention.cu $C/; cp build/ab_old/tcgen05.cuh $C/;
  else cp build/ab_old/prefill_attention.new.cu $C/prefill_attention.cu; cp build/ab_old/tcgen05.new.cuh $C/tcgen05.cuh; fi
  touch $C/prefill_attention.cu
  python -m paper_2410_18701_b200.build > $O/build_$1.log 2>&1
}
use new
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in old new; do
    use $v
    echo "issuer $v" >> $O/ab.log
    timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
use new
python -m paper_2410_18701_b200.build --experiments > $O/build_exp.log 2>&1
for sh in 70b:3400 7b:1800; do
  timeout 300 python scripts/trace_prefill.py --shape $sh --out $O/trace_${sh/:/_}.json >> $O/trace.log 2>&1
done
python -m paper_2410_18701_b200.build > $O/build_product.log 2>&1
