#!/bin/bash
# (1) GQA decode issuers as converged warps + elect.sync (new) vs lane 0 (old,
#     build/ab_old/): GQA parity tests on the new build, then 70b bench lines alternating.
# (2) prefill: a quarter of the off-diagonal exponentials on the FMA pipe
#     (BATON_PF_POLY=1): parity of every a8 path, then graph-timed A/B.
cd "$(dirname "$0")/.."
O=gpurun_out/gep
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {
  if [ "$1" = old ]; then cp build/ab_old/decode_gqa_tc.cu $C/decode_gqa_tc.cu;
  else cp build/ab_old/decode_gqa_tc.new.cu $C/decode_gqa_tc.cu; fi
  touch $C/decode_gqa_tc.cu
  python -m paper_2410_18701_b200.build > $O/build_$1.log 2>&1
}
use new
timeout 1200 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py::test_70b_gqa_shard_full_size -q -x -k "gqa or GQA or 70b or tc" > $O/gqa_tests.log 2>&1
echo "rc=$?" >> $O/gqa_tests.log
: > $O/gqa_ab.log
for rep in 1 2; do
  for v in old new; do
    use $v
    echo "gqa $v" >> $O/gqa_ab.log
    timeout 600 python bench.py --config 70b --windows 3 --steps 100 --warmup 10 --no-cpu-baseline --no-full-run --no-e2e 2>/dev/null | grep '^{' >> $O/gqa_ab.log
  done
done
use new
BATON_PF_POLY=1 timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py -q -x > $O/poly_tests.log 2>&1
echo "rc=$?" >> $O/poly_tests.log
: > $O/poly_ab.log
for rep in 1 2; do
  for v in 0 1; do
    echo "poly $v" >> $O/poly_ab.log
    BATON_PF_POLY=$v timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/poly_ab.log 2>&1
  done
done
