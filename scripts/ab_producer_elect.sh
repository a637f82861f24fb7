#!/bin/bash
# Producers (TMA issue) as converged warps + elect.sync, GQA decode and prefill: new vs
# old (build/ab_old/), parity on the new build, 70b bench lines and prefill shapes
# alternating builds.
cd "$(dirname "$0")/.."
O=gpurun_out/pre
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {
  if [ "$1" = old ]; then cp build/ab_old/decode_gqa_tc.cu $C/; cp build/ab_old/prefill_attention.cu $C/;
  else cp build/ab_old/decode_gqa_tc.new.cu $C/decode_gqa_tc.cu; cp build/ab_old/prefill_attention.new.cu $C/prefill_attention.cu; fi
  touch $C/decode_gqa_tc.cu $C/prefill_attention.cu
  python -m paper_2410_18701_b200.build > $O/build_$1.log 2>&1
}
use new
timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py tests/test_gpu_fullsize.py::test_70b_gqa_shard_full_size -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in old new; do
    use $v
    echo "build $v" >> $O/ab.log
    timeout 600 python bench.py --config 70b --windows 3 --steps 100 --warmup 10 --no-cpu-baseline --no-full-run --no-e2e 2>/dev/null | grep '^{' >> $O/ab.log
    timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
use new
