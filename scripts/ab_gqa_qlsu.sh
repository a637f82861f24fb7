#!/bin/bash
# GQA decode: q through cp.async (LSU) on its own barrier (new) vs TMA on the stage
# barrier (old, build/ab_old/): GQA parity tests, 70b bench lines alternating builds,
# and the chain trace of the new build.
cd "$(dirname "$0")/.."
O=gpurun_out/gql
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {
  if [ "$1" = old ]; then cp build/ab_old/decode_gqa_tc.cu $C/decode_gqa_tc.cu;
  else cp build/ab_old/decode_gqa_tc.new.cu $C/decode_gqa_tc.cu; fi
  touch $C/decode_gqa_tc.cu
  python -m paper_2410_18701_b200.build > $O/build_$1.log 2>&1
}
use new
timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py::test_70b_gqa_shard_full_size tests/test_gpu_multirank.py tests/test_gpu_handoff.py -q -x > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
: > $O/ab.log
for rep in 1 2; do
  for v in old new; do
    use $v
    echo "build $v" >> $O/ab.log
    timeout 600 python bench.py --config 70b --windows 3 --steps 100 --warmup 10 --no-cpu-baseline --no-full-run --no-e2e 2>/dev/null | grep '^{' >> $O/ab.log
  done
done
use new
OUT=$O/trg bash scripts/gpu_trace_gqa_r02.sh
