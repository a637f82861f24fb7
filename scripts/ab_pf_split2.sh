#!/bin/bash
# prefill: K and V rings on two producer lanes (new) vs one (old, build/ab_old/), after
# the elect.sync MMA issuer: parity, alternating-build A/B, clock64 trace of the new one
cd "$(dirname "$0")/.."
O=gpurun_out/pfs2
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {
  if [ "$1" = old ]; then cp build/ab_old/prefill_attention.cu $C/prefill_attention.cu;
  else cp build/ab_old/prefill_attention.new.cu $C/prefill_attention.cu; fi
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
    echo "build $v" >> $O/ab.log
    timeout 300 python scripts/bench_prefill.py --iters 20 >> $O/ab.log 2>&1
  done
done
use new
OUT=$O/tr bash scripts/gpu_trace_pf.sh
