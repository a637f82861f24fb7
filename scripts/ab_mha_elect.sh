#!/bin/bash
# MHA decode producer as a converged warp + elect.sync: new vs old (build/ab_old/),
# parity on the new build, then 7b and stress bench lines alternating builds.
cd "$(dirname "$0")/.."
O=gpurun_out/mhe
mkdir -p $O
C=paper_2410_18701_b200/csrc
use() {
  if [ "$1" = old ]; then cp build/ab_old/decode_attention.cu $C/decode_attention.cu;
  else cp build/ab_old/decode_attention.new.cu $C/decode_attention.cu; fi
  touch $C/decode_attention.cu
  python -m paper_2410_18701_b200.build > $O/build_$1.log 2>&1
}
use new
timeout 2400 python -m pytest tests -m gpu -q -x -k "not stress_shard_full_size" > $O/tests.log 2>&1
echo "rc=$?" >> $O/tests.log
: > $O/ab.log
for rep in 1 2; do
  for v in old new; do
    use $v
    for c in 7b stress; do
      echo "build $v $c" >> $O/ab.log
      timeout 600 python bench.py --config $c --windows 3 --steps 100 --warmup 10 --no-cpu-baseline --no-full-run --no-e2e 2>/dev/null | grep '^{' >> $O/ab.log
    done
  done
done
use new
