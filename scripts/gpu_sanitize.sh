#!/bin/bash
# compute-sanitizer over the CUDA path: smoke() (W1 toy replay, MHA d16 + splice +
# metadata kernels) and small parity tests of every other kernel family (MHA d128,
# GQA tcgen05 + combine, tcgen05 prefill, shaping).  One log per tool.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
SMOKE='import __graft_entry__ as g; g.smoke()'
TESTS="tests/test_gpu_decode.py::test_matches_oracle tests/test_gpu_decode.py::test_gqa_matches_oracle tests/test_gpu_prefill.py::test_prefill_matches_oracle tests/test_gpu_prefill.py::test_prefill_varlen_matches_oracle tests/test_gpu_shaping.py::test_w1_shaping_replay"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "$SMOKE" \
    > gpurun_out/sanitize/smoke_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize/smoke_$tool.log
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider $TESTS \
    > gpurun_out/sanitize/tests_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize/tests_$tool.log
done
