#!/bin/bash
# compute-sanitizer over the round-2 GPU paths: the decode-step graph with the deferred
# GQA merge (engine replay of a GQA-8 random stream), the hybrid K/V store (spill +
# prefetch), the paper-baseline policies, the handoff-free engine paths.  One log per tool.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize_r02
TESTS="tests/test_gpu_engine.py::test_gqa_graph_step_deferred_merge_equals_eager_and_oracle tests/test_gpu_engine.py::test_graph_step_equals_eager_layers_bitwise tests/test_gpu_engine.py::test_random_stream_replay_hybrid_store tests/test_gpu_policies.py tests/test_gpu_abi_contract.py"
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider $TESTS \
    > gpurun_out/sanitize_r02/tests_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_r02/tests_$tool.log
done
