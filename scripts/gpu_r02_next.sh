#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_long.py tests/test_gpu_shaping.py tests/test_gpu_engine.py tests/test_gpu_decode.py tests/test_gpu_abi_contract.py tests/test_gpu_multirank.py -q -x > gpurun_out/r02/prefill_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02/prefill_tests.log
for rep in 1 2; do timeout 300 python scripts/bench_prefill.py > gpurun_out/r02/prefill_bench_$rep.log 2>&1; done
bash scripts/gpu_sanitize_r02.sh
