set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q --timeout 120 > gpurun_out/pytest_prefill.log 2>&1; echo "exit $?" >> gpurun_out/pytest_prefill.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attention -s 2 -c 1 -o gpurun_out/decode_full -f python scripts/profile_decode.py --iters 2 --layers 2 > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_attention -s 1 -c 1 -o gpurun_out/prefill_full -f python -m pytest tests/test_gpu_prefill.py -x -q -k "32-32-260" > gpurun_out/ncu_prefill.log 2>&1
timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -k "splice_error" > gpurun_out/pytest_fix.log 2>&1
