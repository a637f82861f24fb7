set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q --timeout 120 > gpurun_out/pytest_prefill.log 2>&1; echo "exit $?" >> gpurun_out/pytest_prefill.log
timeout 300 python scripts/bench_prefill.py > gpurun_out/bench_prefill.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill -s 5 -c 1 -o gpurun_out/prefill_v1b -f python scripts/bench_prefill.py --iters 1 > gpurun_out/ncu_prefill.log 2>&1
