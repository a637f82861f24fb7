set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q --timeout 300 -k "graph or w1" > gpurun_out/pytest_e.log 2>&1; echo "exit $?" >> gpurun_out/pytest_e.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench6.log 2>&1; echo "exit $?" >> gpurun_out/bench6.log
