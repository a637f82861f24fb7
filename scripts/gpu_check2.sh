set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_decode.py -x -q --timeout 120 > gpurun_out/pytest_a.log 2>&1; echo "exit $?" >> gpurun_out/pytest_a.log
python scripts/profile_decode.py --iters 20 > gpurun_out/prof_decode.log 2>&1
python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/prof_decode.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench2.log 2>&1; echo "exit $?" >> gpurun_out/bench2.log
