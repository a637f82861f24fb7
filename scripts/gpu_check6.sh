set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q --timeout 300 > gpurun_out/pytest_c.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_decode.py -x -q -k "gqa_matches or matches_oracle" > gpurun_out/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/memcheck.log
python scripts/profile_decode.py --iters 20 --config 70b > gpurun_out/prof_decode.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_gqa -s 2 -c 1 -o gpurun_out/gqa_v3 -f python scripts/profile_decode.py --iters 2 --layers 2 --config 70b > gpurun_out/ncu_gqa.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
python scripts/bench_prefill.py > gpurun_out/bench_prefill.log 2>&1
