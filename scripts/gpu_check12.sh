set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fullsize.py tests/test_gpu_engine.py -x -q --timeout 300 -k "gqa or 70b or stream_replay or multirank" > gpurun_out/pytest_gqa.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gqa.log
python scripts/profile_decode.py --iters 20 --config 70b > gpurun_out/prof_gqa.log 2>&1
BATON_GQA_VARIANT=1 python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/prof_gqa.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_gqa -s 2 -c 1 -o gpurun_out/gqa_v4 -f python scripts/profile_decode.py --iters 2 --layers 2 --config 70b > gpurun_out/ncu_gqa.log 2>&1
timeout 600 python scripts/bench_configs.py --only 70b >> gpurun_out/prof_gqa.log 2>&1
