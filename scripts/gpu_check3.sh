set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q --timeout 300 -k "graph or w1 or splice or stream_replay and (0 or 5)" > gpurun_out/pytest_b.log 2>&1; echo "exit $?" >> gpurun_out/pytest_b.log
python scripts/profile_decode.py --iters 20 > gpurun_out/prof_decode.log 2>&1
python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/prof_decode.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attention -s 2 -c 1 -o gpurun_out/decode_v2 -f python scripts/profile_decode.py --iters 2 --layers 2 > gpurun_out/ncu_v2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_gqa -s 2 -c 1 -o gpurun_out/gqa_v1 -f python scripts/profile_decode.py --iters 2 --layers 2 --config 70b > gpurun_out/ncu_gqa.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill -s 0 -c 1 -o gpurun_out/prefill_v1 -f python -m pytest tests/test_gpu_prefill.py -x -q -k "32-32-260" > gpurun_out/ncu_prefill.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench3.log 2>&1; echo "exit $?" >> gpurun_out/bench3.log
