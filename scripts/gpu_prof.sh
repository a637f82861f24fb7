set -x
cd $GRAFT_REPO_ROOT
python scripts/profile_decode.py --iters 20 > gpurun_out/prof_decode.log 2>&1
python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/prof_decode.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attention -s 4 -c 1 -o gpurun_out/decode_full -f python scripts/profile_decode.py --iters 2 --layers 2 > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
