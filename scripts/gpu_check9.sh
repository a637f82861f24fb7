set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench4.log 2>&1; echo "exit $?" >> gpurun_out/bench4.log
python scripts/profile_decode.py --iters 20 --config 70b > gpurun_out/prof_gqa.log 2>&1
BATON_GQA_VARIANT=1 python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/prof_gqa.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attention -s 40 -c 1 -o gpurun_out/bench_decode_full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_full.log 2>&1
