set -x
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench7.log 2>&1; echo "exit $?" >> gpurun_out/bench7.log
timeout 1200 python scripts/policy_compare.py --dataset d2 --batches 2,4,6,8,10 > gpurun_out/policy_d2.log 2>&1; echo "exit $?" >> gpurun_out/policy_d2.log
timeout 1500 python scripts/policy_compare.py --dataset d1 --batches 4,8 > gpurun_out/policy_d1.log 2>&1; echo "exit $?" >> gpurun_out/policy_d1.log
