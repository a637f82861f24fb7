# sweep the head_dim-128 MHA pipeline variants on the cfg2 state
cd $GRAFT_REPO_ROOT
for v in 0 3 5 6 7 8; do
  echo "variant $v" >> gpurun_out/sweep.log
  BATON_MHA_VARIANT=$v python scripts/profile_decode.py --iters 30 >> gpurun_out/sweep.log 2>&1
  BATON_MHA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_decode.py -q -x -k "matches_oracle or repeat or invariance" >> gpurun_out/sweep.log 2>&1
done
