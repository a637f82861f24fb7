# sweep the head_dim-128 MHA pipeline variants on the cfg2 state
# (BATON_MHA_VARIANT: 0 = default (4,2,3); 1 = (4,3,2); 5 = (2,2,5); 6 = (2,2,4);
#  other values fall back to the default -- decode_attention.cu)
cd $GRAFT_REPO_ROOT
# the sweep variants exist in experiment builds only
python -m paper_2410_18701_b200.build --experiments > /dev/null
for v in 0 1 5 6; do
  echo "variant $v" >> gpurun_out/sweep.log
  BATON_MHA_VARIANT=$v python scripts/profile_decode.py --iters 30 >> gpurun_out/sweep.log 2>&1
  BATON_MHA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_decode.py -q -x -k "matches_oracle or repeat or invariance" >> gpurun_out/sweep.log 2>&1
done
