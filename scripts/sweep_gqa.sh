cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4; do
  echo "gqa variant $v" >> gpurun_out/sweep_gqa.log
  BATON_GQA_VARIANT=$v python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/sweep_gqa.log 2>&1
  BATON_GQA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_decode.py -q -x -k "gqa" >> gpurun_out/sweep_gqa.log 2>&1
done
