cd $GRAFT_REPO_ROOT
for v in 0 5; do
  echo "gqa variant $v" >> gpurun_out/sweep_gqa.log
  BATON_GQA_VARIANT=$v python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/sweep_gqa.log 2>&1
  BATON_GQA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_decode.py -q -x -k "gqa" >> gpurun_out/sweep_gqa.log 2>&1
done
BATON_GQA_VARIANT=5 timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_gqa -s 2 -c 1 -o gpurun_out/gqa_v5 -f python scripts/profile_decode.py --iters 2 --layers 2 --config 70b > gpurun_out/ncu_gqa.log 2>&1
