set -x
cd $GRAFT_REPO_ROOT
bash scripts/sweep_mha.sh
python scripts/profile_decode.py --iters 20 --config 70b >> gpurun_out/sweep.log 2>&1
