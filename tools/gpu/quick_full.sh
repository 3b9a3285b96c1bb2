# quick_c4 + the full-size parity tests and the multi-process K7 tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}
bash tools/gpu/quick_c4.sh $TAG
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_dist_mp.py -x -q > gpurun_out/${TAG}_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/${TAG}_full.log
