set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python tools/gpu/probe_c5_group.py > gpurun_out/c5group.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_r2a.log 2>&1
echo pytest_rc=$?
tail -30 gpurun_out/pytest_r2a.log
cat gpurun_out/c5group.log
