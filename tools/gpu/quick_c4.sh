# merge-pipeline parity tests + C4 stage times (quick check of a kernel change)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_combine.py tests/test_gpu_dist.py tests/test_gpu_f12.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python tools/gpu/probe_step.py 4 > gpurun_out/${TAG}_c4.log 2>&1; tail -2 gpurun_out/${TAG}_c4.log
timeout 300 python tools/gpu/probe_step.py 2 > gpurun_out/${TAG}_c2.log 2>&1; tail -1 gpurun_out/${TAG}_c2.log
timeout 300 python tools/gpu/probe_c5.py > gpurun_out/${TAG}_c5.log 2>&1; tail -2 gpurun_out/${TAG}_c5.log
