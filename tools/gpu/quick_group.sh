# grouping parity tests + C3 / f3 / C5 grouping timings
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-g}
timeout 900 python -m pytest tests/test_gpu_grouping.py -x -q > gpurun_out/${TAG}_gtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_gtests.log
timeout 300 python tools/gpu/probe_c3.py > gpurun_out/${TAG}_c3.log 2>&1; tail -2 gpurun_out/${TAG}_c3.log
timeout 300 python tools/gpu/probe_f3.py > gpurun_out/${TAG}_f3.log 2>&1; tail -1 gpurun_out/${TAG}_f3.log
timeout 600 python tools/gpu/probe_c5_group.py > gpurun_out/${TAG}_c5g.log 2>&1; tail -2 gpurun_out/${TAG}_c5g.log
