# quick GPU iteration: merge-path parity tests + per-stage timings of C4 and C2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_combine.py tests/test_gpu_dist.py tests/test_gpu_api_r2.py -x -q -p no:cacheprovider > gpurun_out/quick_pytest.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/quick_pytest.log
timeout 300 python tools/gpu/probe_step.py 4 2>&1 | tail -3
timeout 300 python tools/gpu/probe_step.py 2 2>&1 | tail -2
timeout 300 python tools/gpu/probe_c5.py 2>&1 | tail -2
