# session re-entry check: GPU suite, f3 probe, ncu source pages of the leaf / split kernels, sanitizer attempt
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
timeout 300 python tools/gpu/probe_f3.py > gpurun_out/r2d_f3.log 2>&1; tail -3 gpurun_out/r2d_f3.log
bash tools/gpu/prof_r2.sh "k_leaf_sort" r2d_leaf 1
bash tools/gpu/prof_r2.sh "k_split_scatter|k_split_count|k_scatter|k_count" r2d_part 4
timeout 400 compute-sanitizer --tool memcheck --print-limit 50 --log-file gpurun_out/r2d_memcheck.log python -m pytest -q -x -p no:cacheprovider tests/test_gpu_combine.py::test_outer_c2_golden tests/test_gpu_combine.py::test_runs_longer_than_leaf > gpurun_out/r2d_memcheck_pytest.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2d_memcheck_pytest.log; tail -5 gpurun_out/r2d_memcheck.log
