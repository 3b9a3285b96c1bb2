# compute-sanitizer memcheck / racecheck / synccheck over the golden-sized GPU
# tests of every kernel family (merge pipeline incl. runs longer than a leaf and
# sparse keys, grouping + f3 merge, bitmatrix, batched multiply, gates, K7).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SEL="tests/test_gpu_combine.py::test_outer_c2_golden tests/test_gpu_combine.py::test_outer_hh_golden \
tests/test_gpu_combine.py::test_simplify_golden tests/test_gpu_combine.py::test_runs_longer_than_leaf \
tests/test_gpu_combine.py::test_sparse_keys_plan_and_parity tests/test_gpu_combine.py::test_leaf_window_ties_fall_back \
tests/test_gpu_combine.py::test_eps_and_cancellation tests/test_gpu_combine.py::test_empty_and_single \
tests/test_gpu_grouping.py::test_grouping_golden tests/test_gpu_grouping.py::test_batch_boundaries \
tests/test_gpu_grouping.py::test_group_greedy_parallel_golden \
tests/test_gpu_bitmatrix.py::test_bitmatrix_golden tests/test_gpu_multiply.py::test_batch_multiply_golden \
tests/test_gpu_multiply.py::test_batch_multiply_unaligned_views tests/test_gpu_multiply.py::test_outer_raw_golden \
tests/test_gpu_f12.py::test_clifford_golden_soa tests/test_gpu_f12.py::test_rotation_golden \
tests/test_gpu_dist.py::test_sharded_hh_cancellation tests/test_gpu_api_r2.py"
for TOOL in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --target-processes all --print-limit 200 \
     --log-file gpurun_out/sanitize_$TOOL.log python -m pytest -q -x -p no:cacheprovider $SEL \
     > gpurun_out/sanitize_${TOOL}_pytest.log 2>&1
  echo "$TOOL rc=$?"
  tail -2 gpurun_out/sanitize_${TOOL}_pytest.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitize_$TOOL.log | sort | uniq -c | head -10
done
