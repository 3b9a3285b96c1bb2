// Temporary entry points for kernels not yet landed (return PL_ERR_ARG).
#include "common.cuh"
using namespace plb;
extern "C" int pl_outer_plan(int, int64_t, int64_t, const uint64_t*, const uint64_t*, int64_t,
                             const uint64_t*, const uint64_t*, int64_t, pl_merge_plan*, void*) {
  set_error("pl_outer_plan: not implemented yet"); return PL_ERR_ARG; }
extern "C" int pl_sort_plan(int, int64_t, const uint64_t*, const uint64_t*, int64_t, pl_merge_plan*, void*) {
  set_error("pl_sort_plan: not implemented yet"); return PL_ERR_ARG; }
extern "C" int pl_outer_multiply_combine(const pl_merge_plan*, const uint64_t*, const uint64_t*, const uint8_t*,
    const double*, int64_t, const uint64_t*, const uint64_t*, const uint8_t*, const double*, int64_t, double,
    void*, size_t, uint64_t*, uint64_t*, uint8_t*, double*, int64_t, int64_t*, void*) {
  set_error("not implemented yet"); return PL_ERR_ARG; }
extern "C" int pl_sort_combine(const pl_merge_plan*, const uint64_t*, const uint64_t*, const uint8_t*, const double*,
    int64_t, double, void*, size_t, uint64_t*, uint64_t*, uint8_t*, double*, int64_t, int64_t*, void*) {
  set_error("not implemented yet"); return PL_ERR_ARG; }
extern "C" int64_t pl_group_workspace_bytes(int, int64_t) { return 0; }
extern "C" int pl_group_greedy(int, int64_t, const uint64_t*, const uint64_t*, int64_t, int32_t*, int32_t*,
    int64_t*, void*, size_t, void*) { set_error("not implemented yet"); return PL_ERR_ARG; }
