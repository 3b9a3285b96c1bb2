// K6 greedy grouping — placeholder until the batched kernel lands.
#include "common.cuh"
using namespace plb;
extern "C" int64_t pl_group_workspace_bytes(int, int64_t) { return 0; }
extern "C" int pl_group_greedy(int, int64_t, const uint64_t*, const uint64_t*, int64_t, int32_t*,
                               int32_t*, int64_t*, void*, size_t, void*) {
  set_error("pl_group_greedy: not implemented yet");
  return PL_ERR_ARG;
}
