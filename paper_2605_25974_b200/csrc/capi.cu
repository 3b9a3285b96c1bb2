// Error state and version of the C ABI (include/paulib_b200.h).
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace plb {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return PL_ERR_CUDA;
}

}  // namespace plb

extern "C" const char* pl_last_error(void) { return plb::g_last_error; }

extern "C" int pl_abi_version(void) { return PL_ABI_VERSION; }
