// Error state and version of the C ABI (include/paulib_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

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

struct StageRec {
  char name[32];
  cudaEvent_t a, b;
};
static std::mutex g_stage_mu;
static std::vector<StageRec> g_stages;
static bool g_stage_on = false;

bool stage_timing_enabled() { return g_stage_on; }

void stage_record(const char* name, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  StageRec r;
  snprintf(r.name, sizeof(r.name), "%s", name);
  r.a = a;
  r.b = b;
  g_stages.push_back(r);
}

}  // namespace plb

extern "C" int pl_stage_timing(int enable) {
  std::lock_guard<std::mutex> lk(plb::g_stage_mu);
  plb::g_stage_on = enable != 0;
  return PL_OK;
}

extern "C" int pl_stage_times(char* names, float* ms, int max) {
  std::lock_guard<std::mutex> lk(plb::g_stage_mu);
  int n = 0;
  for (auto& r : plb::g_stages) {
    cudaEventSynchronize(r.b);
    if (n < max) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      if (names) memcpy(names + 32 * n, r.name, 32);
      if (ms) ms[n] = t;
      ++n;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  plb::g_stages.clear();
  return n;
}

extern "C" const char* pl_last_error(void) { return plb::g_last_error; }

extern "C" int pl_abi_version(void) { return PL_ABI_VERSION; }
