// Shared helpers for the paulib_b200 sm_100a kernels.
//
// Storage convention (the north-star SoA layout, reference sums.py:429-450):
//   x, z : W planes of M uint64 words each; word w of term t lives at
//          plane[w * ld + t]  (ld >= M, the plane stride in words)
//   k    : M uint8 phase exponents (i^k)
//   c    : M complex128 coefficients, interleaved (re, im) doubles
// W = tier / 64 in {1, 2, 4, 8, 16} (reference bits.py:12, :34-46).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "paulib_b200.h"

namespace plb {

typedef unsigned long long u64;
typedef unsigned int u32;

// ------------------------------------------------------------- error state
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define PLB_CHECK_LAUNCH(what)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::plb::cuda_status(_e, what);  \
  } while (0)

#define PLB_CUDA(call)                                           \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::plb::cuda_status(_e, #call); \
  } while (0)

// ------------------------------------------------------------ stage timing
// RAII event pair around one kernel launch when pl_stage_timing(1) is on.
bool stage_timing_enabled();
void stage_record(const char* name, cudaEvent_t a, cudaEvent_t b);
struct StageTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  const char* name;
  StageTimer(cudaStream_t s, const char* n) : st(s), name(n) {
    if (stage_timing_enabled()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~StageTimer() {
    if (a) {
      cudaEventRecord(b, st);
      stage_record(name, a, b);
    }
  }
};

// ----------------------------------------------------------- bit helpers
__device__ __forceinline__ int popc64(u64 v) { return __popcll(v); }

// Per-word contribution to the product phase exponent of a*b
// (reference strings.py:32-44):
//   popc(ax&az) + popc(bx&bz) + 2 popc(az&bx) - popc((ax^bx)&(az^bz)).
__device__ __forceinline__ int phase_word(u64 ax, u64 az, u64 bx, u64 bz) {
  return popc64(ax & az) + popc64(bx & bz) + 2 * popc64(az & bx) -
         popc64((ax ^ bx) & (az ^ bz));
}

// Symplectic inner product contribution of one word pair (strings.py:47-51);
// the parity of the sum over words is 1 when the strings anti-commute.
__device__ __forceinline__ u64 sip_word(u64 ax, u64 az, u64 bx, u64 bz) {
  return (ax & bz) ^ (az & bx);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline bool valid_words(int W) { return W == 1 || W == 2 || W == 4 || W == 8 || W == 16; }

// Dispatch a templated launcher on the word count W.
#define PLB_DISPATCH_W(W, FN, ...)                         \
  [&]() -> int {                                           \
    switch (W) {                                           \
      case 1: return FN<1>(__VA_ARGS__);                   \
      case 2: return FN<2>(__VA_ARGS__);                   \
      case 4: return FN<4>(__VA_ARGS__);                   \
      case 8: return FN<8>(__VA_ARGS__);                   \
      case 16: return FN<16>(__VA_ARGS__);                 \
      default:                                             \
        ::plb::set_error("unsupported word count W=%d", W); \
        return PL_ERR_TIER;                                \
    }                                                      \
  }()

}  // namespace plb
