// Multi-block exclusive scan of uint32 counts (3 phases: block sums, scan of
// block sums, block-local scan + offset).  Used to build CSR offsets.
#pragma once
#include "common.cuh"

namespace plb {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;                       // per thread
constexpr int kScanTile = kScanThreads * kScanItems;  // per block

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan; returns the thread's exclusive prefix and the
// block total via *total.  blockDim.x must be a multiple of 32, <= 1024.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? warp_sums[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < nw) warp_sums[lane] = s;
  }
  __syncthreads();
  const uint32_t before = wid ? warp_sums[wid - 1] : 0;
  if (total) *total = warp_sums[nw - 1];
  __syncthreads();
  return before + inc - v;
}

static __global__ void k_scan_block_sums(const uint32_t* __restrict__ in, int64_t n,
                                  uint32_t* __restrict__ block_sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  uint32_t tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of nb block sums in place; total -> *total.
static __global__ void k_scan_partials(uint32_t* __restrict__ sums, int64_t nb, uint32_t* total) {
  uint32_t carry = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? sums[i] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// out[i] = exclusive prefix of in[i]; in and out may alias.
static __global__ void k_scan_apply(const uint32_t* in, int64_t n, const uint32_t* __restrict__ block_off,
                             uint32_t* out) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  uint32_t ex = block_excl_scan(s, nullptr) + block_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
}

inline int64_t scan_scratch_words(int64_t n) { return ceil_div(n > 0 ? n : 1, kScanTile) + 1; }

// Exclusive scan of n uint32 values (in place allowed); the grand total is
// written to *total (device).  scratch holds scan_scratch_words(n) words.
inline int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* scratch,
                              uint32_t* total, cudaStream_t st) {
  const int64_t nb = ceil_div(n > 0 ? n : 1, kScanTile);
  k_scan_block_sums<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, scratch);
  k_scan_partials<<<1, 1024, 0, st>>>(scratch, nb, total);
  k_scan_apply<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, scratch, out);
  PLB_CHECK_LAUNCH("exclusive_scan_u32");
  return PL_OK;
}

}  // namespace plb
