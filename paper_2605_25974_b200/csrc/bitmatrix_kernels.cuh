// Bitmatrix kernels shared by bitmatrix.cu (K5) and grouping.cu (K6 uses
// the row-list kernel for its intra-batch anti-commutation rows).  See
// bitmatrix.cu for the method description.
#pragma once
#include "common.cuh"

namespace plb {

constexpr int kColsPerCta = 1024;  // 32 groups x 32 columns
constexpr int kTPad = 1;           // row pad of T (conflict-free lane reads)

// ---------------------------------------------------------------- CSR lists
template <int W>
__global__ void k_row_weight(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld,
                             int64_t row0, int64_t rows, uint32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = row0 + i;
  int c = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) c += popc64(__ldg(x + w * ld + r)) + popc64(__ldg(z + w * ld + r));
  cnt[i] = (uint32_t)c;
}

template <int W>
__global__ void k_row_fill(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld,
                           int64_t row0, int64_t rows, const uint32_t* __restrict__ off,
                           uint16_t* __restrict__ list) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = row0 + i;
  uint32_t o = off[i];
#pragma unroll
  for (int u = 0; u < 2 * W; ++u) {
    u64 v = u < W ? __ldg(x + u * ld + r) : __ldg(z + (u - W) * ld + r);
    while (v) {
      const int b = __ffsll((long long)v) - 1;
      v &= v - 1;
      list[o++] = (uint16_t)(u * 64 + b);
    }
  }
}

// --------------------------------------------------------- method 1 kernel
template <int W>
__global__ void __launch_bounds__(1024, 1)
k_bitmatrix_lists(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
                  int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                  const uint32_t* __restrict__ off, const uint16_t* __restrict__ list,
                  uint32_t* __restrict__ bits, int64_t ld_bits, int64_t rows_per_split) {
  constexpr int E = 128 * W;  // key bits per term
  constexpr int TS = E + kTPad;
  extern __shared__ uint32_t T[];  // [32][TS]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = col0 + (int64_t)blockIdx.x * kColsPerCta;

  // ---- transpose this CTA's 1024 columns into T (warp g -> group g)
  {
    const int g = warp;
    const int64_t c = c0 + 32 * g + lane;
    const bool valid = c < col0 + cols && c < M;
#pragma unroll 1
    for (int u = 0; u < 2 * W; ++u) {
      const u64 v = valid ? (u < W ? __ldg(z + u * ld + c) : __ldg(x + (u - W) * ld + c)) : 0ull;
      uint32_t mlo = 0, mhi = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const uint32_t m = __ballot_sync(0xffffffffu, (uint32_t)(v >> b) & 1u);
        if (lane == b) mlo = m;
      }
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const uint32_t m = __ballot_sync(0xffffffffu, (uint32_t)(v >> (32 + b)) & 1u);
        if (lane == b) mhi = m;
      }
      T[g * TS + u * 64 + lane] = mlo;
      T[g * TS + u * 64 + 32 + lane] = mhi;
    }
    if (lane == 0) T[g * TS + E] = 0;  // sentinel slice (all zero)
  }
  __syncthreads();

  const int64_t words_here = ceil_div(cols - (c0 - col0) < kColsPerCta ? cols - (c0 - col0)
                                                                       : kColsPerCta, 32);
  const int64_t wcol = (c0 - col0) / 32;
  const uint32_t* Tl = T + lane * TS;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_split;
  int64_t r_end = r_begin + rows_per_split;
  if (r_end > rows) r_end = rows;

  for (int64_t i = r_begin + warp; i < r_end; i += 32) {
    const uint32_t o = off[i], cnt = off[i + 1] - o;
    uint32_t acc = 0;
    for (uint32_t base = 0; base < cnt; base += 32) {
      const uint32_t e_l = base + lane < cnt ? (uint32_t)list[o + base + lane] : (uint32_t)E;
      const uint32_t n = cnt - base < 32 ? cnt - base : 32;
      uint32_t k = 0;
      for (; k + 4 <= n; k += 4) {
        const uint32_t e0 = __shfl_sync(0xffffffffu, e_l, k);
        const uint32_t e1 = __shfl_sync(0xffffffffu, e_l, k + 1);
        const uint32_t e2 = __shfl_sync(0xffffffffu, e_l, k + 2);
        const uint32_t e3 = __shfl_sync(0xffffffffu, e_l, k + 3);
        acc ^= Tl[e0] ^ Tl[e1];
        acc ^= Tl[e2] ^ Tl[e3];
      }
      for (; k < n; ++k) acc ^= Tl[__shfl_sync(0xffffffffu, e_l, k)];
    }
    if (lane < words_here) bits[i * ld_bits + wcol + lane] = acc;
  }
}

// --------------------------------------------------------- method 2 kernel
constexpr int kDirectRows = 256;  // one row per thread
template <int W> struct DirectCols { static constexpr int value = W >= 16 ? 128 : 256; };

template <int W>
__global__ void __launch_bounds__(kDirectRows)
k_bitmatrix_direct(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
                   int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                   uint32_t* __restrict__ bits, int64_t ld_bits) {
  constexpr int kDirectCols = DirectCols<W>::value;  // columns staged per CTA
  __shared__ u64 sx[W][kDirectCols], sz[W][kDirectCols];
  const int64_t cb = col0 + (int64_t)blockIdx.x * kDirectCols;
  for (int t = threadIdx.x; t < W * kDirectCols; t += blockDim.x) {
    const int w = t / kDirectCols, j = t % kDirectCols;
    const int64_t c = cb + j;
    const bool ok = c < col0 + cols && c < M;
    sx[w][j] = ok ? __ldg(x + w * ld + c) : 0ull;
    sz[w][j] = ok ? __ldg(z + w * ld + c) : 0ull;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.y * kDirectRows + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = row0 + i;
  u64 rx[W], rz[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    rx[w] = __ldg(x + w * ld + r);
    rz[w] = __ldg(z + w * ld + r);
  }
  const int64_t remaining = cols - (cb - col0);
  const int nwords = (int)ceil_div(remaining < kDirectCols ? remaining : kDirectCols, 32);
  uint32_t* out = bits + i * ld_bits + (cb - col0) / 32;
  for (int q = 0; q < nwords; ++q) {
    uint32_t word = 0;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
      const int j = q * 32 + t;
      u64 acc = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) acc ^= (rx[w] & sz[w][j]) ^ (rz[w] & sx[w][j]);
      const uint32_t p = __popc((uint32_t)acc ^ (uint32_t)(acc >> 32)) & 1u;
      word |= p << t;
    }
    out[q] = word;
  }
}

}  // namespace plb
