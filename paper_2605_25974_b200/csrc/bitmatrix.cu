// K5 — all-pairs commutation bitmatrix (restates grouping.py:136-140, the
// parity popc(x_r & z_c) + popc(z_r & x_c) of strings.py:47-51).
//
// Method 1 (row-list XOR over transposed column slices).  A CTA owns a block
// of 1024 columns and transposes it in shared memory into bit slices
//   T[g][e]  (g = 32-column group, e = key bit),  bit t of T[g][e] = bit e of
//   column c0 + 32g + t,  where e = 64u + b addresses z-word u (u < W) or
//   x-word u - W (u >= W) of the column.
// A row r anti-commutes with column c iff the XOR over the row's set bits of
// the swapped partner slice is 1:   sip(r, c) = XOR_{b in x_r} z_c[b] ^
// XOR_{b in z_r} x_c[b].  Each warp takes one row (its set-bit list is warp
// uniform, so there is no divergence) and every lane produces 32 column bits
// with one LDS + one XOR per set bit: cost per 1024 checks is proportional to
// the row weight, which makes sparse Hamiltonians (config 5, weight 2-12)
// bound by the 1-bit-per-check output stream instead of the INT pipe.
//
// Method 2 (direct).  One thread per row, the row's 2W words in registers,
// columns broadcast from shared memory: 4W LOP3 + POPC per check.  Used for
// dense rows and W = 16 (whose slices exceed shared memory).
#include "common.cuh"
#include "scan.cuh"

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

// ------------------------------------------------------------- launchers
static inline int64_t list_capacity_entries(int64_t rows) { return rows * 64; }

template <int W>
static int launch_bitmatrix(int64_t M, const u64* x, const u64* z, int64_t ld, int64_t row0,
                            int64_t rows, int64_t col0, int64_t cols, uint32_t* bits,
                            int64_t ld_bits, int method, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (W == 16 && method == 1) {
    set_error("bitmatrix method 1 supports W <= 8");
    return PL_ERR_ARG;
  }
  if (method != 2 && W <= 8) {
    // CSR row lists: off (rows+1) u32 | scan scratch | list u16
    const int64_t need_min = (rows + 1) * 4 + scan_scratch_words(rows) * 4 + 16;
    if (ws == nullptr || (int64_t)ws_bytes < need_min) {
      if (method == 1) {
        set_error("bitmatrix: workspace too small (%lld < %lld)", (long long)ws_bytes,
                  (long long)need_min);
        return PL_ERR_WORKSPACE;
      }
      method = 2;
    }
  }
  if constexpr (W <= 8) if (method != 2) {
    uint8_t* p = (uint8_t*)ws;
    uint32_t* off = (uint32_t*)p;
    p += (rows + 1) * 4;
    uint32_t* scratch = (uint32_t*)p;
    p += scan_scratch_words(rows) * 4;
    p = (uint8_t*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    uint16_t* list = (uint16_t*)p;
    const int64_t cap = ((int64_t)ws_bytes - (p - (uint8_t*)ws)) / 2;
    const unsigned nb = (unsigned)ceil_div(rows, 256);
    k_row_weight<W><<<nb, 256, 0, st>>>(x, z, ld, row0, rows, off);
    PLB_CHECK_LAUNCH("k_row_weight");
    int rc = exclusive_scan_u32(off, off, rows, scratch, off + rows, st);
    if (rc) return rc;
    uint32_t total = 0;
    PLB_CUDA(cudaMemcpyAsync(&total, off + rows, 4, cudaMemcpyDeviceToHost, st));
    PLB_CUDA(cudaStreamSynchronize(st));
    const double avg = rows ? (double)total / (double)rows : 0.0;
    // method 1 costs ~1 LDS per set bit per 32 checks; method 2 ~4W LOP3 per check
    const bool dense = avg > 48.0 * W;
    if ((int64_t)total > cap || (method == 0 && dense)) {
      if (method == 1) {
        set_error("bitmatrix: list workspace too small (%u entries > %lld)", total,
                  (long long)cap);
        return PL_ERR_WORKSPACE;
      }
      method = 2;
    } else {
      k_row_fill<W><<<nb, 256, 0, st>>>(x, z, ld, row0, rows, off, list);
      PLB_CHECK_LAUNCH("k_row_fill");
      const int64_t colblocks = ceil_div(cols, kColsPerCta);
      int64_t splits = ceil_div(2 * num_sms(), colblocks);
      const int64_t max_splits = ceil_div(rows, 256);
      if (splits > max_splits) splits = max_splits;
      if (splits < 1) splits = 1;
      if (splits > 65535) splits = 65535;
      const int64_t rps = ceil_div(rows, splits);
      const size_t smem = (size_t)32 * (128 * W + kTPad) * 4;
      auto kern = k_bitmatrix_lists<W>;
      PLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int64_t cbase = 0; cbase < colblocks; cbase += 65535) {
        const int64_t nblk = colblocks - cbase < 65535 ? colblocks - cbase : 65535;
        dim3 grid((unsigned)nblk, (unsigned)splits);
        StageTimer t_(st, "k_bitmatrix_lists");
        kern<<<grid, 1024, smem, st>>>(x, z, ld, M, row0, rows, col0 + cbase * kColsPerCta,
                                       cols - cbase * kColsPerCta, off, list,
                                       bits + cbase * (kColsPerCta / 32), ld_bits, rps);
        PLB_CHECK_LAUNCH("k_bitmatrix_lists");
      }
      return PL_OK;
    }
  }
  // method 2
  constexpr int kDirectCols = DirectCols<W>::value;
  const int64_t colblocks = ceil_div(cols, kDirectCols);
  const int64_t rowblocks = ceil_div(rows, kDirectRows);
  for (int64_t rb = 0; rb < rowblocks; rb += 65535) {
    const int64_t nrb = rowblocks - rb < 65535 ? rowblocks - rb : 65535;
    dim3 grid((unsigned)colblocks, (unsigned)nrb);
    StageTimer t_(st, "k_bitmatrix_direct");
    k_bitmatrix_direct<W><<<grid, kDirectRows, 0, st>>>(
        x, z, ld, M, row0 + rb * kDirectRows, rows - rb * kDirectRows, col0, cols,
        bits + rb * kDirectRows * ld_bits, ld_bits);
    PLB_CHECK_LAUNCH("k_bitmatrix_direct");
  }
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int64_t pl_bitmatrix_workspace_bytes(int W, int64_t rows) {
  (void)W;
  if (rows < 0) return 0;
  return (rows + 1) * 4 + scan_scratch_words(rows) * 4 + 16 + list_capacity_entries(rows) * 2;
}

extern "C" int pl_commutation_bitmatrix(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                                        int64_t ld, int64_t row0, int64_t rows, int64_t col0,
                                        int64_t cols, uint32_t* bits, int64_t ld_bits, int method,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (M < 0 || ld < M || row0 < 0 || rows < 0 || row0 + rows > M || col0 < 0 || cols < 0 ||
      col0 + cols > M || (col0 % 32) != 0 || ld_bits < ceil_div(cols, 32) || method < 0 ||
      method > 2) {
    set_error("pl_commutation_bitmatrix: bad arguments");
    return PL_ERR_ARG;
  }
  if (rows * 128LL * (W > 0 ? W : 1) >= 0xFFFFFFFFLL) {
    set_error("pl_commutation_bitmatrix: too many rows per call (split the row range)");
    return PL_ERR_CAPACITY;
  }
  if (rows == 0 || cols == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_bitmatrix, M, (const u64*)x, (const u64*)z, ld, row0, rows,
                        col0, cols, bits, ld_bits, method, workspace, workspace_bytes,
                        (cudaStream_t)stream);
}
