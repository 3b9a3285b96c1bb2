// Bitmatrix kernels shared by bitmatrix.cu (K5) and grouping.cu (K6 uses
// the generic row-list kernel for its intra-batch anti-commutation rows).
// See bitmatrix.cu for the method description.
#pragma once
#include "common.cuh"

namespace plb {

constexpr int kColsPerCta = 1024;  // 32 groups x 32 columns
constexpr int kTPad = 1;           // row pad of T (conflict-free lane reads)
constexpr int kEBuf = 1024;        // per-warp staged entries of 32 rows (uint16)

// ---------------------------------------------------------------- CSR lists
// FMT 0 (grouping): uint16 entry e = 64u + b for set bit b of canonical word
// u (u < W: x word u, u >= W: z word u - W).  FMT 2 (bitmatrix letter
// kernel): one uint32 entry per letter, the byte offset of its slice row (z,
// x or z^x slice of the qubit), every row padded to a multiple of 4 entries
// with the all-zero sentinel slice 192W.
template <int W, int FMT = 0>
__global__ void k_row_weight(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld,
                             int64_t row0, int64_t rows, uint32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = row0 + i;
  int c = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const u64 xv = __ldg(x + w * ld + r), zv = __ldg(z + w * ld + r);
    c += FMT == 2 ? popc64(xv | zv) : popc64(xv) + popc64(zv);  // FMT 2: one entry per letter
  }
  cnt[i] = FMT == 2 ? (uint32_t)((c + 3) & ~3) : (uint32_t)c;
}

template <int W, int FMT = 0>
__global__ void k_row_fill(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld,
                           int64_t row0, int64_t rows, const uint32_t* __restrict__ off,
                           void* __restrict__ list_) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = row0 + i;
  uint32_t o = off[i];
  uint16_t* l16 = reinterpret_cast<uint16_t*>(list_);
  uint32_t* l32 = reinterpret_cast<uint32_t*>(list_);
  if (FMT == 2) {
    // one entry per letter, byte offsets of 128-byte slice rows: X at q -> z
    // slice q, Z -> x slice 64W + q, Y -> (z ^ x) slice 128W + q
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 xv = __ldg(x + w * ld + r), zv = __ldg(z + w * ld + r);
      const u64 cls[3] = {xv & ~zv, zv & ~xv, xv & zv};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        u64 v = cls[k];
        while (v) {
          const int b = __ffsll((long long)v) - 1;
          v &= v - 1;
          l32[o++] = 128u * (uint32_t)(k * 64 * W + w * 64 + b);
        }
      }
    }
    const uint32_t end = off[i + 1];
    while (o < end) l32[o++] = 128u * (uint32_t)(192 * W);
    return;
  }
#pragma unroll
  for (int u = 0; u < 2 * W; ++u) {
    u64 v = u < W ? __ldg(x + u * ld + r) : __ldg(z + (u - W) * ld + r);
    while (v) {
      const int b = __ffsll((long long)v) - 1;
      v &= v - 1;
      l16[o++] = (uint16_t)(u * 64 + b);
    }
  }
}

// ---- transpose 1024 columns into T (warp g -> 32-column group g)
template <int W>
__device__ __forceinline__ void build_slices(uint32_t* T, const u64* __restrict__ x,
                                             const u64* __restrict__ z, int64_t ld, int64_t M,
                                             int64_t c0, int64_t cend) {
  constexpr int E = 128 * W;
  constexpr int TS = E + kTPad;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t c = c0 + 32 * g + lane;
  const bool valid = c < cend && c < M;
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

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ unsigned long long lds64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

// --------------------------------------------- method 1, generic lists
template <int W>
__device__ __forceinline__ void bitmatrix_lists_body(
    const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M, int64_t row0,
    int64_t rows, int64_t col0, int64_t cols, const uint32_t* __restrict__ off,
    const uint16_t* __restrict__ list, uint32_t* __restrict__ bits, int64_t ld_bits,
    int64_t rows_per_split) {
  constexpr int E = 128 * W;
  constexpr int TS = E + kTPad;
  extern __shared__ uint32_t T[];  // [32][TS]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = col0 + (int64_t)blockIdx.x * kColsPerCta;
  build_slices<W>(T, x, z, ld, M, c0, col0 + cols);
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
      for (uint32_t k = 0; k < n; ++k) acc ^= Tl[__shfl_sync(0xffffffffu, e_l, k)];
    }
    if (lane < words_here) bits[i * ld_bits + wcol + lane] = acc;
  }
}

template <int W>
__global__ void __launch_bounds__(1024, 1)
k_bitmatrix_lists(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
                  int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                  const uint32_t* __restrict__ off, const uint16_t* __restrict__ list,
                  uint32_t* __restrict__ bits, int64_t ld_bits, int64_t rows_per_split) {
  bitmatrix_lists_body<W>(x, z, ld, M, row0, rows, col0, cols, off, list, bits, ld_bits,
                          rows_per_split);
}

// ------------------- method 1, letter slices (fast path)
// Per CTA 1024 columns; slices are stored entry-major as TY[e][h] (uint64, h =
// 16 groups of 64 columns) for three entry kinds per qubit q: the z slice (a
// row letter X at q), the x slice (Z) and their XOR (Y), so a row costs one
// 64-bit shared load per letter instead of one per set bit.  Each warp stages
// the entries of blocks of 16 rows and processes two rows per pass (half-warp
// per row, each lane producing 64 column bits).
constexpr int kColsY = 1024;
constexpr int kRowsY = 16;     // rows staged per warp block
constexpr int kEBufY = 240;    // staged entries per warp (<= 15 letters per row on average)

template <int W>
__global__ void __launch_bounds__(1024, 1)
k_bitmatrix_letters(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
                    int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                    const uint32_t* __restrict__ off, const uint32_t* __restrict__ list,
                    uint32_t* __restrict__ bits, int64_t ld_bits, int64_t rows_per_split) {
  constexpr int E = 192 * W;  // slices: z (64W) | x (64W) | z^x (64W), + sentinel
  extern __shared__ __align__(16) uint32_t TY32[];  // [E+1][16] u64 | ebuf [32][kEBufY] u32
  u64* TY = reinterpret_cast<u64*>(TY32);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = col0 + (int64_t)blockIdx.x * kColsY;
  {  // transpose: warp g ballots columns c0+32g.. -> h = g/2, 32-bit half g&1
    const int64_t c = c0 + 32 * warp + lane;
    const bool valid = c < col0 + cols && c < M;
    const int h = warp >> 1, part = warp & 1;
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
      TY32[((u * 64 + lane) * 16 + h) * 2 + part] = mlo;
      TY32[((u * 64 + 32 + lane) * 16 + h) * 2 + part] = mhi;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 64 * W * 16; t += blockDim.x) {  // Y slices
    const int q = t >> 4, h = t & 15;
    TY[(128 * W + q) * 16 + h] = TY[q * 16 + h] ^ TY[(64 * W + q) * 16 + h];
  }
  if (threadIdx.x < 16) TY[E * 16 + threadIdx.x] = 0ull;  // sentinel slice
  __syncthreads();
  const int words_here = (int)ceil_div(cols - (c0 - col0) < kColsY ? cols - (c0 - col0) : kColsY,
                                       32);
  const int64_t wcol = (c0 - col0) / 32;
  const int half = lane >> 4, hl = lane & 15;
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(TY) + (uint32_t)(hl * 8);
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_split;
  int64_t r_end = r_begin + rows_per_split;
  if (r_end > rows) r_end = rows;
  constexpr int kTBytes = (((E + 1) * 16 * 8 + 15) / 16) * 16;
  uint32_t* ebuf = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(TY32) + kTBytes) +
                   warp * kEBufY;
  const uint32_t ebuf_s = (uint32_t)__cvta_generic_to_shared(ebuf);
  const bool w0 = 2 * hl < words_here, w1 = 2 * hl + 1 < words_here;
  const int64_t nblk = ceil_div(r_end - r_begin, kRowsY);
  // Software pipeline over this warp's row blocks (blk, blk+32, ...): the
  // offsets of block i+2 and the entries of block i+1 are loaded into
  // registers while block i is computed from the staged entries.
  constexpr int kEVec = kEBufY / 4 / 32 + 1;  // uint4 entry vectors per lane (>= kEBufY/4/32)
  auto load_off = [&](int64_t blk) -> uint32_t {
    if (blk >= nblk) return 0u;
    const int64_t rb = r_begin + blk * kRowsY;
    const int nr = (int)(r_end - rb < kRowsY ? r_end - rb : kRowsY);
    return lane <= nr ? __ldg(off + rb + lane) : 0u;  // lane nr holds the block end
  };
  auto block_nr = [&](int64_t blk) -> int {
    const int64_t rb = r_begin + blk * kRowsY;
    return (int)(r_end - rb < kRowsY ? r_end - rb : kRowsY);
  };
  auto load_entries = [&](int64_t blk, uint32_t offv, uint4 (&ev)[kEVec]) {
    if (blk >= nblk) return;
    const int nr = block_nr(blk);
    const uint32_t o_first = __shfl_sync(0xffffffffu, offv, 0);
    const uint32_t total = __shfl_sync(0xffffffffu, offv, nr) - o_first;
    if (total > (uint32_t)kEBufY) return;
    const uint4* srcl = reinterpret_cast<const uint4*>(list + o_first);
#pragma unroll
    for (int v = 0; v < kEVec; ++v) {
      const uint32_t k = lane + 32 * v;
      if (k < total / 4) ev[v] = __ldg(srcl + k);
    }
  };
  uint32_t off_cur = load_off(warp);
  uint32_t off_nxt = load_off(warp + 32);
  uint4 ev[kEVec];
  load_entries(warp, off_cur, ev);
  for (int64_t blk = warp; blk < nblk; blk += 32) {
    const int64_t rb = r_begin + blk * kRowsY;
    const int nr = block_nr(blk);
    const uint32_t my_off = off_cur;
    const uint32_t o_first = __shfl_sync(0xffffffffu, my_off, 0);
    const uint32_t o_end = __shfl_sync(0xffffffffu, my_off, nr);
    const uint32_t total = o_end - o_first;  // multiple of 4
    const bool staged = total <= (uint32_t)kEBufY;
    if (staged) {
      uint4* dst = reinterpret_cast<uint4*>(ebuf);
#pragma unroll
      for (int v = 0; v < kEVec; ++v) {
        const uint32_t k = lane + 32 * v;
        if (k < total / 4) dst[k] = ev[v];
      }
      __syncwarp();
    }
    // prefetch: offsets two blocks ahead, entries of the next block
    const uint32_t off_nn = load_off(blk + 64);
    load_entries(blk + 32, off_nxt, ev);
    for (int j = 0; j < nr; j += 2) {
      const int jr = j + half;  // this half-warp's row
      const uint32_t a = __shfl_sync(0xffffffffu, my_off, jr & 31);
      const uint32_t bnx = __shfl_sync(0xffffffffu, my_off, (jr + 1) & 31);
      const bool live = jr < nr;
      const uint32_t beg = live ? a - o_first : 0u;
      const uint32_t end = live ? bnx - o_first : 0u;
      unsigned long long acc = 0;
      if (staged) {
        uint4 e = make_uint4(0, 0, 0, 0);
        if (beg < end)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                       : "r"(ebuf_s + 4 * beg));
        unsigned long long acc1 = 0;
        for (uint32_t k = beg; k < end; k += 4) {
          uint4 en = e;
          if (k + 4 < end)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(en.x), "=r"(en.y), "=r"(en.z), "=r"(en.w)
                         : "r"(ebuf_s + 4 * (k + 4)));
          const unsigned long long t0 = lds64(tb + e.x), t1 = lds64(tb + e.y);
          const unsigned long long t2 = lds64(tb + e.z), t3 = lds64(tb + e.w);
          acc ^= t0 ^ t1;
          acc1 ^= t2 ^ t3;
          e = en;
        }
        acc ^= acc1;
      } else {
        for (uint32_t k = beg; k < end; ++k) acc ^= lds64(tb + list[o_first + k]);
      }
      if (live) {
        uint32_t* out = bits + (rb + jr) * ld_bits + wcol + 2 * hl;
        if (w0) out[0] = (uint32_t)acc;
        if (w1) out[1] = (uint32_t)(acc >> 32);
      }
    }
    __syncwarp();
    off_cur = off_nxt;
    off_nxt = off_nn;
  }
}

template <int W>
constexpr size_t letters_smem_bytes() {
  return (size_t)((((192 * W + 1) * 16 * 8) + 15) / 16) * 16 + (size_t)32 * kEBufY * 4;
}

// dynamic shared memory of the list kernels
template <int W>
constexpr size_t lists_smem_bytes() {
  return (size_t)32 * (128 * W + kTPad) * 4;
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
