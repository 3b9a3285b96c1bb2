// K5 method 3: the commutation bitmatrix on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8, accumulators in TMEM).
//
//   sip(r, c) = (popc(x_r & z_c) + popc(z_r & x_c)) & 1      (strings.py:47-51)
//             = (A_r . B_c) & 1,  A_r = [x_r | z_r], B_c = [z_c | x_c]
//
// as 0/1 bytes, K = 128 W (grouping.py:136-140's all-pairs block as an int8
// GEMM; 2K = 256 W ops per check).  A CTA (4 warps) owns 128 rows: their
// expanded A operand (128 x K bytes) stays in shared memory; the columns
// stream through in N-tiles of 256, each tile's B operand expanded chunk by
// chunk (KC bytes of K) into a double buffer while the previous chunk's MMAs
// run; thread 0 issues the MMAs (M=128, N=256, K=32 each) and commits them to
// an mbarrier per buffer.  The epilogue reads each row's 256 int32 dot
// products from TMEM (tcgen05.ld 32x32b), keeps bit 0 and packs 32 checks per
// word.  Operands use the K-major no-swizzle core-matrix layout (8 rows x 16
// bytes per 128-byte core matrix).  The bit -> byte expansion order is the
// same for A and B, so the dot products are exact.
#pragma once

namespace plb {

constexpr int kTcRows = 128;   // UMMA M
constexpr int kTcN = 256;      // UMMA N (columns per tile)
constexpr int kTcKC = 128;     // B chunk: bytes of K per buffer
constexpr int kTcCols = 4096;  // columns per CTA

__device__ __forceinline__ uint32_t tc_saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t addr, uint32_t sbo) {
  // start >> 4 | LBO = 128 B (K-adjacent core matrices) | SBO (8-row groups) | version 1
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// 16 bits -> 16 bytes of 0/1 (byte i = bit i)
__device__ __forceinline__ uint4 tc_expand16(uint32_t v) {
  auto e8 = [](uint32_t b) -> unsigned long long {
    unsigned long long x = (unsigned long long)(b & 0xFF) * 0x0101010101010101ull;
    x &= 0x8040201008040201ull;
    x = (x + 0x7F7F7F7F7F7F7F7Full) & 0x8080808080808080ull;
    return x >> 7;
  };
  const unsigned long long lo = e8(v), hi = e8(v >> 8);
  return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
}

template <int W>
struct TcSmem {
  static constexpr int K = 128 * W;                 // bytes per operand row
  static constexpr uint32_t SBO_A = (K / 16) * 128;  // A: 8-row group stride
  static constexpr uint32_t SBO_B = (kTcKC / 16) * 128;
  static constexpr size_t A_BYTES = (size_t)kTcRows * K;
  static constexpr size_t B_BYTES = (size_t)kTcN * kTcKC;
  static constexpr size_t BYTES = A_BYTES + 2 * B_BYTES + 1024;  // + alignment slack
};

__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tTC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TC_WAIT_%=;\n\t}\n" ::"r"(tc_saddr(bar)),
      "r"(phase)
      : "memory");
}

// operand word (plane p of x/z) of term t: x for p < W, z for p >= W (A: [x|z]);
// B swaps the halves ([z|x])
template <int W>
__device__ __forceinline__ u64 tc_word(const u64* x, const u64* z, int64_t ld, int64_t t, int p,
                                       bool swap) {
  const bool use_x = (p < W) != swap;
  const int w = p < W ? p : p - W;
  return __ldg((use_x ? x : z) + (int64_t)w * ld + t);
}

constexpr int kTcThreads = 256;

template <int W>
__global__ void __launch_bounds__(kTcThreads, 1)
k_bitmatrix_tc(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
               int64_t row0, int64_t rows, int64_t col0, int64_t cols,
               uint32_t* __restrict__ bits, int64_t ld_bits) {
  using S = TcSmem<W>;
  constexpr int K = S::K;
  constexpr int NCH = K / kTcKC;  // B chunks per tile
  extern __shared__ uint8_t tc_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB[2] = {smem + S::A_BYTES, smem + S::A_BYTES + S::B_BYTES};
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rb = (int64_t)blockIdx.y * kTcRows;        // first row of the block (in the row range)
  const int64_t cbeg = (int64_t)blockIdx.x * kTcCols;      // first column (relative to col0)
  if (cbeg >= cols) return;
  const int64_t cend = min(cols, cbeg + kTcCols);
  const int ntiles = (int)ceil_div(cend - cbeg, kTcN);
  const int G = ntiles * NCH;

  // A: row r, K-segment s (16 bits of operand plane s / 4): one word per
  // (row, plane) loaded once and expanded into its 4 segments
  for (int e = tid; e < kTcRows * 2 * W; e += blockDim.x) {
    const int r = e % kTcRows, p = e / kTcRows;
    const int64_t i = rb + r;
    const u64 v = i < rows ? tc_word<W>(x, z, ld, row0 + i, p, false) : 0ull;
    uint8_t* dst = sA + (r >> 3) * S::SBO_A + (r & 7) * 16 + 4 * p * 128;
#pragma unroll
    for (int h = 0; h < 4; ++h)
      *reinterpret_cast<uint4*>(dst + h * 128) = tc_expand16((uint32_t)(v >> (16 * h)) & 0xFFFF);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_saddr(&bar[1])));
  }
  if (warp == 0) {  // two accumulators (tiles alternate): 2 x 256 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc_saddr(&tbase)),
                 "r"(2 * kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B chunk g (tile g / NCH, K range (g % NCH) * KC ..) into buffer g & 1:
  // work item e = (column j, operand plane of the chunk) -> one word, 4
  // segments.  The words are fetched one iteration before they are expanded
  // (software pipelining hides the L2 latency behind a chunk of MMAs).
  constexpr int kItems = kTcN * (kTcKC / 64) / kTcThreads;
  static_assert(kItems * kTcThreads == kTcN * (kTcKC / 64), "chunk work items");
  auto fetch_chunk = [&](int g, u64 (&v)[kItems]) {
    const int64_t c0 = cbeg + (int64_t)(g / NCH) * kTcN;
    const int q = g % NCH;
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int e = tid + u * kTcThreads;
      const int j = e % kTcN, pw = e / kTcN;  // consecutive threads: consecutive columns
      const int64_t c = c0 + j;
      v[u] = c < cend ? tc_word<W>(x, z, ld, col0 + c, q * (kTcKC / 64) + pw, true) : 0ull;
    }
  };
  auto store_chunk = [&](int g, const u64 (&v)[kItems]) {
    uint8_t* buf = sB[g & 1];
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int e = tid + u * kTcThreads;
      const int j = e % kTcN, pw = e / kTcN;
      uint8_t* dst = buf + (j >> 3) * S::SBO_B + (j & 7) * 16 + 4 * pw * 128;
#pragma unroll
      for (int h = 0; h < 4; ++h)
        *reinterpret_cast<uint4*>(dst + h * 128) = tc_expand16((uint32_t)(v[u] >> (16 * h)) & 0xFFFF);
    }
  };
  u64 pre[kItems];
  constexpr uint32_t idesc = (2u << 4) | ((uint32_t)(kTcN >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
  uint32_t waits[2] = {0u, 0u};  // commits consumed per barrier (its phase parity)
  fetch_chunk(0, pre);
  store_chunk(0, pre);
  if (G > 1) fetch_chunk(1, pre);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;

  // epilogue of tile t: warps 0-3 take columns 0-127, warps 4-7 columns 128-255
  // of their TMEM lane quarter (rows 32 (warp % 4) ..)
  auto epilogue = [&](int t) {
    const int64_t c0 = cbeg + (int64_t)t * kTcN;
    const int64_t i = rb + 32 * (warp & 3) + lane;
    const int half = warp >> 2;
    for (int cc = half * (kTcN / 2); cc < (half + 1) * (kTcN / 2); cc += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (t & 1) * kTcN + cc;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) word |= (v[b] & 1u) << b;
      const int64_t cw = c0 + cc;
      if (i < rows && cw < cend) bits[i * ld_bits + cw / 32] = word;
    }
  };

  for (int g = 0; g < G; ++g) {
    const int b = g & 1, t = g / NCH, q = g % NCH;
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dcol = tmem + (t & 1) * kTcN;
#pragma unroll
      for (int s = 0; s < kTcKC / 32; ++s) {
        const uint64_t ad = tc_desc(tc_saddr(sA) + (q * (kTcKC / 16) + 2 * s) * 128, S::SBO_A);
        const uint64_t bd = tc_desc(tc_saddr(sB[b]) + 2 * s * 128, S::SBO_B);
        const uint32_t acc = (q > 0 || s > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dcol),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              tc_saddr(&bar[b]))
          : "memory");
    }
    if (g >= 1) {
      // chunk g-1 complete: its buffer is free and, if it ended a tile, that
      // tile's dot products are final (MMAs complete in issue order)
      tc_mbar_wait(&bar[b ^ 1], waits[b ^ 1] & 1u);
      ++waits[b ^ 1];
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (q == 0) epilogue(t - 1);  // overlaps the MMAs of chunk g (other accumulator)
    }
    if (g + 1 < G) {
      store_chunk(g + 1, pre);
      if (g + 2 < G) fetch_chunk(g + 2, pre);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  tc_mbar_wait(&bar[(G - 1) & 1], waits[(G - 1) & 1] & 1u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  epilogue(G / NCH - 1);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kTcN));
}

}  // namespace plb
