// Leaf stage of the merge pipeline (included by combine_impl.cuh, which
// defines the key helpers, RunSum, Source and keep_sum).
//
//   k_leaf_sort  one CTA per leaf (<= leaf_cap items staged in shared memory):
//                radix sort on a 24-bit key window below the leaf's common
//                prefix, ties finished on the full (key, ik) (bitonic network
//                when a tie segment is long); run heads; each run summed in
//                numpy reduceat order by one thread (RunSum); |sum| <= eps
//                dropped; kept (key, sum) written compacted at the leaf's
//                offset in the idle item buffer + C.sums; kept count per leaf.
//   k_leaf_scan  exclusive scan of the kept counts -> output offset per leaf.
//   k_emit       warp per leaf: unpack each kept key into the 2W plane words
//                and write the SoA output term (planes, phase 0, coefficient).
// Leaves larger than leaf_cap (one key repeated more than leaf_cap times,
// which no splitter can divide) are sorted in place in global memory.
#pragma once

// Shared-memory items per leaf for key width KW (a multiple of the CTA size;
// about 32 KB of shared memory per CTA with the radix scratch -> 7 CTAs/SM).
__host__ __device__ constexpr int leaf_cap_for(int KW) {
  return KW <= 2 ? 768 : KW == 4 ? 384 : KW == 8 ? 256 : 128;
}

__host__ __device__ constexpr size_t leaf_buf_stride(int KW) {
  return ((size_t)leaf_cap_for(KW) * (8 * KW + 4 + 2 + 1) + 15) & ~(size_t)15;
}

constexpr int kLeafThreads2 = 128;
constexpr int kLeafWarps2 = kLeafThreads2 / 32;
constexpr int kRadixBits = 8, kRadixBins = 1 << kRadixBits, kRadixPasses = 3;
constexpr int kRadixWindow = kRadixBits * kRadixPasses;
constexpr int kRadixTieMax = 32;

__host__ __device__ constexpr size_t radix_smem_bytes(int cap) {
  // window keys x2 | perm x2 (u16) | per-warp bin counters (u16)
  return (size_t)cap * 4 * 2 + (size_t)cap * 2 * 2 + (size_t)kLeafWarps2 * kRadixBins * 2 + 16;
}



// Straight-line compare-exchange with a compile-time stride: both items are
// loaded once, compared branch-free and written back only when out of order.
template <int KW, int STRIDE>
__device__ __forceinline__ void cex(u64* __restrict__ K, uint32_t* __restrict__ I, int i, int p) {
  u64 a[KW], b[KW];
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    a[d] = K[d * STRIDE + i];
    b[d] = K[d * STRIDE + p];
  }
  const uint32_t ia = I[i], ib = I[p];
  // b < a ?  (lexicographic over key words, then ik)
  bool lt = ib < ia, eq = true;
#pragma unroll
  for (int d = KW - 1; d >= 0; --d) {
    lt = (b[d] < a[d]) || (b[d] == a[d] && lt);
    (void)eq;
  }
  if (lt) {
#pragma unroll
    for (int d = 0; d < KW; ++d) {
      K[d * STRIDE + i] = b[d];
      K[d * STRIDE + p] = a[d];
    }
    I[i] = ib;
    I[p] = ia;
  }
}

// Fully unrolled bitonic network for NPOW (power of two) slots: every stage's
// partner distance and locality are compile-time constants.
template <int KW, int STRIDE, int NPOW>
__device__ __forceinline__ void bitonic_fixed(u64* K, uint32_t* I, int n) {
  constexpr int HALF = NPOW / 2;
  constexpr int SEG = NPOW / kLeafWarps2;  // elements owned by one warp
  constexpr int PER = HALF / kLeafWarps2;  // pairs per warp in local stages
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool prev_local = false;  // folded to constants: both loops are fully unrolled
#pragma unroll
  for (int k = 2; k <= NPOW; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const bool flip = j == (k >> 1);
      const int xr = flip ? (k - 1) : j;
      const bool local = SEG >= 2 && (flip ? k : 2 * j) <= SEG;
      if (local) {
        if (PER >= 1) {
#pragma unroll
          for (int t0 = 0; t0 < (PER + 31) / 32; ++t0) {
            const int t = warp * PER + t0 * 32 + lane;
            if (t0 * 32 + lane < PER) {
              const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
              const int p = i ^ xr;
              if (p < n) cex<KW, STRIDE>(K, I, i, p);
            }
          }
        }
        __syncwarp();
      } else {
        if (prev_local) __syncthreads();
#pragma unroll
        for (int t0 = 0; t0 < (HALF + kLeafThreads2 - 1) / kLeafThreads2; ++t0) {
          const int t = t0 * kLeafThreads2 + threadIdx.x;
          if (t < HALF) {
            const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
            const int p = i ^ xr;
            if (p < n) cex<KW, STRIDE>(K, I, i, p);
          }
        }
        __syncthreads();
      }
      prev_local = local;
    }
  }
  __syncthreads();
}

// Bitonic sort of n items in shared memory with warp-local stages
// (STRIDE = leaf capacity, a compile-time constant).
template <int KW, int STRIDE>
__device__ __noinline__ void bitonic_sort_local(u64* K, uint32_t* I, int n) {
  int npow = 1;
  while (npow < n) npow <<= 1;
  switch (npow) {
    case 2: bitonic_fixed<KW, STRIDE, 2>(K, I, n); return;
    case 4: bitonic_fixed<KW, STRIDE, 4>(K, I, n); return;
    case 8: bitonic_fixed<KW, STRIDE, 8>(K, I, n); return;
    case 16: bitonic_fixed<KW, STRIDE, 16>(K, I, n); return;
    case 32: bitonic_fixed<KW, STRIDE, 32>(K, I, n); return;
    case 64: bitonic_fixed<KW, STRIDE, 64>(K, I, n); return;
    case 128: bitonic_fixed<KW, STRIDE, 128>(K, I, n); return;
    case 256: if (STRIDE >= 256) { bitonic_fixed<KW, STRIDE, (STRIDE >= 256 ? 256 : 2)>(K, I, n); return; } break;
    case 512: if (STRIDE >= 512) { bitonic_fixed<KW, STRIDE, (STRIDE >= 512 ? 512 : 2)>(K, I, n); return; } break;
    case 1024: if (STRIDE >= 1024) { bitonic_fixed<KW, STRIDE, (STRIDE >= 1024 ? 1024 : 2)>(K, I, n); return; } break;
    default: break;
  }
  const int half = npow >> 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = npow / kLeafWarps2;  // elements owned by one warp
  const int per = half / kLeafWarps2;  // pairs per warp in local stages
  bool prev_local = false;
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const bool flip = j == (k >> 1);
      const int blk = flip ? k : 2 * j;
      const bool local = seg >= 2 && blk <= seg;
      const int xr = flip ? (k - 1) : j;
      if (local) {
        for (int t = warp * per + lane; t < (warp + 1) * per; t += 32) {
          const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
          const int p = i ^ xr;
          if (p < n) cex<KW, STRIDE>(K, I, i, p);
        }
        __syncwarp();
      } else {
        if (prev_local) __syncthreads();
        for (int t = threadIdx.x; t < half; t += kLeafThreads2) {
          const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
          const int p = i ^ xr;
          if (p < n) cex<KW, STRIDE>(K, I, i, p);
        }
        __syncthreads();
      }
      prev_local = local;
    }
  }
  if (prev_local) __syncthreads();
}

// Block-wide exclusive scan of one uint32 per thread (kLeafThreads2 threads).
__device__ __forceinline__ uint32_t leaf_excl_scan(uint32_t v, uint32_t* s_warp,
                                                   uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kLeafWarps2; ++w) {
    const uint32_t s = s_warp[w];
    before += w < wid ? s : 0;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return before + inc - v;
}

// ---------------------------------------------------------------- leaf radix sort
// The items of one leaf lie in a narrow key range, so after the bits they all
// share, a 24-bit window starting at their highest differing bit orders them
// almost completely.  The leaf is sorted by that window with a stable LSD
// radix sort (3 passes of 8 bits, warp multisplit with match.any), then every
// segment of equal windows is finished by an insertion sort on the full
// (key, ik); a segment longer than kRadixTieMax (many equal keys) makes the
// caller fall back to the bitonic network.  Result: identical order to the
// bitonic sort, about a tenth of its shared-memory traffic.


// bits [p, p + kRadixWindow) of the key (bit 0 = MSB of word 0), zero-padded
template <int KW>
__device__ __forceinline__ uint32_t key_window(const u64* K, int stride, int t, int p) {
  const int d = p >> 6, o = p & 63;
  const u64 hi = K[d * stride + t];
  const u64 lo = d + 1 < KW ? K[(d + 1) * stride + t] : 0ull;
  const u64 v = o ? ((hi << o) | (lo >> (64 - o))) : hi;
  return (uint32_t)(v >> (64 - kRadixWindow));
}

// (key, ik) order of items a, b of a tie segment; *dup set when the keys are equal
template <int KW>
__device__ __forceinline__ bool item_lt_dup(const u64* K, const uint32_t* I, int stride, int a,
                                            int b, int* dup) {
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    const u64 ka = K[d * stride + a], kb = K[d * stride + b];
    if (ka != kb) return ka < kb;
  }
  *dup = 1;
  return I[a] < I[b];
}

// Result of radix_rank_leaf
constexpr int kRankFallback = 0;  // no order produced (equal keys / long window ties)
constexpr int kRankDistinct = 1;  // *perm holds the order, every key differs
constexpr int kRankDups = 2;      // *perm holds the order, some keys are equal

// Ranks the n items of a leaf by (key, ik) without moving them: (*perm)[t] is
// the position of the item of rank t.  The first pass takes its window keys
// straight from the leaf's keys (no staging pass), per-warp bin counters are
// read and written as packed pairs, and the block scan alternates between two
// warp-total buffers (four barriers per pass).
template <int KW, int CAP>
__device__ __noinline__ int radix_rank_leaf(const u64* K, const uint32_t* I, int n,
                                            uint8_t* scratch, uint16_t** perm,
                                            const u64 (&diff)[KW]) {
  static_assert(CAP % kLeafThreads2 == 0, "leaf capacity must be a multiple of the CTA size");
  constexpr int SEG = CAP / kLeafWarps2;             // max positions owned by one warp
  constexpr int SLOTS = SEG >= 32 ? SEG / 32 : 1;
  // only the first npos positions take part: warps own seg = npos / 4 each
  const int npos = SEG >= 32 ? (n + kLeafThreads2 - 1) / kLeafThreads2 * kLeafThreads2 : CAP;
  const int seg = SEG >= 32 ? npos / kLeafWarps2 : SEG;
  const int slots = SEG >= 32 ? seg / 32 : 1;
  uint32_t* wk[2] = {reinterpret_cast<uint32_t*>(scratch),
                     reinterpret_cast<uint32_t*>(scratch) + CAP};
  uint16_t* wp[2] = {reinterpret_cast<uint16_t*>(scratch + 8 * CAP),
                     reinterpret_cast<uint16_t*>(scratch + 8 * CAP) + CAP};
  uint16_t* hist = reinterpret_cast<uint16_t*>(scratch + 12 * CAP);  // [warp][bin]
  __shared__ u64 s_or[kLeafWarps2][KW];
  __shared__ int s_flag, s_dup;
  __shared__ uint32_t s_scan[2][kLeafWarps2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // 1. highest bit at which any key differs from item 0 (diff: this thread's
  //    OR of key ^ key 0 over the items it staged)
  u64 acc[KW];
#pragma unroll
  for (int d = 0; d < KW; ++d) acc[d] = diff[d];
#pragma unroll
  for (int d = 0; d < KW; ++d) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[d] |= __shfl_xor_sync(0xffffffffu, acc[d], o);
    if (lane == 0) s_or[warp][d] = acc[d];
  }
  if (tid == 0) {
    s_flag = 0;
    s_dup = 0;
  }
  __syncthreads();
  int p = -1;
#pragma unroll
  for (int d = KW - 1; d >= 0; --d) {
    u64 v = 0;
#pragma unroll
    for (int w = 0; w < kLeafWarps2; ++w) v |= s_or[w][d];
    if (v) p = d * 64 + __clzll(v);
  }
  if (p < 0) return kRankFallback;  // every key equal: order is by ik alone (bitonic)

  // 2. LSD passes; warp w owns positions [w*seg, (w+1)*seg), slot-major.
  //    Positions >= n carry the maximal window and sort last (stable).
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool lane_on = SEG >= 32 || lane < SEG;
  const unsigned wmask = SEG >= 32 ? 0xffffffffu : ((1u << SEG) - 1u);
  int cur = 0;
#pragma unroll 1
  for (int pass = 0; pass < kRadixPasses; ++pass) {
    const int sh = pass * kRadixBits;
    uint16_t* hw = hist + warp * kRadixBins;
    {
      uint32_t* hz = reinterpret_cast<uint32_t*>(hw);
      for (int b = lane; b < kRadixBins / 2; b += 32) hz[b] = 0u;
    }
    __syncwarp();
    uint32_t key[SLOTS];
    uint16_t pm[SLOTS], rk[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int pos = warp * seg + s * 32 + lane;
      if (lane_on && s < slots) {
        if (pass == 0) {
          key[s] = pos < n ? key_window<KW>(K, CAP, pos, p) : 0xFFFFFFFFu >> (32 - kRadixWindow);
          pm[s] = (uint16_t)pos;
        } else {
          key[s] = wk[cur][pos];
          pm[s] = wp[cur][pos];
        }
        const uint32_t dg = (key[s] >> sh) & (kRadixBins - 1);
        const unsigned grp = __match_any_sync(wmask, dg);
        const uint16_t prev = hw[dg];
        __syncwarp(wmask);
        if ((grp & lt_mask) == 0) hw[dg] = (uint16_t)(prev + __popc(grp));
        __syncwarp(wmask);
        rk[s] = (uint16_t)(prev + __popc(grp & lt_mask));
      }
    }
    __syncthreads();
    // bin-major offsets: bin b's start, then warps in order inside the bin;
    // thread t owns the adjacent bins 2t, 2t+1 (one packed word per warp)
    {
      static_assert(kRadixBins == 2 * kLeafThreads2, "two bins per thread");
      uint32_t* h32 = reinterpret_cast<uint32_t*>(hist);
      uint32_t c[kLeafWarps2];
      uint32_t tot = 0;
#pragma unroll
      for (int w = 0; w < kLeafWarps2; ++w) {
        c[w] = h32[w * (kRadixBins / 2) + tid];
        tot += (c[w] & 0xFFFFu) + (c[w] >> 16);
      }
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      uint32_t* sc = s_scan[pass & 1];
      if (lane == 31) sc[warp] = inc;
      __syncthreads();
      uint32_t run = inc - tot;
#pragma unroll
      for (int w = 0; w < kLeafWarps2; ++w) run += w < warp ? sc[w] : 0u;
      uint32_t lo_off[kLeafWarps2];
#pragma unroll
      for (int w = 0; w < kLeafWarps2; ++w) {
        lo_off[w] = run;
        run += c[w] & 0xFFFFu;
      }
#pragma unroll
      for (int w = 0; w < kLeafWarps2; ++w) {
        h32[w * (kRadixBins / 2) + tid] = lo_off[w] | (run << 16);
        run += c[w] >> 16;
      }
    }
    __syncthreads();
    if (lane_on) {
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        if (s >= slots) break;
        const uint32_t dg = (key[s] >> sh) & (kRadixBins - 1);
        const int np = hw[dg] + rk[s];
        wk[cur ^ 1][np] = key[s];
        wp[cur ^ 1][np] = pm[s];
      }
    }
    cur ^= 1;
    __syncthreads();
  }

  // 3. finish segments of equal windows on the full (key, ik)
  const uint32_t* sk = wk[cur];
  uint16_t* sp = wp[cur];
  for (int q = tid; q < n; q += kLeafThreads2) {
    if ((q > 0 && sk[q - 1] == sk[q]) || q + 1 >= n || sk[q + 1] != sk[q]) continue;
    int e = q + 1;
    while (e < n && sk[e] == sk[q] && e - q <= kRadixTieMax) ++e;
    if (e - q > kRadixTieMax) {
      s_flag = 1;
      continue;
    }
    int dup = 0;
    for (int a = q + 1; a < e; ++a) {  // insertion sort of sp[q..e)
      const uint16_t v = sp[a];
      int b = a;
      while (b > q && item_lt_dup<KW>(K, I, CAP, v, sp[b - 1], &dup)) {
        sp[b] = sp[b - 1];
        --b;
      }
      sp[b] = v;
    }
    if (dup) s_dup = 1;
  }
  __syncthreads();
  if (s_flag) return kRankFallback;
  *perm = sp;
  return s_dup ? kRankDups : kRankDistinct;
}

// Moves K, I into the order perm[0..n) in place (perm[t] = source of rank t).
template <int KW, int CAP>
__device__ __forceinline__ void apply_leaf_perm(u64* K, uint32_t* I, int n, const uint16_t* sp) {
  const int tid = threadIdx.x;
  constexpr int PER = (CAP + kLeafThreads2 - 1) / kLeafThreads2;
  u64 gk[PER][KW];
  uint32_t gi[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int t = r * kLeafThreads2 + tid;
    if (t < n) {
      const int src = sp[t];
#pragma unroll
      for (int d = 0; d < KW; ++d) gk[r][d] = K[d * CAP + src];
      gi[r] = I[src];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int t = r * kLeafThreads2 + tid;
    if (t < n) {
#pragma unroll
      for (int d = 0; d < KW; ++d) K[d * CAP + t] = gk[r][d];
      I[t] = gi[r];
    }
  }
  __syncthreads();
}

// Sorts the leaf in place; false = not sorted (the caller runs the bitonic network).
template <int KW, int CAP>
__device__ __forceinline__ bool radix_sort_leaf(u64* K, uint32_t* I, int n, uint8_t* scratch,
                                                const u64 (&diff)[KW]) {
  uint16_t* sp = nullptr;
  if (radix_rank_leaf<KW, CAP>(K, I, n, scratch, &sp, diff) == kRankFallback) return false;
  apply_leaf_perm<KW, CAP>(K, I, n, sp);
  return true;
}

// ------------------------------------------------------------ leaf sort
// One CTA per leaf (grid = the plan's leaf bound; CTAs past n_leaves record an
// empty leaf).  Load the leaf's items into shared memory, sort by (key, ik),
// mark run heads, sum each run in numpy reduceat order (RunSum, one thread per
// run), drop |sum| <= eps, and write the kept runs compacted -- key words to
// the idle item buffer at the leaf's own offset, sums to C.sums -- plus the
// leaf's kept count.  Leaves larger than the shared-memory capacity (one key
// repeated more than leaf_cap times) are sorted in place in global memory.
// Oversized leaf (a key repeated more than leaf_cap times, which no splitter
// can divide), sorted by the CTA in global memory:
//   1. tiles of `cap` items sorted in shared memory exactly like a normal leaf
//      (radix window sort, bitonic fallback) and written back;
//   2. merge passes over the sorted tiles (width cap, 2 cap, ...), ping-pong
//      between the leaf's items and the idle buffer at the same offset: each
//      thread takes an equal share of the output, finds its start by a
//      merge-path binary search and merges sequentially;
//   3. run heads, each run's end by binary search on the sorted keys, its sum
//      (RunSum, numpy's order) computed once, |sum| <= eps dropped, kept
//      (key, sum) compacted into the idle buffer / C.sums.
// Round 1 used one global-memory bitonic network (H*H with |H| = 10^4: the
// identity run of 10^4 items cost ~10 ms on one CTA).  Returns the kept count
// (valid in thread 0).
// (key, ik) order / key equality of items a, b of a row-major global key buffer
template <int KW>
__device__ __forceinline__ bool item_lt2(const u64* K, const uint32_t* I, int64_t a, int64_t b) {
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    const u64 ka = K[a * KW + d], kb = K[b * KW + d];
    if (ka != kb) return ka < kb;
  }
  return I[a] < I[b];
}

template <int KW>
__device__ __forceinline__ bool row_eq(const u64* K, int64_t a, int64_t b) {
#pragma unroll
  for (int d = 0; d < KW; ++d)
    if (K[a * KW + d] != K[b * KW + d]) return false;
  return true;
}

template <int W, int KW, int MODE>
__device__ __noinline__ uint32_t leaf_sort_global(const Dims& D, const SrcA& S, u64* K,
                                                  uint32_t* I, u64* K2, uint32_t* I2,
                                                  double2* DS, int n, double eps,
                                                  uint32_t* s_warp, u64* SK, uint32_t* SI,
                                                  uint8_t* scratch) {
  using RS = RunSum<W, KW, MODE>;
  constexpr int cap = leaf_cap_for(KW);
  const int tid = threadIdx.x;
  // 1. sorted tiles
  for (int t0 = 0; t0 < n; t0 += cap) {
    const int m = min(cap, n - t0);
    u64 diff[KW];
#pragma unroll
    for (int d = 0; d < KW; ++d) diff[d] = 0;
    for (int t = tid; t < m; t += kLeafThreads2) {
#pragma unroll
      for (int d = 0; d < KW; ++d) {
        const u64 v = K[(int64_t)(t0 + t) * KW + d];
        SK[d * cap + t] = v;
        diff[d] |= v ^ K[(int64_t)t0 * KW + d];
      }
      SI[t] = I[t0 + t];
    }
    __syncthreads();
    if (m > 1 && !radix_sort_leaf<KW, cap>(SK, SI, m, scratch, diff))
      bitonic_sort_local<KW, cap>(SK, SI, m);
    for (int t = tid; t < m; t += kLeafThreads2) {
#pragma unroll
      for (int d = 0; d < KW; ++d) K[(int64_t)(t0 + t) * KW + d] = SK[d * cap + t];
      I[t0 + t] = SI[t];
    }
    __syncthreads();
  }
  // 2. merge passes
  u64* sk = K;
  uint32_t* si = I;
  u64* dk = K2;
  uint32_t* di = I2;
  for (int w = cap; w < n; w *= 2) {
    for (int a0 = 0; a0 < n; a0 += 2 * w) {
      const int la = min(w, n - a0), lb = max(0, min(w, n - a0 - w));
      const int64_t A = a0, B = a0 + la;
      const int L = la + lb;
      const int chunk = (L + kLeafThreads2 - 1) / kLeafThreads2;
      const int d0 = min(L, tid * chunk), d1 = min(L, d0 + chunk);
      if (d0 < d1) {
        int lo = max(0, d0 - lb), hi = min(d0, la);  // A items before output d0
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (item_lt2<KW>(sk, si, A + mid, B + (d0 - 1 - mid))) lo = mid + 1;
          else hi = mid;
        }
        int i = lo, j = d0 - lo;
        for (int o = d0; o < d1; ++o) {
          const bool take_a = j >= lb || (i < la && item_lt2<KW>(sk, si, A + i, B + j));
          const int64_t src = take_a ? A + i++ : B + j++;
#pragma unroll
          for (int d = 0; d < KW; ++d) dk[(int64_t)(a0 + o) * KW + d] = sk[src * KW + d];
          di[a0 + o] = si[src];
        }
      }
    }
    __syncthreads();
    u64* tk = sk; sk = dk; dk = tk;
    uint32_t* ti = si; si = di; di = ti;
  }
  if (sk != K) {  // sorted data back into the leaf's own buffer
    for (int t = tid; t < n; t += kLeafThreads2) {
#pragma unroll
      for (int d = 0; d < KW; ++d) K[(int64_t)t * KW + d] = sk[(int64_t)t * KW + d];
      I[t] = si[t];
    }
    __syncthreads();
  }
  // 3. runs: sums once per head, compaction by tiles
  const int tile = kLeafThreads2 * 8;
  uint32_t base = 0;
  for (int t0 = 0; t0 < n; t0 += tile) {
    double2 sv[8];
    uint32_t keepm = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = t0 + tid * 8 + u;
      if (p >= n || (p != 0 && row_eq<KW>(K, p, p - 1))) continue;
      int lo = p + 1, hi = n;  // first position with a different (greater) key
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (row_eq<KW>(K, mid, p)) lo = mid + 1;
        else hi = mid;
      }
      sv[u] = RS::run(S, D.ma, I, p, lo - p);
      if (keep_sum(sv[u], eps)) keepm |= 1u << u;
    }
    uint32_t tt;
    uint32_t pos = base + leaf_excl_scan((uint32_t)__popc(keepm), s_warp, &tt);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!(keepm >> u & 1)) continue;
      const int p = t0 + tid * 8 + u;
#pragma unroll
      for (int d = 0; d < KW; ++d) K2[(int64_t)pos * KW + d] = K[(int64_t)p * KW + d];
      DS[pos] = sv[u];
      ++pos;
    }
    base += tt;
  }
  return base;
}

// runs of two or more items (kept out of line: rare in most workloads)
template <int W, int KW, int MODE>
__device__ __noinline__ double2 run_sum_multi(const SrcA& S, int64_t ma, const uint32_t* I,
                                              int p, int m) {
  return RunSum<W, KW, MODE>::run(S, ma, I, p, m);
}

constexpr int kSortCtasPerSm = 7;  // bounded by shared memory (~32 KB per CTA)

template <int W, int KW, int MODE>
__global__ void __launch_bounds__(kLeafThreads2, kSortCtasPerSm)
k_leaf_sort(Layout L, Dims D, SrcA S, Ctl C, double eps) {
  extern __shared__ u64 sm[];
  constexpr int cap = leaf_cap_for(KW);  // == D.leaf_cap
  __shared__ uint32_t s_warp[kLeafWarps2];
  const int tid = threadIdx.x;
  const uint32_t leaf = blockIdx.x;
#ifdef PLB_LEAF_PROF
  long long tp[8];
  tp[0] = clock64();
#define LEAF_T(i) tp[i] = clock64()
#else
#define LEAF_T(i)
#endif
  const uint4 dsc = C.leaf_desc[leaf];  // (in bounds: grid = max_leaves) issued with n_leaves
  if (leaf >= *C.n_leaves) {
    if (tid == 0) C.kept[leaf] = 0;
    return;
  }
  const int n = (int)dsc.z;
  const uint32_t off = dsc.y;
  const u64* GK = (dsc.x == 1 ? C.k1 : C.k2) + (int64_t)off * KW;  // row-major item keys
  const uint32_t* GI = (dsc.x == 1 ? C.i1 : C.i2) + off;
  u64* DK = (dsc.x == 1 ? C.k2 : C.k1) + (int64_t)off * KW;  // idle buffer at the same offset
  double2* DS = C.sums + off;

  // shared memory: K [KW][cap] | I [cap] | POS u16 [cap] | HEAD u8 [cap] | scratch
  u64* K = sm;
  uint32_t* I = reinterpret_cast<uint32_t*>(K + (int64_t)KW * cap);
  uint16_t* POS = reinterpret_cast<uint16_t*>(I + cap);
  uint8_t* HEAD = reinterpret_cast<uint8_t*>(POS + cap);
  uint8_t* scratch = reinterpret_cast<uint8_t*>(sm) + leaf_buf_stride(KW);
  if (n > cap) {
    uint32_t* DI = (dsc.x == 1 ? C.i2 : C.i1) + off;
    const uint32_t kept = leaf_sort_global<W, KW, MODE>(
        D, S, const_cast<u64*>(GK), const_cast<uint32_t*>(GI), DK, DI, DS, n, eps, s_warp, K, I,
        scratch);
    if (tid == 0) C.kept[leaf] = kept;
    return;
  }
  double2* SUM = reinterpret_cast<double2*>(scratch);  // reuses the radix scratch
  u64 diff[KW];  // OR of key ^ key 0 over this thread's items (the radix window start)
  {
    u64 k0[KW];
    load_row<KW>(GK, 0, k0);
#pragma unroll
    for (int d = 0; d < KW; ++d) diff[d] = 0;
    for (int t = tid; t < n; t += kLeafThreads2) {
      u64 v[KW];
      load_row<KW>(GK, t, v);
#pragma unroll
      for (int d = 0; d < KW; ++d) {
        K[d * cap + t] = v[d];
        diff[d] |= v[d] ^ k0[d];
      }
      I[t] = GI[t];
    }
  }
  __syncthreads();
  LEAF_T(1);
  if (n > 1) {
    uint16_t* sp = nullptr;
    const int rank = radix_rank_leaf<KW, cap>(K, I, n, scratch, &sp, diff);
    if (rank == kRankDistinct) {
      // Every key of the leaf differs: each item is its own run, so nothing is
      // moved in shared memory -- rank t's key and coefficient go straight to
      // the leaf's output slots (kept = n) unless a coefficient is dropped.
      constexpr int PERF = cap / kLeafThreads2;
      double2 cf[PERF];
      int src[PERF];
      bool drop = false;
      // the keys go out first (asynchronous stores; the general path below
      // rewrites the leaf's slots if a term is dropped), then the coefficients
#pragma unroll
      for (int r = 0; r < PERF; ++r) {
        const int t = r * kLeafThreads2 + tid;
        src[r] = t < n ? (int)sp[t] : -1;
        if (src[r] < 0) continue;
        u64 kv[KW];
#pragma unroll
        for (int d = 0; d < KW; ++d) kv[d] = K[d * cap + src[r]];
        store_row<KW>(DK, t, kv);
      }
#pragma unroll
      for (int r = 0; r < PERF; ++r)
        if (src[r] >= 0) cf[r] = Source<W, KW, MODE>::coef(S, D.ma, I[src[r]]);
#pragma unroll
      for (int r = 0; r < PERF; ++r)
        if (src[r] >= 0 && !keep_sum(cf[r], eps)) drop = true;
      if (!__syncthreads_or(drop)) {
#pragma unroll
        for (int r = 0; r < PERF; ++r)
          if (src[r] >= 0) DS[r * kLeafThreads2 + tid] = cf[r];
        if (tid == 0) C.kept[leaf] = (uint32_t)n;
        return;
      }
    }
    if (rank == kRankFallback) bitonic_sort_local<KW, cap>(K, I, n);
    else apply_leaf_perm<KW, cap>(K, I, n, sp);
  }
  LEAF_T(2);
  for (int p = tid; p < n; p += kLeafThreads2)
    HEAD[p] = (p == 0 || !key_eq<KW>(K, cap, p, p - 1)) ? 1 : 0;
  __syncthreads();
  LEAF_T(3);
  constexpr int CH = cap / kLeafThreads2;  // max items per thread
  const int ch = (n + kLeafThreads2 - 1) / kLeafThreads2;
  const int p0 = tid * ch, p1 = min(n, p0 + ch);
  // coefficients of the chunk's items, all gathers in flight together; a run
  // of one item is its coefficient (RunSum::run with m == 1), longer runs
  // are summed by RunSum in numpy's order
  double2 cf[CH];
  uint8_t hd[CH];
#pragma unroll
  for (int u = 0; u < CH; ++u) {
    hd[u] = 0;
    if (u < ch && p0 + u < p1) {
      hd[u] = HEAD[p0 + u];
      cf[u] = Source<W, KW, MODE>::coef(S, D.ma, I[p0 + u]);
    }
  }
  uint32_t keepbits = 0;
#pragma unroll
  for (int u = 0; u < CH; ++u) {
    const int p = p0 + u;
    if (u >= ch || p >= p1 || !hd[u]) continue;
    int q = p + 1;
    while (q < n && !HEAD[q]) ++q;
    const double2 s = q == p + 1 ? cf[u] : run_sum_multi<W, KW, MODE>(S, D.ma, I, p, q - p);
    if (keep_sum(s, eps)) {
      keepbits |= 1u << u;
      SUM[p] = s;
    }
  }
  LEAF_T(4);
  uint32_t kept;
  uint32_t slot = leaf_excl_scan(__popc(keepbits), s_warp, &kept);
  for (uint32_t bb = keepbits; bb; bb &= bb - 1) POS[slot++] = (uint16_t)(p0 + __ffs(bb) - 1);
  __syncthreads();
  LEAF_T(5);
  for (uint32_t q = tid; q < kept; q += kLeafThreads2) {
    const int p = POS[q];
    u64 kv[KW];
#pragma unroll
    for (int d = 0; d < KW; ++d) kv[d] = K[d * cap + p];
    store_row<KW>(DK, q, kv);
    DS[q] = SUM[p];
  }
  if (tid == 0) C.kept[leaf] = kept;
#ifdef PLB_LEAF_PROF
  LEAF_T(6);
  if (tid == 0 && (leaf % 20011) == 5)
    printf("LEAFPROF n=%d load=%lld sort=%lld head=%lld sums=%lld scan=%lld write=%lld\n", n,
           tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5]);
#endif
}

// leaf buffer + scratch (radix sort, then the run sums SUM[cap])
__host__ __device__ constexpr size_t leaf_sort_smem_bytes(int KW) {
  return leaf_buf_stride(KW) +
         (radix_smem_bytes(leaf_cap_for(KW)) > 16 * (size_t)leaf_cap_for(KW)
              ? radix_smem_bytes(leaf_cap_for(KW))
              : 16 * (size_t)leaf_cap_for(KW)) +
         64;
}

// ------------------------------------------------------------ emit
// Streams the merged terms out in output order: a CTA owns the output range
// [o0, o0 + T) (T = emit_tile(KW) terms), finds the leaves covering it
// (range map + binary search on the kept-count prefix), stages the range's
// (key, sum) entries in shared memory, then builds the SoA output one plane
// at a time in a double-buffered shared tile that a TMA bulk store
// (cp.async.bulk) writes out: T*8 contiguous, 16-byte aligned bytes per plane
// per CTA, so every DRAM sector is written whole exactly once and the SM does
// not issue the global stores itself.  The coefficients go out of the staging
// buffer the same way and the phase bytes from a zero tile.  Partial (last)
// tiles and unaligned outputs use plain coalesced stores.
constexpr int kEmitThreads = 256;
__host__ __device__ constexpr int emit_tile(int KW) {
  return KW <= 4 ? 1024 : KW <= 8 ? 512 : 256;  // >= kEmitThreads
}
// staged (key, sum) | leaf metadata | two plane buffers + zero phase bytes
// for the TMA bulk stores
__host__ __device__ constexpr size_t emit_smem_bytes(int KW) {
  return (size_t)emit_tile(KW) * (8 * KW + 16) + (size_t)kEmitThreads * 12 + 64 +
         (size_t)emit_tile(KW) * (2 * 8 + 1) + 16;
}

// TMA (cp.async.bulk) store of `bytes` from shared to global memory, one
// bulk group per call (issued by one thread)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
               "cp.async.bulk.commit_group;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// last leaf l in [lo, hi] with pre[l] <= v (pre non-decreasing, pre[lo] <= v)
__device__ __forceinline__ uint32_t leaf_at(const uint32_t* pre, uint32_t lo, uint32_t hi,
                                            uint32_t v) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= v) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// rmap[r] = the leaf holding output position r*T (every position lies in
// exactly one leaf with kept > 0)
template <int KW>
__global__ void k_range_map(Dims D, Ctl C) {
  constexpr uint32_t T = emit_tile(KW);
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= *C.n_leaves) return;
  const uint32_t k = C.kept[l];
  if (k == 0) return;
  const uint32_t pre = C.kprefix[l];
  for (uint32_t r = (pre + T - 1) / T; r * T < pre + k; ++r) C.rmap[r] = l;
}

// Small merges (<= kScanSmallLeaves leaf slots): the scan of the kept counts,
// its total and the range map in ONE single-CTA launch instead of four (the
// three-kernel scan + k_range_map); a 10^6-item merge is bound by its ~15
// dependent launches, not by bandwidth.
constexpr int kScanSmallItems = 16;
constexpr int kScanSmallLeaves = 1024 * kScanSmallItems;

template <int KW>
__global__ void __launch_bounds__(1024) k_leaf_scan_small(Dims D, Ctl C) {
  constexpr uint32_t T = emit_tile(KW);
  const uint32_t n_leaves = *C.n_leaves;
  const int base = threadIdx.x * kScanSmallItems;
  uint32_t v[kScanSmallItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanSmallItems; ++k) {
    const int l = base + k;
    v[k] = l < D.max_leaves ? C.kept[l] : 0u;  // (leaf slots past n_leaves hold 0)
    s += v[k];
  }
  uint32_t total;
  uint32_t pre = block_excl_scan(s, &total);
  if (threadIdx.x == 0) *C.scan_total = total;
#pragma unroll
  for (int k = 0; k < kScanSmallItems; ++k) {
    const int l = base + k;
    if (l < D.max_leaves) C.kprefix[l] = pre;
    if ((uint32_t)l < n_leaves && v[k])
      for (uint32_t r = (pre + T - 1) / T; r * T < pre + v[k]; ++r) C.rmap[r] = (uint32_t)l;
    pre += v[k];
  }
}

template <int W, int KW>
__global__ void __launch_bounds__(kEmitThreads)
k_emit(Layout L, Dims D, Ctl C, OutP O) {
  constexpr int T = emit_tile(KW);
  constexpr int TM = T;  // granularity of the range map
  constexpr int PER = T / kEmitThreads;
  extern __shared__ u64 sm[];
  u64* KS = sm;                                              // [KW][T]
  double2* SS = reinterpret_cast<double2*>(KS + (int64_t)KW * T);  // [T]
  uint32_t* m_pre = reinterpret_cast<uint32_t*>(SS + T);     // leaf chunk metadata
  uint32_t* m_end = m_pre + kEmitThreads;
  uint32_t* m_src = m_end + kEmitThreads;                    // buffer << 31 | offset
  u64* PB = reinterpret_cast<u64*>(
      (reinterpret_cast<uintptr_t>(m_src + kEmitThreads) + 15) & ~(uintptr_t)15);  // [2][T]
  uint8_t* ZB = reinterpret_cast<uint8_t*>(PB + 2 * T);      // [T] zero phase bytes
  const int tid = threadIdx.x;
  const uint32_t n_leaves = *C.n_leaves;
  const uint32_t total_all = *C.scan_total;
  if (blockIdx.x == 0 && tid == 0) *O.count = (int64_t)total_all;
  // never write past the caller's columns (phase 2 sizes them from phase 1)
  const uint32_t total = (int64_t)total_all < O.capacity ? total_all : (uint32_t)O.capacity;
  for (int e = tid; e < T; e += kEmitThreads) ZB[e] = 0;
  fence_async_smem();
  // full tiles go out through TMA bulk stores when every destination is
  // 16-byte aligned (planes: even leading dimension)
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(O.oz) | reinterpret_cast<uintptr_t>(O.ox) |
                         reinterpret_cast<uintptr_t>(O.oc) | reinterpret_cast<uintptr_t>(O.ok)) &
                        15) == 0 && (O.ldo & 1) == 0;
  for (uint64_t o0 = (uint64_t)blockIdx.x * T; o0 < total; o0 += (uint64_t)gridDim.x * T) {
    const uint32_t o1 = (uint32_t)(o0 + T < total ? o0 + T : total);
    const bool bulk = bulk_ok && o1 - (uint32_t)o0 == (uint32_t)T;
    if (tid == 0) bulk_wait_read_all();  // previous tile's bulk stores done reading KS/SS/PB
    __syncthreads();
    const uint32_t l0 = C.rmap[(uint32_t)(o0 / TM)];
    const uint64_t rl = (uint64_t)(o1 - 1) / TM + 1;  // first range-map block past the tile
    const uint32_t l1 = rl * TM < total ? C.rmap[rl] : n_leaves - 1;
    for (uint32_t lb = l0; lb <= l1; lb += kEmitThreads) {
      const uint32_t nl = l1 - lb + 1 < (uint32_t)kEmitThreads ? l1 - lb + 1 : (uint32_t)kEmitThreads;
      if (tid < (int)nl) {
        const uint32_t l = lb + tid;
        const uint4 dsc = C.leaf_desc[l];
        const uint32_t pre = C.kprefix[l];
        m_pre[tid] = pre;
        m_end[tid] = pre + C.kept[l];
        m_src[tid] = (dsc.x == 1 ? 0x80000000u : 0u) | dsc.y;  // kept entries live in the idle buffer
      }
      __syncthreads();
      const uint32_t c_lo = m_pre[0], c_hi = m_end[nl - 1];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const uint32_t p = (uint32_t)o0 + u * kEmitThreads + tid;
        if (p >= o1 || p < c_lo || p >= c_hi) continue;
        const uint32_t j = leaf_at(m_pre, 0, nl - 1, p);
        if (p >= m_end[j]) continue;  // (cannot happen: leaves tile the output)
        const uint32_t src = m_src[j];
        const int64_t row = (int64_t)(src & 0x7FFFFFFFu) + (p - m_pre[j]);
        const int e = u * kEmitThreads + tid;
        u64 kv[KW];
        load_row<KW>((src >> 31) ? C.k2 : C.k1, row, kv);
#pragma unroll
        for (int d = 0; d < KW; ++d) KS[d * T + e] = kv[d];
        SS[e] = __ldg(C.sums + (src & 0x7FFFFFFFu) + (p - m_pre[j]));
      }
      __syncthreads();
    }
    // plane-major stores: each plane gets T*8 contiguous bytes from this CTA
    // (sparse keys: the slots are sorted by packed position and the planes
    // cover ascending position ranges, so one cursor per term walks them once)
    int cur[PER], curp[PER];  // sparse keys: slot cursor and its decoded position
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      cur[u] = 0;
      curp[u] = L.sparse ? sparse_slot_pos(L, KS, T, u * kEmitThreads + tid, 0) : 0;
    }
    for (int q = 0; q < 2 * W; ++q) {
      const int len = L.len[q];
      u64* dst = (q < W ? O.oz + (int64_t)q * O.ldo : O.ox + (int64_t)(q - W) * O.ldo) + o0;
      const int pos = L.pos[q], lo = L.lo[q];
      const int wi = pos >> 6, off = pos & 63;
      u64* pb = PB + (q & 1) * T;
      if (bulk && q >= 2) {  // plane buffer q&1 free once the store of plane q-2 has read it
        if (tid == 0) bulk_wait_read_le1();
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = u * kEmitThreads + tid;
        if ((uint32_t)o0 + e >= o1) break;
        u64 w = 0;
        if (L.sparse) {
          if (len) w = sparse_plane_next(L, KS, T, e, q, cur[u], curp[u]);
        } else if (len) {
          const u64 a = KS[wi * T + e];
          const u64 b = (off && wi + 1 < KW) ? KS[(wi + 1) * T + e] : 0ull;
          const u64 hi = off ? ((a << off) | (b >> (64 - off))) : a;
          w = (hi >> (64 - len)) << lo;
        }
        if (bulk) pb[e] = w;
        else dst[e] = w;
      }
      if (bulk) {
        fence_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(dst, pb, (uint32_t)T * 8);
      }
    }
    if (bulk) {  // coefficients straight from the staging buffer, phases from zeros
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        bulk_store(O.oc + o0, SS, (uint32_t)T * 16);
        bulk_store(O.ok + o0, ZB, (uint32_t)T);
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = u * kEmitThreads + tid;
      if ((uint32_t)o0 + e >= o1) break;
      O.oc[o0 + e] = SS[e];
    }
    for (int e = tid * 4; e < T; e += kEmitThreads * 4) {
      if ((uint32_t)o0 + e + 4 <= o1 && ((o0 + e) & 3) == 0 &&
          (reinterpret_cast<uintptr_t>(O.ok + o0 + e) & 3) == 0) {
        *reinterpret_cast<uint32_t*>(O.ok + o0 + e) = 0u;
      } else {
        for (int f = e; f < e + 4 && (uint32_t)o0 + f < o1; ++f) O.ok[o0 + f] = 0;
      }
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait_all();
}

template <int W, int KW>
static int launch_emit(const Layout& L, const Dims& D, const Ctl& C, const OutP& O,
                       cudaStream_t st);

template <int W, int KW, int MODE>
static int launch_leaves(const Layout& L, const Dims& D, const SrcA& S, const Ctl& C,
                         const OutP& O, cudaStream_t st) {
  const size_t lsm = leaf_sort_smem_bytes(KW);
  auto ks = k_leaf_sort<W, KW, MODE>;
  if (lsm > 48 * 1024)
    PLB_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
  {
    StageTimer t_(st, "k_leaf_sort");
    ks<<<(unsigned)D.max_leaves, kLeafThreads2, lsm, st>>>(L, D, S, C, O.eps);
    PLB_CHECK_LAUNCH("k_leaf_sort");
  }
  if (D.max_leaves <= kScanSmallLeaves) {
    StageTimer t_(st, "k_leaf_scan_small");
    k_leaf_scan_small<KW><<<1, 1024, 0, st>>>(D, C);
    PLB_CHECK_LAUNCH("k_leaf_scan_small");
  } else {
    {
      StageTimer t_(st, "k_leaf_scan");
      int rc = exclusive_scan_u32(C.kept, C.kprefix, D.max_leaves, C.scan_scratch, C.scan_total, st);
      if (rc) return rc;
    }
    StageTimer t_(st, "k_range_map");
    k_range_map<KW><<<(unsigned)ceil_div(D.max_leaves, 256), 256, 0, st>>>(D, C);
    PLB_CHECK_LAUNCH("k_range_map");
  }
  if (O.phase == 1) {  // merged count only (count's high word was zeroed by k_buckets)
    PLB_CUDA(cudaMemcpyAsync(O.count, C.scan_total, 4, cudaMemcpyDeviceToDevice, st));
    return PL_OK;
  }
  return launch_emit<W, KW>(L, D, C, O, st);
}

template <int W, int KW>
static int launch_emit(const Layout& L, const Dims& D, const Ctl& C, const OutP& O,
                       cudaStream_t st) {
  const size_t esm = emit_smem_bytes(KW);
  auto ke = k_emit<W, KW>;
  if (esm > 48 * 1024)
    PLB_CUDA(cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
  StageTimer t_(st, "k_emit");
  ke<<<(unsigned)(4 * num_sms()), kEmitThreads, esm, st>>>(L, D, C, O);
  PLB_CHECK_LAUNCH("k_emit");
  return PL_OK;
}
