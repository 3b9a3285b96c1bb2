// Leaf stage of the merge pipeline (included by combine.cu, which defines the
// key helpers, RunSum, Source, keep_sum and the relaxed gpu-scope loads).
//
// Persistent CTAs of kLeafThreads2 threads (4 per SM) take leaves in order
// from an atomic counter.  Each leaf (<= leaf_cap items, staged in shared
// memory) goes through two phases, software-pipelined over two buffers so a
// CTA never idles waiting for a predecessor:
//   phase A (leaf i):  load; bitonic sort by (key, ik) -- stages whose blocks
//       fit in one warp's contiguous segment run warp-synchronously; run heads;
//       pass 1 sums each run in numpy reduceat order (RunSum) and keeps those
//       with |sum| > eps; a block scan fills POS[q] = head of kept run q; the
//       kept count is published as the leaf's aggregate.
//   phase B (leaf i, after phase A of leaf i+1):  warp-parallel decoupled
//       look-back -> global output base; publish the inclusive prefix; pass 2
//       writes merged term q from thread q (coalesced plane stores),
//       recomputing the run sum.
// Leaves larger than leaf_cap (one key repeated more than leaf_cap times,
// which no splitter can divide) are sorted in place in global memory and
// processed synchronously, tile by tile.
#pragma once

// Shared-memory items per leaf buffer for key width KW (two buffers of about
// 23 KB per CTA so four CTAs fit on one SM).
__host__ __device__ constexpr int leaf_cap_for(int KW) {
  return KW <= 2 ? 1024 : KW == 4 ? 512 : KW == 8 ? 256 : KW == 16 ? 128 : 64;
}

__host__ __device__ constexpr size_t leaf_smem_bytes(int KW) {
  return 2 * (((size_t)leaf_cap_for(KW) * (8 * KW + 4 + 2 + 1) + 15) & ~(size_t)15) + 64;
}

constexpr int kLeafThreads2 = 256;
constexpr int kLeafCtasPerSm = 3;  // 85 registers per thread, no spills in the hot path
constexpr int kLeafWarps2 = kLeafThreads2 / 32;

template <int KW>
__device__ __forceinline__ void cmp_swap(u64* K, uint32_t* I, int64_t stride, int i, int p) {
  if (item_lt<KW>(K, I, stride, p, i)) {
#pragma unroll
    for (int d = 0; d < KW; ++d) {
      const u64 t = K[d * stride + i];
      K[d * stride + i] = K[d * stride + p];
      K[d * stride + p] = t;
    }
    const uint32_t t = I[i];
    I[i] = I[p];
    I[p] = t;
  }
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
__device__ void bitonic_sort_local(u64* K, uint32_t* I, int n) {
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

template <int W, int KW>
__device__ __forceinline__ void write_term(const Layout& L, const OutP& O, uint64_t pos,
                                           const u64 (&key)[KW], double2 s) {
#pragma unroll
  for (int q = 0; q < 2 * W; ++q) {
    const int len = L.len[q];
    const u64 w = len ? (get_seg<KW>(key, L.pos[q], len) << L.lo[q]) : 0ull;
    if (q < W) O.oz[q * O.ldo + pos] = w;
    else O.ox[(q - W) * O.ldo + pos] = w;
  }
  O.ok[pos] = 0;
  O.oc[pos] = s;
}

constexpr unsigned long long kLbAgg = 1ull << 62, kLbPre = 2ull << 62,
                             kLbVal = (1ull << 62) - 1;

// Publish a leaf's kept count (inclusive prefix for leaf 0).
__device__ __forceinline__ void leaf_publish(unsigned long long* status, uint32_t leaf,
                                             uint64_t agg) {
  st_relaxed_gpu(&status[leaf], (leaf == 0 ? kLbPre : kLbAgg) | agg);
}

// Warp-parallel look-back for a leaf whose aggregate is already published:
// scan predecessors 32 at a time until the nearest inclusive prefix, then
// publish this leaf's inclusive prefix.  Returns the exclusive prefix.
static __device__ uint64_t leaf_lookback_pub(unsigned long long* status, uint32_t leaf, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (leaf == 0) return 0;
  uint64_t excl = 0;
  int64_t base = (int64_t)leaf - 1;
  for (;;) {
    const int64_t idx = base - lane;
    const unsigned long long v = idx >= 0 ? ld_relaxed_gpu(&status[idx]) : kLbPre;
    const unsigned f = (unsigned)(v >> 62);
    const unsigned inc = __ballot_sync(0xffffffffu, f == 2);
    const unsigned zero = __ballot_sync(0xffffffffu, f == 0);
    const int first = inc ? __ffs(inc) - 1 : 32;
    const unsigned need = first == 32 ? 0xffffffffu : ((2u << first) - 1u);
    if (zero & need) continue;
    unsigned long long c = (lane <= first) ? (v & kLbVal) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    excl += c;
    if (first < 32) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_gpu(&status[leaf], kLbPre | (excl + agg));
  return excl;
}

template <int KW>
struct LeafBuf {
  u64* K;         // [KW][cap]
  uint32_t* I;    // [cap]
  uint16_t* POS;  // [cap]
  uint8_t* HEAD;  // [cap]
};

template <int KW>
__device__ __forceinline__ LeafBuf<KW> leaf_buf(u64* sm, int cap, int b) {
  const size_t bytes = (size_t)cap * (8 * KW + 4 + 2 + 1);
  const size_t stride = (bytes + 15) & ~(size_t)15;
  uint8_t* base = reinterpret_cast<uint8_t*>(sm) + b * stride;
  LeafBuf<KW> lb;
  lb.K = reinterpret_cast<u64*>(base);
  lb.I = reinterpret_cast<uint32_t*>(lb.K + (int64_t)KW * cap);
  lb.POS = reinterpret_cast<uint16_t*>(lb.I + cap);
  lb.HEAD = reinterpret_cast<uint8_t*>(lb.POS + cap);
  return lb;
}

template <int W, int KW, int MODE>
__global__ void __launch_bounds__(kLeafThreads2, kLeafCtasPerSm)
k_leaves(Layout L, Dims D, SrcA S, Ctl C, OutP O) {
  extern __shared__ u64 sm[];
  constexpr int cap = leaf_cap_for(KW);  // == D.leaf_cap
  __shared__ uint32_t s_leaf;
  __shared__ uint32_t s_warp[kLeafWarps2];
  __shared__ uint64_t s_base;
  const int tid = threadIdx.x;
  const uint32_t n_leaves = *C.n_leaves;
  using RS = RunSum<W, KW, MODE>;

  // pending phase-B work
  bool have_prev = false;
  uint32_t prev_leaf = 0, prev_kept = 0;
  int prev_n = 0, prev_buf = 0, cur = 0;

  auto phase_b = [&](uint32_t leaf, uint32_t kept, int n, int b) {
    const LeafBuf<KW> B = leaf_buf<KW>(sm, cap, b);
    if (tid < 32) {
      const uint64_t excl = leaf_lookback_pub(C.leaf_status, leaf, kept);
      if (tid == 0) {
        s_base = excl;
        if (leaf == n_leaves - 1) *O.count = (int64_t)(excl + kept);
      }
    }
    __syncthreads();
    const uint64_t base = s_base;
    for (uint32_t q = tid; q < kept; q += kLeafThreads2) {
      const int p = B.POS[q];
      int e = p + 1;
      while (e < n && !B.HEAD[e]) ++e;
      const double2 s = RS::run(S, D.ma, B.I, p, e - p);
      u64 key[KW];
      load_key<KW>(B.K, cap, p, key);
      write_term<W, KW>(L, O, base + q, key, s);
    }
    __syncthreads();
  };

  for (;;) {
    if (tid == 0) s_leaf = atomicAdd(C.leaf_ctr, 1u);
    __syncthreads();
    const uint32_t leaf = s_leaf;
    const bool done = leaf >= n_leaves;
    if (!done) {
      const uint4 dsc = C.leaf_desc[leaf];
      const int n = (int)dsc.z;
      const u64* GK = (dsc.x == 1 ? C.k1 : C.k2) + dsc.y;
      const uint32_t* GI = (dsc.x == 1 ? C.i1 : C.i2) + dsc.y;
      if (n > cap) {
        // ---------------------------------- oversized leaf, synchronous
        if (have_prev) {
          phase_b(prev_leaf, prev_kept, prev_n, prev_buf);
          have_prev = false;
        }
        u64* K = const_cast<u64*>(GK);
        uint32_t* I = const_cast<uint32_t*>(GI);
        const int64_t stride = D.n;
        bitonic_sort<KW>(K, I, stride, n);
        const int tile = kLeafThreads2 * 8;
        uint32_t total = 0;
        for (int t0 = 0; t0 < n; t0 += tile) {
          uint32_t mine = 0;
          for (int p = t0 + tid * 8; p < min(n, t0 + tid * 8 + 8); ++p) {
            if (p != 0 && key_eq<KW>(K, stride, p, p - 1)) continue;
            int q = p + 1;
            while (q < n && key_eq<KW>(K, stride, q, q - 1)) ++q;
            if (keep_sum(RS::run(S, D.ma, I, p, q - p), O.eps)) ++mine;
          }
          uint32_t tt;
          leaf_excl_scan(mine, s_warp, &tt);
          total += tt;
        }
        if (tid < 32) {
          if (tid == 0) leaf_publish(C.leaf_status, leaf, total);
          __syncwarp();
          const uint64_t excl = leaf_lookback_pub(C.leaf_status, leaf, total);
          if (tid == 0) {
            s_base = excl;
            if (leaf == n_leaves - 1) *O.count = (int64_t)(excl + total);
          }
        }
        __syncthreads();
        uint64_t base = s_base;
        for (int t0 = 0; t0 < n; t0 += tile) {
          uint32_t mine = 0;
          for (int p = t0 + tid * 8; p < min(n, t0 + tid * 8 + 8); ++p) {
            if (p != 0 && key_eq<KW>(K, stride, p, p - 1)) continue;
            int q = p + 1;
            while (q < n && key_eq<KW>(K, stride, q, q - 1)) ++q;
            if (keep_sum(RS::run(S, D.ma, I, p, q - p), O.eps)) ++mine;
          }
          uint32_t tt;
          uint64_t pos = base + leaf_excl_scan(mine, s_warp, &tt);
          for (int p = t0 + tid * 8; p < min(n, t0 + tid * 8 + 8); ++p) {
            if (p != 0 && key_eq<KW>(K, stride, p, p - 1)) continue;
            int q = p + 1;
            while (q < n && key_eq<KW>(K, stride, q, q - 1)) ++q;
            const double2 s = RS::run(S, D.ma, I, p, q - p);
            if (keep_sum(s, O.eps)) {
              u64 key[KW];
              load_key<KW>(K, stride, p, key);
              write_term<W, KW>(L, O, pos++, key, s);
            }
          }
          base += tt;
        }
        __syncthreads();
        continue;
      }
      // -------------------------------------------- phase A (buffer cur)
      const LeafBuf<KW> B = leaf_buf<KW>(sm, cap, cur);
      for (int t = tid; t < n; t += kLeafThreads2) {
#pragma unroll
        for (int d = 0; d < KW; ++d) B.K[d * cap + t] = GK[d * D.n + t];
        B.I[t] = GI[t];
      }
      __syncthreads();
      if (n > 1) bitonic_sort_local<KW, cap>(B.K, B.I, n);
      for (int p = tid; p < n; p += kLeafThreads2)
        B.HEAD[p] = (p == 0 || !key_eq<KW>(B.K, cap, p, p - 1)) ? 1 : 0;
      __syncthreads();
      const int ch = (n + kLeafThreads2 - 1) / kLeafThreads2;  // <= 8
      const int p0 = tid * ch, p1 = min(n, p0 + ch);
      uint32_t keepbits = 0;
      for (int p = p0; p < p1; ++p) {
        if (!B.HEAD[p]) continue;
        int q = p + 1;
        while (q < n && !B.HEAD[q]) ++q;
        if (keep_sum(RS::run(S, D.ma, B.I, p, q - p), O.eps)) keepbits |= 1u << (p - p0);
      }
      uint32_t kept;
      uint32_t slot = leaf_excl_scan(__popc(keepbits), s_warp, &kept);
      for (uint32_t bb = keepbits; bb; bb &= bb - 1) B.POS[slot++] = (uint16_t)(p0 + __ffs(bb) - 1);
      if (tid == 0) leaf_publish(C.leaf_status, leaf, kept);
      __syncthreads();
      // ------------------------------- phase B of the previous leaf
      if (have_prev) phase_b(prev_leaf, prev_kept, prev_n, prev_buf);
      have_prev = true;
      prev_leaf = leaf;
      prev_kept = kept;
      prev_n = n;
      prev_buf = cur;
      cur ^= 1;
    } else {
      if (have_prev) phase_b(prev_leaf, prev_kept, prev_n, prev_buf);
      break;
    }
  }
}

