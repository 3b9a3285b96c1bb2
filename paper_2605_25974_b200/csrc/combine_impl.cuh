// K2-K4: outer product + simplify, and sort_and_combine (kernel templates).
//
// Included by combine.cu (the C ABI, declarations only: extern templates) and
// by combine_w{1,2,4,8,16}.cu, which each instantiate one word count W so the
// five heavy instantiation sets compile in parallel.
//
// Restates _combine_columns (sums.py:94-120) applied to the raw outer product
// of _multiply_columns (sums.py:144-174), without ever materialising the raw
// 145-byte records:
//
//   item      = (packed key, ik)  where ik = raw_row << 2 | k,
//               raw_row = j*Ma + i (the reference's j-major row, sums.py:137)
//   key       = the canonical (z0..z{W-1}, x0..x{W-1}) big-endian string
//               (sums.py:104-106, strings.py:165-167) with every bit range that
//               is zero in all operands removed; removal of constant bits keeps
//               the lexicographic order, so sorting packed keys sorts terms.
//
// Pipeline (sample sort, every stage a pure function of its input):
//   1. k_sample   : S deterministic sample keys, bitonic-sorted in one CTA,
//                   -> nb1-1 splitters (ranges of the key space)
//   2. k_count    : key of every item -> bucket (binary search) -> counts
//   3. k_buckets  : scan counts -> bucket bases, leaves per bucket
//   4. k_scatter  : items -> bucket-contiguous buffer 1 (per-CTA reservation)
//   5. k_split    : buckets larger than a shared-memory leaf are re-partitioned
//                   by a CTA-local sample into sub-buckets (buffer 2)
//   6. k_leaf_sort: per leaf (<= leaf_cap items in shared memory, otherwise
//                   in place in global memory): sort by (key, ik), detect runs
//                   of equal keys, sum each run's coefficients
//                   a_c[i]*b_c[j]*i^k in raw-row order with numpy's reduceat
//                   summation tree (one thread per run, bit-exact), drop
//                   |sum| <= eps, write the kept (key, sum) compacted.
//   7. scan of kept counts per leaf; 8. k_emit: stream the merged terms out.
// Runs never straddle buckets (splitters compare keys only) and each run is
// summed by one thread in ik order, so the output is bit-identical whatever
// the bucket structure, CTA schedule or GPU count.
#pragma once
#include <algorithm>
#include <climits>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace plb {

constexpr int kGenThreads = 256;
constexpr int kGenTB = 16;        // items per thread: b-terms of its group (outer) / terms (sort)
// outer-product tiles: kTileA sorted A-terms x kTileB sorted B-terms per CTA;
// thread t takes A-term t % kTileA and the kGenTB B-terms of group t / kTileA
constexpr int kTileA = 64;
constexpr int kTileB = kGenThreads / kTileA * kGenTB;  // 64
constexpr int kSortOpsChunk = 16384;  // operand terms per k_sort_ops CTA (14-bit local index)
constexpr int kLeafThreads = 1024;  // k_sample (one-CTA sample sort)
constexpr int kSplitThreads = 1024;
constexpr int kSortSmemBytes = 200 * 1024;
constexpr int kSampleOversample = 16;  // level-2 samples per sub-bucket
constexpr int kSample1Oversample = 16;  // level-1 samples per bucket
constexpr int kLeavesPerBucket = 32;
constexpr int kTabBits = 13;  // level-1 prefix table: splitters per top-13-bit key prefix
constexpr int kMaxBuckets = 2048;
constexpr int kSplitTile = 2048;     // items per level-2 classification tile
constexpr int kSplitTileThreads = 256;

// ---------------------------------------------------------------- layout
struct Layout {
  int W, KW, active;  // active: bit w set if z-word w or x-word w is used
  int lo[PL_PLAN_MAX_SEG], len[PL_PLAN_MAX_SEG], pos[PL_PLAN_MAX_SEG];
  // sparse keys (wide, sparse sort keys): the key is the list of the packed
  // key's set-bit positions p, most significant first, each stored as the
  // sbits-wide value key_bits - p, terminated by 0; lexicographic order on
  // these slot sequences equals the packed keys' order
  int sparse, sbits, nslots, key_bits;
};

struct Ctl {  // control arrays inside the workspace
  u64* split;            // [KW][nb1]
  uint32_t* bcount;      // nb1
  uint32_t* bbase;       // nb1 + 1
  uint32_t* bcursor;     // nb1
  uint32_t* leaf_off;    // nb1 + 1
  uint32_t* n_leaves;    // 1
  uint32_t* leaf_ctr;    // 1
  uint4* leaf_desc;      // max_leaves: (buffer 1|2, offset, size, 0)
  u64* split2;           // [nb1][KW][max_sub] level-2 splitters per bucket
  u64* split2w;          // [nb1][max_sub] 64-bit window of each level-2 splitter (after bcp bits)
  int32_t* bcp;          // nb1: bits shared by every key of the bucket (window offset)
  uint16_t* bid;         // level-1 bucket of every generated item (k_count -> k_scatter)
  uint16_t* sid;         // [n] level-2 sub-bucket of every item (k_split_count -> k_split_scatter)
  uint32_t* sub_count;   // [nb1][max_sub] first output position of every sub-bucket
  uint4* tile_desc;      // per level-2 tile: (bucket, first item, items, sub-buckets)
  uint16_t* thist;       // [tiles][max_sub] items of the tile per sub-bucket
  uint32_t* toff;        // [tiles][max_sub] offset of the tile's run inside the sub-bucket
  uint32_t* tile_off;    // nb1 + 1: first split tile of each bucket
  uint32_t* n_tiles;     // 1
  uint32_t* kept;         // max_leaves: merged terms per leaf
  uint32_t* kprefix;      // max_leaves: exclusive prefix of kept
  uint32_t* scan_scratch; // scan_scratch_words(max_leaves)
  uint32_t* scan_total;   // 1: total merged terms
  double2* sums;          // [n] run sums, compacted per leaf
  uint32_t* rmap;         // emit range -> first leaf
  u64* opk;               // [KW][ma (+ mb)] packed operand keys
  uint8_t* opb;           // [ma (+ mb)] operand base phases
  uint16_t* l1tab;        // 2^kTabBits + 1: first splitter per top-bit prefix
  int32_t* perm;          // outer: [ma + mb] sorted position -> operand index (A, then B)
  u64* k1;               // [n][KW] item keys (row-major), buffer 1
  uint32_t* i1;          // [n]
  u64* k2;               // buffer 2
  uint32_t* i2;
};

struct Dims {
  int64_t n, ma, mb;     // items held here; |A|; B columns generated here
  int64_t n_space, j0;   // full raw-product size (sampling space); first B column
  int64_t mb_all;        // |B| (all columns; packed operand keys cover A then all of B)
  int nb1, nsamp, leaf_cap, leaf_target, max_sub, max_leaves;
};

struct SrcA {  // operands (outer: A and B; sort: A only)
  const u64 *ax, *az;
  const uint8_t* ak;
  const double2* ac;
  int64_t lda;
  const u64 *bx, *bz;
  const uint8_t* bk;
  const double2* bc;
  int64_t ldb;
  u64 ma_inv;  // outer: ceil(2^62 / |A|), raw row -> j by multiply (div_ma)
};

// ceil(2^62 / ma): floor(r * inv / 2^62) == r / ma for every r < 2^30
inline u64 ma_inverse(int64_t ma) { return ma > 0 ? ((1ull << 62) - 1) / (u64)ma + 1 : 0; }

__device__ __forceinline__ uint32_t div_ma(uint32_t r, u64 inv) {
  const u64 lo = (u64)r * inv;
  const u64 hi = __umul64hi((u64)r, inv);
  return (uint32_t)((hi << 2) | (lo >> 62));
}

struct OutP {
  u64 *ox, *oz;
  uint8_t* ok;
  double2* oc;
  int64_t ldo;
  int64_t* count;
  double eps;
  // 0: sort + emit; 1: sort only (*count = merged terms, the (key, sum)
  // entries stay in the workspace); 2: emit only, from a phase-1 workspace
  int phase = 0;
  int64_t capacity = INT64_MAX;  // output columns available (emit clamps)
};

__host__ __device__ inline int key_words_for_bits(int bits) {
  const int kw = (bits + 63) / 64;
  int p = 1;
  while (p < kw) p <<= 1;
  return p;
}

__host__ __device__ inline u64 low_mask(int len) { return len >= 64 ? ~0ull : ((1ull << len) - 1); }

template <int KW>
__device__ __forceinline__ void put_seg(u64 (&key)[KW], u64 v, int pos, int len) {
  const int wi = pos >> 6, off = pos & 63;
  const int shift = 64 - off - len;
  const u64 a = shift >= 0 ? (v << shift) : (v >> (-shift));
  const u64 b = shift >= 0 ? 0ull : (v << (64 + shift));
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    if (d == wi) key[d] |= a;
    if (d == wi + 1) key[d] |= b;
  }
}

template <int KW>
__device__ __forceinline__ u64 get_seg(const u64 (&key)[KW], int pos, int len) {
  const int wi = pos >> 6, off = pos & 63;
  u64 a = 0, b = 0;
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    if (d == wi) a = key[d];
    if (d == wi + 1) b = key[d];
  }
  const u64 hi = off ? ((a << off) | (b >> (64 - off))) : a;
  return hi >> (64 - len);
}

// canonical words (z[W], x[W]) -> packed key
template <int W, int KW>
__device__ __forceinline__ void pack_key(const Layout& L, const u64 (&zc)[W], const u64 (&xc)[W],
                                         u64 (&key)[KW]) {
#pragma unroll
  for (int d = 0; d < KW; ++d) key[d] = 0;
  if (L.sparse) {
    int k = 0;
#pragma unroll
    for (int s = 0; s < 2 * W; ++s) {
      const int len = L.len[s];
      if (!len) continue;
      u64 w = ((s < W ? zc[s] : xc[s - W]) >> L.lo[s]) & low_mask(len);
      while (w) {  // segment bits, most significant first
        const int hb = 63 - __clzll((long long)w);
        w ^= 1ull << hb;
        const int p = L.pos[s] + (len - 1 - hb);
        put_seg<KW>(key, (u64)(L.key_bits - p), k * L.sbits, L.sbits);
        ++k;
      }
    }
    return;
  }
#pragma unroll
  for (int s = 0; s < 2 * W; ++s) {
    const int len = L.len[s];
    if (len) {
      const u64 w = s < W ? zc[s] : xc[s - W];
      put_seg<KW>(key, (w >> L.lo[s]) & low_mask(len), L.pos[s], len);
    }
  }
}

// Packed position of slot k of the sparse key staged at KS[d * T + e]
// (INT_MAX past the last slot / at the terminator).
__device__ __forceinline__ int sparse_slot_pos(const Layout& L, const u64* KS, int T, int e, int k) {
  if (k >= L.nslots) return INT_MAX;
  const int bit = k * L.sbits, wi = bit >> 6, off = bit & 63;
  const u64 a = KS[wi * T + e];
  const u64 b = off + L.sbits > 64 ? KS[(wi + 1) * T + e] : 0ull;
  const u64 hiw = off ? ((a << off) | (b >> (64 - off))) : a;
  const u64 v = hiw >> (64 - L.sbits);
  return v == 0 ? INT_MAX : L.key_bits - (int)v;
}

// Plane word q of a sparse key, consuming the slots from cursor k on (planes
// are visited in order, so every slot whose position precedes plane q's range
// was consumed by an earlier plane).  p is the decoded position of slot k:
// a slot is decoded once, not once per plane it is compared with.
__device__ __forceinline__ u64 sparse_plane_next(const Layout& L, const u64* KS, int T, int e,
                                                 int q, int& k, int& p) {
  const int len = L.len[q];
  const int lo = L.pos[q], hi = L.pos[q] + len;
  u64 w = 0;
  while (p < hi) {
    w |= 1ull << (L.lo[q] + len - 1 - (p - lo));
    p = sparse_slot_pos(L, KS, T, e, ++k);
  }
  return w;
}

template <int KW>
__device__ __forceinline__ void load_key(const u64* k, int64_t stride, int64_t i, u64 (&key)[KW]) {
#pragma unroll
  for (int d = 0; d < KW; ++d) key[d] = k[d * stride + i];
}

template <int KW>
__device__ __forceinline__ void store_key(u64* k, int64_t stride, int64_t i, const u64 (&key)[KW]) {
#pragma unroll
  for (int d = 0; d < KW; ++d) k[d * stride + i] = key[d];
}

// Item keys in global memory (buffers k1 / k2) are stored row-major: the KW
// words of item i at k[i * KW .. i * KW + KW), 16-byte aligned for KW >= 2,
// so an item's key moves as 128-bit accesses and a run of items scattered to
// one bucket fills whole sectors (plane-major runs of 2-4 items left every
// sector a quarter full: k_split_scatter 1.43 -> 1.02 ms).
template <int KW>
__device__ __forceinline__ void load_row(const u64* k, int64_t i, u64 (&key)[KW]) {
  if constexpr (KW == 1) {
    key[0] = k[i];
  } else {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(k + i * KW);
#pragma unroll
    for (int d = 0; d < KW / 2; ++d) {
      const ulonglong2 v = p[d];
      key[2 * d] = v.x;
      key[2 * d + 1] = v.y;
    }
  }
}

template <int KW>
__device__ __forceinline__ void store_row(u64* k, int64_t i, const u64 (&key)[KW]) {
  if constexpr (KW == 1) {
    k[i] = key[0];
  } else {
    ulonglong2* p = reinterpret_cast<ulonglong2*>(k + i * KW);
#pragma unroll
    for (int d = 0; d < KW / 2; ++d) p[d] = make_ulonglong2(key[2 * d], key[2 * d + 1]);
  }
}

// key <= splitter[b] ?  (lexicographic)
template <int KW>
__device__ __forceinline__ bool key_lt(const u64 (&a)[KW], const u64* s, int64_t stride, int b) {
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    const u64 v = s[d * stride + b];
    if (a[d] != v) return a[d] < v;
  }
  return false;
}

// number of splitters <= key  (upper bound); splitters s[0..nsp)
template <int KW>
__device__ __forceinline__ int bucket_of(const u64 (&key)[KW], const u64* s, int64_t stride,
                                         int nsp) {
  int lo = 0, hi = nsp;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key_lt<KW>(key, s, stride, mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// item order: (key, ik)
template <int KW>
__device__ __forceinline__ bool item_lt(const u64* K, const uint32_t* I, int64_t stride, int a,
                                        int b) {
#pragma unroll
  for (int d = 0; d < KW; ++d) {
    const u64 ka = K[d * stride + a], kb = K[d * stride + b];
    if (ka != kb) return ka < kb;
  }
  return I[a] < I[b];
}

template <int KW>
__device__ __forceinline__ bool key_eq(const u64* K, int64_t stride, int a, int b) {
#pragma unroll
  for (int d = 0; d < KW; ++d)
    if (K[d * stride + a] != K[d * stride + b]) return false;
  return true;
}

// Block-wide bitonic sort (all comparators ascending; elements at index >= n
// behave as +inf so no padding is stored).  Works on shared or global memory.
template <int KW>
__device__ void bitonic_sort(u64* K, uint32_t* I, int64_t stride, int n) {
  int npow = 1;
  while (npow < n) npow <<= 1;
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (npow >> 1); t += blockDim.x) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i + j);
        if (p < n && item_lt<KW>(K, I, stride, p, i)) {
#pragma unroll
          for (int d = 0; d < KW; ++d) {
            const u64 tmp = K[d * stride + i];
            K[d * stride + i] = K[d * stride + p];
            K[d * stride + p] = tmp;
          }
          const uint32_t ti = I[i];
          I[i] = I[p];
          I[p] = ti;
        }
      }
      __syncthreads();
    }
  }
}

// Complex product rounded exactly like numpy's complex128 multiply on
// FMA-capable x86 hosts (the reference's sums.py:141):
//   re = fma(ar, br, -(ai*bi)),  im = fma(ar, bi, ai*br)
// (verified bit-for-bit against numpy 2.3.5).
__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

// c * i^k  (exact)
__device__ __forceinline__ double2 rot_ik(double2 c, int k) {
  switch (k & 3) {
    case 0: return c;
    case 1: return make_double2(-c.y, c.x);
    case 2: return make_double2(-c.x, -c.y);
    default: return make_double2(c.y, -c.x);
  }
}

// ------------------------------------------------------------ item sources
// MODE 0: outer product A*B; MODE 1: one sum (sort_and_combine).
template <int W, int KW, int MODE>
struct Source {
  // key + phase of raw item r (used by the sampler; slow path, global loads)
  static __device__ __forceinline__ void item_at(const Layout& L, const SrcA& S, int64_t ma,
                                                 int64_t r, u64 (&key)[KW], int& k) {
    u64 zc[W], xc[W];
    if (MODE == 0) {
      const int64_t j = (uint32_t)r / (uint32_t)ma, i = r - j * ma;
      k = (S.ak ? S.ak[i] : 0) + (S.bk ? S.bk[j] : 0);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (L.active >> w & 1) {
          const u64 a_x = S.ax[w * S.lda + i], a_z = S.az[w * S.lda + i];
          const u64 b_x = S.bx[w * S.ldb + j], b_z = S.bz[w * S.ldb + j];
          k += phase_word(a_x, a_z, b_x, b_z);
          xc[w] = a_x ^ b_x;
          zc[w] = a_z ^ b_z;
        } else {
          xc[w] = zc[w] = 0;
        }
      }
    } else {
      k = S.ak ? S.ak[r] : 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const bool on = L.active >> w & 1;
        xc[w] = on ? S.ax[w * S.lda + r] : 0ull;
        zc[w] = on ? S.az[w * S.lda + r] : 0ull;
      }
    }
    pack_key<W, KW>(L, zc, xc, key);
  }

  static __device__ __forceinline__ double2 coef(const SrcA& S, int64_t ma, uint32_t ik) {
    const int64_t r = ik >> 2;
    if (MODE == 0) {
      const int64_t j = div_ma((uint32_t)r, S.ma_inv), i = r - j * ma;
      return rot_ik(cmul_np(S.ac[i], S.bc[j]), (int)(ik & 3));
    } else {
      return rot_ik(S.ac[r], (int)(ik & 3));
    }
  }
};

// Sum of one run of equal keys in raw-row order, reproducing numpy's
// np.add.reduceat (sums.py:112) bit for bit: out = c0 + pairwise(c1..c{m-1}),
// where numpy's pairwise sum (complex128, PW_BLOCKSIZE 128 doubles) adds
// fewer than 4 elements left to right from -0.0, blocks of <= 64 elements
// with 4 interleaved accumulators ((r0+r1)+(r2+r3)) plus a sequential tail,
// and splits longer ranges at a multiple of 4 elements near the middle.
// Verified against numpy 2.3.5.
template <int W, int KW, int MODE>
struct RunSum {
  static __device__ __forceinline__ double2 c(const SrcA& S, int64_t ma, const uint32_t* I,
                                              int64_t e) {
    return Source<W, KW, MODE>::coef(S, ma, I[e]);
  }
  static __device__ double2 block(const SrcA& S, int64_t ma, const uint32_t* I, int64_t b,
                                  int64_t L) {
    if (L < 4) {
      double rr = -0.0, ri = -0.0;
      for (int64_t e = 0; e < L; ++e) {
        const double2 v = c(S, ma, I, b + e);
        rr = __dadd_rn(rr, v.x);
        ri = __dadd_rn(ri, v.y);
      }
      return make_double2(rr, ri);
    }
    double2 r0 = c(S, ma, I, b), r1 = c(S, ma, I, b + 1), r2 = c(S, ma, I, b + 2),
            r3 = c(S, ma, I, b + 3);
    int64_t i = 4;
    const int64_t lim = L - (L % 4);
    for (; i < lim; i += 4) {
      const double2 v0 = c(S, ma, I, b + i), v1 = c(S, ma, I, b + i + 1);
      const double2 v2 = c(S, ma, I, b + i + 2), v3 = c(S, ma, I, b + i + 3);
      r0.x = __dadd_rn(r0.x, v0.x); r0.y = __dadd_rn(r0.y, v0.y);
      r1.x = __dadd_rn(r1.x, v1.x); r1.y = __dadd_rn(r1.y, v1.y);
      r2.x = __dadd_rn(r2.x, v2.x); r2.y = __dadd_rn(r2.y, v2.y);
      r3.x = __dadd_rn(r3.x, v3.x); r3.y = __dadd_rn(r3.y, v3.y);
    }
    double rr = __dadd_rn(__dadd_rn(r0.x, r1.x), __dadd_rn(r2.x, r3.x));
    double ri = __dadd_rn(__dadd_rn(r0.y, r1.y), __dadd_rn(r2.y, r3.y));
    for (; i < L; ++i) {
      const double2 v = c(S, ma, I, b + i);
      rr = __dadd_rn(rr, v.x);
      ri = __dadd_rn(ri, v.y);
    }
    return make_double2(rr, ri);
  }
  // numpy's recursive split, evaluated with an explicit stack (depth <= 25
  // for runs < 2^30; device recursion would overflow the default stack)
  static __device__ __noinline__ double2 pairwise(const SrcA& S, int64_t ma, const uint32_t* I,
                                                  int64_t b, int64_t L) {
    int64_t sb[32], sl[32];
    double2 left[32];
    int sp = 0;
    sb[0] = b;
    sl[0] = L;
    for (;;) {
      while (sl[sp] > 64) {  // descend into left halves
        sb[sp + 1] = sb[sp];
        sl[sp + 1] = (sl[sp] - (sl[sp] % 8)) / 2;
        left[sp].x = __longlong_as_double(-1);  // marker: left half pending
        ++sp;
      }
      double2 r = block(S, ma, I, sb[sp], sl[sp]);
      for (;;) {  // ascend
        if (sp == 0) return r;
        --sp;
        if (__double_as_longlong(left[sp].x) == -1LL) {  // r is the left half: go right
          left[sp] = r;
          const int64_t e1 = (sl[sp] - (sl[sp] % 8)) / 2;
          sb[sp + 1] = sb[sp] + e1;
          sl[sp + 1] = sl[sp] - e1;
          ++sp;
          break;
        }
        r = make_double2(__dadd_rn(left[sp].x, r.x), __dadd_rn(left[sp].y, r.y));
      }
    }
  }
  static __device__ __forceinline__ double2 run(const SrcA& S, int64_t ma, const uint32_t* I,
                                                int64_t p, int64_t m) {
    const double2 c0 = c(S, ma, I, p);
    if (m == 1) return c0;
    const double2 r = m - 1 <= 64 ? block(S, ma, I, p + 1, m - 1) : pairwise(S, ma, I, p + 1, m - 1);
    return make_double2(__dadd_rn(c0.x, r.x), __dadd_rn(c0.y, r.y));
  }
};

// ------------------------------------------------- sample sorting (one CTA)
// Sorts ns keys K[KW][ns] (shared memory) through 64-bit composites CK[npow]:
// the 64 key bits after the first cp bits (a prefix every key shares) with the
// low 13 bits replaced by the sample index -- one compare per exchange
// instead of KW words + index -- then finishes every run of equal composite
// prefixes on the full keys by insertion sort.  A run longer than 64 (keys
// equal over those 64 bits) makes it fall back to a full-key bitonic sort.
// Returns (all threads) the sorted position -> sample index map via `order`:
// order(p) = CK[p] & 0x1FFF, or p itself after the fallback (K then sorted).
template <int KW>
__device__ bool sort_samples(u64* K, int ns, u64* CK, int cp) {
  int npow = 1;
  while (npow < ns) npow <<= 1;
  for (int s = threadIdx.x; s < npow; s += blockDim.x) {
    if (s < ns) {
      u64 key[KW];
      load_key<KW>(K, ns, s, key);
      CK[s] = (get_seg<KW>(key, cp, 64) & ~0x1FFFull) | (u64)s;
    } else {
      CK[s] = ~0ull;
    }
  }
  __syncthreads();
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (npow >> 1); t += blockDim.x) {
        const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int b = (j == (k >> 1)) ? (a ^ (k - 1)) : (a + j);
        const u64 va = CK[a], vb = CK[b];
        if (vb < va) {
          CK[a] = vb;
          CK[b] = va;
        }
      }
      __syncthreads();
    }
  }
  __shared__ int s_long;
  if (threadIdx.x == 0) s_long = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < ns; q += blockDim.x) {
    const u64 pre = CK[q] >> 13;
    if ((q > 0 && (CK[q - 1] >> 13) == pre) || q + 1 >= ns || (CK[q + 1] >> 13) != pre) continue;
    int e = q + 1;
    while (e < ns && (CK[e] >> 13) == pre && e - q <= 64) ++e;
    if (e - q > 64) {
      s_long = 1;
      continue;
    }
    for (int a = q + 1; a < e; ++a) {
      const u64 v = CK[a];
      const int va = (int)(v & 0x1FFF);
      int b = a;
      while (b > q) {
        const int vb = (int)(CK[b - 1] & 0x1FFF);
        bool lt = false;
#pragma unroll
        for (int d = 0; d < KW; ++d) {
          const u64 x = K[d * ns + va], y = K[d * ns + vb];
          if (x != y) {
            lt = x < y;
            break;
          }
        }
        if (!lt) break;
        CK[b] = CK[b - 1];
        --b;
      }
      CK[b] = v;
    }
  }
  __syncthreads();
  if (!s_long) return true;
  uint32_t* I = reinterpret_cast<uint32_t*>(CK);
  for (int t = threadIdx.x; t < ns; t += blockDim.x) I[t] = (uint32_t)t;
  __syncthreads();
  bitonic_sort<KW>(K, I, ns, ns);
  return false;
}

__host__ __device__ inline int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

static inline size_t sample_smem_bytes(int ns, int KW) {
  return (size_t)ns * 8 * KW + (size_t)pow2_ceil(ns) * 8 + 16;
}

// level-1 prefix table: tab[h] = number of splitters whose top kTabBits bits
// are < h (h = 0 .. 2^kTabBits); a key with prefix h lies after splitter
// tab[h]-1 and before splitter tab[h+1], so only [tab[h], tab[h+1]) is searched
__device__ __forceinline__ void l1_table_fill(const Dims& D, const Ctl& C, int first, int stride) {
  const int nsp = D.nb1 - 1;
  for (int h = first; h <= (1 << kTabBits); h += stride) {
    int lo = 0, hi = nsp;  // first splitter with prefix >= h
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)(C.split[mid] >> (64 - kTabBits)) < (int64_t)h) lo = mid + 1;
      else hi = mid;
    }
    C.l1tab[h] = (uint16_t)lo;
  }
}

// ------------------------------------------------------------- 1. sampler
// One CTA: ns deterministic sample keys of the product (raw rows spread
// evenly), sorted, every (ns/nb1)-th taken as a level-1 splitter.  The sort
// runs on 64-bit composites (key word 0 with its low 13 bits replaced by the
// sample index: one compare per exchange instead of KW words + index), then
// every run of equal composite prefixes is finished on the full keys by
// insertion sort (rare), so the splitters are exactly the sorted samples.
template <int W, int KW, int MODE>
__global__ void __launch_bounds__(kLeafThreads)
k_sample(Layout L, Dims D, SrcA S, Ctl C) {
  extern __shared__ u64 sm[];
  const int ns = D.nsamp;
  u64* K = sm;                        // [KW][ns] sample keys
  u64* CK = K + (int64_t)KW * ns;     // [npow] composites
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const int64_t r = ((2 * (int64_t)s + 1) * D.n_space) / (2 * (int64_t)ns);
    u64 key[KW];
    // packed keys of the operands are already in C.opk (k_pack_ops)
    if (MODE == 1) {
#pragma unroll
      for (int d = 0; d < KW; ++d) key[d] = C.opk[d * D.ma + r];
    } else {
      const int64_t nops = D.ma + D.mb_all;
      const int64_t j = r / D.ma, i = r - j * D.ma;
#pragma unroll
      for (int d = 0; d < KW; ++d) key[d] = C.opk[d * nops + i] ^ C.opk[d * nops + D.ma + j];
    }
    store_key<KW>(K, ns, s, key);
  }
  __syncthreads();
  const bool composite = sort_samples<KW>(K, ns, CK, 0);
  for (int b = 1 + threadIdx.x; b < D.nb1; b += blockDim.x) {
    const int pos = (int)(((int64_t)b * ns) / D.nb1);
    const int src = composite ? (int)(CK[pos] & 0x1FFF) : pos;
#pragma unroll
    for (int d = 0; d < KW; ++d) C.split[d * D.nb1 + (b - 1)] = K[d * ns + src];
  }
  // level-1 prefix table in the same launch (the splitters are this CTA's own writes)
  __syncthreads();
  l1_table_fill(D, C, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------- 2./4. count, scatter
// Packing is a fixed bit permutation, so it commutes with XOR: the key of the
// product a_i*b_j is pack(a_i) ^ pack(b_j).  k_pack_ops packs every operand
// term once (and its base phase k + popc(x&z), sums.py:156-157); the item
// generators then need KW XORs for the key and, per active word, the cross
// phase 2popc(az&bx) - popc((ax^bx)&(az^bz)) (sums.py:134-136).
// Sparse key of one term (Layout::sparse): its set bits in packed order (the
// segments in order, each from its high bit down) appended as sbits-wide
// values key_bits - p into a bit stream, MSB first, 0-terminated.  One loop
// over the term's set bits with a segment cursor (the segment words staged in
// shared memory, so no divergent per-segment loops), a 64-bit accumulator
// flushed into the key words by a static select.
template <int W, int KW>
__device__ __forceinline__ void pack_sparse(const Layout& L, const u64 (&seg)[2 * W],
                                            u64 (&key)[KW]) {
#pragma unroll
  for (int d = 0; d < KW; ++d) key[d] = 0;
  u64 acc = 0;
  int fill = 0, wi = 0;  // bits in acc, key word being filled
  auto flush = [&](u64 v) {
#pragma unroll
    for (int d = 0; d < KW; ++d)
      if (d == wi) key[d] = v;
    ++wi;
  };
  const int nb = L.sbits;
  // the segments in order (a uniform, unrolled loop: the words stay in
  // registers), each from its high bit down
#pragma unroll
  for (int s = 0; s < 2 * W; ++s) {
    u64 w = seg[s];
    const int top = L.key_bits - (L.pos[s] + L.len[s] - 1);  // value of the segment's bit 0 ... + hb
    while (w) {
      const int hb = 63 - __clzll((long long)w);
      w ^= 1ull << hb;
      const u64 v = (u64)(top + hb);  // = key_bits - p with p = pos + (len - 1 - hb)
      if (fill + nb < 64) {
        acc |= v << (64 - fill - nb);
        fill += nb;
      } else {
        const int r = fill + nb - 64;  // bits spilling into the next word
        acc |= v >> r;
        flush(acc);
        acc = r ? v << (64 - r) : 0ull;
        fill = r;
      }
    }
  }
  if (fill && wi < KW) flush(acc);  // the zero terminator is the zero tail
}

template <int W, int KW, int MODE>
__global__ void __launch_bounds__(256, 4) k_pack_ops(Layout L, SrcA S, int64_t ma, int64_t mb, Ctl C) {
  const int64_t n = ma + (MODE == 0 ? mb : 0);
  if constexpr (MODE == 1 && W <= 8) if (L.sparse) {
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < n; t0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t t = t0 + threadIdx.x;
      if (t < n) {
        int base = S.ak ? S.ak[t] : 0;
        u64 seg[2 * W];
#pragma unroll
        for (int q = 0; q < 2 * W; ++q) {  // all plane loads in flight together
          const int w = q < W ? q : q - W;
          seg[q] = L.len[q] ? (q < W ? S.az : S.ax)[w * S.lda + t] : 0ull;
        }
#pragma unroll
        for (int q = 0; q < 2 * W; ++q) seg[q] = (seg[q] >> L.lo[q]) & low_mask(L.len[q]);
        u64 key[KW];
        pack_sparse<W, KW>(L, seg, key);
#pragma unroll
        for (int d = 0; d < KW; ++d) C.opk[d * n + t] = key[d];
        C.opb[t] = (uint8_t)(base & 3);
      }
    }
    return;
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const bool isb = t >= ma;
    const int64_t r = isb ? t - ma : t;
    const u64* X = isb ? S.bx : S.ax;
    const u64* Z = isb ? S.bz : S.az;
    const uint8_t* K = isb ? S.bk : S.ak;
    const int64_t ld = isb ? S.ldb : S.lda;
    u64 zc[W], xc[W];
    int base = K ? K[r] : 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const bool on = L.active >> w & 1;
      xc[w] = on ? X[w * ld + r] : 0ull;
      zc[w] = on ? Z[w * ld + r] : 0ull;
      if (MODE == 0) base += popc64(xc[w] & zc[w]);
    }
    u64 key[KW];
    pack_key<W, KW>(L, zc, xc, key);
#pragma unroll
    for (int d = 0; d < KW; ++d) C.opk[d * n + t] = key[d];
    C.opb[t] = (uint8_t)(base & 3);
  }
}

// Shared memory: splitters [KW][nb1] | hist nb1 | gbase nb1 | b tile | (b, r) per item
struct GenSmem {
  u64* split;
  uint32_t* hist;
  uint32_t* gbase;
  u64* tile;       // outer: [2W][kTileB] b-term words (z then x)
  u64* tkey;       // outer: [KW][kTileB] packed b-term keys
  uint32_t* tpb;   // outer: [kTileB] b-term base phases
  uint32_t* tj;    // outer: [kTileB] b-term operand index (raw row = j * ma + i)
  uint32_t* slot;  // per item: bucket << 16 | rank  (scatter only)
  uint16_t* tab;   // level-1 prefix table (2^kTabBits + 1)
};

// search = false (k_scatter): no splitters and no prefix table
template <int W>
__device__ __forceinline__ GenSmem gen_smem(u64* sm, int nb1, int KW, bool search = true) {
  GenSmem g;
  g.split = sm;
  g.hist = reinterpret_cast<uint32_t*>(sm + (search ? (int64_t)KW * nb1 : 0));
  g.gbase = g.hist + nb1;
  g.tile = reinterpret_cast<u64*>(g.gbase + nb1);  // 2*nb1 u32 keeps 8-byte alignment
  g.tkey = g.tile + 2 * W * kTileB;
  g.tpb = reinterpret_cast<uint32_t*>(g.tkey + KW * kTileB);
  g.tj = g.tpb + kTileB;
  g.slot = g.tj + kTileB;
  g.tab = reinterpret_cast<uint16_t*>(g.slot + kGenTB * kGenThreads);
  return g;
}

__host__ __device__ constexpr size_t gen_smem_bytes(int W, int KW, int nb1, bool search = true) {
  return (search ? (size_t)8 * KW * nb1 : 0) + 8 * (size_t)nb1 + 8 + (size_t)16 * W * kTileB +
         (size_t)8 * KW * kTileB + 8 * (size_t)kTileB + (size_t)4 * kGenTB * kGenThreads +
         (search ? 2 * (size_t)((1 << kTabBits) + 1) : 0) + 64;
}

template <int KW>
__device__ __forceinline__ void gen_prologue(const GenSmem& g, const Ctl& C, int nb1) {
  for (int h = threadIdx.x; h <= (1 << kTabBits); h += blockDim.x) g.tab[h] = C.l1tab[h];
  for (int b = threadIdx.x; b < nb1; b += blockDim.x) {
    g.hist[b] = 0;
    if (b < nb1 - 1) {
#pragma unroll
      for (int d = 0; d < KW; ++d) g.split[d * nb1 + b] = C.split[d * nb1 + b];
    }
  }
}

// Per-thread item generator.
// Outer: the CTA owns the tile (sorted A positions [blockIdx.x*kTileA, +kTileA)) x
// (sorted B positions [blockIdx.y*kTileB, +kTileB)).  Operands are visited in
// packed-key order (C.perm, k_sort_ops), so a tile's products share a long key
// prefix and land in a few level-1 buckets: the bucket runs written per CTA are
// long (coalesced) instead of ~8 items in each of 512 buckets.  Thread t takes
// A-term t % kTileA and the kGenTB B-terms of group t / kTileA; a warp's lanes
// share the B-term of every step (shared-memory broadcast).  Raw rows use the
// ORIGINAL operand indices (raw row j*Ma + i, sums.py:137), so the (key, ik)
// order and every run sum are unchanged.
// Sort: thread handles terms base + jj*blockDim + tid.
template <int W, int KW, int MODE>
struct Gen {
  u64 ax[W], az[W], ka[KW];
  int pa;
  int64_t i;
  bool valid_i;

  __device__ __forceinline__ void init(const Layout& L, const Dims& D, const SrcA& S,
                                       const Ctl& C, const GenSmem& g) {
    if (MODE == 0) {
      const int64_t is = (int64_t)blockIdx.x * kTileA + (threadIdx.x % kTileA);
      valid_i = is < D.ma;
      i = valid_i ? C.perm[is] : 0;
      const int64_t nops = D.ma + D.mb_all;
      const int64_t js0 = (int64_t)blockIdx.y * kTileB;  // local sorted B position
      // b tile into shared memory: operand index, active z words then x words,
      // packed keys, base phases
      for (int jj = threadIdx.x; jj < kTileB; jj += blockDim.x) {
        const int64_t js = js0 + jj;
        g.tj[jj] = js < D.mb ? (uint32_t)C.perm[D.ma + js] : 0u;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < 2 * W * kTileB; t += blockDim.x) {
        const int s = t / kTileB, jj = t % kTileB;
        const int w = s < W ? s : s - W;
        const int64_t j = g.tj[jj];
        u64 v = 0;
        if (js0 + jj < D.mb && (L.active >> w & 1))
          v = s < W ? S.bz[w * S.ldb + j] : S.bx[w * S.ldb + j];
        g.tile[s * kTileB + jj] = v;
      }
      for (int t = threadIdx.x; t < KW * kTileB; t += blockDim.x) {
        const int d = t / kTileB, jj = t % kTileB;
        g.tkey[t] = js0 + jj < D.mb ? C.opk[d * nops + D.ma + g.tj[jj]] : 0ull;
      }
      for (int jj = threadIdx.x; jj < kTileB; jj += blockDim.x)
        g.tpb[jj] = js0 + jj < D.mb ? C.opb[D.ma + g.tj[jj]] : 0u;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const bool on = valid_i && (L.active >> w & 1);
        ax[w] = on ? S.ax[w * S.lda + i] : 0ull;
        az[w] = on ? S.az[w * S.lda + i] : 0ull;
      }
#pragma unroll
      for (int d = 0; d < KW; ++d) ka[d] = valid_i ? C.opk[d * nops + i] : 0ull;
      pa = valid_i ? C.opb[i] : 0;
    }
  }

  // whether item jj of this thread exists (no loads)
  __device__ __forceinline__ bool valid(const Dims& D, int jj) const {
    if (MODE == 0) {
      const int bb = (threadIdx.x / kTileA) * kGenTB + jj;
      return valid_i && (int64_t)blockIdx.y * kTileB + bb < D.mb;
    }
    return (int64_t)blockIdx.x * blockDim.x * kGenTB + (int64_t)jj * blockDim.x + threadIdx.x < D.n;
  }
  // slot of item jj in the per-item bucket-id array (coalesced over threads)
  static __device__ __forceinline__ int64_t slot_of(int jj) {
    const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    return (blk * kGenTB + jj) * kGenThreads + threadIdx.x;
  }

  // item jj of this thread: returns false when out of range
  __device__ __forceinline__ bool item(const Layout& L, const Dims& D, const Ctl& C,
                                       const GenSmem& g, int jj, u64 (&key)[KW], uint32_t& ik) {
    int64_t r;
    int k;
    if (MODE == 0) {
      const int bb = (threadIdx.x / kTileA) * kGenTB + jj;  // slot in the B tile
      if (!valid_i || (int64_t)blockIdx.y * kTileB + bb >= D.mb) return false;
      k = pa + (int)g.tpb[bb];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (L.active >> w & 1) {
          const u64 b_z = g.tile[w * kTileB + bb], b_x = g.tile[(W + w) * kTileB + bb];
          k += 2 * popc64(az[w] & b_x) - popc64((ax[w] ^ b_x) & (az[w] ^ b_z));
        }
      }
#pragma unroll
      for (int d = 0; d < KW; ++d) key[d] = ka[d] ^ g.tkey[d * kTileB + bb];
      r = (int64_t)g.tj[bb] * D.ma + i;
    } else {
      r = (int64_t)blockIdx.x * blockDim.x * kGenTB + (int64_t)jj * blockDim.x + threadIdx.x;
      if (r >= D.n) return false;
      k = C.opb[r];
#pragma unroll
      for (int d = 0; d < KW; ++d) key[d] = C.opk[d * D.ma + r];
    }
    ik = ((uint32_t)r << 2) | (uint32_t)(k & 3);
    return true;
  }
};

// Operand order for the outer-product tiles: each CTA sorts one chunk of up
// to kSortOpsChunk terms of A (blocks [0, nca)) or of B's local columns (the
// rest) by the top 50 bits of packed key word 0, via a shared-memory bitonic
// sort of (key & ~0x3FFF) | local index, and writes sorted position ->
// operand index into C.perm.  Only the locality of the tiles depends on it.
template <int KW>
__global__ void __launch_bounds__(1024) k_sort_ops(Dims D, Ctl C) {
  extern __shared__ u64 sm[];
  const int64_t nops = D.ma + D.mb_all;
  const int nca = (int)ceil_div(D.ma, kSortOpsChunk);
  const bool isb = (int)blockIdx.x >= nca;
  const int64_t c0 = (int64_t)(isb ? blockIdx.x - nca : blockIdx.x) * kSortOpsChunk;
  const int64_t n_all = isb ? D.mb : D.ma;
  const int n = (int)min((int64_t)kSortOpsChunk, n_all - c0);
  if (n <= 0) return;
  // operand index of local position e: A term c0 + e, or B column j0 + c0 + e
  const int64_t op0 = isb ? D.ma + D.j0 + c0 : c0;
  int npow = 1;
  while (npow < n) npow <<= 1;
  for (int e = threadIdx.x; e < npow; e += blockDim.x)
    sm[e] = e < n ? ((C.opk[op0 + e] & ~0x3FFFull) | (u64)e) : ~0ull;
  __syncthreads();
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (npow >> 1); t += blockDim.x) {
        const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int b = (j == (k >> 1)) ? (a ^ (k - 1)) : (a + j);
        const u64 va = sm[a], vb = sm[b];
        if (vb < va) {
          sm[a] = vb;
          sm[b] = va;
        }
      }
      __syncthreads();
    }
  }
  int32_t* out = C.perm + (isb ? D.ma : 0) + c0;
  const int64_t base = isb ? D.j0 + c0 : c0;  // B: global column index
  for (int e = threadIdx.x; e < n; e += blockDim.x) out[e] = (int32_t)(base + (sm[e] & 0x3FFF));
  (void)nops;
}

__device__ __forceinline__ int pow2_floor(int v) { return v > 0 ? 1 << (31 - __clz(v)) : 0; }

constexpr int kGenIlp = 4;  // independent items per thread in flight

template <int W, int KW, int MODE>
__global__ void __launch_bounds__(kGenThreads)
k_count(Layout L, Dims D, SrcA S, Ctl C) {
  extern __shared__ u64 sm[];
  const GenSmem g = gen_smem<W>(sm, D.nb1, KW);
  gen_prologue<KW>(g, C, D.nb1);
  Gen<W, KW, MODE> gen;
  gen.init(L, D, S, C, g);
  __syncthreads();
#pragma unroll 1
  for (int j0 = 0; j0 < kGenTB; j0 += kGenIlp) {
    u64 key[kGenIlp][KW];
    bool ok[kGenIlp];
    int pos[kGenIlp];
#pragma unroll
    for (int u = 0; u < kGenIlp; ++u) {
      uint32_t ik;
      ok[u] = gen.item(L, D, C, g, j0 + u, key[u], ik);
      pos[u] = 0;
    }
    // the prefix table narrows each search to the splitters sharing the
    // key's top kTabBits bits (usually none or a few)
    int hi[kGenIlp], step[kGenIlp];
    int smax = 0;
#pragma unroll
    for (int u = 0; u < kGenIlp; ++u) {
      const int h = (int)(key[u][0] >> (64 - kTabBits));
      pos[u] = g.tab[h];
      hi[u] = g.tab[h + 1];
      step[u] = pow2_floor(hi[u] - pos[u]);
      smax = step[u] > smax ? step[u] : smax;
    }
    for (int st = smax; st > 0; st >>= 1) {
#pragma unroll
      for (int u = 0; u < kGenIlp; ++u) {
        if (step[u] >= st) {
          const int c = pos[u] + st;
          if (c <= hi[u] && !key_lt<KW>(key[u], g.split, D.nb1, c - 1)) pos[u] = c;
        }
      }
    }
    // the bucket of every item is kept for k_scatter (no second search)
#pragma unroll
    for (int u = 0; u < kGenIlp; ++u)
      C.bid[Gen<W, KW, MODE>::slot_of(j0 + u)] = (uint16_t)pos[u];
    // warp-aggregated histogram: a tile's items share few buckets
#pragma unroll
    for (int u = 0; u < kGenIlp; ++u) {
      const unsigned act = __ballot_sync(0xffffffffu, ok[u]);
      if (ok[u]) {
        const unsigned peers = __match_any_sync(act, pos[u]);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&g.hist[pos[u]], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < D.nb1; b += blockDim.x)
    if (g.hist[b]) atomicAdd(&C.bcount[b], g.hist[b]);
}

template <int W, int KW, int MODE>
__global__ void __launch_bounds__(kGenThreads, W <= 8 ? 4 : 3)
k_scatter(Layout L, Dims D, SrcA S, Ctl C) {
  extern __shared__ u64 sm[];
  const GenSmem g = gen_smem<W>(sm, D.nb1, KW, false);
  for (int b = threadIdx.x; b < D.nb1; b += blockDim.x) g.hist[b] = 0;
  Gen<W, KW, MODE> gen;
  gen.init(L, D, S, C, g);
  __syncthreads();
  // bucket ids come from k_count (a single bucket needs none); lanes with the
  // same bucket get consecutive slots (warp-aggregated ranks)
  const bool one = D.nb1 == 1;
  const int lane = threadIdx.x & 31;
  uint16_t bids[kGenTB];  // all id loads in flight together
#pragma unroll
  for (int jj = 0; jj < kGenTB; ++jj)
    bids[jj] = (!one && gen.valid(D, jj)) ? C.bid[Gen<W, KW, MODE>::slot_of(jj)] : (uint16_t)0;
#pragma unroll
  for (int jj = 0; jj < kGenTB; ++jj) {
    const bool ok = gen.valid(D, jj);
    const int pos = bids[jj];
    uint32_t code = 0xFFFFFFFFu;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const unsigned peers = __match_any_sync(act, pos);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(&g.hist[pos], (uint32_t)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      code = ((uint32_t)pos << 16) | (base + __popc(peers & ((1u << lane) - 1u)));
    }
    g.slot[jj * kGenThreads + threadIdx.x] = code;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < D.nb1; b += blockDim.x)
    if (g.hist[b]) g.gbase[b] = atomicAdd(&C.bcursor[b], g.hist[b]);
  __syncthreads();
#pragma unroll 4
  for (int jj = 0; jj < kGenTB; ++jj) {
    const uint32_t code = g.slot[jj * kGenThreads + threadIdx.x];
    if (code == 0xFFFFFFFFu) continue;
    u64 key[KW];
    uint32_t ik;
    gen.item(L, D, C, g, jj, key, ik);
    const uint32_t pos = g.gbase[code >> 16] + (code & 0xFFFFu);
    store_row<KW>(C.k1, pos, key);
    C.i1[pos] = ik;
  }
}

// ------------------------------------------------------------ 3. buckets
__device__ __forceinline__ int leaves_for(uint32_t size, const Dims& D) {
  if (size == 0) return 0;
  if ((int)size <= D.leaf_cap) return 1;
  int64_t s = ((int64_t)size + D.leaf_target - 1) / D.leaf_target;
  return (int)(s < D.max_sub ? s : D.max_sub);
}

static __global__ void __launch_bounds__(1024) k_buckets(Dims D, Ctl C, int64_t* out_count) {
  __shared__ uint32_t wsum[32], wsum2[32], wsum3[32];
  __shared__ uint32_t carry, carry2, carry3;
  if (threadIdx.x == 0) {
    carry = 0;
    carry2 = 0;
    carry3 = 0;
    if (D.nb1 == 1) C.bcount[0] = (uint32_t)D.n;
    *C.leaf_ctr = 0;
    *out_count = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < D.nb1; base += blockDim.x) {
    const int b = base + threadIdx.x;
    const uint32_t v = b < D.nb1 ? C.bcount[b] : 0;
    const uint32_t nl = b < D.nb1 ? (uint32_t)leaves_for(v, D) : 0;
    const uint32_t nt = (b < D.nb1 && (int)v > D.leaf_cap) ? (v + kSplitTile - 1) / kSplitTile : 0;
    uint32_t a = v, c = nl, e = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ta = __shfl_up_sync(0xffffffffu, a, o);
      const uint32_t tc = __shfl_up_sync(0xffffffffu, c, o);
      const uint32_t te = __shfl_up_sync(0xffffffffu, e, o);
      if (lane >= o) { a += ta; c += tc; e += te; }
    }
    if (lane == 31) { wsum[wid] = a; wsum2[wid] = c; wsum3[wid] = e; }
    __syncthreads();
    if (wid == 0) {
      uint32_t s = wsum[lane], s2 = wsum2[lane], s3 = wsum3[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
        const uint32_t t2 = __shfl_up_sync(0xffffffffu, s2, o);
        const uint32_t t3 = __shfl_up_sync(0xffffffffu, s3, o);
        if (lane >= o) { s += t; s2 += t2; s3 += t3; }
      }
      wsum[lane] = s;
      wsum2[lane] = s2;
      wsum3[lane] = s3;
    }
    __syncthreads();
    const uint32_t ex = carry + (wid ? wsum[wid - 1] : 0) + a - v;
    const uint32_t ex2 = carry2 + (wid ? wsum2[wid - 1] : 0) + c - nl;
    const uint32_t ex3 = carry3 + (wid ? wsum3[wid - 1] : 0) + e - nt;
    if (b < D.nb1) {
      C.bbase[b] = ex;
      C.bcursor[b] = ex;
      C.leaf_off[b] = ex2;
      C.tile_off[b] = ex3;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry = ex + v;
      carry2 = ex2 + nl;
      carry3 = ex3 + nt;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    C.bbase[D.nb1] = carry;
    C.leaf_off[D.nb1] = carry2;
    C.tile_off[D.nb1] = carry3;
    *C.n_leaves = carry2;
    *C.n_tiles = carry3;
  }
}

template <typename K>
static int set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) {
    PLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  return PL_OK;
}

// -------------------------------------------------------------- 5. split
// Level 2: buckets larger than a shared-memory leaf are cut into nsub
// sub-buckets (leaves) by splitters from a bucket-local sample.
//   k_split_prep    CTA per bucket: leaf descriptor of an unsplit bucket, or
//                   sample + sort + nsub-1 splitters (C.split2)
//   k_split_count   CTA per tile of kSplitTile items of a split bucket:
//                   classify (binary search in shared memory), histogram,
//                   add into the bucket's sub-bucket counts
//   k_split_bases   CTA per bucket: scan of sub-bucket counts -> leaf
//                   descriptors and scatter cursors
//   k_split_scatter same tiles: classify again, reserve per (tile, sub-bucket)
//                   ranges, write the items into buffer 2
template <int KW>
__global__ void __launch_bounds__(kSplitThreads)
k_split_prep(Dims D, Ctl C, int s2cap) {
  extern __shared__ u64 sm[];
  const int b = blockIdx.x;
  const uint32_t size = C.bcount[b], base = C.bbase[b];
  const uint32_t lo = C.leaf_off[b];
  if (size == 0) return;
  if ((int)size <= D.leaf_cap) {
    if (threadIdx.x == 0) C.leaf_desc[lo] = make_uint4(1u, base, size, 0u);
    return;
  }
  const int nsub = leaves_for(size, D);
  {  // descriptors of the bucket's level-2 tiles
    const uint32_t nt = (size + kSplitTile - 1) / kSplitTile, t_first = C.tile_off[b];
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
      const uint32_t first = i * kSplitTile;
      C.tile_desc[t_first + i] = make_uint4((uint32_t)b, base + first,
                                            min((uint32_t)kSplitTile, size - first), (uint32_t)nsub);
    }
  }
  int ns = nsub * kSampleOversample;
  if (ns > s2cap) ns = s2cap;
  if ((uint32_t)ns > size) ns = (int)size;
  u64* SK = sm;
  u64* CK = SK + (int64_t)KW * ns;
  const u64* K1 = C.k1 + (int64_t)base * KW;
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const int64_t r = ((2 * (int64_t)s + 1) * size) / (2 * (int64_t)ns);
    u64 key[KW];
    load_row<KW>(K1, r, key);
#pragma unroll
    for (int d = 0; d < KW; ++d) SK[d * ns + s] = key[d];
  }
  // the bucket's keys lie between its level-1 splitters: sort on the 64 bits
  // after the prefix those two share
  int cp = 0;
  {
    bool found = false;
#pragma unroll
    for (int d = 0; d < KW; ++d) {
      const u64 lo_k = b > 0 ? C.split[d * D.nb1 + b - 1] : 0ull;
      const u64 hi_k = b < D.nb1 - 1 ? C.split[d * D.nb1 + b] : ~0ull;
      const u64 x = lo_k ^ hi_k;
      if (!found) {
        if (x) {
          cp += __clzll((long long)x);
          found = true;
        } else {
          cp += 64;
        }
      }
    }
  }
  __syncthreads();
  const bool composite = sort_samples<KW>(SK, ns, CK, cp);
  u64* SP = C.split2 + (int64_t)b * KW * D.max_sub;
  u64* SPW = C.split2w + (int64_t)b * D.max_sub;
  if (threadIdx.x == 0) C.bcp[b] = cp;
  for (int q = 1 + threadIdx.x; q < nsub; q += blockDim.x) {
    const int pos = (int)(((int64_t)q * ns) / nsub);
    const int src = composite ? (int)(CK[pos] & 0x1FFF) : pos;
    u64 key[KW];
#pragma unroll
    for (int d = 0; d < KW; ++d) {
      key[d] = SK[d * ns + src];
      SP[d * D.max_sub + (q - 1)] = key[d];
    }
    SPW[q - 1] = get_seg<KW>(key, cp, 64);  // the 64 key bits after the bucket's shared prefix
  }
}

// One level-2 tile: kSplitTile consecutive items of a split bucket
// (descriptors written by k_split_prep).
struct SplitTile {
  int b, nsub;
  uint32_t first, count;  // first item (absolute) and number of items
};

__device__ __forceinline__ bool split_tile_load(const Ctl& C, SplitTile& T) {
  const uint32_t t = blockIdx.x;
  const uint4 d = C.tile_desc[t];  // in bounds (grid = the tile bound); valid below n_tiles
  if (t >= *C.n_tiles) return false;
  T.b = (int)d.x;
  T.first = d.y;
  T.count = d.z;
  T.nsub = (int)d.w;
  return true;
}

constexpr int kSplitIpt = kSplitTile / kSplitTileThreads;  // items per thread
constexpr int kSplitIlp = 4;                                // searches interleaved per thread
constexpr int kSplitWinSlots = 1024;                        // padded window table (>= max_sub)
static_assert(kSplitIpt % kSplitIlp == 0, "tile items per thread");

// Level-2 classification searches 32-bit windows: the key bits after the
// prefix every key of the bucket shares (C.bcp) -- one shared-memory word and
// one compare per step of a fixed ten-step search over a table padded with
// the maximal window, four items interleaved.  Splitters whose window equals
// the key's (rare) are compared in full from global memory.  Every item's
// sub-bucket goes to C.sid (k_split_scatter does not search again) and the
// tile's histogram to C.thist: k_split_bases turns the histograms of a bucket
// into the position of every (tile, sub-bucket) run, so no global atomics.
template <int KW>
__global__ void __launch_bounds__(kSplitTileThreads)
k_split_count(Dims D, Ctl C) {
  extern __shared__ u64 sm[];
  uint32_t* SPW = reinterpret_cast<uint32_t*>(sm);  // [kSplitWinSlots] splitter windows
  uint32_t* hist = SPW + kSplitWinSlots;
  SplitTile T;
  if (!split_tile_load(C, T)) return;
  const int nsp = T.nsub - 1;
  {
    const u64* G = C.split2w + (int64_t)T.b * D.max_sub;
    for (int q = threadIdx.x; q < kSplitWinSlots; q += blockDim.x) {
      SPW[q] = q < nsp ? (uint32_t)(G[q] >> 32) : 0xFFFFFFFFu;
      if (q < D.max_sub) hist[q] = 0;
    }
  }
  const int cp = C.bcp[T.b];
  const u64* K1 = C.k1 + (int64_t)T.first * KW;
  const u64* SPF = C.split2 + (int64_t)T.b * KW * D.max_sub;
  uint16_t* SID = C.sid + T.first;
  __syncthreads();
#pragma unroll 1
  for (int h = 0; h < kSplitIpt; h += kSplitIlp) {
    u64 key[kSplitIlp][KW];
    uint32_t w[kSplitIlp];
    int pos[kSplitIlp];
#pragma unroll
    for (int u = 0; u < kSplitIlp; ++u) {
      const uint32_t t = (h + u) * kSplitTileThreads + threadIdx.x;
      if (t < T.count) {
        load_row<KW>(K1, t, key[u]);
      } else {
#pragma unroll
        for (int d = 0; d < KW; ++d) key[u][d] = 0ull;
      }
    }
#pragma unroll
    for (int u = 0; u < kSplitIlp; ++u) {
      w[u] = (uint32_t)(get_seg<KW>(key[u], cp, 64) >> 32);
      pos[u] = 0;
    }
    // number of splitter windows <= w (padding compares greater unless w is maximal)
#pragma unroll
    for (int st = kSplitWinSlots / 2; st > 0; st >>= 1) {
#pragma unroll
      for (int u = 0; u < kSplitIlp; ++u)
        if (SPW[pos[u] + st - 1] <= w[u]) pos[u] += st;
    }
#pragma unroll
    for (int u = 0; u < kSplitIlp; ++u) {
      const uint32_t t = (h + u) * kSplitTileThreads + threadIdx.x;
      if (t >= T.count) continue;
      int q = pos[u] < nsp ? pos[u] : nsp;
      // splitters with the key's own window count only if they are <= the key
      while (q > 0 && SPW[q - 1] == w[u] && key_lt<KW>(key[u], SPF, D.max_sub, q - 1)) --q;
      SID[t] = (uint16_t)q;
      atomicAdd(&hist[q], 1u);
    }
  }
  __syncthreads();
  uint16_t* th = C.thist + (int64_t)blockIdx.x * D.max_sub;
  for (int q = threadIdx.x; q < T.nsub; q += kSplitTileThreads) th[q] = (uint16_t)hist[q];
}

// CTA per split bucket, thread per sub-bucket: walks the bucket's tiles in
// order, turning each tile's count into the offset of its run inside the
// sub-bucket (C.toff), then scans the sub-bucket totals into the leaf
// descriptors and the sub-buckets' first positions (C.sub_count).
static __global__ void __launch_bounds__(1024) k_split_bases(Dims D, Ctl C) {
  const int b = blockIdx.x;
  const uint32_t size = C.bcount[b];
  if ((int)size <= D.leaf_cap) return;
  const uint32_t base = C.bbase[b], lo = C.leaf_off[b];
  const int nsub = leaves_for(size, D);
  const uint32_t t0 = C.tile_off[b], nt = (size + kSplitTile - 1) / kSplitTile;
  uint32_t* g = C.sub_count + (int64_t)b * D.max_sub;
  uint32_t carry = 0;
  for (int q0 = 0; q0 < nsub; q0 += blockDim.x) {
    const int q = q0 + threadIdx.x;
    uint32_t h = 0;
    if (q < nsub) {
      const uint16_t* th = C.thist + (int64_t)t0 * D.max_sub + q;
      uint32_t* to = C.toff + (int64_t)t0 * D.max_sub + q;
      uint32_t i = 0;
      for (; i + 4 <= nt; i += 4) {  // four tiles' counts in flight
        uint32_t c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = th[(int64_t)(i + u) * D.max_sub];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          to[(int64_t)(i + u) * D.max_sub] = h;
          h += c[u];
        }
      }
      for (; i < nt; ++i) {
        const uint32_t c = th[(int64_t)i * D.max_sub];
        to[(int64_t)i * D.max_sub] = h;
        h += c;
      }
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan(h, &tot) + carry;
    if (q < nsub) {
      C.leaf_desc[lo + q] = make_uint4(2u, base + ex, h, 0u);
      g[q] = base + ex;
    }
    carry += tot;
  }
}

// Scatter of a tile into the sub-buckets.  Every load of the tile (sub-bucket
// ids, ik, the keys when they are narrow, and the positions of the tile's
// runs) is issued up front and the items wait in registers, so a CTA exposes
// one memory latency after its descriptor; ranks inside a run come from
// shared-memory atomics.
template <int KW>
__global__ void __launch_bounds__(kSplitTileThreads)
k_split_scatter(Dims D, Ctl C) {
  extern __shared__ u64 sm[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm);
  uint32_t* gbase = hist + D.max_sub;
  constexpr bool STAGE = KW <= 2;  // wider keys are re-read when written
  SplitTile T;
  if (!split_tile_load(C, T)) return;
  const u64* K1 = C.k1 + (int64_t)T.first * KW;
  const uint32_t* I1 = C.i1 + T.first;
  const uint16_t* SID = C.sid + T.first;
  uint32_t sub[kSplitIpt], ik[kSplitIpt];
  u64 key[kSplitIpt][STAGE ? KW : 1];
#pragma unroll
  for (int u = 0; u < kSplitIpt; ++u) {
    const uint32_t t = u * kSplitTileThreads + threadIdx.x;
    sub[u] = 0xFFFFFFFFu;
    if (t < T.count) {
      sub[u] = SID[t];
      ik[u] = I1[t];
      if constexpr (STAGE) load_row<KW>(K1, t, key[u]);
    }
  }
  {
    const uint32_t* g = C.sub_count + (int64_t)T.b * D.max_sub;
    const uint32_t* to = C.toff + (int64_t)blockIdx.x * D.max_sub;
    for (int q = threadIdx.x; q < T.nsub; q += kSplitTileThreads) {
      hist[q] = 0;
      gbase[q] = g[q] + to[q];
    }
  }
  __syncthreads();
  uint32_t rank[kSplitIpt];
#pragma unroll
  for (int u = 0; u < kSplitIpt; ++u)
    if (sub[u] != 0xFFFFFFFFu) rank[u] = atomicAdd(&hist[sub[u]], 1u);
#pragma unroll
  for (int u = 0; u < kSplitIpt; ++u) {
    if (sub[u] == 0xFFFFFFFFu) continue;
    const uint32_t pos = gbase[sub[u]] + rank[u];
    if constexpr (STAGE) {
      store_row<KW>(C.k2, pos, key[u]);
    } else {
      const uint32_t t = u * kSplitTileThreads + threadIdx.x;
      u64 kk[KW];
      load_row<KW>(K1, t, kk);
      store_row<KW>(C.k2, pos, kk);
    }
    C.i2[pos] = ik[u];
  }
}

template <int KW>
static int launch_split(const pl_merge_plan& P, const Dims& D, const Ctl& C, cudaStream_t st) {
  const int s2cap = (int)P.reserved[1];
  const size_t psm = sample_smem_bytes(s2cap, KW);
  if (set_smem(k_split_prep<KW>, psm)) return PL_ERR_CUDA;
  const size_t csm = 4 * (size_t)kSplitWinSlots + 4 * (size_t)D.max_sub + 64;  // windows | histogram
  const size_t tsm = 8 * (size_t)D.max_sub + 64;  // histogram | bases
  if (set_smem(k_split_count<KW>, csm)) return PL_ERR_CUDA;
  if (set_smem(k_split_scatter<KW>, tsm)) return PL_ERR_CUDA;
  const unsigned max_tiles = (unsigned)(ceil_div(D.n, (int64_t)kSplitTile) + D.nb1);  // = plan_max_tiles of the layout's plan
  {
    StageTimer t_(st, "k_split_prep");
    k_split_prep<KW><<<D.nb1, kSplitThreads, psm, st>>>(D, C, s2cap);
    PLB_CHECK_LAUNCH("k_split_prep");
  }
  {
    StageTimer t_(st, "k_split_count");
    k_split_count<KW><<<max_tiles, kSplitTileThreads, csm, st>>>(D, C);
    PLB_CHECK_LAUNCH("k_split_count");
  }
  {
    StageTimer t_(st, "k_split_bases");
    k_split_bases<<<D.nb1, 1024, 0, st>>>(D, C);
    PLB_CHECK_LAUNCH("k_split_bases");
  }
  StageTimer t_(st, "k_split_scatter");
  k_split_scatter<KW><<<max_tiles, kSplitTileThreads, tsm, st>>>(D, C);
  PLB_CHECK_LAUNCH("k_split_scatter");
  return PL_OK;
}

// ------------------------------------------------------------ 6. leaves
__device__ __forceinline__ bool keep_sum(double2 s, double eps) {
  if (eps == 0.0) return s.x != 0.0 || s.y != 0.0;
  return hypot(s.x, s.y) > eps;
}

#include "merge_leaves.cuh"

// ============================================================== host side
static inline int64_t align256(int64_t v) { return (v + 255) & ~(int64_t)255; }

struct WsLayout {
  int64_t split, bcount, bbase, bcursor, leaf_off, n_leaves, leaf_ctr, tile_off, n_tiles,
      sub_count, leaf_desc, split2, kept, kprefix, scan, k1, i1, k2, i2, sums, rmap, opk, opb, l1tab,
      perm, split2w, bcp, bid, sid, tile_desc, thist, toff, total;
};

// Bound on the number of leaves: a bucket of s items gets at most
// ceil(s / leaf_target) leaves, so the total is <= n / leaf_target + nb1.
static inline int64_t plan_max_leaves(const pl_merge_plan& P) {
  const int64_t by_sub = (int64_t)P.n_buckets * P.max_sub;
  const int64_t by_size = P.n_items / std::max(1, P.leaf_target) + P.n_buckets + 1;
  return std::min(by_sub, by_size);
}

// Bound on the level-2 tiles: every split bucket has ceil(size / kSplitTile).
static inline int64_t plan_max_tiles(const pl_merge_plan& P) {
  return ceil_div(P.n_items, (int64_t)kSplitTile) + P.n_buckets;
}

// Slots of the per-item level-1 bucket ids: whole generator CTAs (kTileA x
// kTileB tiles of the outer product, kGenThreads * kGenTB terms of a sort).
static inline int64_t gen_slots(const pl_merge_plan& P) {
  const int64_t per = (int64_t)kGenThreads * kGenTB;
  if (P.mode == 0 && P.ma > 0) {
    const int64_t cols = ceil_div(P.n_items, P.ma);  // B columns generated here
    return ceil_div(P.ma, (int64_t)kTileA) * ceil_div(cols, (int64_t)kTileB) * per;
  }
  return ceil_div(P.n_items, per) * per;
}

static WsLayout ws_layout(const pl_merge_plan& P) {
  WsLayout w{};
  const int64_t KW = P.key_words, nb1 = P.n_buckets, n = P.n_items;
  const int64_t sub_slots = nb1 * (int64_t)P.max_sub;  // [bucket][sub] tables
  const int64_t max_leaves = plan_max_leaves(P);
  int64_t o = 0;
  w.split = o; o = align256(o + 8 * KW * nb1);
  w.bcount = o; o = align256(o + 4 * nb1);
  w.bbase = o; o = align256(o + 4 * (nb1 + 1));
  w.bcursor = o; o = align256(o + 4 * nb1);
  w.leaf_off = o; o = align256(o + 4 * (nb1 + 1));
  w.n_leaves = o; o = align256(o + 4);
  w.leaf_ctr = o; o = align256(o + 4);
  w.tile_off = o; o = align256(o + 4 * (nb1 + 1));
  w.n_tiles = o; o = align256(o + 4);
  w.sub_count = o; o = align256(o + 4 * sub_slots);
  const int64_t ctl_end = o;  // everything above is zeroed per call
  w.leaf_desc = o; o = align256(o + 16 * max_leaves);
  w.split2 = o; o = align256(o + 8 * KW * sub_slots);
  w.kept = o; o = align256(o + 4 * max_leaves);
  w.kprefix = o; o = align256(o + 4 * max_leaves);
  w.scan = o; o = align256(o + 4 * (scan_scratch_words(max_leaves) + 1));
  w.k1 = o; o = align256(o + 8 * KW * n);
  w.i1 = o; o = align256(o + 4 * n);
  w.k2 = o; o = align256(o + 8 * KW * n);
  w.i2 = o; o = align256(o + 4 * n);
  w.sums = o; o = align256(o + 16 * n);
  w.rmap = o; o = align256(o + 4 * (n / 128 + 2));
  w.opk = o; o = align256(o + 8 * KW * (P.ma + P.mb));
  w.opb = o; o = align256(o + (P.ma + P.mb));
  w.l1tab = o; o = align256(o + 2 * ((1 << kTabBits) + 1));
  w.perm = o; o = align256(o + 4 * (P.ma + P.mb));
  w.split2w = o; o = align256(o + 8 * sub_slots);
  w.bcp = o; o = align256(o + 4 * nb1);
  w.bid = o; o = align256(o + 2 * gen_slots(P));
  w.sid = o; o = align256(o + 2 * n);
  const int64_t max_tiles = plan_max_tiles(P);
  w.tile_desc = o; o = align256(o + 16 * max_tiles);
  w.thist = o; o = align256(o + 2 * max_tiles * P.max_sub);
  w.toff = o; o = align256(o + 4 * max_tiles * P.max_sub);
  w.total = o;
  (void)ctl_end;
  return w;
}

static void finish_plan(pl_merge_plan* P, const u64* masks /* z[W] then x[W] */) {
  const int W = P->W;
  int pos = 0, active = 0;
  for (int s = 0; s < 2 * W; ++s) {
    const u64 m = masks[s];
    if (m == 0) {
      P->seg_lo[s] = 0;
      P->seg_len[s] = 0;
      P->seg_pos[s] = pos;
      continue;
    }
    const int lo = __builtin_ctzll(m), hi = 63 - __builtin_clzll(m);
    P->seg_lo[s] = lo;
    P->seg_len[s] = hi - lo + 1;
    P->seg_pos[s] = pos;
    pos += hi - lo + 1;
    active |= 1 << (s < W ? s : s - W);
  }
  for (int s = 2 * W; s < PL_PLAN_MAX_SEG; ++s) P->seg_lo[s] = P->seg_len[s] = P->seg_pos[s] = 0;
  P->key_bits = pos;
  P->key_words = key_words_for_bits(pos > 0 ? pos : 1);
  P->reserved[0] = active;
  // sort_and_combine of wide, sparse keys: the set-bit position list is
  // shorter than the packed bit string (config 5: 1000-bit keys with <= 24
  // set bits -> 250 bits, KW 16 -> 4)
  P->reserved[4] = P->reserved[5] = P->reserved[6] = 0;
  if (P->mode == 1 && pos > 0) {
    const int maxbits = (int)masks[2 * W];
    int sb = 1;
    while ((1 << sb) <= pos) ++sb;  // values key_bits - p in [1, key_bits]
    const int nslots = maxbits + 1;  // + the 0 terminator
    const int kw_sparse = key_words_for_bits(nslots * sb);
    if (kw_sparse < P->key_words) {
      P->key_words = kw_sparse;
      P->reserved[4] = 1;
      P->reserved[5] = sb;
      P->reserved[6] = nslots;
    }
  }
  const int KW = P->key_words;
  const int cap = leaf_cap_for(KW);
  P->leaf_cap = cap;
  P->leaf_target = KW <= 2 ? cap / 2 : cap / 3;  // headroom for the sampled splitters
  // one-CTA sample capacity: the sampler sorts in up to kSortSmemBytes
  int scap = 8192;  // a power of two (13-bit sample index) whose keys + composites fit
  while ((int64_t)scap * (8 * KW + 8) > kSortSmemBytes) scap >>= 1;
  const int64_t n = P->n_items;
  int64_t nb1 = 1;
  if (n > cap) {
    // level 1 aims at ~kLeavesPerBucket leaves per bucket (fewer, cheaper
    // samples for small inputs); level 2 adapts to the exact bucket sizes
    nb1 = ceil_div(n, (int64_t)kLeavesPerBucket * P->leaf_target);
    const int64_t nb_max = std::min<int64_t>(kMaxBuckets, scap / kSample1Oversample);
    if (nb1 > nb_max) nb1 = nb_max;
    if (nb1 < 2) nb1 = 2;
  }
  P->n_buckets = (int)nb1;
  P->n_samples = nb1 > 1 ? (int)std::min<int64_t>(n, std::min<int64_t>(scap, nb1 * kSample1Oversample)) : 0;
  // level-2 sample capacity bounds the sub-bucket count
  // level-2 sample (one CTA, <= 160 KB): >= 8 samples per sub-bucket
  int s2cap = 8192;  // power of two (13-bit sample index); keys + composites in 200 KB
  while (s2cap > 64 && (int64_t)s2cap * (8 * KW + 8) > 200 * 1024) s2cap >>= 1;
  P->max_sub = std::max(1, std::min(1024, s2cap / 8));
  P->reserved[1] = s2cap;
  P->workspace_bytes = ws_layout(*P).total;
}

// OR of every operand word per plane (z[W] then x[W]) and the most set bits
// (x and z) of any term.  Warp shuffles, then one shared-memory reduction per
// CTA, then one global atomic per word per CTA.
template <int W>
__global__ void __launch_bounds__(256) k_or_masks(const u64* __restrict__ x,
                                                  const u64* __restrict__ z, int64_t ld,
                                                  int64_t m, u64* out) {
  __shared__ u64 red[8][2 * W + 1];
  u64 mz[W], mx[W];
  unsigned long long maxbits = 0;  // most set bits (x and z) of any term
#pragma unroll
  for (int w = 0; w < W; ++w) mz[w] = mx[w] = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    u64 zv[W], xv[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {  // all 2W loads in flight together
      zv[w] = __ldg(z + w * ld + t);
      xv[w] = __ldg(x + w * ld + t);
    }
    int bitsum = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      mz[w] |= zv[w];
      mx[w] |= xv[w];
      bitsum += popc64(zv[w]) + popc64(xv[w]);
    }
    maxbits = maxbits > (unsigned long long)bitsum ? maxbits : (unsigned long long)bitsum;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, maxbits, o);
    maxbits = v > maxbits ? v : maxbits;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      mz[w] |= __shfl_xor_sync(0xffffffffu, mz[w], o);
      mx[w] |= __shfl_xor_sync(0xffffffffu, mx[w], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      red[warp][w] = mz[w];
      red[warp][W + w] = mx[w];
    }
    red[warp][2 * W] = maxbits;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= 2 * W; e += blockDim.x) {
    u64 v = 0;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q)
      v = e < 2 * W ? (v | red[q][e]) : (red[q][e] > v ? red[q][e] : v);
    if (e < 2 * W) {
      if (v) atomicOr(&out[e], v);
    } else if (v) {
      atomicMax(&out[2 * W], v);
    }
  }
}

template <int W>
static int launch_masks(const u64* x, const u64* z, int64_t ld, int64_t m, u64* out,
                        cudaStream_t st) {
  if (m == 0) return PL_OK;
  int64_t blocks = ceil_div(m, 256);
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  StageTimer t_(st, "k_or_masks");
  k_or_masks<W><<<(unsigned)blocks, 256, 0, st>>>(x, z, ld, m, out);
  PLB_CHECK_LAUNCH("k_or_masks");
  return PL_OK;
}

// OR-masks of the operands' words (the plan's key layout).  One small
// device + pinned host buffer per device, reused under a lock, so planning
// costs one tiny kernel and one stream sync (no allocation per call).
static int compute_masks(int W, const u64* x1, const u64* z1, int64_t ld1, int64_t m1,
                         const u64* x2, const u64* z2, int64_t ld2, int64_t m2, u64* host_masks,
                         cudaStream_t st) {
  static std::mutex mtx;
  static u64* dbuf[64] = {nullptr};
  static u64* hbuf[64] = {nullptr};
  int dev = 0;
  PLB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device index %d out of range", dev);
    return PL_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(mtx);
  if (!dbuf[dev]) {
    PLB_CUDA(cudaMalloc((void**)&dbuf[dev], (2 * PL_PLAN_MAX_SEG + 1) * sizeof(u64)));
    PLB_CUDA(cudaMallocHost((void**)&hbuf[dev], (2 * PL_PLAN_MAX_SEG + 1) * sizeof(u64)));
  }
  u64* dmask = dbuf[dev];
  PLB_CUDA(cudaMemsetAsync(dmask, 0, (2 * W + 1) * sizeof(u64), st));
  int rc = PLB_DISPATCH_W(W, launch_masks, x1, z1, ld1, m1, dmask, st);
  if (rc == PL_OK && x2) rc = PLB_DISPATCH_W(W, launch_masks, x2, z2, ld2, m2, dmask, st);
  if (rc == PL_OK) {
    PLB_CUDA(cudaMemcpyAsync(hbuf[dev], dmask, (2 * W + 1) * sizeof(u64), cudaMemcpyDeviceToHost,
                             st));
  }
  PLB_CUDA(cudaStreamSynchronize(st));
  if (rc == PL_OK) memcpy(host_masks, hbuf[dev], (2 * W + 1) * sizeof(u64));
  return rc;
}

static Layout to_layout(const pl_merge_plan& P) {
  Layout L{};
  L.W = P.W;
  L.KW = P.key_words;
  L.active = (int)P.reserved[0];
  L.sparse = (int)P.reserved[4];
  L.sbits = (int)P.reserved[5];
  L.nslots = (int)P.reserved[6];
  L.key_bits = P.key_bits;
  for (int s = 0; s < PL_PLAN_MAX_SEG; ++s) {
    L.lo[s] = P.seg_lo[s];
    L.len[s] = P.seg_len[s];
    L.pos[s] = P.seg_pos[s];
  }
  return L;
}

static Dims to_dims(const pl_merge_plan& P) {
  Dims D{};
  D.n = P.n_items;
  D.ma = P.ma;
  D.mb = P.mb;
  D.n_space = P.n_items;
  D.j0 = 0;
  D.mb_all = P.mb;
  D.nb1 = P.n_buckets;
  D.nsamp = P.n_samples;
  D.leaf_cap = P.leaf_cap;
  D.leaf_target = P.leaf_target;
  D.max_sub = P.max_sub;
  D.max_leaves = (int)plan_max_leaves(P);
  return D;
}

static Ctl to_ctl(const pl_merge_plan& P, void* ws) {
  const WsLayout w = ws_layout(P);
  uint8_t* b = (uint8_t*)ws;
  Ctl C;
  C.split = (u64*)(b + w.split);
  C.bcount = (uint32_t*)(b + w.bcount);
  C.bbase = (uint32_t*)(b + w.bbase);
  C.bcursor = (uint32_t*)(b + w.bcursor);
  C.leaf_off = (uint32_t*)(b + w.leaf_off);
  C.n_leaves = (uint32_t*)(b + w.n_leaves);
  C.leaf_ctr = (uint32_t*)(b + w.leaf_ctr);
  C.leaf_desc = (uint4*)(b + w.leaf_desc);
  C.split2 = (u64*)(b + w.split2);
  C.sub_count = (uint32_t*)(b + w.sub_count);
  C.tile_off = (uint32_t*)(b + w.tile_off);
  C.n_tiles = (uint32_t*)(b + w.n_tiles);
  C.kept = (uint32_t*)(b + w.kept);
  C.kprefix = (uint32_t*)(b + w.kprefix);
  C.scan_scratch = (uint32_t*)(b + w.scan);
  C.scan_total = C.scan_scratch + scan_scratch_words(plan_max_leaves(P));
  C.sums = (double2*)(b + w.sums);
  C.rmap = (uint32_t*)(b + w.rmap);
  C.opk = (u64*)(b + w.opk);
  C.opb = (uint8_t*)(b + w.opb);
  C.l1tab = (uint16_t*)(b + w.l1tab);
  C.perm = (int32_t*)(b + w.perm);
  C.split2w = (u64*)(b + w.split2w);
  C.bcp = (int32_t*)(b + w.bcp);
  C.bid = (uint16_t*)(b + w.bid);
  C.sid = (uint16_t*)(b + w.sid);
  C.tile_desc = (uint4*)(b + w.tile_desc);
  C.thist = (uint16_t*)(b + w.thist);
  C.toff = (uint32_t*)(b + w.toff);
  C.k1 = (u64*)(b + w.k1);
  C.i1 = (uint32_t*)(b + w.i1);
  C.k2 = (u64*)(b + w.k2);
  C.i2 = (uint32_t*)(b + w.i2);
  return C;
}


template <int KW>
static int launch_sort_ops(const Dims& D, const Ctl& C, cudaStream_t st) {
  const int64_t nmax = std::min<int64_t>(kSortOpsChunk, std::max(D.ma, D.mb));
  int npow = 1;
  while (npow < nmax) npow <<= 1;
  const size_t sm = 8 * (size_t)npow;
  if (set_smem(k_sort_ops<KW>, sm)) return PL_ERR_CUDA;
  const unsigned nblk = (unsigned)(ceil_div(D.ma, kSortOpsChunk) + ceil_div(D.mb, kSortOpsChunk));
  StageTimer t_(st, "k_sort_ops");
  k_sort_ops<KW><<<nblk, 1024, sm, st>>>(D, C);
  PLB_CHECK_LAUNCH("k_sort_ops");
  return PL_OK;
}

template <int W, int KW, int MODE>
static int run_pipeline(const pl_merge_plan& P, const SrcA& S0, void* ws, const OutP& O,
                        cudaStream_t st) {
  SrcA S = S0;
  S.ma_inv = ma_inverse(P.ma);
  const Layout L = to_layout(P);
  const Dims D = to_dims(P);
  const Ctl C = to_ctl(P, ws);
  const WsLayout wl = ws_layout(P);
  if (O.phase == 2) return launch_emit<W, KW>(L, D, C, O, st);
  PLB_CUDA(cudaMemsetAsync(ws, 0, (size_t)wl.leaf_desc, st));  // control region

  {
    StageTimer t_(st, "k_pack_ops");
    const int64_t nops = D.ma + (MODE == 0 ? D.mb_all : 0);
    k_pack_ops<W, KW, MODE><<<(unsigned)std::min<int64_t>(ceil_div(nops, 256), 8 * num_sms()), 256,
                              0, st>>>(L, S, D.ma, D.mb_all, C);
    PLB_CHECK_LAUNCH("k_pack_ops");
  }
  if (MODE == 0) {
    const int rc = launch_sort_ops<KW>(D, C, st);
    if (rc) return rc;
  }
  // 1-2. splitters + counts
  if (D.nb1 > 1) {
    const size_t sm1 = sample_smem_bytes(D.nsamp, KW);
    if (set_smem(k_sample<W, KW, MODE>, sm1)) return PL_ERR_CUDA;
    StageTimer t_(st, "k_sample");
    k_sample<W, KW, MODE><<<1, kLeafThreads, sm1, st>>>(L, D, S, C);
    PLB_CHECK_LAUNCH("k_sample");
  }
  const size_t gsm = gen_smem_bytes(W, KW, D.nb1);
  dim3 ggrid;
  if (MODE == 0) ggrid = dim3((unsigned)ceil_div(D.ma, kTileA), (unsigned)ceil_div(D.mb, kTileB));
  else ggrid = dim3((unsigned)ceil_div(D.n, (int64_t)kGenThreads * kGenTB), 1);
  if (ggrid.y > 65535) {
    set_error("outer product: |B| too large for one call (%lld)", (long long)D.mb);
    return PL_ERR_CAPACITY;
  }
  if (D.nb1 > 1) {
    if (set_smem(k_count<W, KW, MODE>, gsm)) return PL_ERR_CUDA;
    StageTimer t_(st, "k_count");
    k_count<W, KW, MODE><<<ggrid, kGenThreads, gsm, st>>>(L, D, S, C);
    PLB_CHECK_LAUNCH("k_count");
  }
  // 3. bucket bases / leaves
  {
    StageTimer t_(st, "k_buckets");
    k_buckets<<<1, 1024, 0, st>>>(D, C, O.count);
    PLB_CHECK_LAUNCH("k_buckets");
  }
  // 4. scatter
  const size_t ssm = gen_smem_bytes(W, KW, D.nb1, false);
  if (set_smem(k_scatter<W, KW, MODE>, ssm)) return PL_ERR_CUDA;
  {
    StageTimer t_(st, "k_scatter");
    k_scatter<W, KW, MODE><<<ggrid, kGenThreads, ssm, st>>>(L, D, S, C);
    PLB_CHECK_LAUNCH("k_scatter");
  }
  // 5. level-2 split of oversized buckets
  {
    const int rc = launch_split<KW>(P, D, C, st);
    if (rc) return rc;
  }
  // 6. leaves: sort + reduce, scan, emit
  return launch_leaves<W, KW, MODE>(L, D, S, C, O, st);
}

// ------------------------------------------------------ K7 multi-GPU stages
// Record layout exchanged between ranks: KW key words then ik, (KW+1) u64.
template <int KW>
__global__ void k_pack(const Ctl C, int64_t n, u64* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int d = 0; d < KW; ++d) out[t * (KW + 1) + d] = C.k1[t * KW + d];
    out[t * (KW + 1) + KW] = C.i1[t];
  }
}

// counts [G][nbl] -> bucket totals, per-segment source offsets and
// destination offsets inside the bucket (one CTA, nbl <= kMaxBuckets)
static __global__ void __launch_bounds__(1024)
k_regroup_prep(const uint32_t* __restrict__ cnt, int G, int nbl, Ctl C, uint32_t* seg_src,
               uint32_t* seg_dst) {
  __shared__ uint32_t src_base[65];
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int s = 0; s < G; ++s) {
      src_base[s] = acc;
      for (int b = 0; b < nbl; ++b) acc += cnt[s * nbl + b];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbl; b += blockDim.x) {
    uint32_t in_bucket = 0;
    for (int s = 0; s < G; ++s) {
      seg_dst[s * nbl + b] = in_bucket;
      in_bucket += cnt[s * nbl + b];
    }
    C.bcount[b] = in_bucket;
  }
  if (threadIdx.x < G) {
    const int s = threadIdx.x;
    uint32_t acc = src_base[s];
    for (int b = 0; b < nbl; ++b) {
      seg_src[s * nbl + b] = acc;
      acc += cnt[s * nbl + b];
    }
  }
}

template <int KW>
__global__ void k_regroup_copy(const u64* __restrict__ recv, const uint32_t* __restrict__ cnt,
                               int nbl, const uint32_t* __restrict__ seg_src,
                               const uint32_t* __restrict__ seg_dst, Ctl C, int64_t n) {
  const int b = blockIdx.x, s = blockIdx.y;
  const uint32_t c = cnt[s * nbl + b];
  const uint64_t src = seg_src[s * nbl + b];
  const uint64_t dst = (uint64_t)C.bbase[b] + seg_dst[s * nbl + b];
  for (uint32_t t = threadIdx.x; t < c; t += blockDim.x) {
    const u64* r = recv + (src + t) * (KW + 1);
#pragma unroll
    for (int d = 0; d < KW; ++d) C.k1[(dst + t) * KW + d] = r[d];
    C.i1[dst + t] = (uint32_t)r[KW];
  }
}

static pl_merge_plan local_plan(const pl_merge_plan& P, int64_t n_local, int nb) {
  pl_merge_plan Q = P;
  Q.n_items = n_local;
  Q.n_buckets = nb;
  Q.workspace_bytes = ws_layout(Q).total + align256(8LL * 64 * nb);
  return Q;
}

template <int W, int KW>
static int run_partition(const pl_merge_plan& P, const SrcA& S, int64_t j0, int64_t j1, void* ws,
                         void* send, uint32_t* counts_out, cudaStream_t st) {
  const pl_merge_plan Q = local_plan(P, P.ma * (j1 - j0), P.n_buckets);
  const Layout L = to_layout(Q);
  Dims D = to_dims(Q);
  D.n_space = P.n_items;
  D.mb = j1 - j0;
  D.j0 = j0;
  const Ctl C = to_ctl(Q, ws);
  const WsLayout wl = ws_layout(Q);
  PLB_CUDA(cudaMemsetAsync(ws, 0, (size_t)wl.leaf_desc, st));
  if (D.n > 0) {
    {
      StageTimer t_(st, "k_pack_ops");
      const int64_t nops = D.ma + D.mb_all;
      k_pack_ops<W, KW, 0><<<(unsigned)std::min<int64_t>(ceil_div(nops, 256), 8 * num_sms()), 256,
                             0, st>>>(L, S, D.ma, D.mb_all, C);
      PLB_CHECK_LAUNCH("k_pack_ops");
    }
    {
      const int rc = launch_sort_ops<KW>(D, C, st);
      if (rc) return rc;
    }
    if (D.nb1 > 1) {
      const size_t sm1 = sample_smem_bytes(D.nsamp, KW);
      if (set_smem(k_sample<W, KW, 0>, sm1)) return PL_ERR_CUDA;
      StageTimer t_(st, "k_sample");
      k_sample<W, KW, 0><<<1, kLeafThreads, sm1, st>>>(L, D, S, C);
      PLB_CHECK_LAUNCH("k_sample");
    }
    const size_t gsm = gen_smem_bytes(W, KW, D.nb1);
    const dim3 ggrid((unsigned)ceil_div(D.ma, kTileA), (unsigned)ceil_div(D.mb, kTileB));
    if (D.nb1 > 1) {
      if (set_smem(k_count<W, KW, 0>, gsm)) return PL_ERR_CUDA;
      StageTimer t_(st, "k_count");
      k_count<W, KW, 0><<<ggrid, kGenThreads, gsm, st>>>(L, D, S, C);
      PLB_CHECK_LAUNCH("k_count");
    }
    {
      StageTimer t_(st, "k_buckets");
      k_buckets<<<1, 1024, 0, st>>>(D, C, (int64_t*)(C.n_leaves + 2));
      PLB_CHECK_LAUNCH("k_buckets");
    }
    const size_t ssm = gen_smem_bytes(W, KW, D.nb1, false);
    if (set_smem(k_scatter<W, KW, 0>, ssm)) return PL_ERR_CUDA;
    {
      StageTimer t_(st, "k_scatter");
      k_scatter<W, KW, 0><<<ggrid, kGenThreads, ssm, st>>>(L, D, S, C);
      PLB_CHECK_LAUNCH("k_scatter");
    }
    StageTimer t_(st, "k_pack");
    k_pack<KW><<<4 * num_sms(), 256, 0, st>>>(C, D.n, (u64*)send);
    PLB_CHECK_LAUNCH("k_pack");
  }
  PLB_CUDA(cudaMemcpyAsync(counts_out, C.bcount, 4 * (size_t)D.nb1, cudaMemcpyDeviceToDevice, st));
  return PL_OK;
}

template <int W, int KW>
static int run_merge_received(const pl_merge_plan& P, const u64* recv, int64_t n_recv,
                              const uint32_t* cnt, int G, int nbl, const SrcA& S0, void* ws,
                              const OutP& O, cudaStream_t st) {
  SrcA S = S0;
  S.ma_inv = ma_inverse(P.ma);
  const pl_merge_plan Q = local_plan(P, n_recv, nbl);
  const Layout L = to_layout(Q);
  Dims D = to_dims(Q);
  D.n_space = P.n_items;
  const Ctl C = to_ctl(Q, ws);
  const WsLayout wl = ws_layout(Q);
  uint32_t* seg_src = (uint32_t*)((uint8_t*)ws + wl.total);
  uint32_t* seg_dst = seg_src + 64 * nbl;
  PLB_CUDA(cudaMemsetAsync(ws, 0, (size_t)wl.leaf_desc, st));
  PLB_CUDA(cudaMemsetAsync(O.count, 0, sizeof(int64_t), st));
  if (n_recv == 0) return PL_OK;
  {
    StageTimer t_(st, "k_regroup");
    k_regroup_prep<<<1, 1024, 0, st>>>(cnt, G, nbl, C, seg_src, seg_dst);
    PLB_CHECK_LAUNCH("k_regroup_prep");
    k_buckets<<<1, 1024, 0, st>>>(D, C, O.count);
    PLB_CHECK_LAUNCH("k_buckets");
    k_regroup_copy<KW><<<dim3((unsigned)nbl, (unsigned)G), 256, 0, st>>>(recv, cnt, nbl, seg_src,
                                                                        seg_dst, C, n_recv);
    PLB_CHECK_LAUNCH("k_regroup_copy");
  }
  {
    const int rc = launch_split<KW>(P, D, C, st);
    if (rc) return rc;
  }
  return launch_leaves<W, KW, 0>(L, D, S, C, O, st);
}

template <int W>
int dispatch_partition(const pl_merge_plan& P, const SrcA& S, int64_t j0, int64_t j1,
                              void* ws, void* send, uint32_t* counts, cudaStream_t st) {
  switch (P.key_words) {
    case 1: return run_partition<W, 1>(P, S, j0, j1, ws, send, counts, st);
    case 2: return run_partition<W, 2>(P, S, j0, j1, ws, send, counts, st);
    case 4: return run_partition<W, (W >= 2 ? 4 : 1)>(P, S, j0, j1, ws, send, counts, st);
    case 8: return run_partition<W, (W >= 4 ? 8 : 1)>(P, S, j0, j1, ws, send, counts, st);
    case 16: return run_partition<W, (W >= 8 ? 16 : 1)>(P, S, j0, j1, ws, send, counts, st);
    default: return run_partition<W, (W >= 16 ? 32 : 1)>(P, S, j0, j1, ws, send, counts, st);
  }
}

template <int W>
int dispatch_received(const pl_merge_plan& P, const u64* recv, int64_t n_recv,
                             const uint32_t* cnt, int G, int nbl, const SrcA& S, void* ws,
                             const OutP& O, cudaStream_t st) {
  switch (P.key_words) {
    case 1: return run_merge_received<W, 1>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
    case 2: return run_merge_received<W, 2>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
    case 4: return run_merge_received<W, (W >= 2 ? 4 : 1)>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
    case 8: return run_merge_received<W, (W >= 4 ? 8 : 1)>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
    case 16: return run_merge_received<W, (W >= 8 ? 16 : 1)>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
    default: return run_merge_received<W, (W >= 16 ? 32 : 1)>(P, recv, n_recv, cnt, G, nbl, S, ws, O, st);
  }
}

template <int W, int MODE>
static int dispatch_kw(const pl_merge_plan& P, const SrcA& S, void* ws, const OutP& O,
                       cudaStream_t st) {
  switch (P.key_words) {
    case 1: return run_pipeline<W, 1, MODE>(P, S, ws, O, st);
    case 2: return run_pipeline<W, 2, MODE>(P, S, ws, O, st);
    case 4: if (W >= 2) return run_pipeline<W, (W >= 2 ? 4 : 1), MODE>(P, S, ws, O, st); break;
    case 8: if (W >= 4) return run_pipeline<W, (W >= 4 ? 8 : 1), MODE>(P, S, ws, O, st); break;
    case 16: if (W >= 8) return run_pipeline<W, (W >= 8 ? 16 : 1), MODE>(P, S, ws, O, st); break;
    case 32: if (W >= 16) return run_pipeline<W, (W >= 16 ? 32 : 1), MODE>(P, S, ws, O, st); break;
    default: break;
  }
  set_error("unsupported key width %d words", P.key_words);
  return PL_ERR_ARG;
}

template <int W>
int run_outer(const pl_merge_plan& P, const SrcA& S, void* ws, const OutP& O,
                     cudaStream_t st) {
  return dispatch_kw<W, 0>(P, S, ws, O, st);
}
template <int W>
int run_sort(const pl_merge_plan& P, const SrcA& S, void* ws, const OutP& O,
                    cudaStream_t st) {
  return dispatch_kw<W, 1>(P, S, ws, O, st);
}

}  // namespace plb

namespace plb {
// Explicit instantiations live in combine_w<W>_{o,s}.cu: "o" = outer product
// (single GPU and K7 partition/merge), "s" = sort_and_combine.
#define PLB_COMBINE_INST_OUTER(EXT, W)                                                          \
  EXT template int run_outer<W>(const pl_merge_plan&, const SrcA&, void*, const OutP&,        \
                                cudaStream_t);                                                \
  EXT template int dispatch_partition<W>(const pl_merge_plan&, const SrcA&, int64_t, int64_t, \
                                         void*, void*, uint32_t*, cudaStream_t);              \
  EXT template int dispatch_received<W>(const pl_merge_plan&, const u64*, int64_t,            \
                                        const uint32_t*, int, int, const SrcA&, void*,        \
                                        const OutP&, cudaStream_t);
#define PLB_COMBINE_INST_SORT(EXT, W)                                                           \
  EXT template int run_sort<W>(const pl_merge_plan&, const SrcA&, void*, const OutP&,         \
                               cudaStream_t);
#define PLB_COMBINE_INSTANTIATE(EXT, W) PLB_COMBINE_INST_OUTER(EXT, W) PLB_COMBINE_INST_SORT(EXT, W)
}  // namespace plb
