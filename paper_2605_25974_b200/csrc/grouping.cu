// K6 — greedy first-fit commutation grouping, exactly the reference's
// _greedy_over (grouping.py:67-83): term t, in index order, joins the first
// group (creation order) all of whose members commute with it, else opens a
// new group; pair_checks counts the members of every group tried (:75-76).
//
// Group state is kept TRANSPOSED: for group g, member-chunk c (members
// 64c..64c+63) stores one uint64 per key bit e in [0, 128W):
//   T_g[c][e] bit s  =  partner bit of member 64c+s for a term entry e, where
//   a term's x-bit at qubit q (entry e = q) pairs with the member's z-bit at q
//   and a term's z-bit at q (entry e = 64W + q) with the member's x-bit at q.
// "t commutes with every member of g" <=> for every chunk c the XOR over t's
// set-bit entries of T_g[c][e] is zero (bit s = symplectic parity with member
// s).  Cost per (term, group) test = |entries of t| loads of chunk 0 (members
// 0..63); later chunks are only read when chunk 0 already fits.
//
// Exactness under parallelism: terms are processed in batches of B = 1024.
//   fit     : fit0[t][g] for every batch term t and every group g existing at
//             batch start (parallel over groups x terms);
//   firstk  : first 4 fitting groups per term (warp per term);
//   anti    : intra-batch anti-commutation rows (row-list bitmatrix kernel);
//   resolve : one warp replays the batch in order; a candidate group is
//             rejected only if an earlier batch member already placed in it
//             anti-commutes with t (member masks in shared memory), and
//             groups created inside the batch are tried after all older
//             ones, in creation order -- exactly the sequential first-fit;
//   update  : append the batch members to their groups' transposed chunks and
//             add each term's reference pair_checks contribution
//             #{u < t : group(u) <= group(t)}.
#include <algorithm>
#include <cstdlib>

#include "bitmatrix_kernels.cuh"
#include "common.cuh"
#include "scan.cuh"

namespace plb {

constexpr int kGB = 1024;              // batch size (terms)
constexpr int kGAW = kGB / 32;         // anti-row words per term
constexpr int kGK = 16;                // first-k fitting groups listed per term
constexpr int kSlotChunks = kGB / 64 + 2;
constexpr int kHash = 2048;            // resolver hash slots (power of 2)

struct GCtx {
  int W;
  int64_t M;
  int64_t gcap, ccap;                  // group / chunk capacity
  const u64 *x, *z;
  int64_t ld;
  // CSR entries of every term
  const uint32_t* off;                 // M + 1
  const uint16_t* list;
  // groups
  uint32_t* gsize;                     // gcap
  int32_t* gfirst;                     // gcap
  int32_t* glast;                      // gcap
  uint32_t* gpre;                      // gcap: inclusive prefix of sizes at batch start
  // chunk pool: ccap chunks of 128W uint64 + next links
  u64* pool;
  int32_t* cnext;
  // chunk index of every group: linked blocks of 32 chunk ids in chunk order,
  // so a warp tests 32 chunks of a big group per step (deep_fit_warp)
  int32_t* tb_ids;                     // [tcap][32]
  int32_t* tb_next;                    // [tcap]
  int32_t* gtb_first;                  // gcap
  int32_t* gtb_last;                   // gcap
  int64_t tcap;
  uint32_t* tb_pool_next;
  // deep-fit queue: (batch term, group) pairs whose first chunk commutes and
  // whose group has more chunks, finished by k_group_deepfit with every warp
  uint2* dq;
  uint32_t* dq_count;
  uint32_t dq_cap;
  // scalars
  uint32_t* gcur;                      // groups so far
  uint32_t* pool_next;
  uint32_t* overflow;
  unsigned long long* checks;
  // per batch
  uint32_t* fit0;                      // [kGB][gw_stride]
  int64_t gw_stride;
  int32_t* fitk;                       // [kGB][kGK]
  int32_t* nfit;                       // [kGB]
  uint32_t* anti;                      // [kGB][kGAW]
  uint32_t* member;                    // [kGB] member index inside its group
  int32_t* tslot;                      // [kGB] resolver slot of each term
  int32_t* slot_old;                   // [kGB]
  int32_t* slot_chunks;                // [kGB][kSlotChunks]
  int32_t* group_of;                   // M (output)
};

__device__ __forceinline__ int swap_entry(int e, int W) { return e < 64 * W ? e + 64 * W : e - 64 * W; }

// ------------------------------------------------------------ fit tests
// Does the term with entry list lst[0..cnt) commute with every member of group
// g beyond its first chunk?  The whole warp walks the group's chunk index, 32
// chunks per step (lane l XORs the term's entries of chunk 32b + l).  Round 1
// walked the chunk list on the one thread that owned the term: a term
// duplicating a member of a 10^4-member group (config 5 injects 10%
// duplicates) kept one thread busy for ~150 dependent chunk visits while the
// GPU idled (k_group_fit: 1.3% issue utilisation, 69% of config 5 grouping).
template <int W>
__device__ __forceinline__ bool deep_fit_warp(const GCtx& G, int g, const uint16_t* lst,
                                              uint32_t cnt, int nchunks) {
  constexpr int E = 128 * W;
  const int lane = threadIdx.x & 31;
  int blk = G.gtb_first[g];
  bool ok = true;
  for (int o0 = 0; o0 < nchunks && ok && blk >= 0; o0 += 32) {
    const int o = o0 + lane;
    u64 acc = 0;
    if (o >= 1 && o < nchunks) {  // chunk 0 was tested from shared memory
      const u64* T = G.pool + (int64_t)G.tb_ids[(int64_t)blk * 32 + lane] * E;
      for (uint32_t k = 0; k < cnt; ++k) acc ^= T[lst[k]];
    }
    ok = !__any_sync(0xffffffffu, acc != 0ull);
    blk = G.tb_next[blk];
  }
  return ok;
}

// Two launch shapes, chosen on the device by the group count (the host never
// reads it): kFitBigThreads terms per CTA, one CTA per (32 groups, half of the
// batch) -- the staged group chunks are shared by 512 terms and three 64 KB
// CTAs fit an SM at W = 8 -- or kFitThreads-term blocks (4x the CTAs again: a
// few hundred groups -- config 3: 23 words -- still fill the SMs).  Each
// launch returns at once when the other shape applies.
constexpr uint32_t kDeepQueue = 1u << 20;  // deep-fit pairs queued per batch (the rest run inline)
constexpr int kFitThreads = 256;
constexpr int kFitBigThreads = 512;  // many groups: half the batch per CTA (three 64 KB CTAs per SM at W = 8)
constexpr int kFitSplitWords = 96;  // below this many 32-group words the split shape runs

__host__ __device__ constexpr int fit_gpc(int W, int threads) {
  return (W <= 2 && threads == kFitThreads) ? 32 : 8;
}

template <int W, int THREADS>
__global__ void __launch_bounds__(THREADS) k_group_fit(GCtx G, int64_t b0, int bn) {
  constexpr int E = 128 * W;
  // groups per shared-memory pass: 8 (8 KB x W); narrow strings in the split
  // shape stage all 32 groups of the word at once (64 KB at W = 2): one
  // staging + barrier phase per word instead of four, and 32 independent
  // loads per entry (config 3: the kernel is a chain of such phases on 92 CTAs)
  constexpr int GPC = fit_gpc(W, THREADS);
  extern __shared__ u64 S[];  // [GPC][E]
  if (*G.overflow) return;
  const uint32_t G0 = *G.gcur;
  if ((THREADS == kFitBigThreads) == (((int64_t)G0 + 31) / 32 < kFitSplitWords)) return;
  const int t = blockIdx.y * THREADS + threadIdx.x;
  const bool valid = t < bn;
  uint32_t off = 0, cnt = 0;
  if (valid) {
    off = G.off[b0 + t];
    cnt = G.off[b0 + t + 1] - off;
  }
  const uint16_t* lst = G.list + off;
  const int64_t nwords = ((int64_t)G0 + 31) / 32;
  for (int64_t gw = blockIdx.x; gw < nwords; gw += gridDim.x) {
    uint32_t word = 0;
#pragma unroll 1
    for (int h = 0; h < 32 / GPC; ++h) {
      const int64_t g0 = gw * 32 + h * GPC;
      // staging: eight (chunk pointer -> chunk word) load pairs in flight per
      // thread (a rolled loop issued them one pair at a time: a chain of 16
      // dependent HBM round trips per pass on config 5)
      static_assert((GPC * E) % (THREADS * 8) == 0 || GPC * E < THREADS * 8, "staging tiles");
      constexpr int kStageIter = GPC * E / THREADS;
      constexpr int kStageBatch = kStageIter < 8 ? kStageIter : 8;
#pragma unroll 1
      for (int it0 = 0; it0 < kStageIter; it0 += kStageBatch) {
        u64 v[kStageBatch];
#pragma unroll
        for (int u = 0; u < kStageBatch; ++u) {
          const int i = threadIdx.x + (it0 + u) * THREADS;
          const int64_t g = g0 + i / E;
          v[u] = g < G0 ? G.pool[(int64_t)G.gfirst[g] * E + i % E] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kStageBatch; ++u) S[threadIdx.x + (it0 + u) * THREADS] = v[u];
      }
      __syncthreads();
      uint32_t cand = 0;  // staged groups whose first chunk commutes with the term
      if (valid && g0 < G0) {
        u64 acc[GPC];
#pragma unroll
        for (int q = 0; q < GPC; ++q) acc[q] = 0;
        for (uint32_t k = 0; k < cnt; ++k) {
          const int e = lst[k];
#pragma unroll
          for (int q = 0; q < GPC; ++q) acc[q] ^= S[q * E + e];
        }
#pragma unroll
        for (int q = 0; q < GPC; ++q) cand |= (acc[q] == 0 && g0 + q < G0 ? 1u : 0u) << q;
        for (uint32_t cb = cand; cb; cb &= cb - 1) {
          const int q = __ffs(cb) - 1;
          if (G.gsize[g0 + q] <= 64) {  // one-chunk groups are settled
            word |= 1u << (h * GPC + q);
            cand &= ~(1u << q);
          } else {  // the rest of the group's chunks: queued for k_group_deepfit
            const uint32_t slot = atomicAdd(G.dq_count, 1u);
            if (slot < G.dq_cap) {
              G.dq[slot] = make_uint2((uint32_t)t, (uint32_t)(g0 + q));
              cand &= ~(1u << q);
            }
          }
        }
      }
      // (queue full: the warp finishes the remaining pairs itself, one at a time)
      for (unsigned pend = __ballot_sync(0xffffffffu, cand != 0u); pend;
           pend = __ballot_sync(0xffffffffu, cand != 0u)) {
        const int L = __ffs(pend) - 1;
        const int q = __ffs(__shfl_sync(0xffffffffu, cand, L)) - 1;
        const int g = (int)(g0 + q);
        const uint32_t off_l = __shfl_sync(0xffffffffu, off, L);
        const uint32_t cnt_l = __shfl_sync(0xffffffffu, cnt, L);
        const bool fits = deep_fit_warp<W>(G, g, G.list + off_l, cnt_l, (int)((G.gsize[g] + 63) / 64));
        if ((threadIdx.x & 31) == L) {
          if (fits) word |= 1u << (h * GPC + q);
          cand &= ~(1u << q);
        }
      }
      __syncthreads();
    }
    if (valid) G.fit0[(int64_t)t * G.gw_stride + gw] = word;
  }
}

// Deep fits of the queued (term, group) pairs, one pair per warp at a time over
// the whole GPU; a fitting pair sets its bit in the term's fit0 row.  Inside
// k_group_fit the pairs ran between the CTA's barriers on whichever warp owned
// the term: the groups with many chunks sit in the first words, so a few CTAs
// carried most of them.
template <int W>
__global__ void __launch_bounds__(256) k_group_deepfit(GCtx G, int64_t b0) {
  if (*G.overflow) return;
  const uint32_t n = min(*G.dq_count, G.dq_cap);
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nwarps) {
    const uint2 pr = G.dq[i];
    const uint32_t off = G.off[b0 + pr.x], cnt = G.off[b0 + pr.x + 1] - off;
    const int g = (int)pr.y;
    if (deep_fit_warp<W>(G, g, G.list + off, cnt, (int)((G.gsize[g] + 63) / 64)) &&
        (threadIdx.x & 31) == 0)
      atomicOr(&G.fit0[(int64_t)pr.x * G.gw_stride + (g >> 5)], 1u << (g & 31));
  }
}

// first kGK fitting groups of each batch term (warp per term)
__global__ void __launch_bounds__(1024) k_group_firstk(GCtx G, int bn) {
  if (*G.overflow) return;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= bn) return;
  const uint32_t G0 = *G.gcur;
  const int64_t nwords = ((int64_t)G0 + 31) / 32;
  const uint32_t* row = G.fit0 + (int64_t)t * G.gw_stride;
  int found = 0;
  int32_t mine = -1;
  for (int64_t base = 0; base < nwords && found <= kGK; base += 32) {
    const int64_t w = base + lane;
    uint32_t v = w < nwords ? row[w] : 0u;
    unsigned nz = __ballot_sync(0xffffffffu, v != 0);
    while (nz && found <= kGK) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      uint32_t bits = __shfl_sync(0xffffffffu, v, src);
      while (bits && found <= kGK) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        if (found < kGK && lane == found) mine = (int32_t)((base + src) * 32 + b);
        ++found;
      }
    }
  }
  if (lane < kGK) G.fitk[t * kGK + lane] = mine;
  if (lane == 0) G.nfit[t] = found;  // kGK + 1 means "more than kGK"
}

// ------------------------------------------------------------ resolver
// One warp replays the batch in term order, 32 terms (one per lane) at a time.
//
// Per group touched in the batch ("slot") the warp keeps BLOCKED[slot]: the OR
// of the intra-batch anti rows of the batch terms placed in it, so "does a
// batch member of the group anti-commute with term i" is ONE bit test (round
// 1 ANDed the term's anti row with the group's member mask: a 32-word
// reduction per candidate, every candidate a dependent chain on one warp,
// ~1000 cycles per term, 57% of config 3).
//
// Sub-block j = batch terms 32j..32j+31.  Its anti rows and candidate lists
// (the first kGK fitting old groups of every term, k_group_firstk) are staged
// in shared memory.  Rounds until every lane is settled:
//   1. every unsettled lane advances its own cursor over its candidate list
//      to the first group not blocked by the COMMITTED members (bit test);
//   2. a lane's pick is void if an earlier unsettled lane picked the same
//      group and anti-commutes with it (match.any + word j of the anti row),
//      or if it has no old group left ("hard");
//   3. the lanes before the first void one are committed together (slots,
//      member ranks, BLOCKED |= their anti rows).  A void pick becomes blocked
//      by that commit, so its cursor moves on in the next round.  Hard lanes
//      are settled alone: one whose list was complete can only join a group
//      opened in this batch (32 tested per step, one bit test per lane) or
//      open one -- lanes with an old candidate never pick those groups, so
//      such lanes do not end the round and are settled, in order, right after
//      the commit; one that fits more than kGK old groups ends the round and
//      walks the rest of its fit0 row from global memory first.
// Blocked bits only ever get set, so cursors never move back; the outcome is
// exactly the sequential first-fit.
constexpr int kMaskLd = kGAW + 1;  // padded rows: lanes reading one word of 32 rows hit 32 banks

struct ResolveSmem {
  int32_t hkey[kHash];
  int32_t hval[kHash];
  int32_t slot_group[kGB];
  int32_t slot_old[kGB];
  int32_t slot_cnt[kGB];
  int32_t newg[kGB];
  uint32_t aw[32 * kMaskLd];        // anti rows of the current sub-block (whole rows)
  int32_t cl[32 * (kGK + 1)];       // candidate lists of the current sub-block (padded rows)
  uint32_t blocked[kGB * kMaskLd];  // per slot: batch terms anti-commuting with a placed member
};

__device__ __forceinline__ int hfind(const ResolveSmem& R, int g) {
  int h = (int)(((unsigned)g * 2654435761u) >> 21) & (kHash - 1);
  for (;;) {
    const int k = R.hkey[h];
    if (k == g) return R.hval[h];
    if (k < 0) return -1;
    h = (h + 1) & (kHash - 1);
  }
}

__device__ __forceinline__ void hinsert(ResolveSmem& R, int g, int s) {
  int h = (int)(((unsigned)g * 2654435761u) >> 21) & (kHash - 1);
  while (R.hkey[h] >= 0) h = (h + 1) & (kHash - 1);
  R.hkey[h] = g;
  R.hval[h] = s;
}

struct ResolveState {
  uint32_t G0, gcur;
  int nslots, nnew;
  bool ovf;
};

// New slot for group g (warp-uniform): old = 0 for a group opened in this
// batch, -1 for a pre-existing one (its size is loaded after the replay).
__device__ __forceinline__ int new_slot(ResolveSmem& R, ResolveState& T, int g, int old) {
  const int lane = threadIdx.x;
  const int s = T.nslots++;
  if (lane == 0) {
    R.slot_group[s] = g;
    R.slot_old[s] = old;
    R.slot_cnt[s] = 0;
    hinsert(R, g, s);
  }
  R.blocked[s * kMaskLd + lane] = 0u;
  __syncwarp();
  return s;
}

// Settles batch term i alone (warp-uniform): the old groups after its listed
// candidates (last = the last listed one, -1 if the list was complete), the
// groups opened in this batch, else a new group.
__device__ __forceinline__ void resolve_hard(const GCtx& G, ResolveSmem& R, ResolveState& T,
                                             int64_t b0, int i, int64_t nwords, int last) {
  const int lane = threadIdx.x;
  const int l = i & 31, j = i >> 5;
  int chosen = -1, s = -1;
  if (last >= 0) {  // more than kGK fitting old groups: the row after group `last`, 32 words per step
    const uint32_t* row = G.fit0 + (int64_t)i * G.gw_stride;
    const int64_t w0 = (last + 1) / 32;
    for (int64_t base = w0; base < nwords && chosen < 0; base += 32) {
      const int64_t w = base + lane;
      uint32_t v = w < nwords ? row[w] : 0u;
      if (w == w0) v &= ~((1u << ((last + 1) & 31)) - 1u);
      unsigned nz = __ballot_sync(0xffffffffu, v != 0u);
      while (nz && chosen < 0) {
        const int src = __ffs(nz) - 1;
        nz &= nz - 1;
        uint32_t bits = __shfl_sync(0xffffffffu, v, src);
        while (bits && chosen < 0) {
          const int c = (int)((base + src) * 32) + __ffs(bits) - 1;
          bits &= bits - 1;
          const int sl = hfind(R, c);
          if (sl < 0 || !(R.blocked[sl * kMaskLd + j] >> l & 1u)) {
            chosen = c;
            s = sl;
          }
        }
      }
    }
    if (chosen >= 0 && s < 0) s = new_slot(R, T, chosen, -1);
  }
  for (int k0 = 0; k0 < T.nnew && chosen < 0; k0 += 32) {  // opened in this batch, creation order
    const int kk = k0 + lane;
    int sl = -1;
    bool ok = false;
    if (kk < T.nnew) {
      sl = R.newg[kk];
      ok = !(R.blocked[sl * kMaskLd + j] >> l & 1u);
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (m) {
      s = __shfl_sync(0xffffffffu, sl, __ffs(m) - 1);
      chosen = R.slot_group[s];
    }
  }
  if (chosen < 0) {
    if ((int64_t)T.gcur >= G.gcap) {
      T.ovf = true;
      return;
    }
    chosen = (int)T.gcur++;
    s = new_slot(R, T, chosen, 0);
    if (lane == 0) R.newg[T.nnew] = s;
    ++T.nnew;
  }
  R.blocked[s * kMaskLd + lane] |= R.aw[l * kMaskLd + lane];
  if (lane == 0) {
    G.group_of[b0 + i] = chosen;
    G.member[i] = (uint32_t)R.slot_cnt[s];  // rank among this batch's members
    G.tslot[i] = s;
    R.slot_cnt[s] += 1;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32, 1) k_group_resolve(GCtx G, int64_t b0, int bn) {
  extern __shared__ uint8_t smraw[];
  ResolveSmem& R = *reinterpret_cast<ResolveSmem*>(smraw);
  if (*G.overflow) return;
  const int lane = threadIdx.x;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int i = lane; i < kHash; i += 32) R.hkey[i] = -1;
  __syncwarp();
  ResolveState T;
  T.G0 = *G.gcur;
  T.gcur = T.G0;
  T.nslots = 0;
  T.nnew = 0;
  T.ovf = false;
  const int64_t nwords = ((int64_t)T.G0 + 31) / 32;
  // the next sub-block's anti rows and candidate lists wait in registers
  // (coalesced: 32 rows of 32 words; 32 lists of kGK ids = kGK words per lane)
  uint32_t nx[kGAW];
  int32_t ncl[kGK];
  int nnf = lane < bn ? G.nfit[lane] : 0;
#pragma unroll
  for (int r = 0; r < kGAW; ++r) nx[r] = r < bn ? G.anti[(int64_t)r * kGAW + lane] : 0u;
#pragma unroll
  for (int r = 0; r < kGK; ++r) ncl[r] = G.fitk[r * 32 + lane];  // (in bounds: kGB lists)
#ifdef PLB_RES_PROF
  long long tp[6] = {0, 0, 0, 0, 0, 0};
  int nrounds = 0, nhard = 0;
#define RES_T(k, expr) { const long long t0_ = clock64(); expr; tp[k] += clock64() - t0_; }
#else
#define RES_T(k, expr) { expr; }
#endif
  for (int i0 = 0, j = 0; i0 < bn && !T.ovf; i0 += 32, ++j) {
    const int cnt = bn - i0 < 32 ? bn - i0 : 32;
#ifdef PLB_RES_PROF
    const long long ts0 = clock64();
#endif
#pragma unroll
    for (int r = 0; r < kGAW; ++r) R.aw[r * kMaskLd + lane] = nx[r];
#pragma unroll
    for (int r = 0; r < kGK; ++r) {
      const int e = r * 32 + lane;  // list e / kGK, entry e % kGK
      R.cl[(e / kGK) * (kGK + 1) + (e % kGK)] = ncl[r];
    }
    const int nf = nnf;                       // fitting old groups (kGK + 1 = more than listed)
    const int ncand = nf < kGK ? nf : kGK;
    if (i0 + 32 < bn) {
#pragma unroll
      for (int r = 0; r < kGAW; ++r) {
        const int64_t t = i0 + 32 + r;
        nx[r] = t < bn ? G.anti[t * kGAW + lane] : 0u;
      }
#pragma unroll
      for (int r = 0; r < kGK; ++r) ncl[r] = G.fitk[(i0 + 32) * kGK + r * 32 + lane];
      nnf = i0 + 32 + lane < bn ? G.nfit[i0 + 32 + lane] : 0;
    }
    __syncwarp();
    const uint32_t arow_j = R.aw[lane * kMaskLd + j] & lt_mask;  // anti with earlier lanes
    unsigned todo = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);  // unsettled lanes
    int ck = 0;                                                    // cursor into the candidate list
#ifdef PLB_RES_PROF
    tp[0] += clock64() - ts0;
#endif
    while (todo && !T.ovf) {
#ifdef PLB_RES_PROF
      ++nrounds;
      const long long tr0 = clock64();
#endif
      const bool mine = todo >> lane & 1u;
      // 1. first fitting old group not blocked by the committed members
      int cand = -1, cslot = -1;
      if (mine) {
        for (; ck < ncand; ++ck) {
          const int c = R.cl[lane * (kGK + 1) + ck];
          const int sl = hfind(R, c);
          if (sl < 0 || !(R.blocked[sl * kMaskLd + j] >> lane & 1u)) {
            cand = c;
            cslot = sl;
            break;
          }
        }
      }
#ifdef PLB_RES_PROF
      const long long tr1 = clock64();
      tp[1] += tr1 - tr0;
#endif
      // 2. void picks: an earlier unsettled lane took the same group and anti-commutes
      // A lane with no old group left and a complete list can only go to a
      // group opened inside this batch; such groups are never chosen by lanes
      // that still have an old candidate, so it does not end the round: it is
      // deferred and settled (in lane order) after this round's commit.
      const unsigned have = __ballot_sync(0xffffffffu, mine && cand >= 0);
      const bool deferred = mine && cand < 0 && nf <= kGK;
      bool bad = mine && cand < 0 && nf > kGK;  // the rest of its fit0 row holds old groups
      if (mine && cand >= 0) {
        const unsigned peers = __match_any_sync(have, cand);
        bad = (arow_j & peers) != 0u;
      }
      const unsigned badm = __ballot_sync(0xffffffffu, bad);
      const int first_bad = badm ? __ffs(badm) - 1 : 32;
      const unsigned before_bad = first_bad >= 32 ? 0xffffffffu : ((1u << first_bad) - 1u);
      const unsigned okm = have & before_bad;
      const unsigned defm = __ballot_sync(0xffffffffu, deferred) & before_bad;
#ifdef PLB_RES_PROF
      const long long tr2 = clock64();
      tp[2] += tr2 - tr1;
#endif
      // 3. commit the lanes before the first void one
      if (okm) {
        const bool done = okm >> lane & 1u;
        // slots for the groups first touched in this batch, all at once: the
        // lowest lane of every distinct group takes the next slot number,
        // enters it in the hash table (lock-free: atomicCAS on the key) and
        // hands it to its peers; the BLOCKED rows are cleared by the whole warp
        const bool needs = done && cslot < 0;
        const unsigned need = __ballot_sync(0xffffffffu, needs);
        if (need) {
          unsigned peers = 0;
          if (needs) peers = __match_any_sync(need, cand);
          const bool leader = needs && (peers & lt_mask) == 0u;
          const unsigned leaders = __ballot_sync(0xffffffffu, leader);
          const int base_slot = T.nslots;
          int s_new = base_slot + __popc(leaders & lt_mask);
          if (leader) {
            R.slot_group[s_new] = cand;
            R.slot_old[s_new] = -1;  // pre-existing group: size loaded after the replay
            R.slot_cnt[s_new] = 0;
            int h = (int)(((unsigned)cand * 2654435761u) >> 21) & (kHash - 1);
            while (atomicCAS(&R.hkey[h], -1, cand) != -1) h = (h + 1) & (kHash - 1);
            R.hval[h] = s_new;
          }
          if (needs) cslot = __shfl_sync(need, s_new, __ffs(peers) - 1);
          const int n_new = __popc(leaders);
          for (int k = 0; k < n_new; ++k) R.blocked[(base_slot + k) * kMaskLd + lane] = 0u;
          T.nslots = base_slot + n_new;
          __syncwarp();
        }
        if (done) {
          const unsigned peers = __match_any_sync(okm, cslot);
          const int before = __popc(peers & lt_mask);
          const int base = R.slot_cnt[cslot];
          __syncwarp(okm);
          if (before == 0) R.slot_cnt[cslot] = base + __popc(peers);
          const int i = i0 + lane;
          G.group_of[b0 + i] = cand;
          G.member[i] = (uint32_t)(base + before);  // rank among this batch's members
          G.tslot[i] = cslot;
        }
        __syncwarp();
#ifdef PLB_RES_PROF
        const long long tc1 = clock64();
        tp[5] += tc1 - tr2;
#endif
        // BLOCKED[slot] |= the member's anti row, lane = word, two committed
        // terms per step (their read-modify-writes are independent unless they
        // share the slot).  Shared-memory atomics (lane = term, loop over
        // words) cost ~85 cycles each here and do not pipeline: 168k of a
        // batch's 470k cycles on config 3; one term per step 114k.
        for (unsigned m = okm; m;) {  // two committed terms per step
          const int l_a = __ffs(m) - 1;
          m &= m - 1;
          const bool two = m != 0u;
          const int l_b = two ? __ffs(m) - 1 : l_a;
          m &= m - 1;
          const int s_a = __shfl_sync(0xffffffffu, cslot, l_a);
          const int s_b = __shfl_sync(0xffffffffu, cslot, l_b);
          const uint32_t v_a = R.aw[l_a * kMaskLd + lane];
          const uint32_t v_b = two ? R.aw[l_b * kMaskLd + lane] : 0u;
          const uint32_t o_a = R.blocked[s_a * kMaskLd + lane];
          const uint32_t o_b = R.blocked[s_b * kMaskLd + lane];
          if (s_a == s_b) {
            R.blocked[s_a * kMaskLd + lane] = o_a | v_a | v_b;
          } else {
            R.blocked[s_a * kMaskLd + lane] = o_a | v_a;
            R.blocked[s_b * kMaskLd + lane] = o_b | v_b;
          }
        }
        __syncwarp();
        todo &= ~okm;
      }
#ifdef PLB_RES_PROF
      const long long tr3 = clock64();
      tp[3] += tr3 - tr2;
#endif
      for (unsigned m = defm; m && !T.ovf; m &= m - 1) {  // deferred lanes, in order
        resolve_hard(G, R, T, b0, i0 + __ffs(m) - 1, nwords, -1);
#ifdef PLB_RES_PROF
        ++nhard;
#endif
      }
      todo &= ~defm;
      if (first_bad < 32 && !T.ovf) {
        const bool hard = __shfl_sync(0xffffffffu, (int)(cand < 0), first_bad) != 0;
        if (hard) {  // listed candidates exhausted, more old groups in the fit0 row
          const int last = R.cl[first_bad * (kGK + 1) + kGK - 1];
          resolve_hard(G, R, T, b0, i0 + first_bad, nwords, last);
          todo &= ~(1u << first_bad);
        }
        // a void pick is blocked by the commit above: its cursor moves on next round
#ifdef PLB_RES_PROF
        if (hard) ++nhard;
#endif
      }
#ifdef PLB_RES_PROF
      tp[4] += clock64() - tr3;
#endif
    }
  }
#ifdef PLB_RES_PROF
  if (lane == 0 && (b0 == 51200 || b0 == 10240))
    printf("RESPROF b0=%lld stage=%lld cursor=%lld vote=%lld commit=%lld (pre-blocked %lld) hard=%lld rounds=%d nhard=%d nslots=%d nnew=%d\n",
           (long long)b0, tp[0], tp[1], tp[2], tp[3], tp[5], tp[4], nrounds, nhard, T.nslots, T.nnew);
#endif
  if (T.ovf) {
    if (lane == 0) *G.overflow = 1;
    return;
  }
  const int nslots = T.nslots;
  const uint32_t gcur = T.gcur;
  // grow every touched group: allocate chunks, link, record chunk tables
  for (int s = lane; s < nslots; s += 32) {
    const int g = R.slot_group[s];
    const int old = R.slot_old[s] < 0 ? (int)G.gsize[g] : R.slot_old[s];
    const int nw = old + R.slot_cnt[s];
    const int have = (old + 63) / 64, need = (nw + 63) / 64;
    const int add = need - have;
    int base = 0;
    if (add > 0) base = (int)atomicAdd(G.pool_next, (uint32_t)add);
    if ((int64_t)base + add > G.ccap) {
      *G.overflow = 1;
      continue;
    }
    int prev = have > 0 ? G.glast[g] : -1;
    int32_t* tab = G.slot_chunks + (int64_t)s * kSlotChunks;
    int k = 0;
    if (old % 64) tab[k++] = prev;  // partially filled last chunk
    for (int a = 0; a < add; ++a) {
      const int id = base + a;
      G.cnext[id] = -1;
      if (prev < 0) G.gfirst[g] = id;
      else G.cnext[prev] = id;
      prev = id;
      tab[k++] = id;
      // chunk index: ordinal have + a of group g
      const int ord = have + a;
      if ((ord & 31) == 0) {
        const int nb = (int)atomicAdd(G.tb_pool_next, 1u);
        if ((int64_t)nb >= G.tcap) {
          *G.overflow = 1;
          break;
        }
        G.tb_next[nb] = -1;
        if (ord == 0) G.gtb_first[g] = nb;
        else G.tb_next[G.gtb_last[g]] = nb;
        G.gtb_last[g] = nb;
      }
      G.tb_ids[(int64_t)G.gtb_last[g] * 32 + (ord & 31)] = id;
    }
    if (add > 0) G.glast[g] = prev;
    G.gsize[g] = (uint32_t)nw;
    G.slot_old[s] = old;
  }
  if (lane == 0) *G.gcur = gcur;
}

// ------------------------------------------------------------ update
// kUpdCtas CTAs; thread t of CTA c takes batch term kUpdCtas * t + c, so the
// pair_checks loops (u < i) of a CTA's warps have mixed lengths and the O(B^2)
// count is spread over kUpdCtas SMs (one 1024-thread CTA: 39 us per batch).
constexpr int kUpdCtas = 8;
constexpr int kUpdThreads = kGB / kUpdCtas;

template <int W>
__global__ void __launch_bounds__(kUpdThreads) k_group_update(GCtx G, int64_t b0, int bn,
                                                              const uint32_t* g0_snap) {
  constexpr int E = 128 * W;
  __shared__ __align__(16) int32_t sg[kGB];
  __shared__ unsigned long long red[kUpdThreads / 32];
  if (*G.overflow) return;
  const uint32_t g0_batch = *g0_snap;  // groups that existed at batch start
  for (int u = threadIdx.x; u < bn; u += kUpdThreads) sg[u] = G.group_of[b0 + u];
  __syncthreads();
  const int i = threadIdx.x * kUpdCtas + blockIdx.x;
  unsigned long long chk = 0;
  if (i < bn) {
    const int s = G.tslot[i];
    const int old = G.slot_old[s];
    const uint32_t m = (uint32_t)old + G.member[i];  // member index inside the group
    const int chunk = G.slot_chunks[(int64_t)s * kSlotChunks + (int)(m / 64) - old / 64];
    const u64 bit = 1ull << (m & 63);
    const uint32_t off = G.off[b0 + i], cnt = G.off[b0 + i + 1] - off;
    u64* T = G.pool + (int64_t)chunk * E;
    for (uint32_t k = 0; k < cnt; ++k) atomicOr(&T[swap_entry(G.list[off + k], W)], bit);
    // pair_checks: #{u < t : group(u) <= group(t)}
    const int c = sg[i];
    uint32_t cnt_le = 0;
    int u = 0;
    for (; u + 4 <= i; u += 4) {  // sg is 16-byte aligned: one 128-bit load per four terms
      const int4 v = *reinterpret_cast<const int4*>(&sg[u]);
      cnt_le += (v.x <= c) + (v.y <= c) + (v.z <= c) + (v.w <= c);
    }
    for (; u < i; ++u) cnt_le += sg[u] <= c ? 1u : 0u;
    chk = ((uint32_t)c < g0_batch ? (unsigned long long)G.gpre[c] : (unsigned long long)b0) + cnt_le;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) chk += __shfl_xor_sync(0xffffffffu, chk, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = chk;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < kUpdThreads / 32; ++w) s += red[w];
    atomicAdd(G.checks, s);
  }
}

// inclusive prefix of group sizes at batch start (single CTA) + G0 snapshot
__global__ void __launch_bounds__(1024) k_group_prefix(GCtx G, uint32_t* g0_out) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  if (*G.overflow) return;
  const uint32_t G0 = *G.gcur;
  if (threadIdx.x == 0) {
    carry = 0;
    *g0_out = G0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < G0; base += blockDim.x) {
    const uint32_t g = base + threadIdx.x;
    const uint32_t v = g < G0 ? G.gsize[g] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      before += w < wid ? wsum[w] : 0u;
      tot += wsum[w];
    }
    if (g < G0) G.gpre[g] = carry + before + inc;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// Intra-batch anti rows of up to kAntiSuper consecutive batches in one launch
// (blockIdx.z = batch): they do not depend on the grouping state, and one
// batch alone (4 CTAs) leaves the GPU idle (config 3: 33 us per batch, 98
// launches; config 5: 65 ms of 593).
constexpr int kAntiSuper = 64;

template <int W>
__global__ void __launch_bounds__(1024, 1)
k_group_anti_batches(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
                     int64_t b_first, const uint32_t* __restrict__ off,
                     const uint16_t* __restrict__ list, uint32_t* __restrict__ anti_all) {
  const int64_t b0 = b_first + (int64_t)blockIdx.z * kGB;
  if (b0 >= M) return;
  const int64_t bn = M - b0 < kGB ? M - b0 : kGB;
  if ((int64_t)blockIdx.y * 256 >= bn) return;
  bitmatrix_lists_body<W>(x, z, ld, M, b0, bn, b0, bn, off + b0, list,
                          anti_all + (int64_t)blockIdx.z * kGB * kGAW, kGAW, 256);
}

// ------------------------------------------------------------ host side
static inline int64_t a256(int64_t v) { return (v + 255) & ~(int64_t)255; }

struct GLayout {
  int64_t off, scratch, fixed_end;  // after fixed_end: list | groups | pool
};

static int64_t per_group_bytes(int W, int64_t gw_stride_per_group) {
  (void)gw_stride_per_group;
  return 4 * 4 /* gsize gfirst glast gpre */ + kGB / 8 /* fit0 bits */ +
         (128LL * W * 8 + 4) /* one chunk */ + 2 * 4 + 132 + 5 /* chunk index: ends, a block, id */;
}

static int64_t fixed_bytes(int W, int64_t M) {
  (void)W;
  int64_t o = 0;
  o += a256((M + 1) * 4);                       // off
  o += a256(scan_scratch_words(M) * 4);         // scan scratch
  o += a256(64);                                // scalars
  o += a256((int64_t)kGB * kGK * 4) + a256(kGB * 4) + a256((int64_t)kAntiSuper * kGB * kGAW * 4);
  o += a256(kGB * 4) * 3 + a256((int64_t)kGB * kSlotChunks * 4);
  o += a256(16);                                // g0 snapshot
  o += a256((int64_t)kDeepQueue * 8);           // deep-fit queue
  return o;
}

template <int W>
static int run_group(int64_t M, const u64* x, const u64* z, int64_t ld, int32_t* group_of,
                     int32_t* n_groups, int64_t* pair_checks, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  uint8_t* b = (uint8_t*)ws;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    uint8_t* p = b + o;
    o = a256(o + bytes);
    return p;
  };
  GCtx G{};
  G.W = W;
  G.M = M;
  G.x = x;
  G.z = z;
  G.ld = ld;
  uint32_t* off = (uint32_t*)take((M + 1) * 4);
  uint32_t* scratch = (uint32_t*)take(scan_scratch_words(M) * 4);
  uint32_t* scal = (uint32_t*)take(64);
  G.fitk = (int32_t*)take((int64_t)kGB * kGK * 4);
  G.nfit = (int32_t*)take(kGB * 4);
  uint32_t* anti_all = (uint32_t*)take((int64_t)kAntiSuper * kGB * kGAW * 4);
  G.anti = anti_all;
  G.member = (uint32_t*)take(kGB * 4);
  G.tslot = (int32_t*)take(kGB * 4);
  G.slot_old = (int32_t*)take(kGB * 4);
  G.slot_chunks = (int32_t*)take((int64_t)kGB * kSlotChunks * 4);
  uint32_t* g0snap = (uint32_t*)take(16);
  G.dq_cap = kDeepQueue;
  if (const char* e = getenv("PLB_DEEP_QUEUE_CAP")) {  // tests: force the inline deep-fit fallback
    const long v = atol(e);
    if (v >= 0 && (unsigned long)v < kDeepQueue) G.dq_cap = (uint32_t)v;
  }
  G.dq = (uint2*)take((int64_t)kDeepQueue * 8);
  if (o > (int64_t)ws_bytes) {
    set_error("pl_group_greedy: workspace too small");
    return PL_ERR_WORKSPACE;
  }
  PLB_CUDA(cudaMemsetAsync(scal, 0, 64, st));
  G.gcur = scal;
  G.pool_next = scal + 1;
  G.overflow = scal + 2;
  G.tb_pool_next = scal + 8;
  G.dq_count = scal + 9;
  G.checks = (unsigned long long*)(scal + 4);
  // CSR entry lists of every term (same encoding as the bitmatrix)
  const unsigned nb = (unsigned)ceil_div(M, 256);
  {
    StageTimer t_(st, "k_row_weight");
    k_row_weight<W><<<nb, 256, 0, st>>>(x, z, ld, 0, M, off);
    PLB_CHECK_LAUNCH("k_row_weight");
  }
  int rc = exclusive_scan_u32(off, off, M, scratch, off + M, st);
  if (rc) return rc;
  uint32_t total = 0;
  PLB_CUDA(cudaMemcpyAsync(&total, off + M, 4, cudaMemcpyDeviceToHost, st));
  PLB_CUDA(cudaStreamSynchronize(st));
  uint16_t* list = (uint16_t*)take((int64_t)total * 2 + 16);
  G.off = off;
  G.list = list;
  // remaining bytes -> group capacity
  const int64_t rest = (int64_t)ws_bytes - o - 8192;
  const int64_t chunk_bytes = 128LL * W * 8 + 4 + 5;  // chunk, link, share of an index block
  const int64_t member_chunks = (M + 63) / 64;
  int64_t gcap = (rest - member_chunks * chunk_bytes) / per_group_bytes(W, 0);
  if (gcap > M) gcap = M;
  if (gcap < 1) {
    set_error("pl_group_greedy: workspace too small for the entry lists (%u entries)", total);
    return PL_ERR_WORKSPACE;
  }
  G.gcap = gcap;
  G.ccap = gcap + member_chunks;
  G.gw_stride = (gcap + 31) / 32;
  G.gsize = (uint32_t*)take(gcap * 4);
  G.gfirst = (int32_t*)take(gcap * 4);
  G.glast = (int32_t*)take(gcap * 4);
  G.gpre = (uint32_t*)take(gcap * 4);
  G.fit0 = (uint32_t*)take((int64_t)kGB * G.gw_stride * 4);
  G.cnext = (int32_t*)take(G.ccap * 4);
  G.tcap = G.ccap / 32 + gcap + 2;
  G.tb_ids = (int32_t*)take(G.tcap * 32 * 4);
  G.tb_next = (int32_t*)take(G.tcap * 4);
  G.gtb_first = (int32_t*)take(gcap * 4);
  G.gtb_last = (int32_t*)take(gcap * 4);
  G.pool = (u64*)take(G.ccap * 128LL * W * 8);
  if (o > (int64_t)ws_bytes) {
    set_error("pl_group_greedy: workspace layout overflow");
    return PL_ERR_WORKSPACE;
  }
  PLB_CUDA(cudaMemsetAsync(G.gsize, 0, gcap * 4, st));
  PLB_CUDA(cudaMemsetAsync(G.pool, 0, G.ccap * 128LL * W * 8, st));
  G.group_of = group_of;
  {
    StageTimer t_(st, "k_row_fill");
    k_row_fill<W><<<nb, 256, 0, st>>>(x, z, ld, 0, M, off, list);
    PLB_CHECK_LAUNCH("k_row_fill");
  }
  const size_t fit_smem = (size_t)8 * 128 * W * 8;
  const size_t fit_smem_split = (size_t)fit_gpc(W, kFitThreads) * 128 * W * 8;
  PLB_CUDA(cudaFuncSetAttribute(k_group_fit<W, kFitBigThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fit_smem));
  PLB_CUDA(cudaFuncSetAttribute(k_group_fit<W, kFitThreads>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fit_smem_split));
  PLB_CUDA(cudaFuncSetAttribute(k_group_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(ResolveSmem)));
  const size_t lists_smem = lists_smem_bytes<(W <= 8 ? W : 8)>();
  if (W <= 8) {
    PLB_CUDA(cudaFuncSetAttribute(k_group_anti_batches<(W <= 8 ? W : 8)>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lists_smem));
  }
  const int fit_grid = 2 * num_sms();
  for (int64_t b0 = 0; b0 < M; b0 += kGB) {
    const int bn = (int)std::min<int64_t>(kGB, M - b0);
    {
      StageTimer t_(st, "k_group_prefix");
      k_group_prefix<<<1, 1024, 0, st>>>(G, g0snap);
    }
    if (W <= 8) {
      const int64_t bi = (b0 / kGB) % kAntiSuper;  // batch inside the super-batch
      G.anti = anti_all + bi * kGB * kGAW;
      if (bi == 0) {
        StageTimer t_(st, "k_group_anti");
        const int64_t nbatch = std::min<int64_t>(kAntiSuper, ceil_div(M - b0, (int64_t)kGB));
        k_group_anti_batches<(W <= 8 ? W : 8)><<<dim3(1, kGB / 256, (unsigned)nbatch), 1024,
                                                 lists_smem, st>>>(x, z, ld, M, b0, off, list,
                                                                   anti_all);
      }
    } else {
      StageTimer t_(st, "k_group_anti");
      {
        constexpr int kDC = DirectCols<W>::value;
        dim3 grid((unsigned)ceil_div(bn, kDC), (unsigned)ceil_div(bn, kDirectRows));
        k_bitmatrix_direct<W><<<grid, kDirectRows, 0, st>>>(x, z, ld, M, b0, bn, b0, bn, G.anti,
                                                            kGAW);
      }
    }
    if (b0 > 0) {
      PLB_CUDA(cudaMemsetAsync(G.dq_count, 0, 4, st));
      {
      StageTimer t_(st, "k_group_fit");
      k_group_fit<W, kFitThreads><<<dim3((unsigned)fit_grid, kGB / kFitThreads), kFitThreads,
                                    fit_smem_split, st>>>(G, b0, bn);
      k_group_fit<W, kFitBigThreads><<<dim3((unsigned)fit_grid, kGB / kFitBigThreads),
                                       kFitBigThreads, fit_smem, st>>>(G, b0, bn);
      }
      StageTimer t2_(st, "k_group_deepfit");
      k_group_deepfit<W><<<8 * num_sms(), 256, 0, st>>>(G, b0);
    }
    {
      StageTimer t_(st, "k_group_firstk");
      if (b0 > 0) k_group_firstk<<<kGB / 32, 1024, 0, st>>>(G, bn);
      else PLB_CUDA(cudaMemsetAsync(G.nfit, 0, kGB * 4, st));
    }
    {
      StageTimer t_(st, "k_group_resolve");
      k_group_resolve<<<1, 32, sizeof(ResolveSmem), st>>>(G, b0, bn);
    }
    {
      StageTimer t_(st, "k_group_update");
      k_group_update<W><<<kUpdCtas, kUpdThreads, 0, st>>>(G, b0, bn, g0snap);
    }
    PLB_CHECK_LAUNCH("grouping batch");
  }
  uint32_t ovf = 0;
  PLB_CUDA(cudaMemcpyAsync(&ovf, G.overflow, 4, cudaMemcpyDeviceToHost, st));
  PLB_CUDA(cudaMemcpyAsync(n_groups, G.gcur, 4, cudaMemcpyDeviceToDevice, st));
  PLB_CUDA(cudaMemcpyAsync(pair_checks, G.checks, 8, cudaMemcpyDeviceToDevice, st));
  PLB_CUDA(cudaStreamSynchronize(st));
  if (ovf) {
    set_error("pl_group_greedy: group capacity %lld exceeded; pass a larger workspace",
              (long long)gcap);
    return PL_ERR_WORKSPACE;
  }
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int64_t pl_group_workspace_bytes(int W, int64_t M) {
  if (M <= 0 || !valid_words(W)) return 4096;
  // recommended: entry lists for ~24 set bits per term and groups for M/8
  const int64_t lists = M * 48 + 16;
  int64_t groups = M / 8;
  if (groups < 1024) groups = std::min<int64_t>(M, 1024);
  const int64_t chunks = (M + 63) / 64;
  return fixed_bytes(W, M) + a256(lists) + groups * per_group_bytes(W, 0) +
         chunks * (128LL * W * 8 + 4 + 5) + 64 * 256;
}

extern "C" int pl_group_greedy(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                               int64_t ld, int32_t* group_of, int32_t* n_groups,
                               int64_t* pair_checks, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (M < 0 || ld < M || !group_of || !n_groups || !pair_checks) {
    set_error("pl_group_greedy: bad arguments");
    return PL_ERR_ARG;
  }
  if (M * 128LL * (W > 0 ? W : 1) >= 0xFFFFFFFFLL || M >= (1LL << 31)) {
    set_error("pl_group_greedy: too many terms for 32-bit entry offsets");
    return PL_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) {
    PLB_CUDA(cudaMemsetAsync(n_groups, 0, 4, st));
    PLB_CUDA(cudaMemsetAsync(pair_checks, 0, 8, st));
    return PL_OK;
  }
  return PLB_DISPATCH_W(W, run_group, M, (const u64*)x, (const u64*)z, ld, group_of, n_groups,
                        pair_checks, workspace, workspace_bytes, st);
}
