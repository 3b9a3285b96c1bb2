// §8(f) row f3 — merge phase of the two-phase parallel grouping
// (group_greedy_parallel, grouping.py:98-146).  Phase 1 (greedy per
// contiguous chunk) is K6 on each chunk's planes; this file restates the
// sequential merge exactly: local groups, in chunk order and creation order
// inside a chunk, each join the FIRST global group (creation order) with which
// every cross pair commutes, else open a new global group; pair_checks adds
// |local| * |global group| for every global group tried (grouping.py:129-131).
//
// The sequence is ordered, but the pair tests are not: local groups are taken
// kMergeBatch at a time (K6's scheme at group granularity).
//   k_merge_anti  every term already placed, and every term of the batch, is
//                 checked against the batch's members (staged in shared memory
//                 with their local-group index): an anti-commuting pair marks
//                 bad[local][global group of the placed term] or, inside the
//                 batch, cross[earlier local][later local].  A thread skips a
//                 local group once its own group is marked for it.
//   k_merge_pick  one CTA replays the batch in order: the first global group
//                 not marked bad for the local group (bad also receives the
//                 cross marks of batch groups already placed there), else a
//                 new group; pair_checks; then the batch members' group ids.
// Round 1 launched one marking kernel per local group (2,400 launches on
// config 3 with 8 chunks, 28 ms, launch bound).
#include "common.cuh"

namespace plb {

constexpr int kMergeThreads = 256;
constexpr int kMergeBatch = 256;  // local groups per batch
// batch members per shared-memory tile (<= 16 KB of x/z words)
__host__ __device__ constexpr int merge_tile(int W) { return W >= 8 ? 1024 / W : 256; }

// lg[t] = local group of term t (members lists the terms group by group)
__global__ void k_merge_lgof(const int32_t* __restrict__ members, const int64_t* __restrict__ loff,
                             int32_t n_local, int64_t M, int32_t* __restrict__ lg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  int lo = 0, hi = n_local - 1;  // last l with loff[l] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (loff[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  lg[members[i]] = lo;
}

template <int W>
__global__ void __launch_bounds__(kMergeThreads)
k_merge_anti(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
             const int32_t* __restrict__ gid, const int32_t* __restrict__ lg,
             const int32_t* __restrict__ members, int64_t lo, int64_t hi, int32_t l0,
             uint8_t* bad, int64_t gstride, uint8_t* cross) {
  constexpr int kMergeTile = merge_tile(W);
  __shared__ u64 lx[W][kMergeTile], lz[W][kMergeTile];
  __shared__ int32_t ll[kMergeTile];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t g = t < M ? gid[t] : -1;
  const int32_t my = t < M ? lg[t] - l0 : -1;  // batch-local index of the term's own local group
  const bool placed = g >= 0;
  const bool inbatch = !placed && my >= 0 && my < kMergeBatch && t < M;
  const bool role = placed || inbatch;
  u64 tx[W], tz[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    tx[w] = role ? x[w * ld + t] : 0ull;
    tz[w] = role ? z[w * ld + t] : 0ull;
  }
  int cur = -1;      // batch-local group being scanned
  bool skip = true;  // nothing left to learn about `cur`
  volatile uint8_t* vbad = bad;
  volatile uint8_t* vcross = cross;
  for (int64_t b = lo; b < hi; b += kMergeTile) {
    const int n = (int)(hi - b < kMergeTile ? hi - b : kMergeTile);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t m = members[b + i];
      ll[i] = lg[m] - l0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        lx[w][i] = x[w * ld + m];
        lz[w][i] = z[w * ld + m];
      }
    }
    __syncthreads();
    if (!role) continue;
    for (int i = 0; i < n; ++i) {
      const int L = ll[i];
      if (L != cur) {  // next local group: anything to learn?
        cur = L;
        if (placed) skip = vbad[(int64_t)L * gstride + g] != 0;
        else skip = my >= L || vcross[my * kMergeBatch + L] != 0;
      }
      if (skip) continue;
      u64 acc = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) acc ^= (tx[w] & lz[w][i]) ^ (tz[w] & lx[w][i]);
      if (popc64(acc) & 1) {
        if (placed) vbad[(int64_t)L * gstride + g] = 1;
        else vcross[my * kMergeBatch + L] = 1;
        skip = true;
      }
    }
  }
}

// One CTA replays local groups [l0, l1) in order.
__global__ void __launch_bounds__(1024)
k_merge_pick(int32_t* __restrict__ gid, const int32_t* __restrict__ lg,
             const int32_t* __restrict__ members, const int64_t* __restrict__ loff, int32_t l0,
             int32_t l1, uint8_t* bad, int64_t gstride, const uint8_t* __restrict__ cross,
             int32_t* __restrict__ gsize, int32_t* __restrict__ n_global,
             int32_t* __restrict__ global_of_local, int64_t* __restrict__ pair_checks) {
  __shared__ int32_t s_first;
  __shared__ unsigned long long s_tried;
  __shared__ int32_t dest[kMergeBatch];
  int32_t G = *n_global;
  long long checks = 0;
  for (int32_t l = l0; l < l1; ++l) {
    const int b = l - l0;
    if (threadIdx.x == 0) {
      s_first = G;
      s_tried = 0;
    }
    __syncthreads();
    const uint8_t* row = bad + (int64_t)b * gstride;
    int mine = G;  // this thread's first unmarked group (warp minimum, one atomic per warp)
    for (int g = threadIdx.x; g < G && mine == G; g += blockDim.x)
      if (row[g] == 0) mine = g;
    mine = __reduce_min_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine < G) atomicMin(&s_first, mine);
    __syncthreads();
    const int32_t first = s_first;
    // groups tried: 0..first (inclusive) when one fits, all G otherwise
    const int32_t last = first < G ? first : G - 1;
    unsigned int part = 0;  // (sizes sum to at most M < 2^31)
    for (int g = threadIdx.x; g <= last; g += blockDim.x) part += (unsigned int)gsize[g];
    part = __reduce_add_sync(0xffffffffu, part);
    if ((threadIdx.x & 31) == 0 && part) atomicAdd(&s_tried, (unsigned long long)part);
    __syncthreads();
    const int64_t L = loff[l + 1] - loff[l];
    checks += (long long)s_tried * L;
    if (threadIdx.x == 0) {
      if (first == G) gsize[G] = 0;
      gsize[first] += (int32_t)L;
      global_of_local[l] = first;
      dest[b] = first;
    }
    if (first == G) ++G;
    // later batch groups with an anti-commuting pair against this one cannot join `first`
    for (int b2 = b + 1 + threadIdx.x; b2 < l1 - l0; b2 += blockDim.x)
      if (cross[b * kMergeBatch + b2]) bad[(int64_t)b2 * gstride + first] = 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *n_global = G;
    *pair_checks += checks;
  }
  for (int64_t i = loff[l0] + threadIdx.x; i < loff[l1]; i += blockDim.x) {
    const int32_t t = members[i];
    gid[t] = dest[lg[t] - l0];
  }
}

template <int W>
static int run_merge(int64_t M, const u64* x, const u64* z, int64_t ld, const int32_t* members,
                     const int64_t* local_off, int32_t n_local, int32_t* global_of_local,
                     int32_t* n_global, int64_t* pair_checks, void* ws, cudaStream_t st) {
  // workspace: gid | lg | gsize | loff (device copy) | cross | bad
  int32_t* gid = (int32_t*)ws;
  int32_t* lg = gid + M;
  int32_t* gsize = lg + M;
  int64_t* loff = (int64_t*)(((uintptr_t)(gsize + n_local + 1) + 15) & ~(uintptr_t)15);
  uint8_t* cross = (uint8_t*)(loff + n_local + 1);
  uint8_t* bad = cross + (size_t)kMergeBatch * kMergeBatch;
  const int64_t gstride = ((int64_t)n_local + 15) & ~(int64_t)15;  // a global group per local at most
  PLB_CUDA(cudaMemsetAsync(gid, 0xFF, 4 * (size_t)M, st));  // -1: not placed yet
  PLB_CUDA(cudaMemsetAsync(n_global, 0, 4, st));
  PLB_CUDA(cudaMemcpyAsync(loff, local_off, 8 * ((size_t)n_local + 1), cudaMemcpyHostToDevice, st));
  if (n_local == 0) return PL_OK;
  StageTimer t_(st, "k_group_merge");
  k_merge_lgof<<<(unsigned)ceil_div(M, 256), 256, 0, st>>>(members, loff, n_local, M, lg);
  const unsigned grid = (unsigned)ceil_div(M, kMergeThreads);
  for (int32_t l0 = 0; l0 < n_local; l0 += kMergeBatch) {
    const int32_t l1 = std::min<int32_t>(n_local, l0 + kMergeBatch);
    PLB_CUDA(cudaMemsetAsync(cross, 0, (size_t)kMergeBatch * kMergeBatch + (size_t)kMergeBatch * gstride, st));
    k_merge_anti<W><<<grid, kMergeThreads, 0, st>>>(x, z, ld, M, gid, lg, members, local_off[l0],
                                                    local_off[l1], l0, bad, gstride, cross);
    k_merge_pick<<<1, 256, 0, st>>>(gid, lg, members, loff, l0, l1, bad, gstride, cross, gsize,
                                      n_global, global_of_local, pair_checks);
  }
  PLB_CHECK_LAUNCH("k_group_merge");
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int64_t pl_group_merge_workspace_bytes(int64_t M, int32_t n_local) {
  // gid | lg | gsize | loff | cross | bad (see run_merge)
  const int64_t gstride = ((int64_t)n_local + 15) & ~(int64_t)15;
  return 4 * (2 * M + (int64_t)n_local + 1) + 16 + 8 * ((int64_t)n_local + 1) +
         (int64_t)plb::kMergeBatch * plb::kMergeBatch + (int64_t)plb::kMergeBatch * gstride + 256;
}

extern "C" int pl_group_merge(int W, int64_t M, const uint64_t* x, const uint64_t* z, int64_t ld,
                              const int32_t* members, const int64_t* local_off, int32_t n_local,
                              int32_t* global_of_local, int32_t* n_global, int64_t* pair_checks,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (!valid_words(W) || M < 0 || ld < M || n_local < 0 || !local_off || !n_global ||
      !pair_checks || (n_local > 0 && (!members || !global_of_local))) {
    set_error("pl_group_merge: bad arguments");
    return valid_words(W) ? PL_ERR_ARG : PL_ERR_TIER;
  }
  if ((int64_t)workspace_bytes < pl_group_merge_workspace_bytes(M, n_local) || !workspace) {
    set_error("pl_group_merge: workspace too small");
    return PL_ERR_WORKSPACE;
  }
  if (local_off[0] != 0 || (n_local > 0 && local_off[n_local] != M)) {
    set_error("pl_group_merge: local groups must partition the %lld terms", (long long)M);
    return PL_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return PLB_DISPATCH_W(W, run_merge, M, (const u64*)x, (const u64*)z, ld, members, local_off,
                        n_local, global_of_local, n_global, pair_checks, workspace, st);
}
