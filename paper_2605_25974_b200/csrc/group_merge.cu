// §8(f) row f3 — merge phase of the two-phase parallel grouping
// (group_greedy_parallel, grouping.py:98-146).  Phase 1 (greedy per
// contiguous chunk) is K6 on each chunk's planes; this file restates the
// sequential merge exactly: local groups, in chunk order and creation order
// inside a chunk, each join the FIRST global group (creation order) with which
// every cross pair commutes, else open a new global group; pair_checks adds
// |local| * |global group| for every global group tried (grouping.py:129-131).
//
// Per local group L (the sequence is inherently ordered, so one pair of
// launches per local group, no host synchronisation in between):
//   k_merge_anti  every term already placed (gid >= 0) is checked against L's
//                 members (staged in shared memory, tiles of kMergeTile); an
//                 anti-commuting pair marks the term's global group for this
//                 epoch (anti_epoch[g] = epoch); a group already marked is
//                 skipped.
//   pick          the last CTA of k_merge_anti to finish (completion counter):
//                 first unmarked group in creation order (or a new one), the
//                 pair_checks contribution (|L| * sizes of the groups tried),
//                 L's members joined to it -- one launch per local group.
#include "common.cuh"

namespace plb {

constexpr int kMergeThreads = 256;
// L members per shared-memory tile (<= 16 KB of x/z words)
__host__ __device__ constexpr int merge_tile(int W) { return W >= 8 ? 1024 / W : 256; }

// first unmarked global group (or a new one) for local group `epoch`, the
// pair_checks contribution, and the members joined to it (one CTA)
__device__ void merge_pick(int32_t* __restrict__ gid, const int32_t* __restrict__ members,
                           int64_t lo, int64_t hi, int32_t epoch,
                           const int32_t* __restrict__ anti_epoch, int32_t* __restrict__ gsize,
                           int32_t* __restrict__ n_global, int32_t* __restrict__ global_of_local,
                           int64_t* __restrict__ pair_checks) {
  __shared__ int32_t s_first;
  __shared__ unsigned long long s_tried;
  const int32_t G = *(volatile int32_t*)n_global;
  if (threadIdx.x == 0) {
    s_first = G;
    s_tried = 0;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x)
    if (((volatile const int32_t*)anti_epoch)[g] != epoch) atomicMin(&s_first, g);
  __syncthreads();
  const int32_t first = s_first;
  // groups tried: 0..first (inclusive) when one fits, all G otherwise
  const int32_t last = first < G ? first : G - 1;
  unsigned long long part = 0;
  for (int g = threadIdx.x; g <= last; g += blockDim.x) part += (unsigned long long)gsize[g];
  if (part) atomicAdd(&s_tried, part);
  __syncthreads();
  const int64_t L = hi - lo;
  if (threadIdx.x == 0) {
    *pair_checks += (int64_t)s_tried * L;
    if (first == G) {
      gsize[G] = 0;
      *n_global = G + 1;
    }
    gsize[first] += (int32_t)L;
    global_of_local[epoch] = first;
  }
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) gid[members[i]] = first;
}

template <int W>
__global__ void __launch_bounds__(kMergeThreads)
k_merge_anti(const u64* __restrict__ x, const u64* __restrict__ z, int64_t ld, int64_t M,
             int32_t* __restrict__ gid, const int32_t* __restrict__ members, int64_t lo,
             int64_t hi, int32_t epoch, int32_t* __restrict__ anti_epoch,
             int32_t* __restrict__ gsize, int32_t* __restrict__ n_global,
             int32_t* __restrict__ global_of_local, int64_t* __restrict__ pair_checks,
             unsigned int* __restrict__ done) {
  constexpr int kMergeTile = merge_tile(W);
  __shared__ u64 lx[W][kMergeTile], lz[W][kMergeTile];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t g = t < M ? gid[t] : -1;
  bool live = g >= 0 && anti_epoch[g] != epoch;
  u64 tx[W], tz[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    tx[w] = live ? x[w * ld + t] : 0ull;
    tz[w] = live ? z[w * ld + t] : 0ull;
  }
  for (int64_t b = lo; b < hi; b += kMergeTile) {
    const int n = (int)(hi - b < kMergeTile ? hi - b : kMergeTile);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t m = members[b + i];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        lx[w][i] = x[w * ld + m];
        lz[w][i] = z[w * ld + m];
      }
    }
    __syncthreads();
    if (!__syncthreads_or(live)) continue;
    if (live) {
      bool anti = false;
      for (int i = 0; i < n && !anti; ++i) {
        u64 acc = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) acc ^= (tx[w] & lz[w][i]) ^ (tz[w] & lx[w][i]);
        anti = popc64(acc) & 1;
      }
      if (anti) {
        anti_epoch[g] = epoch;
        live = false;
      }
    }
  }
  // the last CTA to finish picks (no second launch per local group)
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  merge_pick(gid, members, lo, hi, epoch, anti_epoch, gsize, n_global, global_of_local,
             pair_checks);
  if (threadIdx.x == 0) *done = 0u;  // ready for the next local group
}

__global__ void __launch_bounds__(1024)
k_merge_pick(int32_t* __restrict__ gid, const int32_t* __restrict__ members, int64_t lo,
             int64_t hi, int32_t epoch, const int32_t* __restrict__ anti_epoch,
             int32_t* __restrict__ gsize, int32_t* __restrict__ n_global,
             int32_t* __restrict__ global_of_local, int64_t* __restrict__ pair_checks) {
  merge_pick(gid, members, lo, hi, epoch, anti_epoch, gsize, n_global, global_of_local,
             pair_checks);
}

template <int W>
static int run_merge(int64_t M, const u64* x, const u64* z, int64_t ld, const int32_t* members,
                     const int64_t* local_off, int32_t n_local, int32_t* global_of_local,
                     int32_t* n_global, int64_t* pair_checks, void* ws, cudaStream_t st) {
  int32_t* gid = (int32_t*)ws;
  int32_t* anti_epoch = gid + M;
  int32_t* gsize = anti_epoch + n_local;
  unsigned int* done = (unsigned int*)(gsize + n_local);
  PLB_CUDA(cudaMemsetAsync(gid, 0xFF, 4 * (size_t)M, st));           // -1: not placed yet
  PLB_CUDA(cudaMemsetAsync(anti_epoch, 0xFF, 4 * (size_t)n_local, st));
  PLB_CUDA(cudaMemsetAsync(n_global, 0, 4, st));
  PLB_CUDA(cudaMemsetAsync(done, 0, 4, st));
  const unsigned grid = (unsigned)ceil_div(M, kMergeThreads);
  StageTimer t_(st, "k_group_merge");
  for (int32_t l = 0; l < n_local; ++l) {
    const int64_t lo = local_off[l], hi = local_off[l + 1];
    if (l > 0)  // marks, then its last CTA picks
      k_merge_anti<W><<<grid, kMergeThreads, 0, st>>>(x, z, ld, M, gid, members, lo, hi, l,
                                                      anti_epoch, gsize, n_global,
                                                      global_of_local, pair_checks, done);
    else
      k_merge_pick<<<1, 1024, 0, st>>>(gid, members, lo, hi, l, anti_epoch, gsize, n_global,
                                        global_of_local, pair_checks);
  }
  PLB_CHECK_LAUNCH("k_group_merge");
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int64_t pl_group_merge_workspace_bytes(int64_t M, int32_t n_local) {
  return 4 * (M + 2 * (int64_t)n_local + 64);  // gid | anti_epoch | gsize | done
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
