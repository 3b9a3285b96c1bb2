// K2-K4 C ABI: plans, workspace checks and the W dispatch into the per-W
// instantiations (combine_w*.cu); kernels are in combine_impl.cuh.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INSTANTIATE(extern, 1)
PLB_COMBINE_INSTANTIATE(extern, 2)
PLB_COMBINE_INSTANTIATE(extern, 4)
PLB_COMBINE_INSTANTIATE(extern, 8)
PLB_COMBINE_INSTANTIATE(extern, 16)
}  // namespace plb

using namespace plb;

extern "C" int pl_outer_plan(int W, int64_t Ma, int64_t Mb, const uint64_t* ax,
                             const uint64_t* az, int64_t lda, const uint64_t* bx,
                             const uint64_t* bz, int64_t ldb, pl_merge_plan* plan, void* stream) {
  if (!plan || !valid_words(W) || Ma < 0 || Mb < 0 || lda < Ma || ldb < Mb) {
    set_error("pl_outer_plan: bad arguments");
    return valid_words(W) ? PL_ERR_ARG : PL_ERR_TIER;
  }
  if (Ma * Mb > (1LL << 30)) {
    set_error("pl_outer_plan: |A|*|B| = %lld exceeds 2^30 raw terms per call",
              (long long)(Ma * Mb));
    return PL_ERR_CAPACITY;
  }
  *plan = pl_merge_plan{};
  plan->W = W;
  plan->mode = 0;
  plan->ma = Ma;
  plan->mb = Mb;
  plan->n_items = Ma * Mb;
  u64 masks[2 * PL_PLAN_MAX_SEG + 1] = {0};
  int rc = compute_masks(W, (const u64*)ax, (const u64*)az, lda, Ma, (const u64*)bx,
                         (const u64*)bz, ldb, Mb, masks, (cudaStream_t)stream);
  if (rc) return rc;
  finish_plan(plan, masks);
  return PL_OK;
}

extern "C" int pl_sort_plan(int W, int64_t M, const uint64_t* x, const uint64_t* z, int64_t ld,
                            pl_merge_plan* plan, void* stream) {
  if (!plan || !valid_words(W) || M < 0 || ld < M) {
    set_error("pl_sort_plan: bad arguments");
    return valid_words(W) ? PL_ERR_ARG : PL_ERR_TIER;
  }
  if (M > (1LL << 30)) {
    set_error("pl_sort_plan: M exceeds 2^30 terms per call");
    return PL_ERR_CAPACITY;
  }
  *plan = pl_merge_plan{};
  plan->W = W;
  plan->mode = 1;
  plan->ma = M;
  plan->mb = 1;
  plan->n_items = M;
  u64 masks[2 * PL_PLAN_MAX_SEG + 1] = {0};
  int rc = compute_masks(W, (const u64*)x, (const u64*)z, ld, M, nullptr, nullptr, 0, 0, masks,
                         (cudaStream_t)stream);
  if (rc) return rc;
  finish_plan(plan, masks);
  return PL_OK;
}

static int check_ws(const pl_merge_plan* plan, void* ws, size_t bytes, int mode) {
  if (!plan || plan->mode != mode) {
    set_error("merge plan missing or built for another operation");
    return PL_ERR_ARG;
  }
  if ((int64_t)bytes < plan->workspace_bytes || (!ws && plan->workspace_bytes > 0)) {
    set_error("workspace %zu bytes < plan requirement %lld", bytes,
              (long long)plan->workspace_bytes);
    return PL_ERR_WORKSPACE;
  }
  return PL_OK;
}

extern "C" int pl_outer_multiply_combine(const pl_merge_plan* plan, const uint64_t* ax,
                                         const uint64_t* az, const uint8_t* ak, const double* ac,
                                         int64_t lda, const uint64_t* bx, const uint64_t* bz,
                                         const uint8_t* bk, const double* bc, int64_t ldb,
                                         double eps, void* workspace, size_t workspace_bytes,
                                         uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc,
                                         int64_t ldo, int64_t* out_count, void* stream) {
  int rc = check_ws(plan, workspace, workspace_bytes, 0);
  if (rc) return rc;
  const bool sort_only = ox == nullptr;  // phase 1: count only, then pl_merge_emit
  if (eps != eps || (!sort_only && ldo < plan->n_items) || !out_count) {
    set_error("pl_outer_multiply_combine: bad arguments");
    return PL_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (plan->n_items == 0) {
    PLB_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int64_t), st));
    return PL_OK;
  }
  SrcA S{(const u64*)ax, (const u64*)az, ak, (const double2*)ac, lda,
         (const u64*)bx, (const u64*)bz, bk, (const double2*)bc, ldb};
  OutP O{(u64*)ox, (u64*)oz, ok, (double2*)oc, ldo, out_count, eps};
  O.phase = sort_only ? 1 : 0;
  return PLB_DISPATCH_W(plan->W, run_outer, *plan, S, workspace, O, st);
}

extern "C" int pl_sort_combine(const pl_merge_plan* plan, const uint64_t* x, const uint64_t* z,
                               const uint8_t* k, const double* c, int64_t ld, double eps,
                               void* workspace, size_t workspace_bytes, uint64_t* ox,
                               uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                               int64_t* out_count, void* stream) {
  int rc = check_ws(plan, workspace, workspace_bytes, 1);
  if (rc) return rc;
  const bool sort_only = ox == nullptr;  // phase 1: count only, then pl_merge_emit
  if (eps != eps || (!sort_only && ldo < plan->n_items) || !out_count) {
    set_error("pl_sort_combine: bad arguments");
    return PL_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (plan->n_items == 0) {
    PLB_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int64_t), st));
    return PL_OK;
  }
  SrcA S{(const u64*)x, (const u64*)z, k, (const double2*)c, ld,
         nullptr, nullptr, nullptr, nullptr, 0};
  OutP O{(u64*)ox, (u64*)oz, ok, (double2*)oc, ldo, out_count, eps};
  O.phase = sort_only ? 1 : 0;
  return PLB_DISPATCH_W(plan->W, run_sort, *plan, S, workspace, O, st);
}

extern "C" int pl_merge_emit(const pl_merge_plan* plan, void* workspace, size_t workspace_bytes,
                             uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                             int64_t capacity, int64_t* out_count, void* stream) {
  if (!plan || (plan->mode != 0 && plan->mode != 1)) {
    set_error("pl_merge_emit: plan missing");
    return PL_ERR_ARG;
  }
  int rc = check_ws(plan, workspace, workspace_bytes, plan->mode);
  if (rc) return rc;
  if (!ox || !oz || !ok || !oc || !out_count || capacity < 0 || ldo < capacity) {
    set_error("pl_merge_emit: bad arguments");
    return PL_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (plan->n_items == 0) return PL_OK;
  SrcA S{};
  OutP O{(u64*)ox, (u64*)oz, ok, (double2*)oc, ldo, out_count, 0.0};
  O.phase = 2;
  O.capacity = capacity;
  return plan->mode == 0 ? PLB_DISPATCH_W(plan->W, run_outer, *plan, S, workspace, O, st)
                         : PLB_DISPATCH_W(plan->W, run_sort, *plan, S, workspace, O, st);
}

// ------------------------------------------------------------ K7 C ABI
extern "C" int pl_dist_item_bytes(const pl_merge_plan* plan) {
  return plan ? 8 * (plan->key_words + 1) : 0;
}

extern "C" int64_t pl_dist_workspace_bytes(const pl_merge_plan* plan, int64_t n_local,
                                           int32_t n_buckets_local) {
  if (!plan) return 0;
  return local_plan(*plan, n_local, n_buckets_local > 0 ? n_buckets_local : plan->n_buckets)
      .workspace_bytes;
}

extern "C" int pl_outer_partition(const pl_merge_plan* plan, const uint64_t* ax,
                                  const uint64_t* az, const uint8_t* ak, int64_t lda,
                                  const uint64_t* bx, const uint64_t* bz, const uint8_t* bk,
                                  int64_t ldb, int64_t j0, int64_t j1, void* workspace,
                                  size_t workspace_bytes, void* send, uint32_t* bucket_counts,
                                  void* stream) {
  if (!plan || plan->mode != 0 || j0 < 0 || j1 < j0 || j1 > plan->mb || !bucket_counts) {
    set_error("pl_outer_partition: bad arguments");
    return PL_ERR_ARG;
  }
  const int64_t need = pl_dist_workspace_bytes(plan, plan->ma * (j1 - j0), plan->n_buckets);
  if ((int64_t)workspace_bytes < need) {
    set_error("pl_outer_partition: workspace %zu < %lld", workspace_bytes, (long long)need);
    return PL_ERR_WORKSPACE;
  }
  SrcA S{(const u64*)ax, (const u64*)az, ak, nullptr, lda,
         (const u64*)bx, (const u64*)bz, bk, nullptr, ldb};
  return PLB_DISPATCH_W(plan->W, dispatch_partition, *plan, S, j0, j1, workspace, send,
                        bucket_counts, (cudaStream_t)stream);
}

extern "C" int pl_merge_received(const pl_merge_plan* plan, const void* recv, int64_t n_recv,
                                 const uint32_t* counts, int n_ranks, int32_t b0, int32_t b1,
                                 const uint64_t* ax, const uint64_t* az, const uint8_t* ak,
                                 const double* ac, int64_t lda, const uint64_t* bx,
                                 const uint64_t* bz, const uint8_t* bk, const double* bc,
                                 int64_t ldb, double eps, void* workspace, size_t workspace_bytes,
                                 uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                                 int64_t* out_count, void* stream) {
  if (!plan || plan->mode != 0 || n_ranks < 1 || n_ranks > 64 || b0 < 0 || b1 <= b0 ||
      b1 > plan->n_buckets || n_recv < 0 || ldo < n_recv || eps != eps || !out_count) {
    set_error("pl_merge_received: bad arguments");
    return PL_ERR_ARG;
  }
  const int nbl = b1 - b0;
  const int64_t need = pl_dist_workspace_bytes(plan, n_recv, nbl);
  if ((int64_t)workspace_bytes < need) {
    set_error("pl_merge_received: workspace %zu < %lld", workspace_bytes, (long long)need);
    return PL_ERR_WORKSPACE;
  }
  SrcA S{(const u64*)ax, (const u64*)az, ak, (const double2*)ac, lda,
         (const u64*)bx, (const u64*)bz, bk, (const double2*)bc, ldb};
  OutP O{(u64*)ox, (u64*)oz, ok, (double2*)oc, ldo, out_count, eps};
  return PLB_DISPATCH_W(plan->W, dispatch_received, *plan, (const u64*)recv, n_recv, counts,
                        n_ranks, nbl, S, workspace, O, (cudaStream_t)stream);
}
