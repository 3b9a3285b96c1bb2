/*
 * paulib_b200 — C ABI of the B200-native Pauli-sum hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every pointer argument
 * except `plan`, `out_count_host` and the *_bytes queries is a DEVICE pointer;
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Functions return PL_OK (0) or a negative PL_ERR_* code; pl_last_error()
 * returns a thread-local message for the last failure.
 *
 * Storage (the reference's PauliSumSoA, sums.py:429-450): for a sum of M
 * terms at W = tier/64 words per plane (bits.py:12, :34-46)
 *   x, z : W planes, word w of term t at plane[w * ld + t] (ld >= M)
 *   k    : M uint8 phase exponents (factor i^k)
 *   c    : M complex128 coefficients, interleaved (re, im) doubles
 * The reference's (M, W) "columns" are the transpose of these planes
 * (sums.py:459-460).
 *
 * Each entry point names the reference interface it replaces (file:line in
 * /root/reference/pkg/src/paulialg/).
 */
#ifndef PAULIB_B200_H
#define PAULIB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PL_OK 0
#define PL_ERR_ARG (-1)       /* bad size / pointer / alignment            */
#define PL_ERR_TIER (-2)      /* W not in {1,2,4,8,16}  (bits.py CapacityError) */
#define PL_ERR_CUDA (-3)      /* CUDA runtime error                         */
#define PL_ERR_CAPACITY (-4)  /* problem larger than the documented limits  */
#define PL_ERR_WORKSPACE (-5) /* workspace smaller than the plan requires   */

#define PL_ABI_VERSION 1

/* Thread-local description of the most recent error. */
const char* pl_last_error(void);
int pl_abi_version(void);

/* ------------------------------------------------------------------------
 * K1 — batched pair multiply.  Replaces bench.py:168-177 (_batch_pair_multiply)
 * and the per-pair math of strings.py:32-44 (_phase_exponent_words) and
 * strings.py:133-137 (PauliString.multiply):
 *   o.x = a.x ^ b.x,  o.z = a.z ^ b.z,
 *   o.k = (a.k + b.k + phase(a, b)) mod 4,
 * for P aligned pairs.  Planes use leading dimensions lda/ldb/ldo (words).
 * ak / bk may be NULL (treated as 0).
 */
int pl_batch_multiply(int W, int64_t P,
                      const uint64_t* ax, const uint64_t* az, const uint8_t* ak, int64_t lda,
                      const uint64_t* bx, const uint64_t* bz, const uint8_t* bk, int64_t ldb,
                      uint64_t* ox, uint64_t* oz, uint8_t* ok, int64_t ldo,
                      void* stream);

/* Batched symplectic inner product parity (strings.py:47-51, :141-147):
 * anti[p] = 1 when pair p anti-commutes, 0 when it commutes. */
int pl_batch_sip(int W, int64_t P,
                 const uint64_t* ax, const uint64_t* az, int64_t lda,
                 const uint64_t* bx, const uint64_t* bz, int64_t ldb,
                 uint8_t* anti, void* stream);

/* One pair from HOST memory (the scalar API: PauliString.multiply,
 * strings.py:133-137, and symplectic_inner_product / commutes, :141-147):
 * o = a * b with o.k = (ak + bk + phase(a, b)) mod 4, and *anti = 1 when a and
 * b anti-commute.  ax..bz and ox, oz are HOST arrays of W words; ox, oz, ok and
 * anti may be NULL.  The operands travel through a mapped pinned buffer the
 * kernel reads and writes directly: one launch and one synchronisation of
 * `stream` per call (the call returns with the results in place). */
int pl_pair_host(int W, const uint64_t* ax, const uint64_t* az, int ak,
                 const uint64_t* bx, const uint64_t* bz, int bk,
                 uint64_t* ox, uint64_t* oz, int* ok, int* anti, void* stream);

/* ------------------------------------------------------------------------
 * K2 raw — outer product without combine.  Replaces sums.py:144-174
 * (_multiply_columns) + sums.py:123-141 (_multiply_block): output row
 * j*Ma + i holds a_i * b_j (j-major), phase exponent
 * (a.k[i] + b.k[j] + phase(a_i, b_j)) mod 4 and coefficient a.c[i] * b.c[j],
 * rounded as numpy's complex128 multiply on FMA hosts: re = fma(ar, br, -(ai*bi)),
 * im = fma(ar, bi, ai*br).  Output planes have Ma*Mb columns.
 */
int pl_outer_multiply_raw(int W, int64_t Ma, int64_t Mb,
                          const uint64_t* ax, const uint64_t* az, const uint8_t* ak,
                          const double* ac, int64_t lda,
                          const uint64_t* bx, const uint64_t* bz, const uint8_t* bk,
                          const double* bc, int64_t ldb,
                          uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                          void* stream);

/* ------------------------------------------------------------------------
 * K2-K4 — multiply + simplify.  A merge "plan" fixes the packed-key layout
 * (bit ranges of the (z0..z{W-1}, x0..x{W-1}) canonical key that can be
 * nonzero, sums.py:104-106 / strings.py:165-167), the bucket count and the
 * workspace size.  pl_*_plan() reads device data and SYNCHRONISES `stream`.
 */
#define PL_PLAN_MAX_SEG 32

typedef struct pl_merge_plan {
  int32_t W;             /* words per plane                                  */
  int32_t mode;          /* 0 = outer product A*B, 1 = sort_and_combine(S)   */
  int64_t ma, mb;        /* outer: |A|, |B|; sort: M, 1                      */
  int64_t n_items;       /* raw terms to merge (ma*mb, or M)                 */
  int32_t key_words;     /* KW: 64-bit words per packed key                  */
  int32_t key_bits;      /* packed key length in bits                        */
  int32_t seg_lo[PL_PLAN_MAX_SEG];  /* per canonical-key word: lowest used bit */
  int32_t seg_len[PL_PLAN_MAX_SEG]; /* number of bits kept (0 = word unused)  */
  int32_t seg_pos[PL_PLAN_MAX_SEG]; /* offset of the segment in the key (MSB first) */
  int32_t n_buckets;     /* level-1 buckets (splitter ranges)                */
  int32_t n_samples;     /* splitter sample size                             */
  int32_t leaf_cap;      /* largest bucket sorted in shared memory           */
  int32_t leaf_target;   /* target size of a level-2 sub-bucket              */
  int32_t max_sub;       /* max sub-buckets per level-1 bucket               */
  int32_t pad0;
  int64_t workspace_bytes;
  int64_t reserved[8];
} pl_merge_plan;

/* Plan for A*B (sums.py:293-305).  Requires Ma*Mb <= 2^30. */
int pl_outer_plan(int W, int64_t Ma, int64_t Mb,
                  const uint64_t* ax, const uint64_t* az, int64_t lda,
                  const uint64_t* bx, const uint64_t* bz, int64_t ldb,
                  pl_merge_plan* plan, void* stream);

/* Plan for sort_and_combine of M terms (sums.py:286-291).  M <= 2^30. */
int pl_sort_plan(int W, int64_t M, const uint64_t* x, const uint64_t* z, int64_t ld,
                 pl_merge_plan* plan, void* stream);

/* Outer product followed by _combine_columns (sums.py:94-120): fold i^k into
 * the coefficient, order by the canonical key, merge equal keys (summing in
 * raw-row order), drop |c| <= eps (any eps, as _combine_columns: a negative
 * eps keeps every merged term, exact zeros included), flags 0.  Output planes need capacity
 * >= plan->n_items columns (ldo); *out_count (device int64) receives the
 * number of merged terms.  Deterministic: bit-identical run to run. */
int pl_outer_multiply_combine(const pl_merge_plan* plan,
                              const uint64_t* ax, const uint64_t* az, const uint8_t* ak,
                              const double* ac, int64_t lda,
                              const uint64_t* bx, const uint64_t* bz, const uint8_t* bk,
                              const double* bc, int64_t ldb,
                              double eps, void* workspace, size_t workspace_bytes,
                              uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                              int64_t* out_count, void* stream);

/* Two-phase form of pl_outer_multiply_combine / pl_sort_combine, for an
 * exactly sized output: called with ox == NULL they stop after merging and
 * write only *out_count (the merged-term count; the merged entries stay in
 * the workspace, which must not be reused in between); pl_merge_emit then
 * writes those terms into output planes of `capacity` >= *out_count columns
 * (ldo >= capacity; terms past `capacity` are not written). */
int pl_merge_emit(const pl_merge_plan* plan, void* workspace, size_t workspace_bytes,
                  uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                  int64_t capacity, int64_t* out_count, void* stream);

/* ------------------------------------------------------------------------
 * K7 — multi-GPU A*B (no reference equivalent; PAPER.md:712-714 lists
 * distributed memory as future work).  Every rank builds the same plan from
 * the replicated A and B, so the key-range splitters (from a deterministic
 * sample of the full product) are identical everywhere without a collective.
 *   1. pl_outer_partition: rank r generates the items of B columns [j0, j1),
 *      buckets them, writes them bucket-contiguous into `send` as records of
 *      pl_dist_item_bytes() bytes and the per-bucket counts (n_buckets u32,
 *      device) into bucket_counts;
 *   2. the caller exchanges bucket ranges (rank q owns buckets [b0_q, b1_q))
 *      with one all-to-all (NCCL, see paper_2605_25974_b200/dist.py);
 *   3. pl_merge_received: merge the received records (source-major; counts is
 *      the device [n_ranks][b1-b0] matrix of per-source, per-bucket counts)
 *      into this rank's slice of the canonical output.
 * Concatenating the ranks' outputs in rank order gives exactly the
 * single-GPU pl_outer_multiply_combine result (runs never straddle buckets,
 * each run is summed in raw-row order by one thread).
 */
int pl_dist_item_bytes(const pl_merge_plan* plan);
int64_t pl_dist_workspace_bytes(const pl_merge_plan* plan, int64_t n_local,
                                int32_t n_buckets_local);
int pl_outer_partition(const pl_merge_plan* plan,
                       const uint64_t* ax, const uint64_t* az, const uint8_t* ak, int64_t lda,
                       const uint64_t* bx, const uint64_t* bz, const uint8_t* bk, int64_t ldb,
                       int64_t j0, int64_t j1, void* workspace, size_t workspace_bytes,
                       void* send, uint32_t* bucket_counts, void* stream);
int pl_merge_received(const pl_merge_plan* plan, const void* recv, int64_t n_recv,
                      const uint32_t* counts, int n_ranks, int32_t b0, int32_t b1,
                      const uint64_t* ax, const uint64_t* az, const uint8_t* ak,
                      const double* ac, int64_t lda,
                      const uint64_t* bx, const uint64_t* bz, const uint8_t* bk,
                      const double* bc, int64_t ldb,
                      double eps, void* workspace, size_t workspace_bytes,
                      uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                      int64_t* out_count, void* stream);

/* sort_and_combine (sums.py:286-291 / :94-120) of one sum. */
int pl_sort_combine(const pl_merge_plan* plan,
                    const uint64_t* x, const uint64_t* z, const uint8_t* k, const double* c,
                    int64_t ld, double eps, void* workspace, size_t workspace_bytes,
                    uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc, int64_t ldo,
                    int64_t* out_count, void* stream);

/* ------------------------------------------------------------------------
 * K5 — commutation bitmatrix.  Restates the all-pairs block of
 * grouping.py:136-140 (parity of popc(x_r & z_c) + popc(z_r & x_c)):
 * bit (c - col0) % 32 of word bits[(r - row0) * ld_bits + (c - col0) / 32]
 * is 1 when term r anti-commutes with term c, for r in [row0, row0+rows),
 * c in [col0, col0+cols).  Rows and columns index the same M-term sum.
 * col0 must be a multiple of 32; trailing bits of the last word are 0.
 * method: 0 = auto, 1 = row-list XOR over transposed column slices
 * (sparse-friendly), 2 = direct LOP3/POPC per pair, 3 = tensor cores
 * (tcgen05.mma.kind::i8 on 0/1 byte expansions, K = 128 W; W <= 8).  Auto
 * takes 1 for sparse rows and 3 above ~24 W letters per row (W <= 8).
 */
int pl_commutation_bitmatrix(int W, int64_t M,
                             const uint64_t* x, const uint64_t* z, int64_t ld,
                             int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                             uint32_t* bits, int64_t ld_bits, int method,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes pl_commutation_bitmatrix needs for `rows` rows. */
int64_t pl_bitmatrix_workspace_bytes(int W, int64_t rows);

/* ------------------------------------------------------------------------
 * K6 — greedy first-fit commutation grouping.  Replaces grouping.py:67-95
 * (_greedy_over / group_greedy): term t (index order) joins the first group
 * (creation order) all of whose members commute with it, else opens a new
 * group.  group_of[t] receives t's group id (ids in creation order);
 * *n_groups the group count; *pair_checks the reference's
 * GroupingStats.pair_checks (grouping.py:75-76).  All three are device
 * pointers.  Deterministic and exactly equal to the reference.
 */
int64_t pl_group_workspace_bytes(int W, int64_t M);
int pl_group_greedy(int W, int64_t M, const uint64_t* x, const uint64_t* z, int64_t ld,
                    int32_t* group_of, int32_t* n_groups, int64_t* pair_checks,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * §8(f) f3 — merge phase of the two-phase parallel grouping.  Replaces the
 * sequential merge of group_greedy_parallel (grouping.py:120-145): the local
 * groups of the chunk-wise greedy runs (K6 on each contiguous chunk), listed
 * in processing order as device `members` (term ids) with HOST offsets
 * `local_off` [n_local + 1] (local_off[n_local] == M), each join the first
 * global group (creation order) whose members all commute with theirs, else
 * open a new one.  global_of_local (device, n_local) receives each local
 * group's global id, *n_global (device) the global group count, and
 * *pair_checks (device) is INCREASED by the reference's merge contribution
 * (|local| * |group| per group tried).  Exact: same partition as the reference.
 */
int64_t pl_group_merge_workspace_bytes(int64_t M, int32_t n_local);
int pl_group_merge(int W, int64_t M, const uint64_t* x, const uint64_t* z, int64_t ld,
                   const int32_t* members, const int64_t* local_off, int32_t n_local,
                   int32_t* global_of_local, int32_t* n_global, int64_t* pair_checks,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * §8(f) f2 — Clifford conjugation in place.  Replaces gates.py:72-102
 * (apply_clifford_inplace, called by _SumBase.apply_clifford, sums.py:309-316):
 * every term P becomes U P U^dagger for gate H (0), S (1), CNOT (2, q0 =
 * control, q1 = target) or CZ (3); x, z, k are device SoA planes / phases,
 * modified in place.  Qubit indices must be < 64*W (the Python layer checks
 * them against n and raises IndexError as the reference does, gates.py:23-24).
 */
int pl_apply_clifford(int W, int64_t M, uint64_t* x, uint64_t* z, uint8_t* k, int64_t ld,
                      int gate, int q0, int q1, void* stream);

/* ------------------------------------------------------------------------
 * §8(f) f1 — Pauli-rotation split, un-combined.  Replaces _rotation_columns
 * (sums.py:177-223).  gen_x / gen_z are HOST arrays of W words (the phase-free
 * generator P); cos_t is the snapped cosine (rotations.py:24-35) and
 * (msin_re, msin_im) the complex factor -1j*sin_t as the reference's Python
 * evaluates it.  Output: M terms (sin == 0 or cos == 0) or M + #anti
 * interleaved terms; ldo >= 2*M in the split case.  *out_count (device) gets
 * the output term count.  Apply pl_sort_combine afterwards for the canonical
 * form (apply_rotation, sums.py:318-325).
 */
int64_t pl_rotation_workspace_bytes(int64_t M);
int pl_rotation_split(int W, int64_t M, const uint64_t* x, const uint64_t* z, const uint8_t* k,
                      const double* c, int64_t ld, const uint64_t* gen_x, const uint64_t* gen_z,
                      double cos_t, double msin_re, double msin_im, void* workspace,
                      size_t workspace_bytes, uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc,
                      int64_t ldo, int64_t* out_count, void* stream);

/* ------------------------------------------------------------------------
 * §8(f) f4 — packed AoS records <-> SoA planes.  Replaces the host transposes
 * of PauliSum.to_soa (sums.py:417-426) and PauliSumSoA.to_aos (sums.py:469-477)
 * for sums that live on (or are headed to) the device.  `records` is a DEVICE
 * array of M packed records of 16W + 17 bytes, the reference's aos_dtype
 * (sums.py:48-57): x[W] u64 | z[W] u64 | flags u8 | coeff (re, im) f64, no
 * padding; it must be 16-byte aligned.  Planes have leading dimension ld >= M.
 * Exact bijection in both directions.  pl_soa_to_aos accepts k == NULL (flags 0).
 */
int pl_aos_to_soa(int W, int64_t M, const void* records,
                  uint64_t* x, uint64_t* z, uint8_t* k, double* c, int64_t ld, void* stream);
int pl_soa_to_aos(int W, int64_t M,
                  const uint64_t* x, const uint64_t* z, const uint8_t* k, const double* c,
                  int64_t ld, void* records, void* stream);

/* ------------------------------------------------------------------------
 * Stage timing (instrumentation for bench.py).  While enabled, multi-kernel
 * entry points record a CUDA event pair around every kernel they launch, on
 * the launching stream.  pl_stage_times() waits for the recorded events and
 * returns up to `max` (name, milliseconds) pairs in launch order (names are
 * NUL-terminated, 32 bytes each), then clears the record.  Returns the count.
 */
int pl_stage_timing(int enable);
int pl_stage_times(char* names, float* ms, int max);

#ifdef __cplusplus
}
#endif

#endif /* PAULIB_B200_H */
