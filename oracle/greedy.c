/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's greedy
 * first-fit grouping (paulialg/grouping.py:67-83, _greedy_over) and its
 * pair_checks counter (grouping.py:75-76), used as the parity oracle for
 * full-size config-3 runs where the numpy loop is too slow.
 *
 * x, z: term-major (M, W) uint64 words (sums.py:240-242 "columns").
 * Term t goes to the first group (creation order) all of whose members
 * commute with it (symplectic parity 0, strings.py:47-51); else it opens a
 * new group.  pair_checks += |g| for every group tried.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n, cap;
  uint64_t* w; /* member words, (n, 2W): x then z */
} group_t;

static int anti(const uint64_t* a, const uint64_t* b, int W) {
  uint64_t acc = 0;
  for (int i = 0; i < W; ++i) acc ^= (a[i] & b[W + i]) ^ (a[W + i] & b[i]);
  return __builtin_popcountll(acc) & 1;
}

/* Returns the number of groups, or -1 on allocation failure. */
int64_t oracle_greedy(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                      int32_t* group_of, int64_t* pair_checks) {
  int64_t ng = 0, gcap = 64;
  group_t* g = (group_t*)calloc((size_t)gcap, sizeof(group_t));
  uint64_t* row = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)W);
  int64_t checks = 0;
  if (!g || !row) return -1;
  for (int64_t t = 0; t < M; ++t) {
    memcpy(row, x + t * W, sizeof(uint64_t) * W);
    memcpy(row + W, z + t * W, sizeof(uint64_t) * W);
    int64_t chosen = -1;
    for (int64_t q = 0; q < ng && chosen < 0; ++q) {
      checks += g[q].n;
      int ok = 1;
      for (int64_t m = 0; m < g[q].n; ++m)
        if (anti(row, g[q].w + m * 2 * W, W)) { ok = 0; break; }
      if (ok) chosen = q;
    }
    if (chosen < 0) {
      if (ng == gcap) {
        gcap *= 2;
        group_t* ng2 = (group_t*)realloc(g, sizeof(group_t) * (size_t)gcap);
        if (!ng2) return -1;
        g = ng2;
        memset(g + ng, 0, sizeof(group_t) * (size_t)(gcap - ng));
      }
      chosen = ng++;
    }
    group_t* gr = &g[chosen];
    if (gr->n == gr->cap) {
      gr->cap = gr->cap ? 2 * gr->cap : 8;
      uint64_t* w2 = (uint64_t*)realloc(gr->w, sizeof(uint64_t) * 2 * (size_t)W * (size_t)gr->cap);
      if (!w2) return -1;
      gr->w = w2;
    }
    memcpy(gr->w + gr->n * 2 * W, row, sizeof(uint64_t) * 2 * W);
    gr->n++;
    group_of[t] = (int32_t)chosen;
  }
  for (int64_t q = 0; q < ng; ++q) free(g[q].w);
  free(g);
  free(row);
  *pair_checks = checks;
  return ng;
}
