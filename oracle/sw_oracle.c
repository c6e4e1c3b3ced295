/*
 * oracle/sw_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU implementation of what the hot path
 * computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, headers,
 * tables or constants with paper_1404_4152_b200/ (the CUDA path); neither
 * includes or links the other.
 *
 * What it computes (§II.A, Eq. 1), for query S1 = q[1..m]
 * and subject S2 = s[1..n], with fsbt(a,b) = M[a*32 + b] (row = query residue,
 * DESIGN.md reading R1):
 *
 *   H(i,j) = max{ 0, H(i-1,j-1) + fsbt(S1[i],S2[j]), E(i,j), F(i,j) }
 *   E(i,j) = max{ E(i-1,j) - alpha, H(i-1,j) - beta }
 *   F(i,j) = max{ F(i,j-1) - alpha, H(i,j-1) - beta }
 *   H(i,0) = H(0,j) = E(0,j) = F(i,0) = 0
 *   score  = max over the whole matrix H (boundary zeros included)
 *
 * "can be calculated in linear space": one row of H and E is
 * kept (§III.A).  int32 throughout (32-bit lanes):
 * E, F >= -beta and H <= qlen * max(0, s_max), so nothing can overflow under
 * the ABI bound qlen * s_max < 2^31.
 *
 * Parity pins (tests/test_oracle.py): brute-force enumeration of all local
 * alignments for |Q|,|S| <= 6, the Gotoh full matrix with -inf boundaries
 * (oracle_sw_full below), closed forms (self-alignment under row dominance,
 * m = 1, ungapped Kadane, linear gap), invariants (score >= 0, symmetry,
 * monotonicity, DUMMY padding).  No function here is "parity unpinned".
 *
 * Build: gcc -O2 -shared -fPIC -pthread -o oracle/_liboracle.so oracle/sw_oracle.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static inline int32_t max2(int32_t a, int32_t b) { return a > b ? a : b; }

/* Eq. 1 as printed, linear space.  Returns the optimal local score (>= 0),
 * or -1 if a buffer cannot be allocated. */
int32_t oracle_sw_score(const uint8_t* q, int32_t m, const uint8_t* s, int32_t n,
                        const int8_t* M, int32_t alpha, int32_t beta) {
  if (m <= 0 || n <= 0) return 0;               /* H is all boundary zeros */
  int32_t* Hrow = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1)); /* H(i-1, j) */
  int32_t* Erow = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1)); /* E(i-1, j) */
  if (!Hrow || !Erow) { free(Hrow); free(Erow); return -1; }
  for (int32_t j = 0; j <= n; j++) { Hrow[j] = 0; Erow[j] = 0; }  /* H(0,j) = E(0,j) = 0 */
  int32_t best = 0;
  for (int32_t i = 1; i <= m; i++) {
    const int8_t* row = M + 32 * q[i - 1];
    int32_t F = 0;          /* F(i,0) = 0 */
    int32_t Hleft = 0;      /* H(i,0) = 0 */
    int32_t Hdiag = Hrow[0];/* H(i-1,0) = 0 */
    for (int32_t j = 1; j <= n; j++) {
      int32_t E = max2(Erow[j] - alpha, Hrow[j] - beta);   /* E(i,j) */
      F = max2(F - alpha, Hleft - beta);                    /* F(i,j) */
      int32_t H = max2(max2(0, Hdiag + row[s[j - 1]]), max2(E, F));
      Hdiag = Hrow[j];      /* H(i-1,j) is the diagonal of (i, j+1) */
      Hrow[j] = H;
      Erow[j] = E;
      Hleft = H;
      if (H > best) best = H;
    }
  }
  free(Hrow);
  free(Erow);
  return best;
}

/* Full-matrix DP with Gotoh's -inf boundaries (E(0,j) = F(i,0) = -inf): an
 * independent formulation used only to pin the printed boundary (reading R2). */
int32_t oracle_sw_full(const uint8_t* q, int32_t m, const uint8_t* s, int32_t n,
                       const int8_t* M, int32_t alpha, int32_t beta) {
  const int32_t NEG = INT32_MIN / 4;
  size_t W = (size_t)n + 1, sz = ((size_t)m + 1) * W;
  int32_t* H = (int32_t*)malloc(sizeof(int32_t) * sz);
  int32_t* E = (int32_t*)malloc(sizeof(int32_t) * sz);
  int32_t* F = (int32_t*)malloc(sizeof(int32_t) * sz);
  if (!H || !E || !F) { free(H); free(E); free(F); return -1; }
  for (size_t k = 0; k < sz; k++) { H[k] = 0; E[k] = NEG; F[k] = NEG; }
  int32_t best = 0;
  for (int32_t i = 1; i <= m; i++)
    for (int32_t j = 1; j <= n; j++) {
      size_t c = (size_t)i * W + j, up = c - W, lf = c - 1, dg = up - 1;
      E[c] = max2(E[up] - alpha, H[up] - beta);
      F[c] = max2(F[lf] - alpha, H[lf] - beta);
      int32_t h = H[dg] + M[32 * q[i - 1] + s[j - 1]];
      h = max2(h, E[c]);
      h = max2(h, F[c]);
      H[c] = max2(h, 0);
      if (H[c] > best) best = H[c];
    }
  free(H); free(E); free(F);
  return best;
}

/* ---- whole-database scoring: one subject per task, thread pool + atomic counter ---- */
typedef struct {
  const uint8_t* q; int32_t m;
  const uint8_t* residues; const int64_t* offsets; const int32_t* lengths; int64_t n_seqs;
  const int8_t* M; int32_t alpha, beta;
  int32_t* out;
  int64_t next;          /* shared work counter */
  int err;
} pool_t;

static void* pool_worker(void* arg) {
  pool_t* P = (pool_t*)arg;
  const int64_t CH = 16;
  for (;;) {
    int64_t a = __atomic_fetch_add(&P->next, CH, __ATOMIC_RELAXED);
    if (a >= P->n_seqs) break;
    int64_t b = a + CH < P->n_seqs ? a + CH : P->n_seqs;
    for (int64_t i = a; i < b; i++) {
      int32_t r = oracle_sw_score(P->q, P->m, P->residues + P->offsets[i], P->lengths[i],
                                  P->M, P->alpha, P->beta);
      if (r < 0) P->err = 1;
      P->out[i] = r;
    }
  }
  return NULL;
}

/* scores[i] = oracle_sw_score(query, db[i]) for i in [0, n_seqs); input order.
 * Returns 0, or -1 on allocation failure. */
int oracle_scores(const uint8_t* q, int32_t m, const uint8_t* residues, const int64_t* offsets,
                  const int32_t* lengths, int64_t n_seqs, const int8_t* M, int32_t alpha,
                  int32_t beta, int nthreads, int32_t* out) {
  pool_t P = {q, m, residues, offsets, lengths, n_seqs, M, alpha, beta, out, 0, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 512) nthreads = 512;
  pthread_t th[512];
  int started = 0;
  for (int t = 1; t < nthreads; t++)
    if (pthread_create(&th[started], NULL, pool_worker, &P) == 0) started++;
  pool_worker(&P);
  for (int t = 0; t < started; t++) pthread_join(th[t], NULL);
  return P.err ? -1 : 0;
}

/* ---- stage (iv): "sort all alignment scores in descending order" ---- */
typedef struct { int32_t score; int64_t id; } hit_t;

static int hit_cmp(const void* a, const void* b) {
  const hit_t* x = (const hit_t*)a;
  const hit_t* y = (const hit_t*)b;
  if (x->score != y->score) return x->score > y->score ? -1 : 1;   /* score descending */
  return x->id < y->id ? -1 : (x->id > y->id);                     /* then id ascending (R7) */
}

/* Full sort of all (score, id) pairs; the first k are returned.  Slots past n
 * are (-1, -1) (reading R8).  ids == NULL means id = index.  Returns 0 / -1. */
int oracle_topk(const int32_t* scores, const int64_t* ids, int64_t n, int32_t k,
                int64_t* out_ids, int32_t* out_scores) {
  hit_t* h = (hit_t*)malloc(sizeof(hit_t) * (size_t)(n > 0 ? n : 1));
  if (!h) return -1;
  for (int64_t i = 0; i < n; i++) { h[i].score = scores[i]; h[i].id = ids ? ids[i] : i; }
  qsort(h, (size_t)n, sizeof(hit_t), hit_cmp);
  for (int32_t t = 0; t < k; t++) {
    out_ids[t] = t < n ? h[t].id : -1;
    out_scores[t] = t < n ? h[t].score : -1;
  }
  free(h);
  return 0;
}
