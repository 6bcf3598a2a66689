/* sro_oracle.c — plain, slow, fp64 CPU oracle for the BCFW semi-relaxed OT
 * hot path (arXiv 2103.05857).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load this library. It shares no code
 * with the CUDA path (paper_2103_05857_b200/csrc) and neither side includes
 * the other.
 *
 * Compiled with -O2 -ffp-contract=off: every floating-point operation below is
 * one IEEE-754 binary64 operation rounded to nearest-even, in the order
 * written. No fused multiply-add, no reassociation, single-threaded.
 *
 * Citations: P:<line> = /root/reference/PAPER.md. Equation numbers follow
 * SURVEY.md's table (Eq. 7 problem, Eq. 9 LMO, Eq. 10 BCFW ELS, Eq. 11 column
 * gap, Eq. 13 away atom, Eq. 14 generalised ELS, Eq. A.1 FW ELS). Where the
 * paper is silent (summation order, tie-breaks, counters, GA constants) the
 * reading R<n> is listed in DESIGN.md §3 and cited here.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_pins*.py
 * against closed forms, brute force, exact-rational replay or values printed
 * in the paper; the GA sampler (fen_build / fen_add / fen_draw, the inner and
 * global refreshes) by an exact-rational replay of Alg. A.4 with the paper's
 * O(n) cumulative-sum draw (tests/test_oracle_pins_ga.py). No function is
 * "parity unpinned".
 */
#include "sro_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

struct or_state {
  int32_t m, n;
  double lambda;
  double* a;            /* source marginal, length m */
  double* b;            /* target marginal, length n */
  int32_t cost_kind;
  double* C;            /* dense column-major, C[i*ld + k] = C_{k,i} */
  int64_t ld;
  double* X;            /* X[3k..3k+2] source colour x_k */
  double* Y;            /* Y[3i..3i+2] target colour y_i */
  uint64_t hash_seed;
  int32_t cap;          /* per-column support capacity */
  int32_t* cnt;         /* |supp(t_i)| */
  int32_t* rows;        /* rows[i*cap + p], ascending in p */
  double* vals;         /* vals[i*cap + p] = T_{rows,i} > 0 */
  double* r;            /* r = T 1_n, maintained (R6) */
  double* h;            /* h = (r - a)/lambda */
  int64_t k;            /* global step counter since reset (R2) */
  /* configuration lock for resumable solves */
  int configured;
  int32_t variant;
  or_options opt;
  uint64_t seed;
  /* P sampling cache */
  int64_t perm_epoch;
  int32_t* perm;
  /* GA (Alg. A.4) */
  double* G;            /* stored per-column gaps */
  double* fen;          /* Fenwick tree, 1-based, fen[1..n] */
  /* scratch */
  double* acc256;       /* 256*m per-chunk row accumulators (allocated on first block step) */
  unsigned char* touched;
  int32_t* trows;       /* touched rows of the current step */
  int32_t ntrows;
  double* xbuf;         /* max(m, n) */
};

/* ------------------------------------------------------------------------ */
/* RNG: SplitMix64 finaliser, counter-based (R21).             */
/* ------------------------------------------------------------------------ */
uint64_t or_splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* t-th value of stream `stream` under `seed`. */
uint64_t or_rng_u64(uint64_t seed, uint32_t stream, uint64_t t) {
  uint64_t key = or_splitmix64_mix(seed ^ (0x5851F42D4C957F2DULL * (uint64_t)(stream + 1)));
  return or_splitmix64_mix(key + (t + 1) * GOLDEN);
}

double or_uniform53(uint64_t x) { return (double)(x >> 11) * 0x1p-53; }

/* floor(u53 * N) computed exactly in integers. */
static int32_t uniform_index(uint64_t x, int32_t N) {
  unsigned __int128 p = (unsigned __int128)(x >> 11) * (unsigned __int128)(uint32_t)N;
  return (int32_t)(uint64_t)(p >> 53);
}

/* Fresh Fisher-Yates permutation of [0, N) for epoch e (R22). */
int or_permutation(uint64_t seed, int64_t epoch, int32_t N, int32_t* perm) {
  for (int32_t q = 0; q < N; q++) perm[q] = q;
  for (int32_t q = N - 1; q >= 1; q--) {
    uint64_t x = or_rng_u64(seed, 2, (uint64_t)epoch * (uint64_t)N + (uint64_t)(N - 1 - q));
    int32_t rr = uniform_index(x, q + 1);
    int32_t tmp = perm[q]; perm[q] = perm[rr]; perm[rr] = tmp;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Summation shapes (R19). chunk_tree_sum: split [0,L) into W contiguous     */
/* chunks [floor(c L/W), floor((c+1) L/W)), sum each sequentially starting   */
/* from +0.0, then combine adjacent pairs level by level.                    */
/* ------------------------------------------------------------------------ */
double or_chunk_tree_sum(const double* x, int64_t L, int32_t W) {
  double part[256];
  for (int32_t c = 0; c < W; c++) {
    int64_t lo = ((int64_t)c * L) / W, hi = ((int64_t)(c + 1) * L) / W;
    double acc = 0.0;
    for (int64_t p = lo; p < hi; p++) acc = acc + x[p];
    part[c] = acc;
  }
  for (int32_t width = W; width > 1; width /= 2)
    for (int32_t c = 0; c < width / 2; c++) part[c] = part[2 * c] + part[2 * c + 1];
  return part[0];
}


/* chunk index of position p among L positions split into W chunks */
static int32_t chunk_of(int64_t p, int64_t L, int32_t W) {
  int32_t c = (int32_t)((p * W) / L);            /* first guess, then fix */
  while (c > 0 && ((int64_t)c * L) / W > p) c--;
  while (c < W - 1 && ((int64_t)(c + 1) * L) / W <= p) c++;
  return c;
}

/* ------------------------------------------------------------------------ */
/* Cost C_{k,i} (Eq. 7; colour costs P:427, squared per BASELINE configs).   */
/* ------------------------------------------------------------------------ */
static double cost(const or_state* s, int32_t k, int32_t i) {
  switch (s->cost_kind) {
    case OR_COST_DENSE:
      return s->C[(int64_t)i * s->ld + k];
    case OR_COST_SQEUCLID_F32:
    case OR_COST_EUCLID_F32: {
      /* binary32 colours evaluated in binary32 arithmetic, same operation
       * order, promoted exactly to binary64 (BASELINE "fp32" configs, R10) */
      float dx = (float)s->X[3 * (int64_t)k + 0] - (float)s->Y[3 * (int64_t)i + 0];
      float dy = (float)s->X[3 * (int64_t)k + 1] - (float)s->Y[3 * (int64_t)i + 1];
      float dz = (float)s->X[3 * (int64_t)k + 2] - (float)s->Y[3 * (int64_t)i + 2];
      float d2 = ((dx * dx) + (dy * dy)) + (dz * dz);
      return s->cost_kind == OR_COST_EUCLID_F32 ? (double)sqrtf(d2) : (double)d2;
    }
    case OR_COST_SQEUCLID:
    case OR_COST_EUCLID: {
      double dx = s->X[3 * (int64_t)k + 0] - s->Y[3 * (int64_t)i + 0];
      double dy = s->X[3 * (int64_t)k + 1] - s->Y[3 * (int64_t)i + 1];
      double dz = s->X[3 * (int64_t)k + 2] - s->Y[3 * (int64_t)i + 2];
      double d2 = ((dx * dx) + (dy * dy)) + (dz * dz);
      return s->cost_kind == OR_COST_EUCLID ? sqrt(d2) : d2;
    }
    default: { /* OR_COST_HASH: C_ki = (splitmix64(seed, i*m + k) >> 40) * 2^-24 */
      uint64_t idx = (uint64_t)i * (uint64_t)s->m + (uint64_t)k;
      uint64_t z = or_splitmix64_mix(s->hash_seed + (idx + 1) * GOLDEN);
      return (double)(z >> 40) * 0x1p-24;
    }
  }
}

double or_cost(or_state* s, int32_t k, int32_t i) { return cost(s, k, i); }

/* ------------------------------------------------------------------------ */
/* LMO, Eq. 9: j = argmin_k (C_ki + h_k), lowest k on ties (R1). */
/* ------------------------------------------------------------------------ */
static int lmo(const or_state* s, int32_t i, int32_t* j_out, double* min_out) {
  double best = INFINITY;
  int32_t j = -1;
  for (int32_t k = 0; k < s->m; k++) {
    double v = cost(s, k, i) + s->h[k];
    if (!isfinite(v)) return OR_ERR_NONFINITE;
    if (v < best) { best = v; j = k; }
  }
  if (j < 0) return OR_ERR_NONFINITE;
  *j_out = j;
  *min_out = best;
  return OR_OK;
}

int or_lmo_column(or_state* s, int32_t i, int32_t* j, double* minval) {
  if (i < 0 || i >= s->n) return OR_ERR_ARG;
  return lmo(s, i, j, minval);
}

/* <t_i, grad_i f> = sum over supp(t_i), rows ascending (R19: sequential). */
static double column_dot_grad(const or_state* s, int32_t i) {
  const int32_t* rw = s->rows + (int64_t)i * s->cap;
  const double* vl = s->vals + (int64_t)i * s->cap;
  double acc = 0.0;
  for (int32_t p = 0; p < s->cnt[i]; p++) {
    double gk = cost(s, rw[p], i) + s->h[rw[p]];
    double prod = vl[p] * gk;
    acc = acc + prod;
  }
  return acc;
}

/* column gap g_i = <t_i - s_i, grad_i f> (Eq. 11) */
static int column_gap(const or_state* s, int32_t i, int32_t* j, double* minval, double* g) {
  int st = lmo(s, i, j, minval);
  if (st) return st;
  double dot = column_dot_grad(s, i);
  double bm = s->b[i] * *minval;
  *g = dot - bm;
  return OR_OK;
}

/* full sweep: per-column gaps, total via the 256-chunk tree (Thm 2 / Eq. 11) */
static int gap_sweep(or_state* s, double* total, double* per_col, int32_t* jrows, double* minvals) {
  double* g = per_col ? per_col : s->xbuf;
  for (int32_t i = 0; i < s->n; i++) {
    int32_t j; double mv, gi;
    int st = column_gap(s, i, &j, &mv, &gi);
    if (st) return st;
    g[i] = gi;
    if (jrows) jrows[i] = j;
    if (minvals) minvals[i] = mv;
  }
  *total = or_chunk_tree_sum(g, s->n, 256);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Creation / reset                                                          */
/* ------------------------------------------------------------------------ */
static void free_state(or_state* s) {
  if (!s) return;
  free(s->a); free(s->b); free(s->C); free(s->X); free(s->Y);
  free(s->cnt); free(s->rows); free(s->vals); free(s->r); free(s->h);
  free(s->perm); free(s->G); free(s->fen); free(s->acc256); free(s->touched); free(s->trows); free(s->xbuf);
  free(s);
}

void or_destroy(or_state* s) { free_state(s); }

/* T^(0) = (b_1 e_1, ..., b_n e_1): all mass on row 0 (R3). */
int or_reset(or_state* s) {
  for (int32_t i = 0; i < s->n; i++) {
    /* t_i = b_i e_1; a zero-mass column (b_i = 0, Eq. 8 allows it) is the zero vector,
     * whose support is empty (exact zeros are not stored, R13) */
    s->cnt[i] = s->b[i] != 0.0 ? 1 : 0;
    s->rows[(int64_t)i * s->cap] = 0;
    s->vals[(int64_t)i * s->cap] = s->b[i];
  }
  for (int32_t k = 0; k < s->m; k++) s->r[k] = 0.0;
  double r0 = 0.0;
  for (int32_t i = 0; i < s->n; i++) r0 = r0 + s->b[i];
  s->r[0] = r0;
  for (int32_t k = 0; k < s->m; k++) s->h[k] = (s->r[k] - s->a[k]) / s->lambda;
  s->k = 0;
  s->configured = 0;
  s->perm_epoch = -1;
  return OR_OK;
}

or_state* or_create(int32_t m, int32_t n, double lambda, const double* a, const double* b,
                    int32_t cost_kind, const double* C, int64_t ld, const double* X, const double* Y,
                    uint64_t hash_seed, int32_t cap, int* status) {
  *status = OR_ERR_ARG;
  if (m < 1 || n < 1 || !(lambda > 0.0) || !isfinite(lambda) || cap < 1 || !a || !b) return NULL;
  if (cost_kind < OR_COST_DENSE || cost_kind > OR_COST_EUCLID_F32) return NULL;
  or_state* s = (or_state*)calloc(1, sizeof(or_state));
  if (!s) return NULL;
  s->m = m; s->n = n; s->lambda = lambda; s->cost_kind = cost_kind; s->cap = cap;
  s->hash_seed = hash_seed;
  s->a = (double*)malloc(sizeof(double) * m);
  s->b = (double*)malloc(sizeof(double) * n);
  memcpy(s->a, a, sizeof(double) * m);
  memcpy(s->b, b, sizeof(double) * n);
  if (cost_kind == OR_COST_DENSE) {
    if (!C || ld < m) { free_state(s); return NULL; }
    s->ld = m;
    s->C = (double*)malloc(sizeof(double) * (size_t)m * (size_t)n);
    if (!s->C) { free_state(s); return NULL; }
    for (int32_t i = 0; i < n; i++) memcpy(s->C + (int64_t)i * m, C + (int64_t)i * ld, sizeof(double) * m);
  } else if (cost_kind != OR_COST_HASH) {
    if (!X || !Y) { free_state(s); return NULL; }
    s->X = (double*)malloc(sizeof(double) * 3 * (size_t)m);
    s->Y = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    memcpy(s->X, X, sizeof(double) * 3 * (size_t)m);
    memcpy(s->Y, Y, sizeof(double) * 3 * (size_t)n);
  }
  /* validation: a, b >= 0 summing to 1 within 1e-12; C finite, >= 0 */
  double sa = 0.0, sb = 0.0;
  for (int32_t k = 0; k < m; k++) { if (!(a[k] >= 0.0) || !isfinite(a[k])) { free_state(s); *status = 4; return NULL; } sa = sa + a[k]; }
  /* b_i >= 0: a zero-mass block b_i Delta_m = {0} is allowed (Eq. 8; R32) */
  for (int32_t i = 0; i < n; i++) { if (!(b[i] >= 0.0) || !isfinite(b[i])) { free_state(s); *status = 4; return NULL; } sb = sb + b[i]; }
  if (fabs(sa - 1.0) > 1e-12 || fabs(sb - 1.0) > 1e-12) { free_state(s); *status = 4; return NULL; }
  if (cost_kind == OR_COST_DENSE) {
    for (int64_t q = 0; q < (int64_t)m * n; q++)
      if (!isfinite(s->C[q]) || !(s->C[q] >= 0.0)) { free_state(s); *status = OR_ERR_NONFINITE; return NULL; }
  } else if (cost_kind != OR_COST_HASH) {
    for (int64_t q = 0; q < 3 * (int64_t)m; q++) if (!isfinite(s->X[q])) { free_state(s); *status = OR_ERR_NONFINITE; return NULL; }
    for (int64_t q = 0; q < 3 * (int64_t)n; q++) if (!isfinite(s->Y[q])) { free_state(s); *status = OR_ERR_NONFINITE; return NULL; }
  }
  s->cnt = (int32_t*)malloc(sizeof(int32_t) * n);
  s->rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * cap);
  s->vals = (double*)malloc(sizeof(double) * (size_t)n * cap);
  s->r = (double*)malloc(sizeof(double) * m);
  s->h = (double*)malloc(sizeof(double) * m);
  s->perm = (int32_t*)malloc(sizeof(int32_t) * n);
  s->G = (double*)malloc(sizeof(double) * n);
  s->fen = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  s->touched = (unsigned char*)calloc((size_t)m, 1);
  s->trows = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  s->xbuf = (double*)malloc(sizeof(double) * (size_t)(m > n ? m : n));
  if (!s->cnt || !s->rows || !s->vals || !s->r || !s->h || !s->perm || !s->G || !s->fen || !s->trows ||
      !s->touched || !s->xbuf) { free_state(s); return NULL; }
  or_reset(s);
  *status = OR_OK;
  return s;
}

/* ------------------------------------------------------------------------ */
/* Objective (Eq. 7), gap forms (Thm 2; Eq. 11; App. D)  */
/* ------------------------------------------------------------------------ */
int or_objective(or_state* s, double* f) {
  double* lin = s->xbuf;
  for (int32_t i = 0; i < s->n; i++) {
    const int32_t* rw = s->rows + (int64_t)i * s->cap;
    const double* vl = s->vals + (int64_t)i * s->cap;
    double acc = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++) acc = acc + vl[p] * cost(s, rw[p], i);
    lin[i] = acc;
  }
  double L = or_chunk_tree_sum(lin, s->n, 256);
  for (int32_t k = 0; k < s->m; k++) { double d = s->r[k] - s->a[k]; lin[k] = d * d; }
  double pen = or_chunk_tree_sum(lin, s->m, 256);
  *f = L + pen / (2.0 * s->lambda);
  return OR_OK;
}

/* dense copy of row k of T (columns 0..n-1; exact zeros off the support) */
static void plan_row(const or_state* s, int32_t k, double* row) {
  for (int32_t i = 0; i < s->n; i++) {
    row[i] = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++)
      if (s->rows[(int64_t)i * s->cap + p] == k) row[i] = s->vals[(int64_t)i * s->cap + p];
  }
}

/* Barycentric projection, Eq. 15; zero rows keep x_k. */
int or_barycentric(or_state* s, const double* X, const double* Y, double* xhat) {
  double* row = (double*)malloc(sizeof(double) * (size_t)s->n);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)s->n);
  if (!row || !tmp) { free(row); free(tmp); return OR_ERR_ARG; }
  for (int32_t k = 0; k < s->m; k++) {
    plan_row(s, k, row);
    double den = or_chunk_tree_sum(row, s->n, 256);               /* sum_i T_ki */
    for (int d = 0; d < 3; d++) {
      if (den == 0.0) { xhat[3 * (int64_t)k + d] = X[3 * (int64_t)k + d]; continue; }
      for (int32_t i = 0; i < s->n; i++) tmp[i] = row[i] * Y[3 * (int64_t)i + d];
      double num = or_chunk_tree_sum(tmp, s->n, 256);             /* sum_i T_ki y_id */
      xhat[3 * (int64_t)k + d] = num / den;
    }
  }
  free(row); free(tmp);
  return OR_OK;
}

/* Metrics (iii), (iv) and <T, C> of (vi). */
int or_metrics(or_state* s, double* e_c, double* sparsity, double* lin) {
  const int32_t mx = s->m > s->n ? s->m : s->n;
  double* row = (double*)malloc(sizeof(double) * (size_t)s->n);
  double* sq = (double*)malloc(sizeof(double) * (size_t)mx);
  if (!row || !sq) { free(row); free(sq); return OR_ERR_ARG; }
  for (int32_t k = 0; k < s->m; k++) {                            /* (T 1 - a)_k^2 */
    plan_row(s, k, row);
    double rk = or_chunk_tree_sum(row, s->n, 256);
    double d = rk - s->a[k];
    sq[k] = d * d;
  }
  double e1 = sqrt(or_chunk_tree_sum(sq, s->m, 256));
  int64_t nnz = 0;
  for (int32_t i = 0; i < s->n; i++) {                            /* (T^T 1 - b)_i^2 */
    double ci = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++) ci = ci + s->vals[(int64_t)i * s->cap + p];
    nnz += s->cnt[i];
    double d = ci - s->b[i];
    sq[i] = d * d;
  }
  double e2 = sqrt(or_chunk_tree_sum(sq, s->n, 256));
  *e_c = e1 + e2;
  *sparsity = 1.0 - (double)nnz / ((double)s->m * (double)s->n);
  for (int32_t i = 0; i < s->n; i++) {                            /* <t_i, c_i>, rows ascending */
    double acc = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++)
      acc = acc + s->vals[(int64_t)i * s->cap + p] * cost(s, s->rows[(int64_t)i * s->cap + p], i);
    sq[i] = acc;
  }
  *lin = or_chunk_tree_sum(sq, s->n, 256);
  free(row); free(sq);
  return OR_OK;
}

/* Metrics (v) and (vi) against a reference plan T* (T*_LP in the paper), given as
 * COO sorted by column then row: e_m = ||T - T*||_F / ||T*||_F, e_v = |<T,C> - <T*,C>| / |<T*,C>|.
 * Per column i, over all rows k ascending: sum (T_ki - T*_ki)^2, sum T*_ki^2, sum T*_ki C_ki;
 * each then a 256-chunk sum over the columns (R19); <T, C> as in or_metrics. */
int or_lp_metrics(or_state* s, const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz,
                  double* e_m, double* e_v) {
  const int32_t m = s->m, n = s->n;
  for (int64_t q = 0; q < nnz; q++)
    if (rows[q] < 0 || rows[q] >= m || cols[q] < 0 || cols[q] >= n || !isfinite(vals[q]) ||
        (q > 0 && (cols[q] < cols[q - 1] || (cols[q] == cols[q - 1] && rows[q] <= rows[q - 1]))))
      return OR_ERR_ARG;
  double* Ts = (double*)calloc((size_t)m * n, sizeof(double));   /* T* dense, column-major */
  double* Tc = (double*)malloc(sizeof(double) * (size_t)m);
  double* dd = (double*)malloc(sizeof(double) * (size_t)n);
  double* ss = (double*)malloc(sizeof(double) * (size_t)n);
  double* cc = (double*)malloc(sizeof(double) * (size_t)n);
  if (!Ts || !Tc || !dd || !ss || !cc) { free(Ts); free(Tc); free(dd); free(ss); free(cc); return OR_ERR_ARG; }
  for (int64_t q = 0; q < nnz; q++) Ts[(int64_t)cols[q] * m + rows[q]] = vals[q];
  for (int32_t i = 0; i < n; i++) {
    for (int32_t k = 0; k < m; k++) Tc[k] = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++) Tc[s->rows[(int64_t)i * s->cap + p]] = s->vals[(int64_t)i * s->cap + p];
    double sd = 0.0, s2 = 0.0, sc = 0.0;
    for (int32_t k = 0; k < m; k++) {
      double ts = Ts[(int64_t)i * m + k];
      double d = Tc[k] - ts;
      sd = sd + d * d;
      s2 = s2 + ts * ts;
      sc = sc + ts * cost(s, k, i);
    }
    dd[i] = sd; ss[i] = s2; cc[i] = sc;
  }
  double D = or_chunk_tree_sum(dd, n, 256), S2 = or_chunk_tree_sum(ss, n, 256), SC = or_chunk_tree_sum(cc, n, 256);
  double e_c, sp, lin;
  or_metrics(s, &e_c, &sp, &lin);
  *e_m = sqrt(D) / sqrt(S2);
  *e_v = fabs(lin - SC) / fabs(SC);
  free(Ts); free(Tc); free(dd); free(ss); free(cc);
  return OR_OK;
}

int or_gap(or_state* s, double* total, double* per_column, int32_t* argmin_rows, double* minvals) {
  return gap_sweep(s, total, per_column, argmin_rows, minvals);
}

/* Theorem 2 form, sequential sums: <T - S, C> + (1/lambda) <r - S1, r - a> */
int or_gap_thm2(or_state* s, double* g) {
  double* S1 = (double*)calloc((size_t)s->m, sizeof(double));
  double A = 0.0;
  for (int32_t i = 0; i < s->n; i++) {
    int32_t j; double mv;
    int st = lmo(s, i, &j, &mv);
    if (st) { free(S1); return st; }
    const int32_t* rw = s->rows + (int64_t)i * s->cap;
    const double* vl = s->vals + (int64_t)i * s->cap;
    double tc = 0.0;
    for (int32_t p = 0; p < s->cnt[i]; p++) tc = tc + vl[p] * cost(s, rw[p], i);
    A = A + (tc - s->b[i] * cost(s, j, i));
    S1[j] = S1[j] + s->b[i];
  }
  double B = 0.0;
  for (int32_t k = 0; k < s->m; k++) B = B + (s->r[k] - S1[k]) * (s->r[k] - s->a[k]);
  *g = A + B / s->lambda;
  free(S1);
  return OR_OK;
}

/* Lagrangian dual value (App. D, min_j reading R4):
 * w = f - sum_i <t_i, grad_i f> + sum_i b_i min_k (grad_i f)_k */
int or_lagrangian_dual(or_state* s, double* w) {
  double f;
  or_objective(s, &f);
  double sdot = 0.0, smin = 0.0;
  for (int32_t i = 0; i < s->n; i++) {
    int32_t j; double mv;
    int st = lmo(s, i, &j, &mv);
    if (st) return st;
    sdot = sdot + column_dot_grad(s, i);
    smin = smin + s->b[i] * mv;
  }
  *w = (f - sdot) + smin;
  return OR_OK;
}

int or_get_plan_dense(or_state* s, double* T) {
  memset(T, 0, sizeof(double) * (size_t)s->m * s->n);
  for (int32_t i = 0; i < s->n; i++)
    for (int32_t p = 0; p < s->cnt[i]; p++)
      T[(int64_t)i * s->m + s->rows[(int64_t)i * s->cap + p]] = s->vals[(int64_t)i * s->cap + p];
  return OR_OK;
}

int or_get_plan_coo(or_state* s, int32_t* rows, int32_t* cols, double* vals, int64_t cap, int64_t* nnz) {
  int64_t q = 0;
  for (int32_t i = 0; i < s->n; i++)
    for (int32_t p = 0; p < s->cnt[i]; p++) {
      if (q < cap) {
        rows[q] = s->rows[(int64_t)i * s->cap + p];
        cols[q] = i;
        vals[q] = s->vals[(int64_t)i * s->cap + p];
      }
      q++;
    }
  *nnz = q;
  return q > cap ? OR_ERR_CAPACITY : OR_OK;
}

int or_get_r(or_state* s, double* r) { memcpy(r, s->r, sizeof(double) * s->m); return OR_OK; }
int64_t or_get_k(or_state* s) { return s->k; }

int or_set_plan_dense(or_state* s, const double* T) {
  for (int32_t i = 0; i < s->n; i++) {
    int32_t c = 0;
    for (int32_t k = 0; k < s->m; k++) {
      double t = T[(int64_t)i * s->m + k];
      if (t < 0.0 || !isfinite(t)) return OR_ERR_ARG;
      if (t != 0.0) {
        if (c >= s->cap) return OR_ERR_CAPACITY;
        s->rows[(int64_t)i * s->cap + c] = k;
        s->vals[(int64_t)i * s->cap + c] = t;
        c++;
      }
    }
    s->cnt[i] = c;
  }
  for (int32_t k = 0; k < s->m; k++) {
    double acc = 0.0;
    for (int32_t i = 0; i < s->n; i++) acc = acc + T[(int64_t)i * s->m + k];
    s->r[k] = acc;
    s->h[k] = (s->r[k] - s->a[k]) / s->lambda;
  }
  s->k = 0;
  s->configured = 0;
  s->perm_epoch = -1;
  return OR_OK;
}

int or_max_cost(or_state* s, double* cmax) {
  double mx = 0.0;
  for (int32_t i = 0; i < s->n; i++)
    for (int32_t k = 0; k < s->m; k++) { double c = cost(s, k, i); if (c > mx) mx = c; }
  *cmax = mx;
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* The unified plain step over a column set U:            */
/*   BCFW (Alg. 1) is U = {i}; FW (Alg. A.1) is U = [n]; batched is a block. */
/* Phase A: LMO + column gaps + G_U. Phase B: direction, step size, update.  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t L;
  const int32_t* U;
  int32_t* j;
  double* minval;
  double* g;
  double G;        /* psum256 of g over U (= g(T) when U = [n]) */
} plain_lmo_out;

static int plain_lmo(or_state* s, plain_lmo_out* o) {
  for (int64_t p = 0; p < o->L; p++) {
    int st = column_gap(s, o->U[p], &o->j[p], &o->minval[p], &o->g[p]);
    if (st) return st;
  }
  o->G = or_chunk_tree_sum(o->g, o->L, 256);
  return OR_OK;
}

/* Build the merged support supp(t_i) U {j} in ascending row order. Returns count. */
static int32_t merged_rows(const or_state* s, int32_t i, int32_t j, int32_t* mr, double* mt) {
  const int32_t* rw = s->rows + (int64_t)i * s->cap;
  const double* vl = s->vals + (int64_t)i * s->cap;
  int32_t c = 0, p = 0, inserted = 0;
  while (p < s->cnt[i] || !inserted) {
    if (!inserted && (p >= s->cnt[i] || j < rw[p])) {
      mr[c] = j; mt[c] = 0.0; c++; inserted = 1;
    } else {
      if (rw[p] == j) inserted = 1;
      mr[c] = rw[p]; mt[c] = vl[p]; c++; p++;
    }
  }
  return c;
}

/* Per-row sums of per-column contributions over U (R19): for row k the
 * contributions of the columns at positions p of U are summed left to right
 * inside each of the 256 position chunks, and the 256 chunk partials are
 * combined by adjacent pairs — chunk_tree_sum over U's positions. acc256[c][k]
 * holds the partial of chunk c for row k (+0.0 when nothing was added). */
static int acc_begin(or_state* s) {
  if (!s->acc256) {
    s->acc256 = (double*)calloc((size_t)256 * s->m, sizeof(double));
    if (!s->acc256) return OR_ERR_ARG;
  }
  s->ntrows = 0;
  return OR_OK;
}

static void acc_add(or_state* s, int32_t c, int32_t k, double v) {
  double* a = &s->acc256[(size_t)c * s->m + k];
  *a = *a + v;
  if (!s->touched[k]) { s->touched[k] = 1; s->trows[s->ntrows++] = k; }
}

static double row_tree256(const or_state* s, int32_t k) {
  double part[256];
  for (int c = 0; c < 256; c++) part[c] = s->acc256[(size_t)c * s->m + k];
  for (int width = 256; width > 1; width /= 2)
    for (int c = 0; c < width / 2; c++) part[c] = part[2 * c] + part[2 * c + 1];
  return part[0];
}

static void acc_clear(or_state* s) {
  for (int32_t t = 0; t < s->ntrows; t++) {
    const int32_t k = s->trows[t];
    for (int c = 0; c < 256; c++) s->acc256[(size_t)c * s->m + k] = 0.0;
    s->touched[k] = 0;
  }
  s->ntrows = 0;
}

static int plain_update(or_state* s, const plain_lmo_out* o, int32_t step_rule, int64_t nprime,
                        double* gamma_out, double* num_out, double* den_out) {
  const int64_t L = o->L;
  const int32_t cap1 = s->cap + 1;
  int32_t* mr = (int32_t*)malloc(sizeof(int32_t) * (size_t)L * cap1);
  double* mt = (double*)malloc(sizeof(double) * (size_t)L * cap1);
  int32_t* mc = (int32_t*)malloc(sizeof(int32_t) * (size_t)L);
  if (!mr || !mt || !mc) { free(mr); free(mt); free(mc); return OR_ERR_ARG; }

  /* 2. direction d_i = s_i - t_i on supp(t_i) U {j_i}; Delta_k = per-row psum256 over U */
  if (acc_begin(s)) { free(mr); free(mt); free(mc); return OR_ERR_ARG; }
  for (int64_t p = 0; p < L; p++) {
    int32_t i = o->U[p];
    int32_t c256 = chunk_of(p, L, 256);
    mc[p] = merged_rows(s, i, o->j[p], mr + p * cap1, mt + p * cap1);
    for (int32_t q = 0; q < mc[p]; q++) {
      int32_t k = mr[p * cap1 + q];
      double sk = (k == o->j[p]) ? s->b[i] : 0.0;
      double d = sk - mt[p * cap1 + q];
      acc_add(s, c256, k, d);
    }
  }
  double* x = s->xbuf;
  for (int32_t k = 0; k < s->m; k++) x[k] = 0.0;
  for (int32_t t = 0; t < s->ntrows; t++) {
    const int32_t k = s->trows[t];
    double D = row_tree256(s, k);
    x[k] = D * D;
  }
  acc_clear(s);
  double den = or_chunk_tree_sum(x, s->m, 256);
  double num = s->lambda * o->G;

  /* 3. step size: ELS (Eq. 10 / Eq. A.1) or DEC 2n'/(k'+2n') (Alg. 1, Alg. A.1) */
  double gamma;
  if (step_rule == OR_STEP_ELS) {
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = num / den; if (gamma > 1.0) gamma = 1.0; }
  } else {
    gamma = (double)(2 * nprime) / (double)(s->k + 2 * nprime);
  }

  /* 4. update t_i <- (1-gamma) t_i + gamma s_i; r += psum256_U(t' - t) */
  double omg = 1.0 - gamma;
  /* capacity check before mutating */
  for (int64_t p = 0; p < L; p++) {
    int32_t i = o->U[p];
    double gb = gamma * s->b[i];
    int32_t keep = 0;
    for (int32_t q = 0; q < mc[p]; q++) {
      int32_t k = mr[p * cap1 + q];
      double tn = omg * mt[p * cap1 + q];
      if (k == o->j[p]) tn = tn + gb;
      if (tn != 0.0) keep++;
    }
    if (keep > s->cap) { free(mr); free(mt); free(mc); return OR_ERR_CAPACITY; }
  }
  acc_begin(s);
  for (int64_t p = 0; p < L; p++) {
    int32_t i = o->U[p];
    int32_t c256 = chunk_of(p, L, 256);
    double gb = gamma * s->b[i];
    int32_t* rw = s->rows + (int64_t)i * s->cap;
    double* vl = s->vals + (int64_t)i * s->cap;
    int32_t keep = 0;
    for (int32_t q = 0; q < mc[p]; q++) {
      int32_t k = mr[p * cap1 + q];
      double told = mt[p * cap1 + q];
      double tn = omg * told;
      if (k == o->j[p]) tn = tn + gb;
      double delta = tn - told;
      acc_add(s, c256, k, delta);
      if (tn != 0.0) { rw[keep] = k; vl[keep] = tn; keep++; }   /* drop exact zeros (R13) */
    }
    s->cnt[i] = keep;
  }
  for (int32_t k = 0; k < s->m; k++) {
    if (!s->touched[k]) continue;
    double D = row_tree256(s, k);
    s->r[k] = s->r[k] + D;
    s->h[k] = (s->r[k] - s->a[k]) / s->lambda;
  }
  acc_clear(s);
  free(mr); free(mt); free(mc);
  *gamma_out = gamma; *num_out = num; *den_out = den;
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Away (Alg. A.2, Eq. 13-14) and pairwise (Alg. A.3) steps on one column.   */
/* ------------------------------------------------------------------------ */
/* single-column r/h update from old/new column values over touched rows */
static void apply_column(or_state* s, int32_t i, const int32_t* mr, const double* told, const double* tnew, int32_t c) {
  int32_t* rw = s->rows + (int64_t)i * s->cap;
  double* vl = s->vals + (int64_t)i * s->cap;
  int32_t keep = 0;
  for (int32_t q = 0; q < c; q++) {
    int32_t k = mr[q];
    double delta = tnew[q] - told[q];
    double D = delta + 0.0;              /* per-row psum256 of a single column's term (R19) */
    s->r[k] = s->r[k] + D;
    s->h[k] = (s->r[k] - s->a[k]) / s->lambda;
    if (tnew[q] != 0.0) { rw[keep] = k; vl[keep] = tnew[q]; keep++; }
  }
  s->cnt[i] = keep;
}

/* den of a single-column direction = psum256 over all m rows of d_k^2 */
static double single_den(or_state* s, const int32_t* mr, const double* d, int32_t c) {
  double* x = s->xbuf;
  for (int32_t k = 0; k < s->m; k++) x[k] = 0.0;
  for (int32_t q = 0; q < c; q++) x[mr[q]] = d[q] * d[q];
  return or_chunk_tree_sum(x, s->m, 256);
}

/* BCAFW step. Returns direction in *dir. */
static int away_step(or_state* s, int32_t i, or_trace_rec* tr, int* dir_out, double* g_pre) {
  int32_t j; double minval;
  int st = lmo(s, i, &j, &minval);
  if (st) return st;
  const int32_t* rw = s->rows + (int64_t)i * s->cap;
  const double* vl = s->vals + (int64_t)i * s->cap;
  const int32_t c0 = s->cnt[i];
  /* away atom v = argmax_{k in supp} grad_ki, lowest k on ties (Eq. 13, R1) */
  int32_t v = -1, vq = -1; double gv = -INFINITY;
  double dot = 0.0;
  for (int32_t p = 0; p < c0; p++) {
    double gk = cost(s, rw[p], i) + s->h[rw[p]];
    if (gk > gv) { gv = gk; v = rw[p]; vq = p; }
    double prod = vl[p] * gk;
    dot = dot + prod;
  }
  double bi = s->b[i];
  double gfw = dot - bi * minval;          /* <-grad, d_FW>  = g_i     */
  *g_pre = gfw;
  if (c0 == 0) {
    /* zero-mass column (b_i = 0, R32): t_i = s_i = 0, every direction is zero, no-op */
    *dir_out = 3;
    if (tr) { tr->i = i; tr->j = j; tr->v = -1; tr->dir = 3; tr->gamma = 0.0; tr->num = 0.0; tr->den = 0.0; tr->minval = minval; }
    return OR_OK;
  }
  double gaw = bi * gv - dot;              /* <-grad, d_Away> = g^A_i   */
  int use_fw = (c0 == 1) || (gfw >= gaw); /* R12: singleton forces FW */
  int32_t cap1 = s->cap + 1;
  int32_t* mr = (int32_t*)malloc(sizeof(int32_t) * cap1);
  double* mt = (double*)malloc(sizeof(double) * cap1);
  double* d = (double*)malloc(sizeof(double) * cap1);
  double* tn = (double*)malloc(sizeof(double) * cap1);
  double gamma, num, den;
  int32_t c;
  if (use_fw) {
    c = merged_rows(s, i, j, mr, mt);
    for (int32_t q = 0; q < c; q++) d[q] = ((mr[q] == j) ? bi : 0.0) - mt[q];
    den = single_den(s, mr, d, c);
    double G = gfw + 0.0;                  /* psum256 of a single term */
    num = s->lambda * G;
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = num / den; if (gamma > 1.0) gamma = 1.0; }
    double omg = 1.0 - gamma, gb = gamma * bi;
    int32_t keep = 0;
    for (int32_t q = 0; q < c; q++) { tn[q] = omg * mt[q]; if (mr[q] == j) tn[q] = tn[q] + gb; if (tn[q] != 0.0) keep++; }
    if (keep > s->cap) { free(mr); free(mt); free(d); free(tn); return OR_ERR_CAPACITY; }
    *dir_out = 0;
  } else {
    c = c0;
    for (int32_t q = 0; q < c; q++) { mr[q] = rw[q]; mt[q] = vl[q]; d[q] = (q == vq) ? (vl[q] - bi) : vl[q]; }
    den = single_den(s, mr, d, c);
    double G = gaw + 0.0;
    num = s->lambda * G;
    double alpha = vl[vq] / bi;
    double gmax = alpha / (1.0 - alpha);
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = num / den; if (gamma > gmax) gamma = gmax; }
    double opg = 1.0 + gamma, gb = gamma * bi;
    for (int32_t q = 0; q < c; q++) {
      tn[q] = opg * mt[q];
      if (q == vq) {
        tn[q] = tn[q] - gb;
        if (gamma == gmax || tn[q] < 0.0) tn[q] = 0.0;   /* drop step (R13) */
      }
    }
    *dir_out = 1;
  }
  apply_column(s, i, mr, mt, tn, c);
  if (tr) { tr->i = i; tr->j = j; tr->v = v; tr->dir = *dir_out; tr->gamma = gamma; tr->num = num; tr->den = den; tr->minval = minval; }
  free(mr); free(mt); free(d); free(tn);
  return OR_OK;
}

/* BCPFW step: d = s_i - v_i, gamma_max = alpha_v. Closed form of
 * Eq. 14 with d = b_i (e_j - e_v): gamma = lambda (grad_v - grad_j) / (2 b_i). */
static int pairwise_step(or_state* s, int32_t i, or_trace_rec* tr, int* dir_out, double* g_pre) {
  int32_t j; double minval;
  int st = lmo(s, i, &j, &minval);
  if (st) return st;
  const int32_t* rw = s->rows + (int64_t)i * s->cap;
  const double* vl = s->vals + (int64_t)i * s->cap;
  const int32_t c0 = s->cnt[i];
  int32_t v = -1, vq = -1; double gv = -INFINITY, dot = 0.0;
  for (int32_t p = 0; p < c0; p++) {
    double gk = cost(s, rw[p], i) + s->h[rw[p]];
    if (gk > gv) { gv = gk; v = rw[p]; vq = p; }
    double prod = vl[p] * gk;
    dot = dot + prod;
  }
  double bi = s->b[i];
  *g_pre = dot - bi * minval;
  double gamma = 0.0, num = 0.0, den = 0.0;
  if (v == j || c0 == 0) {
    *dir_out = 3;                          /* no-op step (c0 == 0: zero-mass column, R32) */
  } else {
    double dv = gv - minval;               /* grad_v - grad_j >= 0 */
    num = s->lambda * dv;
    den = 2.0 * bi;
    double alpha = vl[vq] / bi;
    if (!(num > 0.0)) gamma = 0.0;
    else { gamma = num / den; if (gamma > alpha) gamma = alpha; }
    /* new column: move mu = gamma b_i from v to j */
    int32_t cap1 = s->cap + 1;
    int32_t* mr = (int32_t*)malloc(sizeof(int32_t) * cap1);
    double* mt = (double*)malloc(sizeof(double) * cap1);
    double* tn = (double*)malloc(sizeof(double) * cap1);
    int32_t c = merged_rows(s, i, j, mr, mt);
    double mu = gamma * bi;
    int drop = (gamma == alpha) || (mu >= vl[vq]);
    if (drop) mu = vl[vq];
    int32_t keep = 0;
    for (int32_t q = 0; q < c; q++) {
      tn[q] = mt[q];
      if (mr[q] == j) tn[q] = mt[q] + mu;
      if (mr[q] == v) tn[q] = drop ? 0.0 : (mt[q] - mu);
      if (tn[q] != 0.0) keep++;
    }
    if (keep > s->cap) { free(mr); free(mt); free(tn); return OR_ERR_CAPACITY; }
    apply_column(s, i, mr, mt, tn, c);
    free(mr); free(mt); free(tn);
    *dir_out = 2;
  }
  if (tr) { tr->i = i; tr->j = j; tr->v = v; tr->dir = *dir_out; tr->gamma = gamma; tr->num = num; tr->den = den; tr->minval = minval; }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* GA sampler: Fenwick tree over max(G_i, 0) (Alg. A.4 line 2; R14-17)*/
/* ------------------------------------------------------------------------ */
static double wpos(double g) { return g > 0.0 ? g : 0.0; }

static void fen_build(or_state* s) {
  int32_t n = s->n;
  s->fen[0] = 0.0;
  for (int32_t i = 1; i <= n; i++) s->fen[i] = wpos(s->G[i - 1]);
  for (int32_t i = 1; i <= n; i++) {
    int32_t p = i + (i & -i);
    if (p <= n) s->fen[p] = s->fen[p] + s->fen[i];
  }
}

static void fen_add(or_state* s, int32_t i0, double delta) {
  for (int32_t p = i0 + 1; p <= s->n; p += p & -p) s->fen[p] = s->fen[p] + delta;
}

static double fen_total(const or_state* s) {
  double acc = 0.0;
  for (int32_t p = s->n; p > 0; p -= p & -p) acc = acc + s->fen[p];
  return acc;
}

static int32_t fen_draw(const or_state* s, double u53) {
  int32_t n = s->n;
  double W = fen_total(s);
  if (!(W > 0.0)) {                       /* all-zero weights: uniform fallback (R17) */
    int32_t i = (int32_t)(u53 * (double)n);
    return i >= n ? n - 1 : i;
  }
  double u = u53 * W;
  int32_t pos = 0, bit = 1;
  while (bit * 2 <= n) bit *= 2;
  for (; bit > 0; bit >>= 1) {
    if (pos + bit <= n && s->fen[pos + bit] <= u) { pos += bit; u = u - s->fen[pos]; }
  }
  if (pos >= n) {                         /* rounding fell off the end: last positive weight */
    for (int32_t i = n - 1; i >= 0; i--) if (wpos(s->G[i]) > 0.0) return i;
    return n - 1;
  }
  return pos;
}

int or_fenwick_draw(const double* w, int32_t n, double u53, int32_t* out) {
  or_state tmp;
  memset(&tmp, 0, sizeof(tmp));
  tmp.n = n;
  tmp.G = (double*)w;
  tmp.fen = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  fen_build(&tmp);
  *out = fen_draw(&tmp, u53);
  free(tmp.fen);
  return OR_OK;
}

/* GA state for pins: stored gaps G (n) and the prefix sums of the tree,
 * prefix[i] = sum of the weights of columns 0..i as the tree holds them (n). */
int or_get_ga(or_state* s, double* G, double* prefix) {
  if (!s->G || !s->fen) return OR_ERR_STATE;
  for (int32_t i = 0; i < s->n; i++) {
    if (G) G[i] = s->G[i];
    if (prefix) {
      double acc = 0.0;
      for (int32_t p = i + 1; p > 0; p -= p & -p) acc = acc + s->fen[p];
      prefix[i] = acc;
    }
  }
  return OR_OK;
}

/* Fenwick point updates in isolation (pin of fen_add): build over w0, then for
 * u = 0..nupd-1 set column idx[u] to newval[u] exactly as the GA inner refresh does
 * (delta = max(new,0) - max(old,0) added along the update path); then prefix[i] (n)
 * and one draw per u53s entry (ndraw) from the updated tree. */
int or_fenwick_updates(const double* w0, int32_t n, const int32_t* idx, const double* newval, int32_t nupd,
                       double* prefix, const double* u53s, int32_t ndraw, int32_t* draws) {
  or_state tmp;
  memset(&tmp, 0, sizeof(tmp));
  tmp.n = n;
  tmp.G = (double*)malloc(sizeof(double) * (size_t)n);
  tmp.fen = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  memcpy(tmp.G, w0, sizeof(double) * (size_t)n);
  fen_build(&tmp);
  for (int32_t u = 0; u < nupd; u++) {
    int32_t i = idx[u];
    double delta = wpos(newval[u]) - wpos(tmp.G[i]);
    tmp.G[i] = newval[u];
    fen_add(&tmp, i, delta);
  }
  or_get_ga(&tmp, NULL, prefix);
  for (int32_t d = 0; d < ndraw; d++) draws[d] = fen_draw(&tmp, u53s[d]);
  free(tmp.G); free(tmp.fen);
  return OR_OK;
}

static int ga_global_refresh(or_state* s, int64_t* entries) {
  for (int32_t i = 0; i < s->n; i++) {
    int32_t j; double mv, g;
    int st = column_gap(s, i, &j, &mv, &g);
    if (st) return st;
    s->G[i] = g;
  }
  *entries += (int64_t)s->m * s->n;
  fen_build(s);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Driver (Alg. 1 loop; stopping P:186; R2, R11)   */
/* ------------------------------------------------------------------------ */
static int options_equal(const or_options* x, const or_options* y) {
  return x->step_rule == y->step_rule && x->sampling == y->sampling && x->epsilon == y->epsilon &&
         x->gap_period == y->gap_period && x->ga_M == y->ga_M && x->ga_inner == y->ga_inner &&
         x->ga_post_update == y->ga_post_update && x->block_size == y->block_size && x->nranks == y->nranks;
}

static int32_t draw_unit(or_state* s, int32_t sampling, int64_t nprime) {
  if (sampling == OR_SAMPLE_U) {
    return uniform_index(or_rng_u64(s->seed, 0, (uint64_t)s->k), (int32_t)nprime);
  }
  if (sampling == OR_SAMPLE_P) {
    int64_t e = s->k / nprime;
    if (e != s->perm_epoch) { or_permutation(s->seed, e, (int32_t)nprime, s->perm); s->perm_epoch = e; }
    return s->perm[s->k % nprime];
  }
  /* GA (BCFW family: a column; batched: the block of a column drawn with probability
     proportional to max(G_i, 0), i.e. a block with probability proportional to its columns'
     summed stored gaps — SURVEY NEXT-4, R31) */
  int32_t i = fen_draw(s, or_uniform53(or_rng_u64(s->seed, 1, (uint64_t)s->k)));
  return nprime == s->n ? i : i / (s->n / (int32_t)nprime);
}

int or_solve(or_state* s, int32_t variant, const or_options* o, int64_t iters, uint64_t seed,
             const int32_t* visit, or_result* res, or_trace_rec* trace) {
  memset(res, 0, sizeof(*res));
  res->gap = NAN;
  if (variant < OR_FW || variant > OR_BATCHED || iters < 0) return OR_ERR_ARG;
  if (o->gap_period < 1) return OR_ERR_ARG;
  if ((variant == OR_BCAFW || variant == OR_BCPFW) && o->step_rule != OR_STEP_ELS) return OR_ERR_ARG;
  if (o->sampling == OR_SAMPLE_GA && variant == OR_FW) return OR_ERR_ARG;
  if (o->sampling == OR_SAMPLE_GA && variant == OR_BATCHED && o->nranks > 1) return OR_ERR_ARG;
  if (o->sampling == OR_SAMPLE_GA && o->ga_M < 1) return OR_ERR_ARG;
  int32_t G = o->nranks < 1 ? 1 : o->nranks;
  int64_t nprime;
  if (variant == OR_FW) nprime = 1;
  else if (variant == OR_BATCHED) {
    if (o->block_size < 1 || s->n % G != 0 || (s->n / G) % o->block_size != 0) return OR_ERR_ARG;
    nprime = (s->n / G) / o->block_size;
  } else nprime = s->n;
  if (s->configured) {
    if (s->variant != variant || s->seed != seed || !options_equal(&s->opt, o)) return OR_ERR_STATE;
  } else {
    s->configured = 1; s->variant = variant; s->opt = *o; s->seed = seed;
    if (o->sampling == OR_SAMPLE_GA && variant != OR_FW) {
      double cmax;
      or_max_cost(s, &cmax);
      double cinit = cmax + 2.0 / s->lambda;   /* R14: g(T0) <= max C + 2/lambda (App. C) */
      for (int32_t i = 0; i < s->n; i++) s->G[i] = cinit;
      fen_build(s);
    }
  }
  const int32_t m = s->m, n = s->n;
  int64_t L = (variant == OR_FW) ? n : (variant == OR_BATCHED ? (int64_t)o->block_size * G : 1);
  int32_t* U = (int32_t*)malloc(sizeof(int32_t) * (size_t)L);
  int32_t* jj = (int32_t*)malloc(sizeof(int32_t) * (size_t)L);
  double* mv = (double*)malloc(sizeof(double) * (size_t)L);
  double* gg = (double*)malloc(sizeof(double) * (size_t)L);
  int status = OR_OK;
  int64_t done = 0;
  const int64_t period = (int64_t)o->gap_period * nprime;

  for (;;) {
    /* gap check at epoch boundaries, before the epoch's steps (R11) */
    if (variant != OR_FW && s->k % period == 0) {
      double g;
      status = gap_sweep(s, &g, NULL, NULL, NULL);
      if (status) break;
      res->gap = g; res->gap_checks++;
      res->entries_scanned += (int64_t)m * n;
      if (g <= o->epsilon) { res->converged = 1; break; }
    }
    if (done >= iters) break;
    or_trace_rec* tr = trace ? &trace[done] : NULL;
    if (tr) { memset(tr, 0, sizeof(*tr)); tr->k = s->k; tr->v = -1; }

    if (variant == OR_FW || variant == OR_BATCHED || variant == OR_BCFW) {
      if (variant == OR_FW) {
        for (int32_t i = 0; i < n; i++) U[i] = i;
      } else {
        int32_t unit = visit ? visit[done] : draw_unit(s, o->sampling, nprime);
        if (unit < 0 || unit >= nprime) { status = OR_ERR_ARG; break; }
        if (variant == OR_BCFW) U[0] = unit;
        else {
          int64_t q = 0;
          for (int32_t rr = 0; rr < G; rr++)
            for (int32_t t = 0; t < o->block_size; t++)
              U[q++] = rr * (n / G) + unit * o->block_size + t;
        }
      }
      plain_lmo_out po = {L, U, jj, mv, gg, 0.0};
      status = plain_lmo(s, &po);
      if (status) break;
      res->entries_scanned += (int64_t)m * L;
      if (variant == OR_FW) {
        /* Alg. A.1 line 4: stop check with g(T^k) = G_[n], before the step */
        res->gap = po.G; res->gap_checks++;
        if (po.G <= o->epsilon) { res->converged = 1; break; }
      }
      double gamma, num, den;
      status = plain_update(s, &po, o->step_rule, nprime, &gamma, &num, &den);
      if (status) break;
      if (tr) { tr->i = U[0]; tr->j = jj[0]; tr->dir = 0; tr->gamma = gamma; tr->num = num; tr->den = den; tr->minval = mv[0]; }
      if ((variant == OR_BCFW || variant == OR_BATCHED) && o->sampling == OR_SAMPLE_GA && o->ga_inner) {
        /* stored gaps of the visited columns (Alg. A.4 line 6), columns ascending */
        for (int64_t t = 0; t < L && status == OR_OK; t++) {
          int32_t i = U[t];
          double gnew = gg[t];
          if (o->ga_post_update) {
            int32_t j2; double m2;
            status = column_gap(s, i, &j2, &m2, &gnew);
            res->entries_scanned += m;
          }
          double delta = wpos(gnew) - wpos(s->G[i]);
          s->G[i] = gnew;
          fen_add(s, i, delta);
        }
        if (status) break;
      }
    } else {
      int32_t i = visit ? visit[done] : draw_unit(s, o->sampling, nprime);
      if (i < 0 || i >= n) { status = OR_ERR_ARG; break; }
      int dir; double gpre;
      if (variant == OR_BCAFW) status = away_step(s, i, tr, &dir, &gpre);
      else status = pairwise_step(s, i, tr, &dir, &gpre);
      if (status) break;
      res->entries_scanned += m;
      if (o->sampling == OR_SAMPLE_GA && o->ga_inner) {
        double gnew = gpre;
        if (o->ga_post_update) {
          int32_t j2; double m2;
          status = column_gap(s, i, &j2, &m2, &gnew);
          if (status) break;
          res->entries_scanned += m;
        }
        double delta = wpos(gnew) - wpos(s->G[i]);
        s->G[i] = gnew;
        fen_add(s, i, delta);
      }
    }
    s->k++;
    done++;
    /* GA global refresh after step k when (k+1) mod (M n') == 0 (R16; n' = n for the
       BCFW family, n / B block steps for batched, R31) */
    if (o->sampling == OR_SAMPLE_GA && variant != OR_FW && s->k % ((int64_t)o->ga_M * nprime) == 0) {
      status = ga_global_refresh(s, &res->entries_scanned);
      if (status) break;
    }
  }
  res->iters_done = done;
  res->k = s->k;
  double f = NAN;
  if (status == OR_OK) or_objective(s, &f);
  res->objective = f;
  free(U); free(jj); free(mv); free(gg);
  if (status) return status;
  return res->converged ? OR_OK : OR_NOT_CONVERGED;
}
