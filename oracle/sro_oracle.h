/* sro_oracle.h — interface of the plain fp64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The
 * product path (paper_2103_05857_b200/) never links or imports it, and shares
 * no code, header, table or constant generator with it.
 *
 * This header is the oracle's own; it is NOT include/sro.h (the product
 * boundary). See oracle/sro_oracle.c for the algorithm, written step by step
 * from /root/reference/PAPER.md (cited as P:<line>) with the readings listed
 * in DESIGN.md §3.
 */
#ifndef SRO_ORACLE_H
#define SRO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_NOT_CONVERGED = 1, OR_ERR_ARG = 2, OR_ERR_NONFINITE = 5, OR_ERR_CAPACITY = 6, OR_ERR_STATE = 10 };
enum { OR_COST_DENSE = 0, OR_COST_SQEUCLID = 1, OR_COST_EUCLID = 2, OR_COST_HASH = 3,
       OR_COST_SQEUCLID_F32 = 4, OR_COST_EUCLID_F32 = 5 };
enum { OR_FW = 0, OR_BCFW = 1, OR_BCAFW = 2, OR_BCPFW = 3, OR_BATCHED = 4 };
enum { OR_STEP_DEC = 0, OR_STEP_ELS = 1 };
enum { OR_SAMPLE_U = 0, OR_SAMPLE_P = 1, OR_SAMPLE_GA = 2 };

typedef struct or_state or_state;

typedef struct {
  int32_t step_rule;       /* OR_STEP_* */
  int32_t sampling;        /* OR_SAMPLE_* */
  double epsilon;          /* stop at the first gap check with g <= epsilon */
  int32_t gap_period;      /* epochs between gap checks (>= 1) */
  int32_t ga_M;            /* GA global refresh every M*n steps */
  int32_t ga_inner;        /* 1 = GAD (refresh g_i of the visited column), 0 = GAS */
  int32_t ga_post_update;  /* 1 = store g_i(T^{k+1}) (default), 0 = g_i(T^k) */
  int32_t block_size;      /* batched: B; columns per rank-block */
  int32_t nranks;          /* batched / FW: G, column shards (affects only the batched block map) */
} or_options;

typedef struct {
  int64_t iters_done;
  int64_t k;               /* global step counter after the call */
  double gap;              /* last gap evaluated (NaN if none) */
  double objective;
  int32_t converged;
  int32_t gap_checks;
  int64_t entries_scanned; /* cost entries read by LMO calls (steps + sweeps) */
} or_result;

/* One record per step when tracing is enabled. */
typedef struct {
  int64_t k;
  int32_t i;        /* column (first column of U for block steps) */
  int32_t j;        /* LMO argmin row (for i) */
  int32_t v;        /* away atom row (-1 if none) */
  int32_t dir;      /* 0 FW, 1 away, 2 pairwise, 3 no-op */
  double gamma, num, den, minval;
} or_trace_rec;

or_state* or_create(int32_t m, int32_t n, double lambda, const double* a, const double* b,
                    int32_t cost_kind, const double* C, int64_t ld, const double* X, const double* Y,
                    uint64_t hash_seed, int32_t cap, int* status);
void or_destroy(or_state* s);
int or_reset(or_state* s);

int or_solve(or_state* s, int32_t variant, const or_options* o, int64_t iters, uint64_t seed,
             const int32_t* visit /* optional explicit visit list of length iters, or NULL */,
             or_result* res, or_trace_rec* trace /* NULL or iters records */);

int or_gap(or_state* s, double* total, double* per_column, int32_t* argmin_rows, double* minvals);
int or_gap_thm2(or_state* s, double* g);           /* Thm 2 form */
int or_lagrangian_dual(or_state* s, double* w);    /* App. D */
int or_objective(or_state* s, double* f);
/* Barycentric projection (Eq. 15): xhat_k = (sum_i T_ki y_i) / (sum_i T_ki) for
 * every row with mass; a row without mass keeps x_k. Both sums run over the n columns
 * as R19's 256-chunk pairwise sum over column positions. X: m x 3, Y: n x 3, xhat: m x 3. */
int or_barycentric(or_state* s, const double* X, const double* Y, double* xhat);
/* Metrics (iii), (iv) and the <T, C> of (vi): e_c = ||T 1 - a||_2 + ||T^T 1 - b||_2
 * (row sums as in or_barycentric, column sums over the support rows ascending, each norm the
 * square root of a 256-chunk sum of squares); sparsity = 1 - nnz(T) / (m n);
 * lin = 256-chunk sum over columns of <t_i, c_i>. */
int or_metrics(or_state* s, double* e_c, double* sparsity, double* lin);
/* Metrics (v) e_m = ||T - T*||_F / ||T*||_F and (vi) e_v = |<T,C> - <T*,C>| / |<T*,C>|
 * against T* given as COO sorted by column then row; sums per column over all rows ascending,
 * then 256-chunk sums over columns. */
int or_lp_metrics(or_state* s, const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz,
                  double* e_m, double* e_v);
int or_get_plan_dense(or_state* s, double* T);     /* m*n column-major */
int or_get_plan_coo(or_state* s, int32_t* rows, int32_t* cols, double* vals, int64_t cap, int64_t* nnz);
int or_get_r(or_state* s, double* r);
int or_set_plan_dense(or_state* s, const double* T); /* r := T*1 (sequential), k := 0 */
int64_t or_get_k(or_state* s);
double or_cost(or_state* s, int32_t k, int32_t i);
int or_lmo_column(or_state* s, int32_t i, int32_t* j, double* minval);
int or_max_cost(or_state* s, double* cmax);

/* building blocks exposed for pins */
double or_chunk_tree_sum(const double* x, int64_t L, int32_t W);
uint64_t or_splitmix64_mix(uint64_t z);
uint64_t or_rng_u64(uint64_t seed, uint32_t stream, uint64_t t);
double or_uniform53(uint64_t x);
int or_permutation(uint64_t seed, int64_t epoch, int32_t n, int32_t* perm);
int or_fenwick_draw(const double* w, int32_t n, double u53, int32_t* out);
/* GA state (stored gaps, tree prefix sums) and Fenwick point updates in isolation, for pins */
int or_get_ga(or_state* s, double* G, double* prefix);
int or_fenwick_updates(const double* w0, int32_t n, const int32_t* idx, const double* newval, int32_t nupd,
                       double* prefix, const double* u53s, int32_t ndraw, int32_t* draws);

#ifdef __cplusplus
}
#endif
#endif
