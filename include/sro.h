/* sro.h — C-ABI of the B200-native hot path of block-coordinate Frank-Wolfe
 * for convex semi-relaxed optimal transport (arXiv 2103.05857).
 *
 * Problem (Eq. 7):
 *     minimize_{T >= 0, T^T 1_m = b}  f(T) = <T, C> + 1/(2 lambda) ||T 1_n - a||^2
 * over the Cartesian product of scaled simplices b_1 Delta_m x ... x b_n Delta_m
 * (Eq. 8). Column i of T is the block t_i; its gradient is
 * grad_i f = c_i + h with the shared vector h = (T 1_n - a)/lambda.
 *
 * Every entry point returns an sro_status; no exception crosses the ABI.
 * sro_last_error(h) returns a human-readable message for the last failure.
 * All arrays are plain pointers with explicit sizes; no torch types.
 *
 * Precision: SRO_FP64 evaluates C (or the colour costs) in binary64.
 * SRO_FP32 stores / evaluates C in binary32 and promotes it to binary64 before
 * adding h; every reduction, line search and update is binary64 in both modes.
 * The arithmetic of every step is fixed operation by operation (DESIGN.md §3,
 * readings R1-R22), so a run is bitwise reproducible and matches the oracle.
 *
 * Threading: a handle is single-writer. Distinct handles may run concurrently
 * on distinct CUDA streams.
 */
#ifndef SRO_H
#define SRO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sro_solver* sro_handle;

typedef enum {
  SRO_OK = 0,
  SRO_NOT_CONVERGED = 1,   /* iteration budget exhausted with gap > epsilon (not an error) */
  SRO_ERR_INVALID_ARG = 2, /* bad pointer, size, option combination or layout */
  SRO_ERR_DIMENSION = 3,   /* m, n out of range */
  SRO_ERR_MARGINALS = 4,   /* a or b negative, non-finite, or not summing to 1 within 1e-12 */
  SRO_ERR_NONFINITE = 5,   /* non-finite cost / value met; state left at the last finite iterate */
  SRO_ERR_CAPACITY = 6,    /* a column support would exceed slab_cap; state left before that step */
  SRO_ERR_CUDA = 7,        /* CUDA runtime error (message in sro_last_error) */
  SRO_ERR_NCCL = 8,        /* multi-rank exchange failed */
  SRO_ERR_OOM = 9,         /* device allocation failed */
  SRO_ERR_STATE = 10       /* sro_solve called with a different variant/options/seed without sro_reset */
} sro_status;

/* Cost representation. C_{k,i} is the cost of moving source bin k (row, k < m)
 * to target bin i (column, i < n).                                           */
typedef enum {
  SRO_COST_DENSE = 0,         /* C column-major: element (k,i) at data[i*ld + k], ld >= m */
  SRO_COST_SQEUCLID = 1,      /* colours: C_ki = ((dx*dx + dy*dy) + dz*dz), d = x_k - y_i (BASELINE configs) */
  SRO_COST_EUCLID = 2,        /* colours: C_ki = sqrt(...) */
  SRO_COST_HASH_UNIFORM = 3   /* C_ki = (splitmix64(seed + (i*m + k + 1) * 0x9E3779B97F4A7C15) >> 40) * 2^-24,
                                 iid uniform on [0,1), exact in binary32; materialised on the device
                                 (BASELINE config [3]) */
} sro_cost_kind;

typedef enum { SRO_FP64 = 0, SRO_FP32 = 1 } sro_precision;

typedef struct {
  int32_t kind;         /* sro_cost_kind */
  int32_t prec;         /* sro_precision: element type of data / x / y */
  const void* data;     /* DENSE: m x n column-major, element type by prec */
  int64_t ld;           /* DENSE: leading dimension (elements), >= m */
  const void* x;        /* SQEUCLID/EUCLID: source colours, x[3k + d], d = 0..2 */
  const void* y;        /* SQEUCLID/EUCLID: target colours, y[3i + d] */
  uint64_t hash_seed;   /* HASH_UNIFORM */
  int32_t data_on_device; /* 0: host pointers, copied at sro_create.
                             1: device pointers, BORROWED (must outlive the handle, and their
                             contents must be complete before sro_create: it validates them
                             on the handle's stream, which does not wait on other streams);
                             DENSE requires 16-byte aligned data and ld*elem % 16 == 0 */
} sro_cost;

/* Host all-gather for sharded handles whose ranks exchange through host memory instead of
 * NCCL (sro_params.exchange): buf is host memory holding nranks slots of `count` doubles, slot
 * `rank` written by this process; on return every slot must hold the value its rank wrote
 * (an in-place all-gather, e.g. over a gloo process group). Return 0 on success. The library
 * synchronises the solver stream before the call and copies the buffer back to the device
 * after it, so every exchange is a host round trip (for hosts or tests without NCCL peers;
 * NCCL stays the exchange of a real multi-GPU run). */
typedef int32_t (*sro_exchange_fn)(void* user, double* buf, int64_t count, int32_t nranks, int32_t rank);

typedef struct {
  int32_t m, n;         /* rows (source bins), columns (target bins), each >= 1 */
  double lambda;        /* relaxation parameter (Eq. 7), finite and > 0 */
  int32_t slab_cap;     /* per-column support capacity (<= 31; 0 -> default 31) */
  int32_t device;       /* CUDA device ordinal */
  void* cuda_stream;    /* cudaStream_t to run on (NULL -> a stream owned by the handle) */
  /* Column sharding. The LMO sweeps, full FW (Alg. A.1) and
   * batched steps are independent per column except for the per-row sums
   * r = T 1_n, Delta = sum_i (s_i - t_i) and the scalar sums of the line search
   * (P:1786-1795), so the columns split over G shards; every shard keeps a
   * replica of r and h and the per-row / scalar sums are exchanged as
   * subtrees of the fixed 256-chunk tree (R19): the trajectory is bitwise the
   * unsharded one for every G. The sequential BCFW family (Alg. 1, A.2-A.4)
   * does not shard (each step reads the r of the previous one). */
  int32_t shards;       /* G: number of column shards, a power of two <= 64 (0 or 1: unsharded) */
  int32_t shard_block;  /* B_o: shard s holds, in every group of B_o consecutive columns, the
                           s-th contiguous B_o/G of them. 0 -> n (contiguous column slices, FW).
                           Batched steps need block_size == B_o, FW needs B_o == n. n % B_o == 0,
                           B_o % G == 0. */
  int32_t nranks;       /* processes sharing the G shards: 1 = this process holds all G shards and
                           runs them in sequence on its stream (exchanges are in-place device
                           writes), or G = one shard per process exchanged with NCCL all-gathers
                           on cuda_stream (libnccl.so.2 loaded at run time: the one already in the process, else
                           $SRO_NCCL_LIB, else the loader's default) or with the host
                           all-gather `exchange` */
  int32_t rank;         /* this process's shard when nranks == G */
  const void* nccl_id;  /* 128-byte ncclUniqueId (sro_nccl_unique_id on rank 0, shared by the
                           caller), required when nranks > 1 */
  int32_t max_sms;      /* SM budget of this handle's device-wide kernels (gap / LMO sweeps, block
                           steps, plan kernels): their grids are sized for min(max_sms, SM count)
                           SMs instead of every SM (0: every SM). For several handles sharing one
                           GPU concurrently: it bounds how much of the L2 / HBM bandwidth one
                           handle's sweeps take from the others' latency-bound steps. Results
                           do not depend on it (fixed reduction orders). */
  sro_exchange_fn exchange; /* nranks > 1: NULL -> NCCL all-gathers (nccl_id required); else this
                               host all-gather replaces them (nccl_id ignored, no communicator) */
  void* exchange_user;      /* passed to exchange */
} sro_params;

typedef enum { SRO_FW = 0, SRO_BCFW = 1, SRO_BCAFW = 2, SRO_BCPFW = 3, SRO_BATCHED = 4 } sro_variant;
typedef enum { SRO_STEP_DEC = 0, SRO_STEP_ELS = 1 } sro_step;
typedef enum { SRO_SAMPLE_U = 0, SRO_SAMPLE_P = 1, SRO_SAMPLE_GA = 2 } sro_sampling;

/* One per-step record (optional; tests compare it with the oracle's trace). */
typedef struct {
  int64_t k;            /* step counter before the step */
  int32_t i;            /* column (first column of U for block steps) */
  int32_t j;            /* LMO argmin row of column i (Eq. 9) */
  int32_t v;            /* away / pairwise atom row (Eq. 13), -1 if none */
  int32_t dir;          /* 0 FW direction, 1 away, 2 pairwise, 3 no-op */
  double gamma, num, den, minval;
} sro_trace_rec;

typedef struct {
  int32_t step;           /* sro_step */
  int32_t sampling;       /* sro_sampling (BCFW family and batched; ignored by FW) */
  double epsilon;         /* stop at the first gap check with g <= epsilon */
  int32_t gap_period;     /* epochs between gap checks (>= 1) */
  int32_t ga_M;           /* GA: global refresh of all column gaps every M*n' steps (>= 1; n' = n,
                             batched: n / block_size block steps) */
  int32_t ga_inner;       /* GA: 1 = refresh the visited column's gap each step (GAD), 0 = GAS;
                             batched GA (R31; sharded too): the block of a drawn column,
                             all its columns' gaps refreshed after the step */
  int32_t ga_post_update; /* GA: 1 = store g_i(T^{k+1}), 0 = g_i(T^k) */
  int32_t block_size;     /* BATCHED: columns per block B (B divides n) */
  const int32_t* visit;   /* optional host array of explicit visits (columns, or block indices for
                             BATCHED), length >= iters; NULL -> the sampling rule */
  sro_trace_rec* trace;   /* optional host array receiving one record per step, length >= iters
                             (sharded with nranks > 1: written on the rank holding shard 0, which
                             holds the first column of every U; other ranks' records stay zero) */
} sro_options;

typedef struct {
  int64_t iters_done;     /* steps performed by this call */
  int64_t k;              /* global step counter after the call */
  double gap;             /* last evaluated duality gap g(T) (NaN if none) */
  double objective;       /* f(T) at the end of the call */
  int32_t converged;      /* 1 if a gap check met epsilon */
  int32_t gap_checks;     /* gap evaluations in this call */
  int64_t entries_scanned;/* cost entries evaluated by the method's LMO calls in this call (steps, gap
                             sweeps, GA refreshes — counted as the paper's algorithm calls them) */
  double device_ms;       /* device time of the call (CUDA events on the solver stream) */
  int64_t entries_read;   /* cost entries the kernels actually read: a GAD post-update refresh reuses
                             the step's column, and a GA global refresh due with a gap check is one
                             sweep for both (<= entries_scanned) */
} sro_result;

/* Kernel accounting of a handle (for benchmarks): launches of this library's
 * kernels and, when timing is on, device milliseconds per kernel family,
 * measured with CUDA events on the solver stream around each launch. */
typedef struct {
  int64_t kernel_launches;  /* every kernel this handle launched */
  int64_t bcfw_launches;    /* persistent sequential-BCFW kernel (k_bcfw) */
  int64_t bcfw_steps;
  double bcfw_ms;
  int64_t sweep_launches;   /* LMO sweeps (gap checks, GA refresh, FW / batched LMO) */
  int64_t sweep_columns;
  double sweep_ms;
  int64_t block_steps;      /* FW / batched plain steps (all their kernels) */
  double block_ms;
} sro_stats;

/* Create a solver. a: host fp64[m] (source marginal), b: host fp64[n] (target
 * marginal, all n columns even when sharded), copied. Both >= 0 and summing to 1 within
 * 1e-12; a zero-mass column (b_i = 0, Eq. 8 allows it) stays the zero vector, and a BCFW-family
 * step on it is a no-op (R32). cost as described above;
 * for a sharded handle it covers the columns this process holds ("held
 * columns", ascending global index: all n when nranks == 1, the shard's n/G
 * when nranks == G): DENSE data is m x n_held column-major, colour y is
 * n_held x 3 (x always m x 3), HASH_UNIFORM is generated for the held columns.
 * Borrowed device DENSE / colour data with nranks == 1 and G > 1 needs
 * shard_block == n. T starts at the first-row vertex T^(0) = (b_1 e_1, ...,
 * b_n e_1). With nranks > 1 every rank calls
 * sro_create collectively (NCCL communicator set-up).
 * Errors: INVALID_ARG, DIMENSION, MARGINALS, NONFINITE, OOM, CUDA, NCCL. */
sro_status sro_create(const double* a, const double* b, const sro_cost* cost, const sro_params* params,
                      sro_handle* out);

/* Run `iters` steps of `variant` (Alg. 1 / A.1-A.4, PAPER.md P:189-227,
 * P:1765-1869; BATCHED is the super-block FW step of DESIGN.md R18),
 * continuing from the handle's state. Gap checks at epoch boundaries
 * and, for FW, every iteration. seed selects the sampling
 * stream. Returns OK (converged), NOT_CONVERGED (budget spent) or an error.
 * Two calls with iters a and b equal one call with a + b. Sharded handles
 * run FW and BATCHED only (INVALID_ARG otherwise); with nranks > 1 every rank
 * calls sro_solve collectively with identical arguments; entries_scanned
 * counts the held columns. */
sro_status sro_solve(sro_handle h, int32_t variant, const sro_options* opts, int64_t iters, uint64_t seed,
                     sro_result* out);

/* Duality gap g(T) (Thm 2) as sum_i g_i (Eq. 11).
 * per_column: host fp64[n_held] or NULL; argmin_rows: host int32[n_held] or NULL
 * (held columns in ascending global order; n_held = n when unsharded).
 * Sharded handles with nranks > 1: collective. */
sro_status sro_gap(sro_handle h, double* total, double* per_column, int32_t* argmin_rows);

/* Objective f(T) (Eq. 7). Sharded handles with nranks > 1: collective. */
sro_status sro_objective(sro_handle h, double* f);

/* Plan export of the held columns. dense_colmajor: host fp64[m*n_held] (held
 * columns in ascending global order) or NULL. COO triplets (rows, GLOBAL column
 * indices, vals; host, capacity cap) may be NULL; *nnz receives the number of
 * nonzeros (COO is written column by column, rows ascending). */
sro_status sro_get_plan(sro_handle h, double* dense_colmajor, int32_t* rows, int32_t* cols, double* vals,
                        int64_t cap, int64_t* nnz);

/* Row sums r = T 1_n as maintained by the solver (host fp64[m]). */
sro_status sro_get_rowsums(sro_handle h, double* r);

/* Back to T^(0), k = 0; clears the variant/options/seed lock. */
sro_status sro_reset(sro_handle h);

/* Barycentric projection (Eq. 15) of the source colours
 * through the current plan: xhat_k = (sum_i T_ki y_i) / (sum_i T_ki), both sums
 * over the n columns as the 256-chunk pairwise sums of DESIGN.md R19; a row
 * without mass keeps x_k. x: host fp64 m x 3 (source colours),
 * y: host fp64 n x 3 (target colours), xhat: host fp64 m x 3 (output).
 * Unsharded handles only (INVALID_ARG otherwise). Errors: INVALID_ARG, CUDA, OOM. */
sro_status sro_barycentric(sro_handle h, const double* x, const double* y, double* xhat);

/* Evaluation metrics of P:415-421 on the current plan: *e_c = ||T 1_n - a||_2 +
 * ||T^T 1_m - b||_2 (metric iii; row sums as in sro_barycentric, column sums over
 * each support rows ascending, each norm the square root of a 256-chunk sum of
 * squares), *sparsity = ratio of zero entries of T (metric iv), *lin = <T, C>
 * (the plan's value in metric vi). Unsharded handles only. */
sro_status sro_metrics(sro_handle h, double* e_c, double* sparsity, double* lin);

/* Metrics (v) and (vi) of P:419-421 against a reference plan T* (the paper's T*_LP, the
 * solution of the unregularised, unrelaxed OT linear program, supplied by the caller):
 * *e_m = ||T - T*||_F / ||T*||_F and *e_v = |<T, C> - <T*, C>| / |<T*, C>|. Each squared norm
 * and <T*, C> is a 256-chunk pairwise sum over the n columns (R19) of per-column sums over the
 * rows ascending; <T, C> as in sro_metrics; each norm the correctly rounded square root.
 * T*: host COO (rows, cols, vals; nnz entries) sorted by column, then strictly by row, within
 * [0, m) x [0, n), finite values (copied). Unsharded handles only. A zero ||T*|| or <T*, C>
 * gives inf / NaN as the division does. Errors: INVALID_ARG (unsorted, out of range, non-finite),
 * OOM, CUDA. */
sro_status sro_lp_metrics(sro_handle h, const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz,
                          double* e_m, double* e_v);

/* Global indices (ascending) of the columns this handle holds: cols host
 * int32[n_held] or NULL; *n_held receives the count (n when unsharded). */
sro_status sro_held_columns(sro_handle h, int32_t* cols, int32_t* n_held);

/* A fresh NCCL unique id (128 bytes) for sro_params.nccl_id, to be created on
 * rank 0 and shared with the other ranks by the caller. Errors: NCCL. */
sro_status sro_nccl_unique_id(uint8_t* out128);

/* Colour-transfer front end: k-means
 * quantisation of an 8-bit RGB image. pixels: npix x 3 uint8 (row-major RGB;
 * host memory copied in, or device memory borrowed when pixels_on_device != 0);
 * init_idx: host int32[k], k distinct pixel indices (the initial centres, drawn
 * by the caller); Lloyd iterations with squared-Euclidean fp64 distances and the
 * lowest class index on ties, centroids = exact integer channel sums / count,
 * stop when an assignment repeats the previous one and no class was repaired; an
 * empty class takes the pixel farthest from its own centroid (lowest index on
 * ties; never emptying another class), empty classes in ascending order
 * (R28-R30). Outputs (host): centroids fp64 k x 3 in 0..255 units,
 * labels int32[npix] (or NULL), counts int64[k], *iters (assignment passes run),
 * *converged. cuda_stream: the stream to run on (NULL: the default stream).
 * Errors: INVALID_ARG (sizes, k > npix, init indices), DIMENSION (k > 8192),
 * CUDA; sro_kmeans_error() describes the last failure of this thread. */
sro_status sro_kmeans(const uint8_t* pixels, int64_t npix, int32_t k, const int32_t* init_idx, int32_t max_iters,
                      int32_t pixels_on_device, void* cuda_stream, double* centroids, int32_t* labels,
                      int64_t* counts, int32_t* iters, int32_t* converged);

/* k-means++ seeding of sro_kmeans' init_idx (R34): k distinct pixel
 * indices, centre 0 = min(floor(u[0] npix), npix - 1), centre t the first pixel whose inclusive
 * prefix sum (pixel order) of D2 exceeds min(floor(u[t] * total), total - 1), where D2(p) is the
 * squared RGB distance from pixel p to its nearest chosen centre (exact integers) and total their
 * sum; total = 0 (every pixel repeats a chosen colour) takes the lowest index not yet chosen.
 * pixels: uint8 npix x 3 (host, or device when pixels_on_device; borrowed for the call); u: host
 * fp64[k], each in [0, 1) (the caller's random draw); init_idx: host int32[k] output. Runs on
 * cuda_stream (NULL: the default stream) and returns after it has synchronised. Errors:
 * INVALID_ARG (null pointers, k < 1 or > npix, u outside [0, 1)), DIMENSION (npix > 2^31 - 1),
 * CUDA. */
sro_status sro_kmeanspp(const uint8_t* pixels, int64_t npix, int32_t k, const double* u, int32_t pixels_on_device,
                        void* cuda_stream, int32_t* init_idx);

/* Recolouring: out_pixels[p] = clip(rint(255 * xhat[labels[p]]), 0, 255)
 * per channel. labels: host int32[npix] in [0, k); xhat: host fp64 k x 3 (e.g.
 * sro_barycentric's output); out_pixels: host uint8 npix x 3. Errors:
 * INVALID_ARG, CUDA. */
sro_status sro_recolour(const int32_t* labels, int64_t npix, const double* xhat, int32_t k, void* cuda_stream,
                        uint8_t* out_pixels);

/* The colour-transfer features of a quantisation (R29): colours x_c =
 * centroid_c / 255 (k x 3, in [0, 1]^3) and the histogram a_c = count_c / N, N = sum of the
 * counts (k). centroids: host fp64 k x 3 (sro_kmeans output); counts: host int64[k] (>= 0,
 * not all zero); colours, weights: host outputs. Errors: INVALID_ARG. */
sro_status sro_kmeans_features(const double* centroids, const int64_t* counts, int32_t k, double* colours,
                               double* weights);

/* Text of the last sro_kmeans / sro_recolour / sro_kmeans_features failure on this thread ("" if none). */
const char* sro_kmeans_error(void);

/* Copy the accounting into *out; reset it to zero if reset != 0. */
sro_status sro_get_stats(sro_handle h, sro_stats* out, int32_t reset);

/* Enable (1) / disable (0) per-kernel CUDA-event timing (adds no host syncs). */
sro_status sro_set_timing(sro_handle h, int32_t on);

void sro_destroy(sro_handle h);
const char* sro_last_error(sro_handle h);
const char* sro_version(void);

#ifdef __cplusplus
}
#endif
#endif
