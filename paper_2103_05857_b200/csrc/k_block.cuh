// k_block.cuh — the plain step over a contiguous column set U = [col0, col0+L)
// (R18): FW (Alg. A.1) is
// U = [n], batched BCFW is a B-column block. After the LMO sweep over U
// (k_sweep.cuh) the step needs two per-row sums over the block's columns:
//   Delta_k  = sum_{i in U} (s_ik - t_ik)     (direction, for the Eq. A.1 denominator)
//   Delta'_k = sum_{i in U} (t'_ik - t_ik)    (row-sum update r += Delta')
// Both are segment-reduced, never atomically scattered: the (row, column)
// pairs of the merged supports are grouped by row with a counting sort whose
// within-row order is restored by rank (ascending column position); each
// (row, 256-chunk) run is summed left to right by one thread and a warp per
// row combines the chunk partials with the adjacent-pair tree (R19). The
// result is deterministic and identical to the oracle.
//
// Every phase is a __device__ function over grid-stride loops, so the same
// code runs either as one kernel per phase (large U, many CTAs) or inside the
// single-CTA k_block_tail (small U: one launch for the whole post-LMO step).
#pragma once
#include "sro_device.cuh"

namespace sro {

struct BlockArgs {
  int m, n, cap;
  double lambda;
  const double* a;
  const double* b;
  double* r;
  double* h;
  int* cnt;
  int* srow;
  double* sval;
  const int* col0_dev;   // block index pointer (batched) or nullptr
  int col0_mul;          // B
  int L;
  // LMO outputs over U
  const int* j;
  const double* minval;
  const double* g;       // column gaps over U
  // pair workspace
  int* pcount;           // L
  int* poff;             // L+1
  int* ptotal;           // 1
  int* prow;
  int* ppos;             // the pair's column chunk (R19)
  double* pd;
  double* gsum;          // per-slot run partials
  double* pdelta;
  int* rowcnt;           // m
  int* rowstart;         // m+1
  int* cursor;           // m+1
  int* tmp;              // slot -> pair (unordered), then run-start flags
  int* sorted;
  double* X;             // m (Delta^2 dense)
  int* trows;            // touched rows (unordered; every row's work is independent)
  int* ntouch;           // number of touched rows
  double* scal;          // [0]=G [1]=den [2]=gamma [3]=num
  const double* eps;     // FW stop check (nullptr for batched)
  int* stop;             // FW stop flag (nullptr for batched)
  int* status;
  // step parameters
  int step_rule;
  long long kk, nprime;
  double* trace;
  unsigned long long* dsteps;   // completed steps (device counter; host reads at sync points)
};

__device__ __forceinline__ bool blk_skip(const BlockArgs& A) { return (A.stop && *A.stop) || *A.status; }
__device__ __forceinline__ int block_col0(const BlockArgs& A) { return A.col0_dev ? (*A.col0_dev) * A.col0_mul : 0; }
__device__ __forceinline__ int gtid() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int gstride() { return gridDim.x * blockDim.x; }

// merged support supp(t_i) U {j} in ascending rows: entry e -> (row, told)
__device__ __forceinline__ int merged_count(const BlockArgs& A, int i, int j) {
  const int c0 = A.cnt[i];
  bool in = false;
  for (int e = 0; e < c0; e++) in |= (A.srow[(int64_t)i * A.cap + e] == j);
  return c0 + (in ? 0 : 1);
}
template <class F>
__device__ __forceinline__ void for_merged(const BlockArgs& A, int i, int j, F f) {
  const int c0 = A.cnt[i];
  const int* rw = A.srow + (int64_t)i * A.cap;
  const double* vl = A.sval + (int64_t)i * A.cap;
  int e = 0, p = 0;
  bool inserted = false;
  while (p < c0 || !inserted) {
    if (!inserted && (p >= c0 || j < rw[p])) { f(e++, j, 0.0); inserted = true; }
    else { if (rw[p] == j) inserted = true; f(e++, rw[p], vl[p]); p++; }
  }
}

// ---------------------------------------------------------------------------
// Phases
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dev_zero_int(int* x, int N) {
  for (int q = gtid(); q < N; q += gstride()) x[q] = 0;
}
__device__ __forceinline__ void dev_zero_dbl(double* x, int N) {
  for (int q = gtid(); q < N; q += gstride()) x[q] = 0.0;
}

__device__ __forceinline__ void dev_pairs_count(const BlockArgs& A) {
  const int col0 = block_col0(A);
  for (int p = gtid(); p < A.L; p += gstride()) A.pcount[p] = merged_count(A, col0 + p, A.j[p]);
}

// Exclusive scan of x[0..N) into y[0..N], y[N] = total (integers: order-free).
// One CTA of exactly 1024 threads.
__device__ __forceinline__ void dev_scan_excl(const int* __restrict__ x, int N, int* y, int* y2, int* total) {
  __shared__ int ws[32];
  const int t = threadIdx.x;
  const int per = (N + 1023) / 1024;
  const int lo = min(N, t * per), hi = min(N, lo + per);
  int s = 0;
  for (int q = lo; q < hi; q++) s += x[q];
  int incl = s;
  for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(FULL, incl, o); if ((t & 31) >= o) incl += v; }
  if ((t & 31) == 31) ws[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    int w = ws[t];
    for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(FULL, w, o); if (t >= o) w += v; }
    ws[t] = w;
  }
  __syncthreads();
  int run = incl - s + ((t >> 5) ? ws[(t >> 5) - 1] : 0);
  for (int q = lo; q < hi; q++) { y[q] = run; if (y2) y2[q] = run; run += x[q]; }
  if (t == 1023) { y[N] = run; if (total) *total = run; }
  __syncthreads();
}

// pairs of every merged support: row, column chunk of position p in U, d = s - t
__device__ __forceinline__ void dev_pairs_gen(const BlockArgs& A) {
  const int col0 = block_col0(A);
  for (int p = gtid(); p < A.L; p += gstride()) {
    const int i = col0 + p, j = A.j[p];
    const double bi = A.b[i];
    const int base = A.poff[p];
    const int ch = chunk_index(p, A.L, 256);
    for_merged(A, i, j, [&](int e, int row, double told) {
      const int q = base + e;
      A.prow[q] = row;
      A.ppos[q] = ch;
      A.pd[q] = d_sub(row == j ? bi : 0.0, told);
      if (atomicAdd(&A.rowcnt[row], 1) == 0) A.trows[atomicAdd(A.ntouch, 1)] = row;   // order-free
    });
  }
}

__device__ __forceinline__ void dev_place(const BlockArgs& A) {
  const int P = *A.ptotal;
  for (int q = gtid(); q < P; q += gstride()) {
    const int slot = atomicAdd(&A.cursor[A.prow[q]], 1);
    A.tmp[slot] = q;
  }
}

// Restore ascending pair order (= ascending column position) inside each row segment.
__device__ __forceinline__ void dev_rank(const BlockArgs& A) {
  const int P = *A.ptotal;
  for (int s = gtid(); s < P; s += gstride()) {
    const int q = A.tmp[s];
    const int row = A.prow[q];
    const int lo = A.rowstart[row], c = A.rowcnt[row];
    int rank = 0;
    for (int t = lo; t < lo + c; t++) rank += (A.tmp[t] < q);
    A.sorted[lo + rank] = q;
  }
}

// gsum[s] = left-to-right sum of the run of slots starting at s with the same
// (row, chunk); tmp[s] = 1 at run starts.
__device__ __forceinline__ void dev_row_groups(const BlockArgs& A, const double* __restrict__ val) {
  const int P = *A.ptotal;
  for (int s = gtid(); s < P; s += gstride()) {
    const int q = A.sorted[s];
    const int row = A.prow[q];
    const int lo = A.rowstart[row], hi = lo + A.rowcnt[row];
    const int c = A.ppos[q];
    const bool start = (s == lo) || (A.ppos[A.sorted[s - 1]] != c);
    A.tmp[s] = start;
    if (start) {
      double acc = 0.0;
      for (int t = s; t < hi; t++) {
        const int qt = A.sorted[t];
        if (A.ppos[qt] != c) break;
        acc = d_add(acc, val[qt]);
      }
      A.gsum[s] = acc;
    }
  }
}

// Warp per touched row: scatter the row's run partials into 256 shared slots
// (one per chunk), then the 256-leaf adjacent-pair tree. MODE 0: X[k] = D^2;
// MODE 1: r_k += D, h_k = (r_k - a_k)/lambda.
template <int MODE>
__device__ __forceinline__ void dev_row_tree(const BlockArgs& A, double* slots_all) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  double* slots = slots_all + 256 * warp;
  const int T = *A.ntouch;
  for (int w = blockIdx.x * nwarps + warp; w < T; w += gridDim.x * nwarps) {
    const int k = A.trows[w];
    const int c = A.rowcnt[k];
    const int lo = A.rowstart[k];
    for (int t = lane; t < 256; t += 32) slots[t] = 0.0;
    __syncwarp();
    for (int s = lo + lane; s < lo + c; s += 32)
      if (A.tmp[s]) slots[A.ppos[A.sorted[s]]] = A.gsum[s];
    __syncwarp();
    double x[8];
#pragma unroll
    for (int t = 0; t < 8; t++) x[t] = slots[8 * lane + t];
    const double D = warp_pair_tree(tree8(x));
    __syncwarp();
    if (lane == 0) {
      if (MODE == 0) {
        A.X[k] = d_mul(D, D);
      } else {
        const double rn = d_add(A.r[k], D);
        A.r[k] = rn;
        A.h[k] = d_div(d_sub(rn, A.a[k]), A.lambda);
      }
    }
  }
}

// psum256 (R19) of x[0..L) for a CTA of >= 256 threads (threads >= 256 idle
// but present at the barriers). Result in *out; optional FW stop check.
__device__ __forceinline__ double dev_psum256(const double* __restrict__ x, int64_t L, double* out,
                                              const double* eps, int* stop_flag) {
  __shared__ double red[8];
  const int c = threadIdx.x;
  double acc = 0.0;
  if (c < 256) {
    const int64_t lo = chunk_lo(c, L, 256), hi = chunk_lo(c + 1, L, 256);
    for (int64_t p = lo; p < hi; p++) acc = d_add(acc, x[p]);
    acc = warp_pair_tree(acc);
    if ((c & 31) == 0) red[c >> 5] = acc;
  }
  __syncthreads();
  if (c < 32) {
    double v = (c < 8) ? red[c] : 0.0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
    if (c == 0) {
      red[0] = v;
      *out = v;
      if (stop_flag && eps && v <= *eps) *stop_flag = 1;
    }
  }
  __syncthreads();
  const double v = red[0];
  __syncthreads();
  return v;
}

// Step size: ELS (Eq. 10 / Eq. A.1 / joint block search) or DEC 2n'/(k'+2n').
__device__ __forceinline__ void dev_gamma(const BlockArgs& A) {
  if (gtid() != 0) return;
  const double num = d_mul(A.lambda, A.scal[0]);
  const double den = A.scal[1];
  double gamma;
  if (A.step_rule == 1) {
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = d_div(num, den); if (gamma > 1.0) gamma = 1.0; }
  } else {
    gamma = d_div((double)(2LL * A.nprime), (double)(A.kk + 2LL * A.nprime));
  }
  A.scal[2] = gamma;
  A.scal[3] = num;
  if (A.trace) {
    double* tr = A.trace;
    tr[0] = (double)A.kk; tr[1] = block_col0(A); tr[2] = A.j[0]; tr[3] = -1; tr[4] = 0;
    tr[5] = gamma; tr[6] = num; tr[7] = den; tr[8] = A.minval[0];
  }
}

// Capacity check for every column of U before anything is mutated.
__device__ __forceinline__ void dev_cap_check(const BlockArgs& A) {
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  for (int p = gtid(); p < A.L; p += gstride()) {
    const int i = col0 + p, j = A.j[p];
    const double gb = d_mul(gamma, A.b[i]);
    int keep = 0;
    for_merged(A, i, j, [&](int, int row, double told) {
      double tn = d_mul(omg, told);
      if (row == j) tn = d_add(tn, gb);
      keep += (tn != 0.0);
    });
    if (keep > A.cap) set_status(A.status, 6);
  }
}

// t_i <- (1-gamma) t_i + gamma s_i; exact zeros dropped (R13).
__device__ __forceinline__ void dev_update_cols(const BlockArgs& A) {
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  for (int p = gtid(); p < A.L; p += gstride()) {
    const int i = col0 + p, j = A.j[p];
    const double gb = d_mul(gamma, A.b[i]);
    const int base = A.poff[p];
    int nr[32];
    double nv[32];
    int keep = 0;
    for_merged(A, i, j, [&](int e, int row, double told) {
      double tn = d_mul(omg, told);
      if (row == j) tn = d_add(tn, gb);
      A.pdelta[base + e] = d_sub(tn, told);
      if (tn != 0.0) { nr[keep] = row; nv[keep] = tn; keep++; }
    });
    for (int e = 0; e < keep; e++) {
      A.srow[(int64_t)i * A.cap + e] = nr[e];
      A.sval[(int64_t)i * A.cap + e] = nv[e];
    }
    A.cnt[i] = keep;
  }
}

// ---------------------------------------------------------------------------
// Kernels: one per phase (multi-CTA path) ...
// ---------------------------------------------------------------------------
__global__ void k_pairs_count(BlockArgs A) { if (!blk_skip(A)) dev_pairs_count(A); }
__global__ void __launch_bounds__(1024) k_scan_excl(const int* __restrict__ x, int N, int* y, int* y2, int* total,
                                                    const int* stop, const int* status) {
  if ((stop && *stop) || (status && *status)) return;
  dev_scan_excl(x, N, y, y2, total);
}
__global__ void k_pairs_gen(BlockArgs A) { if (!blk_skip(A)) dev_pairs_gen(A); }
__global__ void k_place(BlockArgs A) { if (!blk_skip(A)) dev_place(A); }
__global__ void k_rank(BlockArgs A) { if (!blk_skip(A)) dev_rank(A); }
__global__ void k_row_groups(BlockArgs A, const double* __restrict__ val) { if (!blk_skip(A)) dev_row_groups(A, val); }
template <int MODE>
__global__ void __launch_bounds__(256) k_row_tree(BlockArgs A) {
  __shared__ double sl[8 * 256];
  if (!blk_skip(A)) dev_row_tree<MODE>(A, sl);
}
__global__ void k_gamma(BlockArgs A) { if (!blk_skip(A)) dev_gamma(A); }
__global__ void k_cap_check(BlockArgs A) { if (!blk_skip(A)) dev_cap_check(A); }
__global__ void k_update_cols(BlockArgs A) { if (!blk_skip(A)) dev_update_cols(A); }

// psum256 of x[0..L) -> *out (one CTA of 256 threads). If stop_flag is given,
// sets *stop_flag = (total <= *eps) (FW stop check, Alg. A.1 line 4).
__global__ void __launch_bounds__(256) k_psum256(const double* __restrict__ x, int64_t L, double* out,
                                                 const double* __restrict__ eps, int* stop_flag,
                                                 const int* __restrict__ stop_in) {
  if (stop_in && *stop_in) return;
  dev_psum256(x, L, out, eps, stop_flag);
}

// ... and the whole post-LMO step in one CTA of 1024 threads (small U).
__global__ void __launch_bounds__(1024, 1) k_block_tail(BlockArgs A) {
  extern __shared__ double tail_slots[];   // 32 warps x 256
  if (*A.status) return;
  dev_psum256(A.g, A.L, A.scal + 0, A.eps, A.stop);        // G_U (FW: stop check)
  if (A.stop && *A.stop) return;
  dev_pairs_count(A);
  dev_zero_int(A.rowcnt, A.m);
  if (threadIdx.x == 0) *A.ntouch = 0;
  __syncthreads();
  dev_scan_excl(A.pcount, A.L, A.poff, nullptr, A.ptotal);
  dev_pairs_gen(A);
  __syncthreads();
  dev_scan_excl(A.rowcnt, A.m, A.rowstart, A.cursor, nullptr);
  dev_place(A);
  dev_zero_dbl(A.X, A.m);
  __syncthreads();
  dev_rank(A);
  __syncthreads();
  dev_row_groups(A, A.pd);
  __syncthreads();
  dev_row_tree<0>(A, tail_slots);
  __syncthreads();
  dev_psum256(A.X, A.m, A.scal + 1, nullptr, nullptr);
  dev_gamma(A);
  __syncthreads();
  dev_cap_check(A);
  __syncthreads();
  if (*A.status) return;
  dev_update_cols(A);
  __syncthreads();
  dev_row_groups(A, A.pdelta);
  __syncthreads();
  dev_row_tree<1>(A, tail_slots);
  if (threadIdx.x == 0) atomicAdd(A.dsteps, 1ULL);
}

__global__ void k_step_done(BlockArgs A) {
  if (!blk_skip(A) && threadIdx.x == 0) atomicAdd(A.dsteps, 1ULL);
}

}  // namespace sro
