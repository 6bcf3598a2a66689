// k_block.cuh — the plain step over a contiguous column set U = [col0, col0+L)
// (R18): FW (Alg. A.1) is
// U = [n], batched BCFW is a B-column block. After the LMO sweep over U
// (k_sweep.cuh) the step needs two per-row sums over the block's columns:
//   Delta_k  = sum_{i in U} (s_ik - t_ik)     (direction, for the Eq. A.1 denominator)
//   Delta'_k = sum_{i in U} (t'_ik - t_ik)    (row-sum update r += Delta')
// Both are segment-reduced, never atomically scattered: the (row, column)
// pairs of the merged supports are grouped by row with a counting sort whose
// within-row order is restored by rank (ascending column position), then one
// thread per touched row sums its segment in column order inside each of 8
// column chunks and combines the chunks with the fixed adjacent-pair tree
// (R19 rowsum8). The result is deterministic and identical to the oracle.
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
  // pair workspace
  int* pcount;           // L
  int* poff;             // L+1
  int* ptotal;           // 1
  int* prow;
  int* ppos;
  double* pd;
  double* pt;
  double* pdelta;
  int* rowcnt;           // m
  int* rowstart;         // m
  int* cursor;           // m
  int* tmp;
  int* sorted;
  double* X;             // m (Delta^2 dense)
  double* scal;          // [0]=G [1]=den [2]=gamma [3]=num
  const int* stop;
  int* status;
};

__device__ __forceinline__ int block_col0(const BlockArgs& A) { return A.col0_dev ? (*A.col0_dev) * A.col0_mul : 0; }

// merged support supp(t_i) U {j} in ascending rows: entry e -> (row, told)
__device__ __forceinline__ int merged_count(const BlockArgs& A, int i, int j) {
  const int c0 = A.cnt[i];
  bool in = false;
  for (int e = 0; e < c0; e++) in |= (A.srow[(int64_t)i * A.cap + e] == j);
  return c0 + (in ? 0 : 1);
}
// Iterate merged entries in order, calling f(e, row, told).
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

__global__ void k_pairs_count(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int col0 = block_col0(A);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < A.L; p += gridDim.x * blockDim.x)
    A.pcount[p] = merged_count(A, col0 + p, A.j[p]);
}

// Exclusive scan of x[0..N) into y[0..N], y[N] = total; optional copy to y2.
// One CTA of 1024 threads (integers: order-free).
__global__ void __launch_bounds__(1024) k_scan_excl(const int* __restrict__ x, int N, int* y, int* y2, int* total,
                                                    const int* stop, const int* status) {
  if ((stop && *stop) || (status && *status)) return;
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
}

// pairs of every merged support: row, position p in U, d = s - t, told
__global__ void k_pairs_gen(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int col0 = block_col0(A);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < A.L; p += gridDim.x * blockDim.x) {
    const int i = col0 + p, j = A.j[p];
    const double bi = A.b[i];
    const int base = A.poff[p];
    for_merged(A, i, j, [&](int e, int row, double told) {
      const int q = base + e;
      A.prow[q] = row;
      A.ppos[q] = p;
      A.pd[q] = d_sub(row == j ? bi : 0.0, told);
      A.pt[q] = told;
      atomicAdd(&A.rowcnt[row], 1);   // integer count: order-free
    });
  }
}

__global__ void k_place(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int P = *A.ptotal;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P; q += gridDim.x * blockDim.x) {
    const int slot = atomicAdd(&A.cursor[A.prow[q]], 1);
    A.tmp[slot] = q;
  }
}

// Restore ascending column order inside each row segment: rank by counting.
__global__ void k_rank(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int P = *A.ptotal;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P; s += gridDim.x * blockDim.x) {
    const int q = A.tmp[s];
    const int row = A.prow[q];
    const int lo = A.rowstart[row], c = A.rowcnt[row];
    int rank = 0;
    for (int t = lo; t < lo + c; t++) rank += (A.tmp[t] < q);
    A.sorted[lo + rank] = q;
  }
}

// rowsum8 (R19) of a per-pair value over U for one row segment.
__device__ __forceinline__ double rowsum8(const BlockArgs& A, const double* __restrict__ val, int lo, int c) {
  double acc[8];
#pragma unroll
  for (int t = 0; t < 8; t++) acc[t] = 0.0;
  for (int s = lo; s < lo + c; s++) {
    const int q = A.sorted[s];
    const int ch = chunk_index(A.ppos[q], A.L, 8);
    acc[ch] = d_add(acc[ch], val[q]);
  }
  return tree8(acc);
}

// Delta_k^2 for every row (0 for rows no column of U touches).
__global__ void k_rowsum_dir(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < A.m; k += gridDim.x * blockDim.x) {
    const int c = A.rowcnt[k];
    double x = 0.0;
    if (c > 0) { double D = rowsum8(A, A.pd, A.rowstart[k], c); x = d_mul(D, D); }
    A.X[k] = x;
  }
}

// Step size: ELS (Eq. 10 / Eq. A.1 / joint block search) or DEC 2n'/(k'+2n').
__global__ void k_gamma(BlockArgs A, int step_rule, long long kk, long long nprime, double* trace) {
  if ((A.stop && *A.stop) || *A.status) return;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double num = d_mul(A.lambda, A.scal[0]);
  const double den = A.scal[1];
  double gamma;
  if (step_rule == 1) {
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = d_div(num, den); if (gamma > 1.0) gamma = 1.0; }
  } else {
    gamma = d_div((double)(2LL * nprime), (double)(kk + 2LL * nprime));
  }
  A.scal[2] = gamma;
  A.scal[3] = num;
  if (trace) {
    trace[0] = (double)kk; trace[1] = block_col0(A); trace[2] = A.j[0]; trace[3] = -1; trace[4] = 0;
    trace[5] = gamma; trace[6] = num; trace[7] = den; trace[8] = A.minval[0];
  }
}

// Capacity check for every column of U before anything is mutated.
__global__ void k_cap_check(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < A.L; p += gridDim.x * blockDim.x) {
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
__global__ void k_update_cols(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < A.L; p += gridDim.x * blockDim.x) {
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

// r_k += Delta'_k, h_k = (r_k - a_k)/lambda on touched rows.
__global__ void k_rowsum_update(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < A.m; k += gridDim.x * blockDim.x) {
    const int c = A.rowcnt[k];
    if (c == 0) continue;
    const double D = rowsum8(A, A.pdelta, A.rowstart[k], c);
    const double rn = d_add(A.r[k], D);
    A.r[k] = rn;
    A.h[k] = d_div(d_sub(rn, A.a[k]), A.lambda);
  }
}

}  // namespace sro
