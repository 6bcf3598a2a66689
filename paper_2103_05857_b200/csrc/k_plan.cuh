// k_plan.cuh — what the paper computes from a transport plan after the solve
// (SURVEY §8(f) NEXT-1): the barycentric projection of Eq. 15 (PAPER.md
// P:427-432) and the metrics (iii), (iv) and <T, C> of (vi).
//
// Per-row sums over the n columns (sum_i T_ki and sum_i T_ki y_i) follow R19
// exactly as the block step's per-row sums do: the plan's nonzeros become
// (row, column position, value) pairs, every (row, 256-chunk) run is summed
// in column order and the chunk partials combine by adjacent pairs — the
// same device phases (k_block.cuh) with U = [n] and the support of T in
// place of the merged support.
#pragma once
#include "k_block.cuh"

namespace sro {

// pairs of the plan: column p's support entries (rows ascending)
__global__ void k_plan_pairs_count(BlockArgs A) {
  for (int p = gtid(); p < A.L; p += gstride()) A.pcount[p] = A.cnt[p];
}
__global__ void k_plan_pairs_gen(BlockArgs A) {
  for (int p = gtid(); p < A.L; p += gstride()) {
    const int base = A.poff[p], c = A.cnt[p];
    for (int e = 0; e < c; e++) {
      const int q = base + e, row = A.srow[(int64_t)p * A.cap + e];
      A.prow[q] = row;
      A.ppos[q] = p;
      A.pd[q] = A.sval[(int64_t)p * A.cap + e];
      if (atomicAdd(&A.rowcnt[row], 1) == 0) {
        const int w = atomicAdd(A.ntouch, 1);
        A.trows[w] = row;
        A.rowidx[row] = w;
      }
    }
  }
}
__global__ void k_plan_begin(BlockArgs A) {
  if (threadIdx.x == 0) { *A.ntouch = 0; A.nbig[0] = 0; A.nbig[1] = 0; }
}
// channel values: t (d < 0) or fl(t * y_{i,d})
__global__ void k_plan_channel(BlockArgs A, const double* __restrict__ y, int d, double* out) {
  const int P = *A.ptotal;
  for (int q = gtid(); q < P; q += gstride())
    out[q] = d < 0 ? A.pd[q] : d_mul(A.pd[q], y[3 * (int64_t)A.ppos[q] + d]);
}
// xhat_k = num_k / den_k, or x_k for a row without mass
__global__ void k_plan_project(int m, const double* __restrict__ den, const double* __restrict__ num0,
                               const double* __restrict__ num1, const double* __restrict__ num2,
                               const double* __restrict__ x, double* xhat) {
  for (int k = gtid(); k < m; k += gstride()) {
    const double dk = den[k];
    if (dk == 0.0) {
      xhat[3 * (int64_t)k] = x[3 * (int64_t)k];
      xhat[3 * (int64_t)k + 1] = x[3 * (int64_t)k + 1];
      xhat[3 * (int64_t)k + 2] = x[3 * (int64_t)k + 2];
    } else {
      xhat[3 * (int64_t)k] = d_div(num0[k], dk);
      xhat[3 * (int64_t)k + 1] = d_div(num1[k], dk);
      xhat[3 * (int64_t)k + 2] = d_div(num2[k], dk);
    }
  }
}
// (r_k - a_k)^2 over rows, (sum of column i's support, rows ascending - b_i)^2 over columns
__global__ void k_plan_sq_rows(int m, const double* __restrict__ rs, const double* __restrict__ a, double* out) {
  for (int k = gtid(); k < m; k += gstride()) {
    const double d = d_sub(rs[k], a[k]);
    out[k] = d_mul(d, d);
  }
}
__global__ void k_plan_sq_cols(int n, int cap, const int* __restrict__ cnt, const double* __restrict__ sval,
                               const double* __restrict__ b, double* out) {
  for (int i = gtid(); i < n; i += gstride()) {
    double c = 0.0;
    for (int e = 0; e < cnt[i]; e++) c = d_add(c, sval[(int64_t)i * cap + e]);
    const double d = d_sub(c, b[i]);
    out[i] = d_mul(d, d);
  }
}

}  // namespace sro
