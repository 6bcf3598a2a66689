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

// Metrics (v) and (vi) against a reference plan T* (P:419-421), one thread per column i: the
// plan's support and T*'s column (both rows ascending) merged, and over the rows ascending
// dd_i = sum_k (T_ki - T*_ki)^2, ss_i = sum_k T*_ki^2, cc_i = sum_k T*_ki C_ki (a row in
// neither support adds an exact +0, so this is the sum over all m rows).
template <class Src>
__global__ void k_lp_cols(Src src, int n, int cap, const int* __restrict__ cnt, const int* __restrict__ srow,
                          const double* __restrict__ sval, const int64_t* __restrict__ colptr,
                          const int* __restrict__ lrow, const double* __restrict__ lval, double* dd, double* ss,
                          double* cc) {
  for (int i = gtid(); i < n; i += gstride()) {
    const int c = cnt[i];
    int e = 0;
    int64_t q = colptr[i];
    const int64_t qe = colptr[i + 1];
    double sd = 0.0, s2 = 0.0, sc = 0.0;
    while (e < c || q < qe) {
      const int re = e < c ? srow[(int64_t)i * cap + e] : 0x7fffffff;
      const int rq = q < qe ? lrow[q] : 0x7fffffff;
      const int k = re < rq ? re : rq;
      const double t = re == k ? sval[(int64_t)i * cap + e] : 0.0;
      const double ts = rq == k ? lval[q] : 0.0;
      const double d = d_sub(t, ts);
      sd = d_add(sd, d_mul(d, d));
      if (rq == k) {
        s2 = d_add(s2, d_mul(ts, ts));
        sc = d_add(sc, d_mul(ts, src.cost(k, i)));
      }
      if (re == k) e++;
      if (rq == k) q++;
    }
    dd[i] = sd;
    ss[i] = s2;
    cc[i] = sc;
  }
}

}  // namespace sro
