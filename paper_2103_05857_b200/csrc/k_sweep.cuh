// k_sweep.cuh — the column LMO sweep (Eq. 9) fused with
// the per-column duality-gap epilogue (Eq. 11).
//
// For a contiguous column range [col0, col0 + L): j_p = argmin_k (C_{k,i} + h_k)
// (lowest k on ties), minval_p, and g_p = <t_i, c_i + h> - b_i minval_p.
//
// Layout: C column-major (each LMO is one contiguous, 128-bit vectorised,
// coalesced column read, BASELINE north_star), h staged per row slab in
// shared memory and reused by every column the CTA visits. One warp owns one
// column at a time; a CTA of 8 warps streams many columns. Rows are split in
// slabs of slab_rows rows (blockIdx.y; the host sizes slabs for occupancy);
// with more than one slab the per-slab (min, row) partials are merged in slab
// order by k_lmo_merge.
// Roofline: HBM (dense, 4 or 8 B per entry) or FP32/FP64 issue (colours).
#pragma once
#include "sro_device.cuh"

namespace sro {

constexpr int SWEEP_THREADS = 256;
constexpr int SWEEP_WARPS = SWEEP_THREADS / 32;
constexpr int SLAB_MAX = 8192;   // rows of h staged per CTA at most (the host picks the slab)

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }

// --------------------------------------------------------------------------
// Cost sources
// --------------------------------------------------------------------------
template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int W = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int W = 2; };

__device__ __forceinline__ void proc4(const float4& v, int k, const double* hs, double& best, int& bj) {
  double x0 = d_add((double)v.x, hs[k]), x1 = d_add((double)v.y, hs[k + 1]);
  double x2 = d_add((double)v.z, hs[k + 2]), x3 = d_add((double)v.w, hs[k + 3]);
  if (x0 < best) { best = x0; bj = k; }
  if (x1 < best) { best = x1; bj = k + 1; }
  if (x2 < best) { best = x2; bj = k + 2; }
  if (x3 < best) { best = x3; bj = k + 3; }
}
__device__ __forceinline__ void proc4(const double2& v, int k, const double* hs, double& best, int& bj) {
  double x0 = d_add(v.x, hs[k]), x1 = d_add(v.y, hs[k + 1]);
  if (x0 < best) { best = x0; bj = k; }
  if (x1 < best) { best = x1; bj = k + 1; }
}

// Dense column-major cost. h is staged in shared memory in W planes
// (plane t holds h[row0 + W v + t], v < rows / W; rows past the last full
// vector follow the planes), so a lane's W consecutive rows read W
// conflict-free doubles (consecutive lanes -> consecutive addresses).
template <typename T>
struct SrcDense {
  const T* C;
  int64_t ld;
  static constexpr int SMEM_PER_ROW = 0;
  static constexpr bool WIDE = false;   // 512-thread multi-column sweeps (k_lmo_sweep NT)
  static constexpr bool PLANAR = true;
  static constexpr int COLS = 1;
  template <int NCOL>
  __device__ __forceinline__ void stage(int, int, char*) const {}
  __device__ __forceinline__ double cost(int k, int i) const { return (double)C[(int64_t)i * ld + k]; }
  // per-column registers of a scan (none) and the raw operands of one cost (loaded early, used late)
  struct ColReg {};
  __device__ __forceinline__ ColReg col(int) const { return {}; }
  struct CostPre { T c; };
  __device__ __forceinline__ CostPre cost_load(int k, int i) const { return {C[(int64_t)i * ld + k]}; }
  __device__ __forceinline__ static double cost_of(const CostPre& q, const ColReg&) { return (double)q.c; }
  // Scan rows [row0, row0+rows) of column i; lane-strided 128-bit vectors,
  // rows ascending within a lane, 8 vectors in flight per lane.
  __device__ __forceinline__ void scan(int i, const ColReg&, int row0, int rows, const double* hs, const char*,
                                       double& best, int& bj) const {
    using V = typename Vec<T>::type;
    constexpr int W = Vec<T>::W;
    const int lane = threadIdx.x & 31;
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld + row0);
    const int nvec = rows / W;
    int q = lane;
    for (; q + 224 < nvec; q += 256) {
      V v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = ld_stream(p + q + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; u++) procW(v[u], q + 32 * u, nvec, hs, best, bj);
    }
    for (; q < nvec; q += 32) procW(ld_stream(p + q), q, nvec, hs, best, bj);
    const int k = nvec * W + lane;
    if (k < rows) {
      double x = d_add((double)C[(int64_t)i * ld + row0 + k], hs[k]);
      if (x < best) { best = x; bj = k; }
    }
    // bj is slab-relative here; caller adds row0
  }
  __device__ __forceinline__ static void procW(const float4& v, int q, int nvec, const double* hs, double& best,
                                               int& bj) {
    const int k = 4 * q;
    double x0 = d_add((double)v.x, hs[q]), x1 = d_add((double)v.y, hs[nvec + q]);
    double x2 = d_add((double)v.z, hs[2 * nvec + q]), x3 = d_add((double)v.w, hs[3 * nvec + q]);
    if (x0 < best) { best = x0; bj = k; }
    if (x1 < best) { best = x1; bj = k + 1; }
    if (x2 < best) { best = x2; bj = k + 2; }
    if (x3 < best) { best = x3; bj = k + 3; }
  }
  __device__ __forceinline__ static void procW(const double2& v, int q, int nvec, const double* hs, double& best,
                                               int& bj) {
    const int k = 2 * q;
    double x0 = d_add(v.x, hs[q]), x1 = d_add(v.y, hs[nvec + q]);
    if (x0 < best) { best = x0; bj = k; }
    if (x1 < best) { best = x1; bj = k + 1; }
  }
  // shared-memory index of slab row k
  __device__ __forceinline__ static int hidx(int k, int rows) {
    constexpr int W = Vec<T>::W;
    const int nvec = rows / W;
    return k < nvec * W ? (k % W) * nvec + k / W : k;
  }
};

// Packed binary32 pairs (sm_100 FADD2 / FMUL2): lane-wise IEEE round-to-nearest, the same
// result as two scalar __fsub_rn / __fmul_rn. ptxas contracts a packed multiply into a following
// packed add even under --fmad=false, so the products are only ever summed with scalar adds.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// (x - y0, x - y1) for one broadcast x (ptxas folds the pack into the .F32 operand form)
__device__ __forceinline__ unsigned long long f2_bsub(float x, unsigned long long y) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(x, x)), "l"(y));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sq(unsigned long long d) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(d));
  return r;
}

template <typename T, bool EUCLID>
struct SrcColour {
  const T* x;   // 3m
  const T* y;   // 3n
  // staged colours: binary32 multi-column sweeps one 16-byte (x0, x1, x2, 0) record per row (one
  // LDS.128 per row), everything else three planes (SMEM_PER_ROW covers both layouts)
  static constexpr bool PACKED = sizeof(T) == 4;
  static constexpr int SMEM_PER_ROW = PACKED ? 16 : 3 * sizeof(T);
  static constexpr bool WIDE = PACKED;   // 512-thread multi-column sweeps (k_lmo_sweep NT)
  static constexpr bool PLANAR = false;
#ifndef SRO_COLOUR_COLS
#define SRO_COLOUR_COLS 4
#endif
// rows per unrolled iteration of the 4-column scan. Unpacked loop, 1 / 2 / 4 / 6 / 8 rows: 1.26 /
// 1.36 / 1.46 / 1.48 / 1.48e12 entries/s at config [2]; packed loop, 2 / 4 / 8: 1.65 / 1.67 / 1.69e12,
// but 8 spills the binary64 and euclid instantiations under the 64-register cap
#ifndef SRO_COLOUR_UNROLL
#define SRO_COLOUR_UNROLL 4
#endif
  static constexpr int COLS = SRO_COLOUR_COLS;   // columns a warp evaluates per loaded row (registers hold their y)
  static constexpr int UNROLL = SRO_COLOUR_UNROLL;
  __device__ __forceinline__ static int hidx(int k, int) { return k; }
  // planes (x0 | x1 | x2) of the slab's colours; binary32 planes start at even offsets so that a
  // lane reads two consecutive rows of a coordinate as one packed pair
  __device__ __forceinline__ static int pstride(int rows) { return PACKED ? ((rows + 1) & ~1) : rows; }
  // multi-column scans of binary32 colours read one 16-byte record per row, everything else planes
  template <int NCOL>
  __device__ __forceinline__ void stage(int row0, int rows, char* sm) const {
    if constexpr (PACKED && NCOL > 1 && NCOL % 2 == 0) {
      float4* xs = reinterpret_cast<float4*>(sm);
      for (int k = threadIdx.x; k < rows; k += blockDim.x) {
        const int64_t o = 3 * (int64_t)(row0 + k);
        xs[k] = make_float4(x[o], x[o + 1], x[o + 2], 0.f);
      }
    } else {
      T* xs = reinterpret_cast<T*>(sm);
      const int ps = pstride(rows);
      for (int k = threadIdx.x; k < rows; k += blockDim.x) {
        xs[k] = x[3 * (int64_t)(row0 + k)];
        xs[ps + k] = x[3 * (int64_t)(row0 + k) + 1];
        xs[2 * ps + k] = x[3 * (int64_t)(row0 + k) + 2];
      }
    }
  }
  __device__ __forceinline__ double cost(int k, int i) const {
    return colour_cost<EUCLID>(x[3 * (int64_t)k], x[3 * (int64_t)k + 1], x[3 * (int64_t)k + 2], y[3 * (int64_t)i],
                               y[3 * (int64_t)i + 1], y[3 * (int64_t)i + 2]);
  }
  struct ColReg { T y0, y1, y2; };
  __device__ __forceinline__ ColReg col(int i) const {
    return {y[3 * (int64_t)i], y[3 * (int64_t)i + 1], y[3 * (int64_t)i + 2]};
  }
  struct CostPre { T x0, x1, x2; };
  __device__ __forceinline__ CostPre cost_load(int k, int) const {
    return {x[3 * (int64_t)k], x[3 * (int64_t)k + 1], x[3 * (int64_t)k + 2]};
  }
  __device__ __forceinline__ static double cost_of(const CostPre& q, const ColReg& c) {
    return colour_cost<EUCLID>(q.x0, q.x1, q.x2, c.y0, c.y1, c.y2);
  }
  // one column against the slab (planes), rows ascending per lane
  __device__ __forceinline__ void scan(int, const ColReg& cr, int, int rows, const double* hs, const char* sm,
                                       double& best, int& bj) const {
    const int lane = threadIdx.x & 31;
    const T* xs = reinterpret_cast<const T*>(sm);
    const int ps = pstride(rows);
    if constexpr (PACKED) {
      // lane q takes the row pairs (2q', 2q'+1), q' = q, q + 32, ...: one packed pair per coordinate
      // (the planes' pairs), the differences and squares of both rows per FADD2 / FMUL2 and the
      // sums as scalar adds in colour_cost's order
      const float2* x0 = reinterpret_cast<const float2*>(xs);
      const float2* x1 = reinterpret_cast<const float2*>(xs + ps);
      const float2* x2 = reinterpret_cast<const float2*>(xs + 2 * ps);
      const double2* h2 = reinterpret_cast<const double2*>(hs);
      const unsigned long long Y0 = f2_pack(cr.y0, cr.y0), Y1 = f2_pack(cr.y1, cr.y1), Y2 = f2_pack(cr.y2, cr.y2);
      const int np = rows >> 1;
#pragma unroll 4
      for (int q = lane; q < np; q += 32) {
        const float2 a0 = x0[q], a1 = x1[q], a2 = x2[q];
        const double2 hh = h2[q];
        const float2 sx = f2_unpack(f2_sq(f2_sub(f2_pack(a0.x, a0.y), Y0)));
        const float2 sy = f2_unpack(f2_sq(f2_sub(f2_pack(a1.x, a1.y), Y1)));
        const float2 sz = f2_unpack(f2_sq(f2_sub(f2_pack(a2.x, a2.y), Y2)));
        float d0 = __fadd_rn(__fadd_rn(sx.x, sy.x), sz.x);
        float d1 = __fadd_rn(__fadd_rn(sx.y, sy.y), sz.y);
        if constexpr (EUCLID) { d0 = __fsqrt_rn(d0); d1 = __fsqrt_rn(d1); }
        const double v0 = d_add((double)d0, hh.x), v1 = d_add((double)d1, hh.y);
        if (v0 < best) { best = v0; bj = 2 * q; }
        if (v1 < best) { best = v1; bj = 2 * q + 1; }
      }
      if ((rows & 1) && lane == 0) {   // the odd last row (the largest index: order kept)
        const int k = rows - 1;
        const double v = d_add(colour_cost<EUCLID>(xs[k], xs[ps + k], xs[2 * ps + k], cr.y0, cr.y1, cr.y2), hs[k]);
        if (v < best) { best = v; bj = k; }
      }
    } else {
#pragma unroll 4
      for (int k = lane; k < rows; k += 32) {
        const double c = colour_cost<EUCLID>(xs[k], xs[ps + k], xs[2 * ps + k], cr.y0, cr.y1, cr.y2);
        const double v = d_add(c, hs[k]);
        if (v < best) { best = v; bj = k; }
      }
    }
  }
  // columns i0 .. i0+nc-1 (nc <= COLS) against every row of the slab: one load of
  // (x_k, h_k) per row serves all of them; rows ascending per lane and column.
  template <int NC>
  __device__ __forceinline__ void scan_multi(int i0, int nc, int rows, const double* hs, const char* sm,
                                             double* best, int* bj) const {
    T yv[NC][3];
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const int i = i0 + (c < nc ? c : 0);
      yv[c][0] = y[3 * (int64_t)i]; yv[c][1] = y[3 * (int64_t)i + 1]; yv[c][2] = y[3 * (int64_t)i + 2];
    }
    const int lane = threadIdx.x & 31;
    if constexpr (PACKED && NC % 2 == 0) {
      // binary32: the three differences and squares of two columns per packed instruction
      // (exactly colour_cost's __fsub_rn / __fmul_rn), the two sums as scalar adds in its order
      unsigned long long yp[NC / 2][3];
#pragma unroll
      for (int c = 0; c < NC / 2; c++)
#pragma unroll
        for (int d = 0; d < 3; d++) yp[c][d] = f2_pack(yv[2 * c][d], yv[2 * c + 1][d]);
      // the NC values of row k (packed pairs)
      auto row_values = [&](int k, double* v) {
        const float4 xk = reinterpret_cast<const float4*>(sm)[k];
        const double hk = hs[k];
#pragma unroll
        for (int c = 0; c < NC / 2; c++) {
          const float2 sx = f2_unpack(f2_sq(f2_bsub(xk.x, yp[c][0])));
          const float2 sy = f2_unpack(f2_sq(f2_bsub(xk.y, yp[c][1])));
          const float2 sz = f2_unpack(f2_sq(f2_bsub(xk.z, yp[c][2])));
          float d0 = __fadd_rn(__fadd_rn(sx.x, sy.x), sz.x);
          float d1 = __fadd_rn(__fadd_rn(sx.y, sy.y), sz.y);
          if constexpr (EUCLID) { d0 = __fsqrt_rn(d0); d1 = __fsqrt_rn(d1); }
          v[2 * c] = d_add((double)d0, hk);
          v[2 * c + 1] = d_add((double)d1, hk);
        }
      };
      int k = lane;
#pragma unroll UNROLL
      for (; k < rows; k += 32) {
        double v[NC];
        row_values(k, v);
#pragma unroll
        for (int c = 0; c < NC; c++)
          if (v[c] < best[c]) { best[c] = v[c]; bj[c] = k; }
      }
    } else {
      const T* xs = reinterpret_cast<const T*>(sm);
      const int ps = pstride(rows);
#pragma unroll UNROLL
      for (int k = lane; k < rows; k += 32) {
        const T x0 = xs[k], x1 = xs[ps + k], x2 = xs[2 * ps + k];
        const double hk = hs[k];
#pragma unroll
        for (int c = 0; c < NC; c++) {
          const double v = d_add(colour_cost<EUCLID>(x0, x1, x2, yv[c][0], yv[c][1], yv[c][2]), hk);
          if (v < best[c]) { best[c] = v; bj[c] = k; }
        }
      }
    }
  }
};

// Per-column gap epilogue (Eq. 11): lanes hold one support entry each;
// dot = sequential sum over supp(t_i), rows ascending (R19).
template <class Src>
__device__ __forceinline__ double column_gap_epilogue(const Src& src, int i, double minval, const int* __restrict__ cnt,
                                                      const int* __restrict__ srow, const double* __restrict__ sval,
                                                      int cap, const double* __restrict__ b,
                                                      const double* __restrict__ h) {
  const int lane = threadIdx.x & 31;
  const int c = cnt[i];
  double term = 0.0;
  if (lane < c) {
    const int k = srow[(int64_t)i * cap + lane];
    const double t = sval[(int64_t)i * cap + lane];
    term = d_mul(t, d_add(src.cost(k, i), h[k]));
  }
  const double dot = warp_seq_sum(term, c);
  return d_sub(dot, d_mul(b[i], minval));
}

constexpr int SW_KP = 4;   // support entries per column staged for the block tail
struct SweepOut {
  int* j;          // [L] final rows (single slab) or partial rows [nslabs*L]
  double* minval;  // [L] or partial [nslabs*L]
  double* g;       // [L] column gaps (single slab only)
  // multi-slab block sweeps (the tail merges): slab 0's warps also stage each column's
  // support size, first SW_KP entries (entry-major [e * L + p], so the single-CTA tail reads
  // them coalesced instead of one scattered slab line per column) and b_i; nullptr: off
  int* st_cnt;
  int* st_row;
  double* st_val;
  double* st_b;
  // ... and every slab's warps the gap terms t_ki (C_ki + h_k) of the first SW_KP support
  // entries whose rows lie in their slab ([e * L + p]; the tail's dot is their sum in e order)
  double* st_term;
};
__device__ __forceinline__ void stage_support(const SweepOut& out, int p, int i, int L, const int* __restrict__ cnt,
                                              const int* __restrict__ srow, const double* __restrict__ sval, int cap,
                                              const double* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const int c = cnt[i];
  if (lane == 0) { out.st_cnt[p] = c; out.st_b[p] = b[i]; }
  if (lane < SW_KP && lane < c) {
    out.st_row[lane * L + p] = srow[(int64_t)i * cap + lane];
    out.st_val[lane * L + p] = sval[(int64_t)i * cap + lane];
  }
}

template <class Src>
__device__ __forceinline__ void stage_terms(const Src& src, const SweepOut& out, int p, int i, int L, int row0,
                                            int rows, const int* __restrict__ cnt, const int* __restrict__ srow,
                                            const double* __restrict__ sval, int cap,
                                            const double* __restrict__ h) {
  const int lane = threadIdx.x & 31;
  const int c = cnt[i];
  if (lane < SW_KP && lane < c) {
    const int k = srow[(int64_t)i * cap + lane];
    if (k >= row0 && k < row0 + rows)
      out.st_term[lane * L + p] = d_mul(sval[(int64_t)i * cap + lane], d_add(src.cost(k, i), h[k]));
  }
}

// grid = (gx, nslabs). col0 = col0_dev ? col0_dev[cur ? *cur : 0] * col0_mul : col0_host
// (cur: a device step cursor, so that the launches of consecutive block steps are identical).
// NT threads per CTA: 256, or 512 for the packed binary32 colour sweep over full slabs (two CTAs of
// 16 warps per SM hide the fp32 -> fp64 add -> compare chains better than two of 8; <= 64 registers,
// so only the packed source takes it: the binary64 euclid scan would spill)
template <class Src, int NCOL = Src::COLS, int NT = SWEEP_THREADS>
__global__ void __launch_bounds__(NT, NT > SWEEP_THREADS ? 2 : 1) k_lmo_sweep(Src src, int m, int slab_rows, const double* __restrict__ h,
                                                             const int* __restrict__ col0_dev, const unsigned* __restrict__ cur, int col0_mul,
                                                             int col0_host, int L, const int* __restrict__ cnt,
                                                             const int* __restrict__ srow,
                                                             const double* __restrict__ sval, int cap,
                                                             const double* __restrict__ b, SweepOut out,
                                                             const int* __restrict__ stop, int* status) { pdl_entry();
  // the step words and the cursor together, then the column offset (an FW stop, or a failed step
  // earlier in the call: nothing to do)
  const int stop_v = stop ? *stop : 0, status_v = *status;
  const unsigned cur_v = cur ? *cur : 0u;
  if (stop_v || status_v) return;
  const int col0 = col0_dev ? col0_dev[cur_v] * col0_mul : col0_host;
  extern __shared__ __align__(16) double sm_h[];
  const int nslabs = gridDim.y, slab = blockIdx.y;
  const int row0 = slab * slab_rows;
  const int rows = min(slab_rows, m - row0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* sm_src = reinterpret_cast<char*>(sm_h + ((rows + 1) & ~1));
  if constexpr (NCOL > 1) {
    for (int k = threadIdx.x; k < rows; k += blockDim.x) sm_h[Src::hidx(k, rows)] = h[row0 + k];
    src.template stage<NCOL>(row0, rows, sm_src);
    __syncthreads();
    constexpr int NC = NCOL;
    for (int p0 = (blockIdx.x * (NT / 32) + warp) * NC; p0 < L; p0 += gridDim.x * (NT / 32) * NC) {
      const int nc = min(NC, L - p0);
      double best[NC];
      int bj[NC];
#pragma unroll
      for (int c = 0; c < NC; c++) { best[c] = __longlong_as_double(0x7ff0000000000000LL); bj[c] = 0x7fffffff; }
      src.template scan_multi<NC>(col0 + p0, nc, rows, sm_h, sm_src, best, bj);
#pragma unroll
      for (int c = 0; c < NC; c++) {
        if (c >= nc) break;
        const int p = p0 + c, i = col0 + p;
        double bv = best[c];
        int bjc = bj[c];
        if (bjc != 0x7fffffff) bjc += row0;
        warp_argmin(bv, bjc);
        if (nslabs == 1) {
          if (!(bv < 1.0e308 && bv > -1.0e308)) { if (lane == 0) set_status(status, 5); }
          const double g = column_gap_epilogue(src, i, bv, cnt, srow, sval, cap, b, h);
          if (lane == 0) { out.j[p] = bjc; out.minval[p] = bv; out.g[p] = g; }
        } else {
          if (lane == 0) {
            out.j[(int64_t)slab * L + p] = bjc;
            out.minval[(int64_t)slab * L + p] = bv;
          }
          if (out.st_cnt && slab == 0) stage_support(out, p, i, L, cnt, srow, sval, cap, b);
          if (out.st_term) stage_terms(src, out, p, i, L, row0, rows, cnt, srow, sval, cap, h);
        }
      }
    }
  } else {
    // One column per warp per pass (block steps: one pass). A column's own data (the source's
    // per-column registers, its support size, support entries and b_i) is requested before the
    // slab is staged, and the operands of its gap terms before the scan, so that their round
    // trips overlap the staging and the scan instead of following them.
    constexpr int Wn = NT / 32;
    int p = blockIdx.x * Wn + warp;
    typename Src::ColReg cr{};
    int pc = 0, pk = 0;
    double pt = 0.0, pb = 0.0;
    auto prefetch = [&](int pp) {
      const int i = col0 + pp;
      cr = src.col(i);
      pc = cnt[i];
      pb = b[i];
      if (lane < cap) { pk = srow[(int64_t)i * cap + lane]; pt = sval[(int64_t)i * cap + lane]; }
    };
    if (p < L) prefetch(p);
    for (int k = threadIdx.x; k < rows; k += blockDim.x) sm_h[Src::hidx(k, rows)] = h[row0 + k];
    src.template stage<1>(row0, rows, sm_src);
    __syncthreads();
    for (; p < L; p += gridDim.x * Wn) {
      const int i = col0 + p;
      // this lane's gap term t_ki (C_ki + h_k): every support entry for the full epilogue, the first
      // SW_KP entries with rows in this slab for the block tail (R19 sums them in entry order)
      const bool need = lane < pc && (nslabs == 1 || (out.st_term && lane < SW_KP && pk >= row0 && pk < row0 + rows));
      typename Src::CostPre q{};
      double hk = 0.0;
      if (need) { q = src.cost_load(pk, i); hk = h[pk]; }
      double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      int bj = 0x7fffffff;
      src.scan(i, cr, row0, rows, sm_h, sm_src, best, bj);
      if (bj != 0x7fffffff) bj += row0;
      warp_argmin(best, bj);
      const double term = need ? d_mul(pt, d_add(Src::cost_of(q, cr), hk)) : 0.0;
      if (nslabs == 1) {
        if (!(best < 1.0e308 && best > -1.0e308)) { if (lane == 0) set_status(status, 5); }
        const double g = d_sub(warp_seq_sum(term, pc), d_mul(pb, best));   // Eq. 11, as column_gap_epilogue
        if (lane == 0) { out.j[p] = bj; out.minval[p] = best; out.g[p] = g; }
      } else {
        if (lane == 0) {
          out.j[(int64_t)slab * L + p] = bj;
          out.minval[(int64_t)slab * L + p] = best;
        }
        if (out.st_cnt && slab == 0) {   // as stage_support
          if (lane == 0) { out.st_cnt[p] = pc; out.st_b[p] = pb; }
          if (lane < SW_KP && lane < pc) { out.st_row[lane * L + p] = pk; out.st_val[lane * L + p] = pt; }
        }
        if (need) out.st_term[lane * L + p] = term;   // as stage_terms
      }
      if (p + gridDim.x * Wn < L) prefetch(p + gridDim.x * Wn);
    }
  }
}

// Merge per-slab partials in slab order and apply the gap epilogue. One warp per column.
template <class Src>
__global__ void __launch_bounds__(SWEEP_THREADS) k_lmo_merge(Src src, int nslabs, const double* __restrict__ h,
                                                             const int* __restrict__ col0_dev, const unsigned* __restrict__ cur, int col0_mul,
                                                             int col0_host, int L, const int* __restrict__ cnt,
                                                             const int* __restrict__ srow,
                                                             const double* __restrict__ sval, int cap,
                                                             const double* __restrict__ b, const int* __restrict__ pj,
                                                             const double* __restrict__ pmin, int* out_j,
                                                             double* out_min, double* out_g,
                                                             const int* __restrict__ stop, int* status) { pdl_entry();
  if ((stop && *stop) || *status) return;   // FW stop, or a failed step earlier in the call
  const int col0 = col0_dev ? col0_dev[cur ? *cur : 0u] * col0_mul : col0_host;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = blockIdx.x * SWEEP_WARPS + warp; p < L; p += gridDim.x * SWEEP_WARPS) {
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bj = 0x7fffffff;
    for (int s = lane; s < nslabs; s += 32) argmin_merge(best, bj, pmin[(int64_t)s * L + p], pj[(int64_t)s * L + p]);
    warp_argmin(best, bj);
    if (!(best < 1.0e308 && best > -1.0e308)) { if (lane == 0) set_status(status, 5); }
    const double g = column_gap_epilogue(src, col0 + p, best, cnt, srow, sval, cap, b, h);
    if (lane == 0) { out_j[p] = bj; out_min[p] = best; out_g[p] = g; }
  }
}

// ---------------------------------------------------------------------------
// Dense sweep with bulk asynchronous copies (TMA engine, cp.async.bulk ->
// SASS UBLKCP): every warp runs its own S-stage ring of 4 KiB shared-memory
// buffers, refilled by one lane with an mbarrier completion per stage, so
// S x 4 KiB per warp are in flight independently of the register file (the
// LDG version issues loads just in time and keeps ~1 KiB per warp in flight).
// Work = (slab, column) items, slab-major, split into one contiguous range per
// CTA of a grid sized to the SM count: a CTA restages h (planar, as
// SrcDense) only when its range enters the next slab.
// ---------------------------------------------------------------------------
// 16 warps x 4 stages x 3 KiB in flight per SM (config [3] gap sweep: 6.70 TB/s, from 5.85 with 8
// warps x 4 x 4 KiB; 12 x 4 x 4 KiB 6.49, 20 x 3 x 3 KiB 6.67, 24 x 3 x 2.5 KiB 6.52, 32 x 2 x 3 KiB
// 6.03, 16 x 6 x 2 KiB 5.72 — tools/sweep3_timing.py); the row slab drops to 4096 to fit
#ifndef SRO_BULK_WARPS
#define SRO_BULK_WARPS 16
#endif
#ifndef SRO_BULK_CH
#define SRO_BULK_CH 3072
#endif
constexpr int BULK_WARPS = SRO_BULK_WARPS;
constexpr int BULK_CH = SRO_BULK_CH;   // bytes per stage

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <typename T, int S>
__global__ void __launch_bounds__(BULK_WARPS * 32, 1)
    k_lmo_sweep_bulk(SrcDense<T> src, int m, int slab_rows, int nslabs, const double* __restrict__ h,
                     const int* __restrict__ col0_dev, const unsigned* __restrict__ cur, int col0_mul, int col0_host, int L,
                     const int* __restrict__ cnt, const int* __restrict__ srow, const double* __restrict__ sval,
                     int cap, const double* __restrict__ b, SweepOut out, const int* __restrict__ stop,
                     int* status) { pdl_entry();
  using V = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  constexpr int CHV = BULK_CH / 16;   // vectors per stage
  if ((stop && *stop) || *status) return;   // FW stop, or a failed step earlier in the call
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned char* bufs = smem + 1024;
  double* hs = reinterpret_cast<double*>(bufs + (size_t)BULK_WARPS * S * BULK_CH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < BULK_WARPS * S) mbar_init(&bars[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t* wb = bars + warp * S;
  unsigned char* wbuf = bufs + (size_t)warp * S * BULK_CH;
  const int col0 = col0_dev ? col0_dev[cur ? *cur : 0u] * col0_mul : col0_host;
  const int64_t ntot = (int64_t)nslabs * L;
  const int64_t lo = ntot * blockIdx.x / gridDim.x, hi = ntot * (blockIdx.x + 1) / gridDim.x;
  long long tcons = 0, tiss = 0;   // per-warp stage counters (uniform across the warp)
  for (int64_t seg = lo; seg < hi;) {
    const int slab = (int)(seg / L);
    const int64_t seg_end = min(hi, (int64_t)(slab + 1) * L);
    const int row0 = slab * slab_rows;
    const int rows = min(slab_rows, m - row0);
    const int nvec = rows / W;
    const int nch = (nvec + CHV - 1) / CHV;
    __syncthreads();
    for (int k = threadIdx.x; k < rows; k += blockDim.x) hs[SrcDense<T>::hidx(k, rows)] = h[row0 + k];
    __syncthreads();
    const int p_first = (int)(seg - (int64_t)slab * L) + warp;
    const int p_end = (int)(seg_end - (int64_t)slab * L);
    const int ncol = p_first < p_end ? (p_end - p_first + BULK_WARPS - 1) / BULK_WARPS : 0;
    const int64_t tot = (int64_t)ncol * nch;
    int64_t e_iss = 0;
    auto issue = [&]() {
      const int jc = (int)(e_iss / nch), c = (int)(e_iss % nch);
      const int i = col0 + p_first + jc * BULK_WARPS;
      const int v0 = c * CHV, nv = min(CHV, nvec - v0);
      const int slot = (int)(tiss % S);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const T* g = src.C + (int64_t)i * src.ld + row0 + (int64_t)v0 * W;
        mbar_expect_tx(&wb[slot], (uint32_t)nv * 16u);
        bulk_g2s(wbuf + (size_t)slot * BULK_CH, g, (uint32_t)nv * 16u, &wb[slot]);
      }
      tiss++;
      e_iss++;
    };
    while (e_iss < tot && e_iss < S) issue();
    for (int jc = 0; jc < ncol; jc++) {
      const int p = p_first + jc * BULK_WARPS;
      const int i = col0 + p;
      double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      int bj = 0x7fffffff;
      for (int c = 0; c < nch; c++) {
        const int slot = (int)(tcons % S);
        const uint32_t parity = (uint32_t)((tcons / S) & 1);
        while (!mbar_try_wait(&wb[slot], parity)) {
        }
        const V* vb = reinterpret_cast<const V*>(wbuf + (size_t)slot * BULK_CH);
        const int v0 = c * CHV, nv = min(CHV, nvec - v0);
#pragma unroll 4
        for (int u = lane; u < nv; u += 32) SrcDense<T>::procW(vb[u], v0 + u, nvec, hs, best, bj);
        tcons++;
        __syncwarp();
        if (e_iss < tot) issue();
      }
      const int k = nvec * W + lane;   // rows past the last full vector
      if (k < rows) {
        const double x = d_add((double)src.C[(int64_t)i * src.ld + row0 + k], hs[k]);
        if (x < best) { best = x; bj = k; }
      }
      if (bj != 0x7fffffff) bj += row0;
      warp_argmin(best, bj);
      if (nslabs == 1) {
        if (!(best < 1.0e308 && best > -1.0e308)) { if (lane == 0) set_status(status, 5); }
        const double g = column_gap_epilogue(src, i, best, cnt, srow, sval, cap, b, h);
        if (lane == 0) { out.j[p] = bj; out.minval[p] = best; out.g[p] = g; }
      } else {
        if (lane == 0) {
          out.j[(int64_t)slab * L + p] = bj;
          out.minval[(int64_t)slab * L + p] = best;
        }
        if (out.st_cnt && slab == 0) stage_support(out, p, i, L, cnt, srow, sval, cap, b);
        if (out.st_term) stage_terms(src, out, p, i, L, row0, rows, cnt, srow, sval, cap, h);
      }
    }
    seg = seg_end;
  }
}

}  // namespace sro
