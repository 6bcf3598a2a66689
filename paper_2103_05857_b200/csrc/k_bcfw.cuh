// k_bcfw.cuh — persistent on-device loop for the sequential BCFW family:
// BCFW (Alg. 1), BCAFW (Alg. A.2), BCPFW
// (Alg. A.3), each with U / P / GA sampling (Alg. A.4,
// P:1848-1869) and the decay or exact line-search step (Eq. 10, Eq. 14).
//
// One CTA runs a whole segment of dependent steps (up to the next gap check
// or GA refresh) with no host round trip. h lives in shared memory; the next
// visited column is prefetched into registers while the current step's
// reduction and update run (U / P / explicit visit orders are known ahead).
// Per step: all warps do the LMO over the column (Eq. 9) and a CTA argmin;
// warp 0 then does the O(|supp|) part — column gap, line search, sparse
// column update and the r/h update of the touched rows — one support entry
// per lane (slab_cap <= 31). Roofline: latency (one dependent step at a time).
#pragma once
#include "k_sweep.cuh"
#include "sro_device.cuh"

namespace sro {

constexpr int BCFW_THREADS = 512;
constexpr int BCFW_WARPS = BCFW_THREADS / 32;

enum { VAR_PLAIN = 0, VAR_AWAY = 1, VAR_PAIR = 2 };

struct BcfwArgs {
  int m, n, cap;
  double lambda;
  const double* a;
  const double* b;
  double* r;
  double* h;
  int* cnt;
  int* srow;
  double* sval;
  const int* visit;      // steps entries (U / P / explicit); unused for GA
  int steps;
  long long k0;          // global step counter at segment start
  int step_rule;         // 0 DEC, 1 ELS
  // GA
  double* G;             // n stored gaps
  double* fen;           // n+1 Fenwick tree
  int ga_inner, ga_post;
  unsigned long long seed;
  int ga_smem;           // 1: G and fen staged in shared memory
  int x_smem;            // colour sources: 1 = x staged in shared memory
  int h_smem;            // 1: h staged in shared memory (m small enough)
  // outputs
  int* status;
  int* steps_done;
  double* trace;         // optional: 9 doubles per step (k,i,j,v,dir,gamma,num,den,minval)
};

// ---------------------------------------------------------------------------
// Column providers: the LMO over one column with rows split across the CTA.
// ---------------------------------------------------------------------------
template <typename T, int MAXV>
struct BcDense {
  using V = typename Vec<T>::type;
  static constexpr int W = Vec<T>::W;
  const T* C;
  int64_t ld;
  int m, nvec;
  V cur[MAXV], nxt[MAXV];
  __device__ void init(const T* C_, int64_t ld_, int m_) { C = C_; ld = ld_; m = m_; nvec = m_ / W; }
  __device__ __forceinline__ void fetch(int i) {
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld);
#pragma unroll
    for (int u = 0; u < MAXV; u++) {
      int q = threadIdx.x + u * BCFW_THREADS;
      if (q < nvec) nxt[u] = __ldg(p + q);
    }
  }
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int u = 0; u < MAXV; u++) cur[u] = nxt[u];
  }
  __device__ __forceinline__ void local_argmin(int i, const double* hs, double& best, int& bj) const {
#pragma unroll
    for (int u = 0; u < MAXV; u++) {
      int q = threadIdx.x + u * BCFW_THREADS;
      if (q < nvec) proc4(cur[u], W * q, hs, best, bj);
    }
    // rows beyond the register-prefetched part: direct loads (large m)
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld);
    for (int q = threadIdx.x + MAXV * BCFW_THREADS; q < nvec; q += BCFW_THREADS) proc4(__ldg(p + q), W * q, hs, best, bj);
    int k = nvec * W + threadIdx.x;  // tail rows (m % W)
    if (k < m) {
      double x = d_add((double)C[(int64_t)i * ld + k], hs[k]);
      if (x < best) { best = x; bj = k; }
    }
  }
  __device__ __forceinline__ double cost(int k, int i) const { return (double)C[(int64_t)i * ld + k]; }
};

template <typename T, bool EUCLID>
struct BcColour {
  const T* x;    // global 3m
  const T* xs;   // SoA in smem (x_smem) or nullptr
  const T* y;
  int m;
  __device__ void init(const T* x_, const T* xs_, const T* y_, int m_) { x = x_; xs = xs_; y = y_; m = m_; }
  __device__ __forceinline__ void fetch(int) {}
  __device__ __forceinline__ void advance() {}
  __device__ __forceinline__ void local_argmin(int i, const double* hs, double& best, int& bj) const {
    const T y0 = y[3 * (int64_t)i], y1 = y[3 * (int64_t)i + 1], y2 = y[3 * (int64_t)i + 2];
    for (int k = threadIdx.x; k < m; k += BCFW_THREADS) {
      T x0, x1, x2;
      if (xs) { x0 = xs[k]; x1 = xs[m + k]; x2 = xs[2 * m + k]; }
      else { x0 = x[3 * (int64_t)k]; x1 = x[3 * (int64_t)k + 1]; x2 = x[3 * (int64_t)k + 2]; }
      double v = d_add(colour_cost<EUCLID>(x0, x1, x2, y0, y1, y2), hs[k]);
      if (v < best) { best = v; bj = k; }
    }
  }
  __device__ __forceinline__ double cost(int k, int i) const {
    return colour_cost<EUCLID>(x[3 * (int64_t)k], x[3 * (int64_t)k + 1], x[3 * (int64_t)k + 2], y[3 * (int64_t)i],
                               y[3 * (int64_t)i + 1], y[3 * (int64_t)i + 2]);
  }
};

// ---------------------------------------------------------------------------
// GA sampler on a Fenwick tree over max(G_i, 0) (Alg. A.4 line 2; R14-R17).
// Single-thread functions; fen is 1-based, fen[1..n].
// ---------------------------------------------------------------------------
__device__ __forceinline__ double wpos(double g) { return g > 0.0 ? g : 0.0; }

__device__ int ga_draw(const double* fen, const double* G, int n, double u53) {
  double W = 0.0;
  for (int p = n; p > 0; p -= p & -p) W = d_add(W, fen[p]);
  if (!(W > 0.0)) {
    int i = (int)d_mul(u53, (double)n);
    return i >= n ? n - 1 : i;
  }
  double u = d_mul(u53, W);
  int pos = 0, bit = 1;
  while (bit * 2 <= n) bit *= 2;
  for (; bit > 0; bit >>= 1) {
    if (pos + bit <= n && fen[pos + bit] <= u) { pos += bit; u = d_sub(u, fen[pos]); }
  }
  if (pos >= n) {
    for (int i = n - 1; i >= 0; i--) if (wpos(G[i]) > 0.0) return i;
    return n - 1;
  }
  return pos;
}

__device__ __forceinline__ void ga_add(double* fen, int n, int i0, double delta) {
  for (int p = i0 + 1; p <= n; p += p & -p) fen[p] = d_add(fen[p], delta);
}

// ---------------------------------------------------------------------------
// The persistent kernel.
// ---------------------------------------------------------------------------
template <class Col, int VAR, bool GA>
__global__ void __launch_bounds__(BCFW_THREADS, 1) k_bcfw(BcfwArgs A, Col col) {
  extern __shared__ __align__(16) double sm[];
  double* sh_h = sm;                                   // m
  double* slots = sh_h + (A.h_smem ? ((A.m + 1) & ~1) : 0);  // 256 (warp 0 sparse psum256)
  double* wbest = slots + 256;                         // BCFW_WARPS
  int* wj = reinterpret_cast<int*>(wbest + BCFW_WARPS); // BCFW_WARPS
  int* misc = wj + BCFW_WARPS;                         // [0]=i [1]=j [2]=abort
  double* miscd = reinterpret_cast<double*>(misc + 4); // [0]=minval [1]=g_pre
  double* ga_base = miscd + 2;
  double* Gs = A.G;
  double* fens = A.fen;
  if (GA && A.ga_smem) { Gs = ga_base; fens = ga_base + A.n; }

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  double* hs = A.h_smem ? sh_h : A.h;   // h staged in shared memory when it fits
  if (A.h_smem) for (int k = tid; k < m; k += BCFW_THREADS) sh_h[k] = A.h[k];
  for (int c = tid; c < 256; c += BCFW_THREADS) slots[c] = 0.0;
  if (GA && A.ga_smem) {
    for (int c = tid; c < n; c += BCFW_THREADS) Gs[c] = A.G[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) fens[c] = A.fen[c];
  }
  if (tid == 0) misc[2] = 0;
  __syncthreads();

  const double lam = A.lambda;
  int done = 0;
  if (!GA && A.steps > 0) col.fetch(A.visit[0]);

  for (int s = 0; s < A.steps; s++) {
    const long long kk = A.k0 + s;
    int i;
    if (GA) {
      if (tid == 0) misc[0] = ga_draw(fens, Gs, n, uniform53(rng_u64(A.seed, 1, (uint64_t)kk)));
      __syncthreads();
      i = misc[0];
      col.fetch(i);
      col.advance();
    } else {
      i = A.visit[s];
      col.advance();
      if (s + 1 < A.steps) col.fetch(A.visit[s + 1]);
    }
    // ---- LMO (Eq. 9): CTA argmin of c_i + h, lowest row on ties
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bj = 0x7fffffff;
    col.local_argmin(i, hs, best, bj);
    warp_argmin(best, bj);
    if (lane == 0) { wbest[warp] = best; wj[warp] = bj; }
    __syncthreads();
    if (warp == 0) {
      double mv = lane < BCFW_WARPS ? wbest[lane] : __longlong_as_double(0x7ff0000000000000LL);
      int j = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
      warp_argmin(mv, j);
      // ---- O(|supp|) part, one support entry per lane
      const double bi = A.b[i];
      const int c0 = A.cnt[i];
      int rw = 0x7fffffff;
      double tv = 0.0, gk = 0.0;
      if (lane < c0) {
        rw = A.srow[(int64_t)i * cap + lane];
        tv = A.sval[(int64_t)i * cap + lane];
        gk = d_add(col.cost(rw, i), hs[rw]);
      }
      const double dot = warp_seq_sum(d_mul(tv, gk), c0);
      const double gfw = d_sub(dot, d_mul(bi, mv));
      bool abort = !(mv < 1.0e308 && mv > -1.0e308);
      // away atom v = argmax_{k in supp} grad_ki (Eq. 13), lowest row on ties
      double gv = __longlong_as_double(0xfff0000000000000LL);  // -inf
      int vrow = 0x7fffffff;
      if (VAR != VAR_PLAIN) {
        double x = lane < c0 ? gk : __longlong_as_double(0xfff0000000000000LL);
        int xr = lane < c0 ? rw : 0x7fffffff;
        gv = x; vrow = xr;
        warp_argmax(gv, vrow);
      }
      const unsigned inmask = __ballot_sync(FULL, lane < c0 && rw == j);
      const bool j_in = inmask != 0u;
      const int ins = __popc(__ballot_sync(FULL, lane < c0 && rw < j));
      // merged support supp(t_i) U {j}, rows ascending, one entry per lane
      const int M = c0 + (j_in ? 0 : 1);
      int src = (j_in || lane < ins) ? lane : lane - 1;
      if (src < 0) src = 0;
      int mrow = __shfl_sync(FULL, rw, src & 31);
      double mt = __shfl_sync(FULL, tv, src & 31);
      if (!j_in && lane == ins) { mrow = j; mt = 0.0; }
      const bool mvalid = lane < M;

      int dir = 0;
      double gamma = 0.0, num = 0.0, den = 0.0;
      double tnew = mt;        // new value of the merged entry (plain / FW / pairwise)
      bool use_merged = true;  // false: away direction over supp only
      if (VAR == VAR_PLAIN) {
        double d = d_sub((mvalid && mrow == j) ? bi : 0.0, mvalid ? mt : 0.0);
        double D = d_add(0.0, d);
        den = warp_sparse_psum256(m, M, mrow, d_mul(D, D), slots);
        num = d_mul(lam, d_add(0.0, gfw));
        if (A.step_rule == 1) {
          if (!(num > 0.0) || den == 0.0) gamma = 0.0;
          else { gamma = d_div(num, den); if (gamma > 1.0) gamma = 1.0; }
        } else {
          gamma = d_div((double)(2LL * n), (double)(kk + 2LL * n));
        }
        const double omg = d_sub(1.0, gamma), gb = d_mul(gamma, bi);
        tnew = d_mul(omg, mt);
        if (mrow == j) tnew = d_add(tnew, gb);
      } else if (VAR == VAR_AWAY) {
        const double gaw = d_sub(d_mul(bi, gv), dot);
        const bool use_fw = (c0 == 1) || (gfw >= gaw);
        if (use_fw) {
          double d = d_sub((mvalid && mrow == j) ? bi : 0.0, mvalid ? mt : 0.0);
          den = warp_sparse_psum256(m, M, mrow, d_mul(d, d), slots);
          num = d_mul(lam, d_add(gfw, 0.0));
          if (!(num > 0.0) || den == 0.0) gamma = 0.0;
          else { gamma = d_div(num, den); if (gamma > 1.0) gamma = 1.0; }
          const double omg = d_sub(1.0, gamma), gb = d_mul(gamma, bi);
          tnew = d_mul(omg, mt);
          if (mrow == j) tnew = d_add(tnew, gb);
        } else {
          dir = 1;
          use_merged = false;
          const double tvv = __shfl_sync(FULL, tv, __ffs(__ballot_sync(FULL, lane < c0 && rw == vrow)) - 1);
          double d = (lane < c0) ? ((rw == vrow) ? d_sub(tv, bi) : tv) : 0.0;
          den = warp_sparse_psum256(m, c0, rw, d_mul(d, d), slots);
          num = d_mul(lam, d_add(gaw, 0.0));
          const double alpha = d_div(tvv, bi);
          const double gmax = d_div(alpha, d_sub(1.0, alpha));
          if (!(num > 0.0) || den == 0.0) gamma = 0.0;
          else { gamma = d_div(num, den); if (gamma > gmax) gamma = gmax; }
          const double opg = d_add(1.0, gamma), gb = d_mul(gamma, bi);
          tnew = d_mul(opg, tv);
          if (lane < c0 && rw == vrow) {
            tnew = d_sub(tnew, gb);
            if (gamma == gmax || tnew < 0.0) tnew = 0.0;
          }
        }
      } else {  // VAR_PAIR
        if (vrow == j) {
          dir = 3;
        } else {
          dir = 2;
          const double tvv = __shfl_sync(FULL, tv, __ffs(__ballot_sync(FULL, lane < c0 && rw == vrow)) - 1);
          const double dv = d_sub(gv, mv);
          num = d_mul(lam, dv);
          den = d_mul(2.0, bi);
          const double alpha = d_div(tvv, bi);
          if (!(num > 0.0)) gamma = 0.0;
          else { gamma = d_div(num, den); if (gamma > alpha) gamma = alpha; }
          double mu = d_mul(gamma, bi);
          const bool drop = (gamma == alpha) || (mu >= tvv);
          if (drop) mu = tvv;
          tnew = mt;
          if (mrow == j) tnew = d_add(mt, mu);
          if (mrow == vrow) tnew = drop ? 0.0 : d_sub(mt, mu);
        }
      }
      // ---- apply: new column (drop exact zeros), r += (t' - t), h refresh
      const bool noop = (VAR == VAR_PAIR && dir == 3);
      const int E = use_merged ? M : c0;
      const int erow = use_merged ? mrow : rw;
      const double eold = use_merged ? mt : tv;
      const bool ev = lane < E;
      const bool keep = ev && tnew != 0.0;
      const unsigned kmask = __ballot_sync(FULL, keep);
      const int nk = __popc(kmask);
      if (!noop && nk > cap) abort = true;
      if (!abort && !noop) {
        if (ev) {
          const double Dp = d_add(0.0, d_sub(tnew, eold));
          const double rn = d_add(A.r[erow], Dp);
          const double hn = d_div(d_sub(rn, A.a[erow]), lam);
          A.r[erow] = rn;
          A.h[erow] = hn;
          if (A.h_smem) sh_h[erow] = hn;
        }
        if (keep) {
          const int pos = __popc(kmask & ((1u << lane) - 1u));
          A.srow[(int64_t)i * cap + pos] = erow;
          A.sval[(int64_t)i * cap + pos] = tnew;
        }
        if (lane == 0) A.cnt[i] = nk;
      }
      if (lane == 0) {
        misc[1] = j;
        miscd[0] = mv;
        miscd[1] = gfw;
        if (abort) {
          misc[2] = 1;
          set_status(A.status, !(mv < 1.0e308 && mv > -1.0e308) ? 5 : 6);
        } else if (A.trace) {
          double* tr = A.trace + 9 * (int64_t)s;
          tr[0] = (double)kk; tr[1] = i; tr[2] = j; tr[3] = (VAR == VAR_PLAIN) ? -1 : vrow;
          tr[4] = dir; tr[5] = gamma; tr[6] = num; tr[7] = den; tr[8] = mv;
        }
      }
    }
    __syncthreads();
    if (misc[2]) break;
    // ---- GA: refresh the visited column's stored gap (Alg. A.4 line 6)
    if (GA && A.ga_inner) {
      double gnew = miscd[1];
      if (A.ga_post) {
        double b2 = __longlong_as_double(0x7ff0000000000000LL);
        int j2 = 0x7fffffff;
        col.local_argmin(i, hs, b2, j2);
        warp_argmin(b2, j2);
        if (lane == 0) { wbest[warp] = b2; wj[warp] = j2; }
        __syncthreads();
        if (warp == 0) {
          double mv2 = lane < BCFW_WARPS ? wbest[lane] : __longlong_as_double(0x7ff0000000000000LL);
          int jj2 = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
          warp_argmin(mv2, jj2);
          const int c1 = A.cnt[i];
          double term = 0.0;
          if (lane < c1) {
            int k2 = A.srow[(int64_t)i * cap + lane];
            term = d_mul(A.sval[(int64_t)i * cap + lane], d_add(col.cost(k2, i), hs[k2]));
          }
          const double dot2 = warp_seq_sum(term, c1);
          gnew = d_sub(dot2, d_mul(A.b[i], mv2));
          if (lane == 0) {
            double delta = d_sub(wpos(gnew), wpos(Gs[i]));
            Gs[i] = gnew;
            ga_add(fens, n, i, delta);
          }
        }
      } else if (tid == 0) {
        double delta = d_sub(wpos(gnew), wpos(Gs[i]));
        Gs[i] = gnew;
        ga_add(fens, n, i, delta);
      }
      __syncthreads();
    }
    done = s + 1;
  }
  if (GA && A.ga_smem) {
    __syncthreads();
    for (int c = tid; c < n; c += BCFW_THREADS) A.G[c] = Gs[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) A.fen[c] = fens[c];
  }
  if (tid == 0) *A.steps_done = done;
}

// Fenwick rebuild after a GA global refresh: fen[i] = max(G_{i-1}, 0), then
// the standard linear build (R14). One thread, in order.
__global__ void k_fen_build(const double* __restrict__ G, double* fen, int n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  fen[0] = 0.0;
  for (int i = 1; i <= n; i++) fen[i] = wpos(G[i - 1]);
  for (int i = 1; i <= n; i++) {
    int p = i + (i & -i);
    if (p <= n) fen[p] = d_add(fen[p], fen[i]);
  }
}

__global__ void k_fill(double* x, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = v;
}

}  // namespace sro
