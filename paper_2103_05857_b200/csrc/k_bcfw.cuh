// k_bcfw.cuh — persistent on-device loop for the sequential BCFW family:
// BCFW (Alg. 1), BCAFW (Alg. A.2), BCPFW
// (Alg. A.3), each with U / P / GA sampling (Alg. A.4,
// P:1848-1869) and the decay or exact line-search step (Eq. 10, Eq. 14).
//
// One CTA runs a whole segment of dependent steps (up to the next gap check or
// GA refresh) with no host round trip. Per step:
//   1. all 16 warps: LMO over the visited column (Eq. 9) -> CTA argmin;
//   2. warp 0: the O(|supp|) part — column gap (Eq. 11), line search (Eq. 10 /
//      Eq. 14), sparse column update and the r/h refresh of the touched rows —
//      one support entry per lane (slab_cap <= 31).
// Fast layout (SMEM = true): h, r and the per-column support counts live in
// shared memory for the whole segment; the next visited column is staged into
// a shared-memory double buffer with cp.async while the current step runs
// (colour costs: the source colours are staged once), and warp 0 prefetches
// the next column's support slab into registers, so the serial part touches
// no global memory on its critical path. Generic layout (SMEM = false): the
// same arithmetic on global arrays, for sizes that do not fit.
// Roofline: latency of one dependent step.
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
  double* G;             // GA stored gaps (n)
  double* fen;           // GA Fenwick tree (n+1)
  int ga_inner, ga_post;
  unsigned long long seed;
  int ga_smem;           // GA arrays staged in shared memory
  int* status;
  int* steps_done;
  double* trace;         // optional: 9 doubles per step (k,i,j,v,dir,gamma,num,den,minval)
  long long* phase;      // SRO_PHASE_TIMING builds only: 8 accumulated clock64 phase totals
  double cmax;           // max_{k,i} |C_ki| (fp32 LMO filter window)
  int a_smem;            // a staged in shared memory
  int visit_smem;        // the segment's visit list staged in shared memory
  int dbg;               // timing experiments only (SRO_DBG): 1 = skip the serial part, 2 = skip the LMO
  int spec;              // GA pipe: speculative next column prefetched and pre-scanned; 0 = off (SRO_NO_SPEC)
  const int* halt;       // device flag: set -> the segment is a no-op (it was enqueued ahead of
                         // the host's check of the previous one, which converged or failed)
};

__device__ __forceinline__ bool bcfw_halted(const BcfwArgs& A) {
  if (A.halt && *(volatile const int*)A.halt) {
    if (threadIdx.x == 0) *A.steps_done = 0;
    return true;
  }
  return false;
}


#ifdef SRO_PHASE_TIMING
struct PhaseState { long long acc[16]; long long t; };
#define PHASE_MARK(idx)                                       \
  do {                                                        \
    if (threadIdx.x == 0) {                                   \
      const long long t_ = clock64();                         \
      g_ph->acc[idx] += t_ - g_ph->t;                         \
      g_ph->t = t_;                                           \
    }                                                         \
  } while (0)
#else
#define PHASE_MARK(idx) do {} while (0)
#endif

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }
__device__ __forceinline__ double dninf() { return __longlong_as_double(0xfff0000000000000LL); }
__host__ __device__ __forceinline__ size_t rup16(size_t x) { return (x + 15) / 16 * 16; }

// ---------------------------------------------------------------------------
// cp.async helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gsrc), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// ---------------------------------------------------------------------------
// Column providers
// ---------------------------------------------------------------------------
// Dense column staged in a shared-memory double buffer by cp.async (fast layout).
template <typename T>
struct ColStaged {
  using V = typename Vec<T>::type;
  static constexpr int W = Vec<T>::W;
  static constexpr bool STAGED = true;
  static constexpr bool FILTER = sizeof(T) == 4;   // binary32 costs: fp32 filter + exact fp64 check
  const T* C;
  int64_t ld;
  int m;
  T* buf0;
  T* buf1;
  static size_t smem_bytes(int m) { return 2 * rup16((size_t)m * sizeof(T)); }
  __device__ __forceinline__ T* buf(int slot) const { return slot ? buf1 : buf0; }
  __device__ __forceinline__ void setup(char* region) {
    buf0 = reinterpret_cast<T*>(region);
    buf1 = reinterpret_cast<T*>(region + rup16((size_t)m * sizeof(T)));
  }
  // every thread issues its share of the copy of column i into buffer `slot`
  __device__ __forceinline__ void issue(int i, int slot) const {
    const T* src = C + (int64_t)i * ld;
    T* dst = buf(slot);
    const int nvec = m / W;
    for (int q = threadIdx.x; q < nvec; q += BCFW_THREADS) cp_async16(dst + W * q, src + W * q);
    const int k = nvec * W + threadIdx.x;
    if (k < m) cp_async_small<sizeof(T)>(dst + k, src + k);
    cp_async_commit();
  }
  __device__ __forceinline__ void local_argmin(int, int slot, const double* hs, double& best, int& bj) const {
    const T* c = buf(slot);
    const V* cv = reinterpret_cast<const V*>(c);
    const int nvec = m / W;
    for (int q = threadIdx.x; q < nvec; q += BCFW_THREADS) proc4(cv[q], W * q, hs, best, bj);
    const int k = nvec * W + threadIdx.x;
    if (k < m) {
      const double x = d_add((double)c[k], hs[k]);
      if (x < best) { best = x; bj = k; }
    }
  }
  __device__ __forceinline__ double cost(int k, int, int slot) const { return (double)buf(slot)[k]; }
  // Exact LMO with a binary32 filter: F_k = fl32(c_k + fl32(h_k)) is within
  // eps = 2^-24 (cmax + (2 + 2^-24) hmax) of c_k + h_k and the exact value
  // V_k = fl64(c_k + h_k) within 2^-53 (cmax + hmax), so every row that ties
  // or beats the thread's exact minimum has F_k <= min F + delta with
  // delta = 2^-22 (cmax + 2 hmax) + 1e-30 >= 2 eps + 2 * 2^-53 (...). Only those
  // candidate rows are evaluated exactly in binary64 (ascending rows, strict <),
  // so the result is the thread's exact lowest-index argmin of V.
  __device__ __forceinline__ void local_argmin_filt(int slot, const double* hs, const float* hs32, float delta,
                                                    double& best, int& bj) const {
    const float4* cv = reinterpret_cast<const float4*>(buf(slot));
    const float4* hv = reinterpret_cast<const float4*>(hs32);
    const int nvec = m / 4;
    float4 cq[4], fq[4];
    float fmin = __int_as_float(0x7f800000);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = threadIdx.x + u * BCFW_THREADS;
      if (q < nvec) {
        cq[u] = reinterpret_cast<const float4*>(cv)[q];
        const float4 hh = hv[q];
        fq[u] = make_float4(__fadd_rn(cq[u].x, hh.x), __fadd_rn(cq[u].y, hh.y), __fadd_rn(cq[u].z, hh.z),
                            __fadd_rn(cq[u].w, hh.w));
        fmin = fminf(fmin, fminf(fminf(fq[u].x, fq[u].y), fminf(fq[u].z, fq[u].w)));
      }
    }
    const int kt = nvec * 4 + threadIdx.x;
    float ct = 0.f, ft = __int_as_float(0x7f800000);
    if (kt < m) { ct = buf(slot)[kt]; ft = __fadd_rn(ct, hs32[kt]); fmin = fminf(fmin, ft); }
    const float thr = __fadd_ru(fmin, delta);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = threadIdx.x + u * BCFW_THREADS;
      if (q < nvec) {
        const int k = 4 * q;
        if (fq[u].x <= thr) { const double v = d_add((double)cq[u].x, hs[k]); if (v < best) { best = v; bj = k; } }
        if (fq[u].y <= thr) { const double v = d_add((double)cq[u].y, hs[k + 1]); if (v < best) { best = v; bj = k + 1; } }
        if (fq[u].z <= thr) { const double v = d_add((double)cq[u].z, hs[k + 2]); if (v < best) { best = v; bj = k + 2; } }
        if (fq[u].w <= thr) { const double v = d_add((double)cq[u].w, hs[k + 3]); if (v < best) { best = v; bj = k + 3; } }
      }
    }
    if (kt < m && ft <= thr) { const double v = d_add((double)ct, hs[kt]); if (v < best) { best = v; bj = kt; } }
  }
};

// Dense column read straight from global memory (generic layout).
template <typename T>
struct ColDirect {
  using V = typename Vec<T>::type;
  static constexpr int W = Vec<T>::W;
  static constexpr bool STAGED = false;
  static constexpr bool FILTER = false;
  const T* C;
  int64_t ld;
  int m;
  static size_t smem_bytes(int) { return 0; }
  __device__ __forceinline__ void local_argmin_filt(int, const double*, const float*, float, double&, int&) const {}
  __device__ __forceinline__ void setup(char*) {}
  __device__ __forceinline__ void issue(int, int) const {}
  __device__ __forceinline__ void local_argmin(int i, int, const double* hs, double& best, int& bj) const {
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld);
    const int nvec = m / W;
    for (int q = threadIdx.x; q < nvec; q += BCFW_THREADS) proc4(__ldg(p + q), W * q, hs, best, bj);
    const int k = nvec * W + threadIdx.x;
    if (k < m) {
      const double x = d_add((double)__ldg(C + (int64_t)i * ld + k), hs[k]);
      if (x < best) { best = x; bj = k; }
    }
  }
  __device__ __forceinline__ double cost(int k, int i, int) const { return (double)__ldg(C + (int64_t)i * ld + k); }
};

// Colour costs computed on the fly; source colours staged (SoA) in shared memory if XS.
template <typename T, bool XS>
struct ColColour {
  static constexpr bool STAGED = false;
  static constexpr bool FILTER = false;
  __device__ __forceinline__ void local_argmin_filt(int, const double*, const float*, float, double&, int&) const {}
  const T* x;
  const T* y;
  int m;
  int euclid;
  T* xs;
  static size_t smem_bytes(int m) { return XS ? rup16((size_t)3 * m * sizeof(T)) : 0; }
  __device__ __forceinline__ void setup(char* region) {
    if (XS) {
      xs = reinterpret_cast<T*>(region);
      for (int k = threadIdx.x; k < m; k += BCFW_THREADS) {
        xs[k] = x[3 * (int64_t)k];
        xs[m + k] = x[3 * (int64_t)k + 1];
        xs[2 * m + k] = x[3 * (int64_t)k + 2];
      }
    }
  }
  __device__ __forceinline__ void issue(int, int) const {}
  __device__ __forceinline__ void xk(int k, T& x0, T& x1, T& x2) const {
    if (XS) { x0 = xs[k]; x1 = xs[m + k]; x2 = xs[2 * m + k]; }
    else { x0 = x[3 * (int64_t)k]; x1 = x[3 * (int64_t)k + 1]; x2 = x[3 * (int64_t)k + 2]; }
  }
  __device__ __forceinline__ double c(T x0, T x1, T x2, T y0, T y1, T y2) const {
    return euclid ? colour_cost<true>(x0, x1, x2, y0, y1, y2) : colour_cost<false>(x0, x1, x2, y0, y1, y2);
  }
  __device__ __forceinline__ void local_argmin(int i, int, const double* hs, double& best, int& bj) const {
    const T y0 = y[3 * (int64_t)i], y1 = y[3 * (int64_t)i + 1], y2 = y[3 * (int64_t)i + 2];
    for (int k = threadIdx.x; k < m; k += BCFW_THREADS) {
      T x0, x1, x2;
      xk(k, x0, x1, x2);
      const double v = d_add(c(x0, x1, x2, y0, y1, y2), hs[k]);
      if (v < best) { best = v; bj = k; }
    }
  }
  __device__ __forceinline__ double cost(int k, int i, int) const {
    T x0, x1, x2;
    xk(k, x0, x1, x2);
    return c(x0, x1, x2, y[3 * (int64_t)i], y[3 * (int64_t)i + 1], y[3 * (int64_t)i + 2]);
  }
};

// psum256 over m rows of a vector that is zero except at up to 32 rows (one per
// lane, rows ascending with the lane): exactly chunk_tree_sum(x, m, 256) of
// R19, with shuffles only. Entries of one chunk are consecutive lanes and are
// summed left to right from +0.0 (a segmented scan, usually of length 1).
// The 256-leaf adjacent-pair tree restricted to the non-empty chunks is the
// tree whose internal node between adjacent non-empty chunks c_u < c_{u+1}
// sits at level hdb(c_u ^ c_{u+1}) (zero leaves are additive identities): every
// lane holds the value of its current subtree and, level by level (only the
// levels that occur), the two subtrees separated by a boundary of that level
// merge as left + right. <= 8 rounds of 2 ballots, 2 shuffles and 1 add.
__device__ __forceinline__ double warp_sparse_psum256_fast(int m, int cnt, int row, double x) {
  const int lane = threadIdx.x & 31;
  const bool valid = lane < cnt;
  // chunk of a row: floor((256 (row + 1) - 1) / m) (R19); for m = 256 * 2^s that is row >> s
  const int dm = m >> 8;
  int c;
  if ((m & 255) == 0 && (dm & (dm - 1)) == 0) c = valid ? (row >> (__ffs(dm) - 1)) : -1 - lane;
  else c = valid ? chunk_index(row, m, 256) : -1 - lane;
  if (cnt <= 3) {
    // the same tree for at most three entries, evaluated directly: runs of one
    // chunk summed left to right from +0.0, distinct chunks merged at their
    // lowest common ancestor (three distinct chunks: the lower of the two
    // adjacent LCAs first; they are never equal)
    const double x0 = __shfl_sync(FULL, x, 0), x1 = __shfl_sync(FULL, x, 1), x2 = __shfl_sync(FULL, x, 2);
    const int c0 = __shfl_sync(FULL, c, 0), c1 = __shfl_sync(FULL, c, 1), c2 = __shfl_sync(FULL, c, 2);
    const double v0 = d_add(0.0, x0);
    if (cnt <= 1) return cnt == 1 ? v0 : 0.0;
    if (cnt == 2) return c0 == c1 ? d_add(v0, x1) : d_add(v0, d_add(0.0, x1));
    if (c0 == c1 && c1 == c2) return d_add(d_add(v0, x1), x2);
    if (c0 == c1) return d_add(d_add(v0, x1), d_add(0.0, x2));
    if (c1 == c2) return d_add(v0, d_add(d_add(0.0, x1), x2));
    const double v1 = d_add(0.0, x1), v2 = d_add(0.0, x2);
    return (31 - __clz(c0 ^ c1)) < (31 - __clz(c1 ^ c2)) ? d_add(d_add(v0, v1), v2) : d_add(v0, d_add(v1, v2));
  }
  const int cprev = __shfl_up_sync(FULL, c, 1);
  const int cnext = __shfl_down_sync(FULL, c, 1);
  const bool start = valid && (lane == 0 || cprev != c);
  const bool last = valid && (lane == cnt - 1 || cnext != c);
  const unsigned smask = __ballot_sync(FULL, start);
  const unsigned lmask = __ballot_sync(FULL, last);
  double v = valid ? d_add(0.0, x) : 0.0;
  if (smask != lmask) {   // some chunk holds several entries: segmented left-to-right sums
    const int seg0 = 31 - __clz(smask & (0xffffffffu >> (31 - lane)));
    const int pos = valid ? lane - seg0 : 0;
    const int maxpos = (int)__reduce_max_sync(FULL, (unsigned)pos);
    for (int t = 1; t <= maxpos; t++) {
      const double prev = __shfl_up_sync(FULL, v, 1);
      if (pos == t) v = d_add(prev, x);
    }
    const unsigned after = lmask & (0xffffffffu << lane);
    v = __shfl_sync(FULL, v, after ? __ffs(after) - 1 : lane);   // segment total to all its lanes
  }
  const int hdb = (last && lane < cnt - 1) ? 31 - __clz((unsigned)(c ^ cnext)) : -1;
  unsigned levels = __reduce_or_sync(FULL, hdb >= 0 ? (1u << hdb) : 0u);
  while (levels) {
    const int b = __ffs(levels) - 1;
    levels &= levels - 1;
    const unsigned ge = __ballot_sync(FULL, hdb >= b);
    const unsigned eq = __ballot_sync(FULL, hdb == b);
    const unsigned rm = ge & (0xffffffffu << lane);
    const unsigned lm = lane ? (ge & (0xffffffffu >> (32 - lane))) : 0u;
    const int rb = rm ? __ffs(rm) - 1 : -1;
    const int lb = lm ? 31 - __clz(lm) : -1;
    int u = -1;
    if (rb >= 0 && ((eq >> rb) & 1u)) u = rb;        // this lane's subtree is the left child
    else if (lb >= 0 && ((eq >> lb) & 1u)) u = lb;   // ... or the right child
    const double vl = __shfl_sync(FULL, v, u < 0 ? lane : u);
    const double vr = __shfl_sync(FULL, v, u < 0 ? lane : u + 1);
    if (u >= 0 && valid) v = d_add(vl, vr);
  }
  return __shfl_sync(FULL, v, 0);
}

// Sequential left-to-right sum (from +0.0) of the values of lanes 0..cnt-1 with
// the first 8 operands fetched by independent shuffles. Result in every lane.
__device__ __forceinline__ double warp_seq_sum_fast(double x, int cnt) {
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; q++) v[q] = __shfl_sync(FULL, x, q);
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 8; q++) if (q < cnt) acc = d_add(acc, v[q]);
  for (int q = 8; q < cnt; q++) acc = d_add(acc, __shfl_sync(FULL, x, q));
  return acc;
}

// Warp argmax of (value, row), lowest row on ties, via REDUX on order keys.
__device__ __forceinline__ void warp_argmax_redux(double& v, int& j, bool valid) {
  const unsigned long long key = valid ? okey(v) : 0ULL;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned m1 = __reduce_max_sync(FULL, hi);
  const unsigned m2 = __reduce_max_sync(FULL, hi == m1 ? lo : 0u);
  const unsigned m3 = __reduce_min_sync(FULL, (valid && hi == m1 && lo == m2) ? (unsigned)j : 0x7fffffffu);
  j = (int)m3;
  v = okey_inv(((unsigned long long)m1 << 32) | m2);
}

// ---------------------------------------------------------------------------
// GA sampler on a Fenwick tree over max(G_i, 0) (Alg. A.4 line 2; R14-R17).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double wpos(double g) { return g > 0.0 ? g : 0.0; }

// fen lives in shared memory: loads through its 32-bit shared address (no
// generic-to-shared conversion per load); clamped address, then the select.
__device__ __forceinline__ double sh_ld_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
// SH: fen is known to be in shared memory (else any generic pointer).
template <bool SH>
__device__ __forceinline__ int ga_draw_t(const double* fen, const double* G, int n, double u53) {
  const uint32_t fb = SH ? (uint32_t)__cvta_generic_to_shared(fen) : 0u;
  auto ldn = [&](int q) { return SH ? sh_ld_f64(fb + 8u * (uint32_t)q) : fen[q]; };
  double W = 0.0;
  for (int p = n; p > 0; p -= p & -p) W = d_add(W, ldn(p));
  if (!(W > 0.0)) {
    int i = (int)d_mul(u53, (double)n);
    return i >= n ? n - 1 : i;
  }
  double u = d_mul(u53, W);
  int pos = 0;
  int bit = 1 << (31 - __clz(n));   // highest power of two <= n
  // Standard descent (if (pos+bit <= n && fen[pos+bit] <= u) { pos += bit; u -= fen[pos]; }),
  // three levels per round: the 1 + 2 + 4 candidates of the round are loaded
  // together, so the dependent shared-memory loads drop to a third; the
  // comparisons and subtractions are the same operations in the same order.
  // (a candidate past n is never taken: level() tests pos + b <= n first, so its
  // clamped load needs no zeroing)
  auto ld = [&](int q) { return ldn(q <= n ? q : n); };
  auto level = [&](int b, double f) {
    const bool t = (pos + b <= n) && f <= u;
    const double un = d_sub(u, f);
    if (t) { pos += b; u = un; }
    return t;
  };
  while (bit >= 4) {
    const int b2 = bit >> 1, b3 = bit >> 2;
    const double fa = ld(pos + bit);
    const double f0 = ld(pos + b2), f1 = ld(pos + bit + b2);
    const double g00 = ld(pos + b3), g01 = ld(pos + b2 + b3), g10 = ld(pos + bit + b3), g11 = ld(pos + bit + b2 + b3);
    const bool t1 = level(bit, fa);
    const bool t2 = level(b2, t1 ? f1 : f0);
    level(b3, t1 ? (t2 ? g11 : g10) : (t2 ? g01 : g00));
    bit >>= 3;
  }
  while (bit >= 1) {
    level(bit, ld(pos + bit));
    bit >>= 1;
  }
  if (pos >= n) {
    for (int i = n - 1; i >= 0; i--) if (wpos(G[i]) > 0.0) return i;
    return n - 1;
  }
  return pos;
}
__device__ __forceinline__ int ga_draw(const double* fen, const double* G, int n, double u53) {
  return ga_draw_t<false>(fen, G, n, u53);
}
__device__ __forceinline__ int ga_draw_sh(const double* fen, const double* G, int n, double u53) {
  return ga_draw_t<true>(fen, G, n, u53);
}

__device__ __forceinline__ void ga_add(double* fen, int n, int i0, double delta) {
  for (int p = i0 + 1; p <= n; p += p & -p) fen[p] = d_add(fen[p], delta);
}
// Same update with lane t of a warp updating the t-th node of the path (the
// nodes are distinct, so each node receives exactly the one add it gets above).
// With x = p - 1 a step p += p & -p sets the lowest zero bit of x (x |= x + 1).
// The node lane t of a warp updates for leaf i0 (> n: none), so that the
// update itself (ga_add_node) is one read-modify-write once delta is known.
__device__ __forceinline__ long long ga_path_node(int n, int i0) {
  const int lane = threadIdx.x & 31;
  unsigned x = (unsigned)i0;
  for (int t = 0; t < lane && x <= (unsigned)n; t++) x |= x + 1u;
  return (long long)x + 1;
}
__device__ __forceinline__ void ga_add_node(double* fen, int n, long long p, double delta) {
  if (p <= n) fen[p] = d_add(fen[p], delta);
  __syncwarp();
}
__device__ __forceinline__ void ga_add_warp(double* fen, int n, int i0, double delta) {
  const int lane = threadIdx.x & 31;
  unsigned x = (unsigned)i0;
  for (int t = 0; t < lane && x <= (unsigned)n; t++) x |= x + 1u;
  const long long p = (long long)x + 1;
  if (p <= n) fen[p] = d_add(fen[p], delta);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Warp 0: the O(|supp|) part of one step (all 32 lanes call it).
// In: column i, LMO result (j, mv), b_i, support size c0 and the lane's slab
// entry (rw, tv) with its gradient gk = C_{rw,i} + h_rw (lanes < c0).
// Applies the update to (r, h) and to the slab of column i.
// Out (per lane): the new entries (erow, tnew, keep) for reuse by the caller.
// ---------------------------------------------------------------------------
struct StepOut {
  int dir, vrow, nk, erow;
  bool abort, keep, noop, ev, merged;   // merged: entries in merged-support lane layout (else slab layout)
  double gamma, num, den, gfw, tnew, hnew;
  unsigned kmask;
};

#ifdef SRO_PHASE_TIMING
#define SP_MARK(idx) do { if (threadIdx.x == 0 && sp_ph) { const long long t_ = clock64(); sp_ph->acc[idx] += t_ - sp_ph->t; sp_ph->t = t_; } } while (0)
#define SP_PARAM , PhaseState* sp_ph
#define SP_ARG , g_ph
#define SP_NULL , nullptr
#else
#define SP_NULL
#define SP_MARK(idx) do {} while (0)
#define SP_PARAM
#define SP_ARG
#endif
// <t_i, grad_i f> over the slab (lanes < c0 hold t_ki (C_ki + h_k), rows ascending),
// summed in slab order; needs no LMO result, so a caller may form it while the LMO runs
__device__ __forceinline__ double slab_dot(double prod, int c0) {
  double dv[8];
#pragma unroll
  for (int q = 0; q < 8; q++) dv[q] = __shfl_sync(FULL, prod, q);
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 8; q++) {
    if (q >= c0) break;
    acc = d_add(acc, dv[q]);
  }
  for (int q = 8; q < c0; q++) acc = d_add(acc, __shfl_sync(FULL, prod, q));
  return acc;
}

// PRE_DOT: the caller passes slab_dot(t_i (C_i + h), c0) in dot_in
template <int VAR, bool PRE_DOT = false>
__device__ __forceinline__ StepOut serial_step(const BcfwArgs& A, long long kk, int i, int j, double mv, double bi,
                                               int c0, int rw, double tv, double gk, double* r, double* h,
                                               float* h32, const double* a, int* cnt2, double* slots,
                                               float* hmax SP_PARAM, double dot_in = 0.0) {
  const int lane = threadIdx.x & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  const double lam = A.lambda;
  StepOut o;
  o.dir = 0; o.vrow = -1; o.gamma = 0.0; o.num = 0.0; o.den = 0.0; o.hnew = 0.0;
  // <t_i, grad_i f>: operands fetched now, summed (rows ascending) once the
  // independent merged-support / denominator work below has been issued
  const double prod = PRE_DOT ? 0.0 : d_mul(tv, gk);
  double dv[8];
#pragma unroll
  for (int q = 0; q < 8; q++) dv[q] = PRE_DOT ? 0.0 : __shfl_sync(FULL, prod, q);
  auto finish_dot = [&]() {
    if (PRE_DOT) return dot_in;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (q >= c0) break;
      acc = d_add(acc, dv[q]);
    }
    for (int q = 8; q < c0; q++) acc = d_add(acc, __shfl_sync(FULL, prod, q));
    return acc;
  };
  double dot = 0.0;
  if (VAR != VAR_PLAIN) {
    dot = finish_dot();
    o.gfw = d_sub(dot, d_mul(bi, mv));
  }
  SP_MARK(8);
  o.abort = !(mv < 1.0e308 && mv > -1.0e308);
  double gv = dninf();
  int vrow = 0x7fffffff;
  if (VAR != VAR_PLAIN) {
    gv = lane < c0 ? gk : dninf();
    vrow = lane < c0 ? rw : 0x7fffffff;
    warp_argmax_redux(gv, vrow, lane < c0);
    o.vrow = vrow;
  }
  const bool j_in = __ballot_sync(FULL, lane < c0 && rw == j) != 0u;
  const int ins = __popc(__ballot_sync(FULL, lane < c0 && rw < j));
  // merged support supp(t_i) U {j}, rows ascending, one entry per lane
  const int M = c0 + (j_in ? 0 : 1);
  int src = (j_in || lane < ins) ? lane : lane - 1;
  if (src < 0) src = 0;
  int mrow = __shfl_sync(FULL, rw, src);
  double mt = __shfl_sync(FULL, tv, src);
  if (!j_in && lane == ins) { mrow = j; mt = 0.0; }
  const bool mvalid = lane < M;
  SP_MARK(9);
  // source marginal and row sum of the rows this lane may update (loads issued early)
  const double a_m = a[mvalid ? mrow : 0];
  const double a_s = (VAR == VAR_AWAY && lane < c0) ? a[rw] : 0.0;
  const double r_m = r[mvalid ? mrow : 0];
  const double r_s = (VAR != VAR_PLAIN && lane < c0) ? r[rw] : 0.0;

  double tnew = mt;
  bool use_merged = true;
  if (VAR == VAR_PLAIN) {
    const double d = d_sub((mvalid && mrow == j) ? bi : 0.0, mvalid ? mt : 0.0);
    const double D = d_add(0.0, d);
    o.den = warp_sparse_psum256_fast(m, M, mrow, d_mul(D, D));
    dot = finish_dot();
    o.gfw = d_sub(dot, d_mul(bi, mv));
    SP_MARK(10);
    o.num = d_mul(lam, d_add(0.0, o.gfw));
    if (A.step_rule == 1) {
      if (!(o.num > 0.0) || o.den == 0.0) o.gamma = 0.0;
      else { o.gamma = d_div(o.num, o.den); if (o.gamma > 1.0) o.gamma = 1.0; }
    } else {
      o.gamma = d_div((double)(2LL * n), (double)(kk + 2LL * n));
    }
    const double omg = d_sub(1.0, o.gamma), gb = d_mul(o.gamma, bi);
    tnew = d_mul(omg, mt);
    if (mrow == j) tnew = d_add(tnew, gb);
    SP_MARK(11);
  } else if (VAR != VAR_PLAIN && c0 == 0) {
    // zero-mass column (b_i = 0, R32): t_i = s_i = v_i = 0, every direction is zero: no-op
    o.dir = 3;
    o.vrow = -1;
  } else if (VAR == VAR_AWAY) {
    const double gaw = d_sub(d_mul(bi, gv), dot);
    const bool use_fw = (c0 == 1) || (o.gfw >= gaw);
    if (use_fw) {
      const double d = d_sub((mvalid && mrow == j) ? bi : 0.0, mvalid ? mt : 0.0);
      o.den = warp_sparse_psum256_fast(m, M, mrow, d_mul(d, d));
      o.num = d_mul(lam, d_add(o.gfw, 0.0));
      if (!(o.num > 0.0) || o.den == 0.0) o.gamma = 0.0;
      else { o.gamma = d_div(o.num, o.den); if (o.gamma > 1.0) o.gamma = 1.0; }
      const double omg = d_sub(1.0, o.gamma), gb = d_mul(o.gamma, bi);
      tnew = d_mul(omg, mt);
      if (mrow == j) tnew = d_add(tnew, gb);
    } else {
      o.dir = 1;
      use_merged = false;
      const double tvv = __shfl_sync(FULL, tv, __ffs(__ballot_sync(FULL, lane < c0 && rw == vrow)) - 1);
      const double d = (lane < c0) ? ((rw == vrow) ? d_sub(tv, bi) : tv) : 0.0;
      o.den = warp_sparse_psum256_fast(m, c0, rw, d_mul(d, d));
      o.num = d_mul(lam, d_add(gaw, 0.0));
      const double alpha = d_div(tvv, bi);
      const double gmax = d_div(alpha, d_sub(1.0, alpha));
      if (!(o.num > 0.0) || o.den == 0.0) o.gamma = 0.0;
      else { o.gamma = d_div(o.num, o.den); if (o.gamma > gmax) o.gamma = gmax; }
      const double opg = d_add(1.0, o.gamma), gb = d_mul(o.gamma, bi);
      tnew = d_mul(opg, tv);
      if (lane < c0 && rw == vrow) {
        tnew = d_sub(tnew, gb);
        if (o.gamma == gmax || tnew < 0.0) tnew = 0.0;
      }
    }
  } else {  // VAR_PAIR
    if (vrow == j) {
      o.dir = 3;
    } else {
      o.dir = 2;
      const double tvv = __shfl_sync(FULL, tv, __ffs(__ballot_sync(FULL, lane < c0 && rw == vrow)) - 1);
      const double dv = d_sub(gv, mv);
      o.num = d_mul(lam, dv);
      o.den = d_mul(2.0, bi);
      const double alpha = d_div(tvv, bi);
      if (!(o.num > 0.0)) o.gamma = 0.0;
      else { o.gamma = d_div(o.num, o.den); if (o.gamma > alpha) o.gamma = alpha; }
      double mu = d_mul(o.gamma, bi);
      const bool drop = (o.gamma == alpha) || (mu >= tvv);
      if (drop) mu = tvv;
      tnew = mt;
      if (mrow == j) tnew = d_add(mt, mu);
      if (mrow == vrow) tnew = drop ? 0.0 : d_sub(mt, mu);
    }
  }
  // apply: new column (exact zeros dropped), r += (t' - t), h refresh
  o.noop = (VAR != VAR_PLAIN && o.dir == 3);
  o.merged = use_merged;
  const int E = use_merged ? M : c0;
  const int erow = use_merged ? mrow : rw;
  const double eold = use_merged ? mt : tv;
  const double aval = use_merged ? a_m : a_s;
  if (o.noop) tnew = eold;
  const bool ev = lane < E;
  const bool keep = ev && tnew != 0.0;
  o.kmask = __ballot_sync(FULL, keep);
  o.nk = __popc(o.kmask);
  if (!o.noop && o.nk > cap) o.abort = true;
  SP_MARK(12);
  if (!o.abort && !o.noop) {
    if (ev) {
      const double Dp = d_add(0.0, d_sub(tnew, eold));
      const double rn = d_add(use_merged ? r_m : r_s, Dp);
      const double hn = lam == 1.0 ? d_sub(rn, aval) : d_div(d_sub(rn, aval), lam);   // x / 1 == x exactly
      r[erow] = rn;
      h[erow] = hn;
      o.hnew = hn;
      if (h32) h32[erow] = __double2float_rn(hn);
    }
    if (hmax) {
      // running upper bound of max_k |h_k| for the LMO filter window
      const float ah = ev ? __double2float_ru(fabs(h[erow])) : 0.f;
      const unsigned mb = __reduce_max_sync(FULL, (unsigned)__float_as_int(ah));
      if (lane == 0) *hmax = fmaxf(*hmax, __int_as_float((int)mb));
    }
    if (keep) {
      const int pos = __popc(o.kmask & ((1u << lane) - 1u));
      A.srow[(int64_t)i * cap + pos] = erow;
      A.sval[(int64_t)i * cap + pos] = tnew;
    }
    if (lane == 0) { A.cnt[i] = o.nk; if (cnt2) cnt2[i] = o.nk; }
  }
  SP_MARK(13);
  o.erow = erow;
  o.tnew = tnew;
  o.keep = keep;
  o.ev = ev && !o.abort && !o.noop;
  return o;
}

// lane p <- the p-th kept entry (ascending rows): the column's new support slab.
__device__ __forceinline__ void new_slab_entry(const StepOut& o, int& rw, double& tv) {
  const int lane = threadIdx.x & 31;
  const int srcl = lane < o.nk ? (int)__fns(o.kmask, 0, lane + 1) : 0;
  const int r2 = __shfl_sync(FULL, o.erow, srcl);
  const double t2 = __shfl_sync(FULL, o.tnew, srcl);
  rw = lane < o.nk ? r2 : 0x7fffffff;
  tv = lane < o.nk ? t2 : 0.0;
}

// Shared-memory layout of the persistent kernel (host and device agree):
// fixed | [SMEM: h, r, counts, h32] | [GA: G, fen] | [a] | [visits] | column region.
struct BcfwLayout {
  size_t fixed, state, ga, a, visit;
  __host__ __device__ static size_t fixed_bytes() {
    return 256 * 8 + BCFW_WARPS * 8 + BCFW_WARPS * 4 + 16 * 4 + 8 * 8;
  }
  __host__ __device__ static size_t state_bytes(int m, int n) {
    return 2 * rup16((size_t)m * 8) + rup16((size_t)n * 4) + rup16((size_t)m * 4);
  }
  __host__ __device__ static size_t ga_bytes(int n) { return rup16((size_t)n * 8) + rup16((size_t)(n + 1) * 8); }
  __host__ __device__ static size_t a_bytes(int m) { return rup16((size_t)m * 8); }
  __host__ __device__ static size_t visit_bytes(int steps) { return rup16((size_t)steps * 4); }
};

// ---------------------------------------------------------------------------
// The persistent kernel.
// ---------------------------------------------------------------------------
template <class Col, int VAR, bool GA, bool SMEM>
__global__ void __launch_bounds__(BCFW_THREADS, 1) k_bcfw(BcfwArgs A, Col col) {
  if (bcfw_halted(A)) return;
  extern __shared__ __align__(16) char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  double* slots = reinterpret_cast<double*>(smraw);                           // 256
  unsigned long long* wkey = reinterpret_cast<unsigned long long*>(slots + 256);  // 16
  int* wj = reinterpret_cast<int*>(wkey + BCFW_WARPS);                        // 16
  int* misc = wj + BCFW_WARPS;                                                // 16 ints
  double* miscd = reinterpret_cast<double*>(misc + 16);                       // 8
  float* hmaxp = reinterpret_cast<float*>(miscd + 6);                         // miscd[6..7] as floats
  char* p = smraw + BcfwLayout::fixed_bytes();
  double* sh_h = nullptr;
  double* sh_r = nullptr;
  int* sh_cnt = nullptr;
  float* sh_h32 = nullptr;
  if (SMEM) {
    sh_h = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
    sh_r = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
    sh_cnt = reinterpret_cast<int*>(p); p += rup16((size_t)n * 4);
    sh_h32 = reinterpret_cast<float*>(p); p += rup16((size_t)m * 4);
  }
  double* Gs = A.G;
  double* fens = A.fen;
  if (GA && A.ga_smem) {
    Gs = reinterpret_cast<double*>(p); p += rup16((size_t)n * 8);
    fens = reinterpret_cast<double*>(p); p += rup16((size_t)(n + 1) * 8);
  }
  const double* aa = A.a;
  if (A.a_smem) {
    double* sa = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
    for (int k = tid; k < m; k += BCFW_THREADS) sa[k] = A.a[k];
    aa = sa;
  }
  const int* vis = A.visit;
  if (!GA && A.visit_smem) {
    int* sv = reinterpret_cast<int*>(p); p += rup16((size_t)A.steps * 4);
    for (int q = tid; q < A.steps; q += BCFW_THREADS) sv[q] = A.visit[q];
    vis = sv;
  }
  col.setup(p);
  double* hs = SMEM ? sh_h : A.h;
  double* rr = SMEM ? sh_r : A.r;
  const int* cnt_rd = SMEM ? sh_cnt : A.cnt;
  const bool FILT = SMEM && Col::FILTER && m <= 4 * 4 * BCFW_THREADS;

  for (int c = tid; c < 256; c += BCFW_THREADS) slots[c] = 0.0;
  float hloc = 0.f;
  if (SMEM) {
    for (int k = tid; k < m; k += BCFW_THREADS) {
      const double hk = A.h[k];
      sh_h[k] = hk; sh_r[k] = A.r[k];
      sh_h32[k] = __double2float_rn(hk);
      hloc = fmaxf(hloc, __double2float_ru(fabs(hk)));
    }
    for (int c = tid; c < n; c += BCFW_THREADS) sh_cnt[c] = A.cnt[c];
  }
  if (GA && A.ga_smem) {
    for (int c = tid; c < n; c += BCFW_THREADS) Gs[c] = A.G[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) fens[c] = A.fen[c];
  }
  if (tid == 0) { misc[2] = 0; *hmaxp = 0.f; }
  __syncthreads();
  if (FILT) {
    const unsigned mb = __reduce_max_sync(FULL, (unsigned)__float_as_int(hloc));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(hmaxp), mb);   // non-negative floats order as ints
  }
  int i_cur = 0, i_nxt = 0;
  if (!GA && A.steps > 0) {
    i_cur = vis[0];
    i_nxt = A.steps > 1 ? vis[1] : i_cur;
    if (Col::STAGED) { col.issue(i_cur, 0); cp_async_wait_all(); }
  }
  __syncthreads();

  // warp 0's register copy of the visited column's support slab (prefetched)
  int rw = 0x7fffffff, c0 = 0;
  double tv = 0.0, bi = 0.0;
  if (!GA && warp == 0 && A.steps > 0) {
    c0 = cnt_rd[i_cur];
    bi = A.b[i_cur];
    if (lane < c0) { rw = A.srow[(int64_t)i_cur * cap + lane]; tv = A.sval[(int64_t)i_cur * cap + lane]; }
  }
  int done = 0;
#ifdef SRO_PHASE_TIMING
  PhaseState ph_state;
  for (int q = 0; q < 16; q++) ph_state.acc[q] = 0;
  ph_state.t = clock64();
  PhaseState* g_ph = &ph_state;
#endif
  for (int s = 0; s < A.steps; s++) {
    const long long kk = A.k0 + s;
    const int slot = s & 1;
    int i;
    if (GA) {
      if (tid == 0) misc[0] = ga_draw(fens, Gs, n, uniform53(rng_u64(A.seed, 1, (uint64_t)kk)));
      __syncthreads();
      i = misc[0];
      if (Col::STAGED) { col.issue(i, slot); cp_async_wait_all(); __syncthreads(); }
    } else {
      i = i_cur;
      if (Col::STAGED && s + 1 < A.steps) col.issue(i_nxt, slot ^ 1);      // lands during this step
    }
    PHASE_MARK(0);
    // ---- LMO (Eq. 9): CTA argmin of c_i + h, lowest row on ties
    double best = dinf();
    int bj = 0x7fffffff;
    if (FILT) {
      const float delta = __double2float_ru(d_add(d_mul(0x1p-22, d_add(A.cmax, d_mul(2.0, (double)*hmaxp))), 1e-30));
      col.local_argmin_filt(slot, hs, sh_h32, delta, best, bj);
    } else {
      col.local_argmin(i, slot, hs, best, bj);
    }
    PHASE_MARK(1);
    unsigned long long key = okey(best);
    warp_argmin_redux(key, bj);
    if (lane == 0) { wkey[warp] = key; wj[warp] = bj; }
    PHASE_MARK(2);
    __syncthreads();
    PHASE_MARK(3);
    if (warp == 0) {
      unsigned long long k2 = lane < BCFW_WARPS ? wkey[lane] : ~0ULL;
      int j = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
      warp_argmin_redux(k2, j);
      const double mv = okey_inv(k2);
      PHASE_MARK(4);
      if (GA) {
        c0 = cnt_rd[i];
        bi = A.b[i];
        rw = 0x7fffffff; tv = 0.0;
        if (lane < c0) { rw = A.srow[(int64_t)i * cap + lane]; tv = A.sval[(int64_t)i * cap + lane]; }
      }
      const double gk = lane < c0 ? d_add(col.cost(rw, i, slot), hs[rw]) : 0.0;
      const StepOut o = serial_step<VAR>(A, kk, i, j, mv, bi, c0, rw, tv, gk, rr, hs, FILT ? sh_h32 : nullptr, aa,
                                         SMEM ? sh_cnt : nullptr, slots, FILT ? hmaxp : nullptr SP_ARG);
      PHASE_MARK(5);
      if (lane == 0) {
        miscd[1] = o.gfw;
        if (o.abort) {
          misc[2] = 1;
          set_status(A.status, !(mv < 1.0e308 && mv > -1.0e308) ? 5 : 6);
        } else if (A.trace) {
          double* tr = A.trace + 9 * (int64_t)s;
          tr[0] = (double)kk; tr[1] = i; tr[2] = j; tr[3] = (VAR == VAR_PLAIN) ? -1 : o.vrow;
          tr[4] = o.dir; tr[5] = o.gamma; tr[6] = o.num; tr[7] = o.den; tr[8] = mv;
        }
      }
      if (!o.abort) {
        if (GA || i_nxt == i) {
          // column i stays in hand (GA post-update refresh, or the same column next)
          new_slab_entry(o, rw, tv);
          c0 = o.nk;
        } else if (s + 1 < A.steps) {
          // prefetch the next visited column's slab into warp-0 registers
          c0 = cnt_rd[i_nxt];
          bi = A.b[i_nxt];
          rw = 0x7fffffff; tv = 0.0;
          if (lane < c0) { rw = A.srow[(int64_t)i_nxt * cap + lane]; tv = A.sval[(int64_t)i_nxt * cap + lane]; }
        }
      }
    }
    if (!GA) { i_cur = i_nxt; i_nxt = (s + 2 < A.steps) ? vis[s + 2] : i_nxt; }
    PHASE_MARK(6);
    if (!GA && Col::STAGED) cp_async_wait_all();
    __syncthreads();
    PHASE_MARK(7);
    if (misc[2]) break;
    // ---- GA: refresh the visited column's stored gap (Alg. A.4 line 6)
    if (GA && A.ga_inner) {
      if (A.ga_post) {
        double b2 = dinf();
        int j2 = 0x7fffffff;
        if (FILT) {
          const float delta = __double2float_ru(d_add(d_mul(0x1p-22, d_add(A.cmax, d_mul(2.0, (double)*hmaxp))), 1e-30));
          col.local_argmin_filt(slot, hs, sh_h32, delta, b2, j2);
        } else {
          col.local_argmin(i, slot, hs, b2, j2);
        }
        unsigned long long key2 = okey(b2);
        warp_argmin_redux(key2, j2);
        if (lane == 0) { wkey[warp] = key2; wj[warp] = j2; }
        __syncthreads();
        if (warp == 0) {
          unsigned long long k3 = lane < BCFW_WARPS ? wkey[lane] : ~0ULL;
          int jj2 = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
          warp_argmin_redux(k3, jj2);
          const double mv2 = okey_inv(k3);
          const double term = lane < c0 ? d_mul(tv, d_add(col.cost(rw, i, slot), hs[rw])) : 0.0;
          const double dot2 = warp_seq_sum(term, c0);
          const double gnew = d_sub(dot2, d_mul(bi, mv2));
          if (lane == 0) {
            const double delta = d_sub(wpos(gnew), wpos(Gs[i]));
            Gs[i] = gnew;
            ga_add(fens, n, i, delta);
          }
        }
      } else if (tid == 0) {
        const double gnew = miscd[1];
        const double delta = d_sub(wpos(gnew), wpos(Gs[i]));
        Gs[i] = gnew;
        ga_add(fens, n, i, delta);
      }
      __syncthreads();
    }
    done = s + 1;
  }
  __syncthreads();
  if (SMEM) {
    for (int k = tid; k < m; k += BCFW_THREADS) { A.h[k] = sh_h[k]; A.r[k] = sh_r[k]; }
  }
  if (GA && A.ga_smem) {
    for (int c = tid; c < n; c += BCFW_THREADS) A.G[c] = Gs[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) A.fen[c] = fens[c];
  }
  if (tid == 0) *A.steps_done = done;
#ifdef SRO_PHASE_TIMING
  if (tid == 0 && A.phase) for (int q = 0; q < 16; q++) A.phase[q] += ph_state.acc[q];
#endif
}

// ---------------------------------------------------------------------------
// Register-file variant for dense costs (the config [0]/[1] path).
// Thread t owns the rows of the 128-bit vectors q = t + u*NT (u < MAXV) plus one
// tail row; it keeps those rows of h (fp64) in registers for the whole segment
// and prefetches its part of the next visited column into registers one step
// ahead, so the LMO touches neither shared nor global memory. Warp 0 keeps the
// master copies of h and r in shared memory; after each update it publishes
// the touched rows in a small list and marks their owners dirty, and each
// owner refreshes its registers at the next step (a shared-memory
// LMO costs ~1250 cycles per step, a register-file LMO ~420).
// ---------------------------------------------------------------------------
template <typename T, int MAXV>
struct RegCol {
  using V = typename Vec<T>::type;
  static constexpr int W = Vec<T>::W;
  const T* C;
  int64_t ld;
  int m, nvec;
  V cur[MAXV], nxt[MAXV];
  T ctail, ntail;
  __device__ __forceinline__ void fetch(int i) {
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld);
#pragma unroll
    for (int u = 0; u < MAXV; u++) {
      const int q = threadIdx.x + u * BCFW_THREADS;
      if (q < nvec) nxt[u] = __ldg(p + q);
    }
    const int kt = nvec * W + threadIdx.x;
    if (kt < m) ntail = __ldg(C + (int64_t)i * ld + kt);
  }
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int u = 0; u < MAXV; u++) cur[u] = nxt[u];
    ctail = ntail;
  }
};

__device__ __forceinline__ void vproc(const float4& v, const double* hd, int k, double& best, int& bj) {
  const double x0 = d_add((double)v.x, hd[0]), x1 = d_add((double)v.y, hd[1]);
  const double x2 = d_add((double)v.z, hd[2]), x3 = d_add((double)v.w, hd[3]);
  if (x0 < best) { best = x0; bj = k; }
  if (x1 < best) { best = x1; bj = k + 1; }
  if (x2 < best) { best = x2; bj = k + 2; }
  if (x3 < best) { best = x3; bj = k + 3; }
}
__device__ __forceinline__ void vproc(const double2& v, const double* hd, int k, double& best, int& bj) {
  const double x0 = d_add(v.x, hd[0]), x1 = d_add(v.y, hd[1]);
  if (x0 < best) { best = x0; bj = k; }
  if (x1 < best) { best = x1; bj = k + 1; }
}

struct RfLayout {
  __host__ __device__ static size_t bytes(int m, int n, int steps, bool ga_smem, bool visit_smem) {
    size_t b = 256 * 8 + BCFW_WARPS * 8 + BCFW_WARPS * 4 + 16 * 4 + 8 * 8;   // fixed
    b += 32 * 4 + 32 * 8 + rup16(BCFW_THREADS);                               // update list + dirty flags
    b += 3 * rup16((size_t)m * 8) + rup16((size_t)n * 4);                     // h, r, a, counts
    if (ga_smem) b += rup16((size_t)n * 8) + rup16((size_t)(n + 1) * 8);
    if (visit_smem) b += rup16((size_t)steps * 4);
    return b;
  }
};

template <typename T, int MAXV, int VAR, bool GA>
__global__ void __launch_bounds__(BCFW_THREADS, 1) k_bcfw_rf(BcfwArgs A, const T* __restrict__ Cg, int64_t ld) {
  if (bcfw_halted(A)) return;
  using Col = RegCol<T, MAXV>;
  constexpr int W = Col::W;
  extern __shared__ __align__(16) char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  double* slots = reinterpret_cast<double*>(smraw);
  unsigned long long* wkey = reinterpret_cast<unsigned long long*>(slots + 256);
  int* wj = reinterpret_cast<int*>(wkey + BCFW_WARPS);
  int* misc = wj + BCFW_WARPS;                                   // [0]=i [2]=abort [3]=upd count
  double* miscd = reinterpret_cast<double*>(misc + 16);
  char* p = smraw + (256 * 8 + BCFW_WARPS * 8 + BCFW_WARPS * 4 + 16 * 4 + 8 * 8);
  int* upd_row = reinterpret_cast<int*>(p); p += 32 * 4;
  double* upd_h = reinterpret_cast<double*>(p); p += 32 * 8;
  unsigned char* dirty = reinterpret_cast<unsigned char*>(p); p += rup16(BCFW_THREADS);
  double* sh_h = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_r = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_a = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  int* sh_cnt = reinterpret_cast<int*>(p); p += rup16((size_t)n * 4);
  // GA: stored gaps and Fenwick tree always in shared memory here (the host
  // falls back to the generic kernel when they do not fit)
  double* Gs = reinterpret_cast<double*>(p);
  double* fens = reinterpret_cast<double*>(p + rup16((size_t)n * 8));
  if (GA) p += rup16((size_t)n * 8) + rup16((size_t)(n + 1) * 8);
  const int* vis = A.visit;
  if (!GA && A.visit_smem) {
    int* sv = reinterpret_cast<int*>(p); p += rup16((size_t)A.steps * 4);
    for (int q = tid; q < A.steps; q += BCFW_THREADS) sv[q] = A.visit[q];
    vis = sv;
  }
  for (int c = tid; c < 256; c += BCFW_THREADS) slots[c] = 0.0;
  for (int k = tid; k < m; k += BCFW_THREADS) { sh_h[k] = A.h[k]; sh_r[k] = A.r[k]; sh_a[k] = A.a[k]; }
  for (int c = tid; c < n; c += BCFW_THREADS) sh_cnt[c] = A.cnt[c];
  if (GA) {
    for (int c = tid; c < n; c += BCFW_THREADS) Gs[c] = A.G[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) fens[c] = A.fen[c];
  }
  dirty[tid] = 0;
  if (tid == 0) { misc[2] = 0; misc[3] = 0; }
  Col col;
  col.C = Cg; col.ld = ld; col.m = m; col.nvec = m / W;
  // owned rows of h in registers
  double hd[MAXV * W];
  double htail = 0.0;
  const int kt = col.nvec * W + tid;
#pragma unroll
  for (int u = 0; u < MAXV; u++) {
    const int q = tid + u * BCFW_THREADS;
#pragma unroll
    for (int t = 0; t < W; t++) hd[u * W + t] = q < col.nvec ? A.h[W * q + t] : 0.0;
  }
  if (kt < m) htail = A.h[kt];
  int i_cur = 0, i_nxt = 0;
  if (!GA && A.steps > 0) {
    i_cur = A.visit[0];
    i_nxt = A.steps > 1 ? A.visit[1] : i_cur;
    col.fetch(i_cur);
  }
  __syncthreads();

  int rw = 0x7fffffff, c0 = 0;
  double tv = 0.0, bi = 0.0, cw = 0.0;
  int rwn = 0x7fffffff, c0n = 0;         // next visited column's slab (prefetched)
  double tvn = 0.0, bin = 0.0;
  if (!GA && warp == 0 && A.steps > 0) {
    c0 = sh_cnt[i_cur];
    bi = A.b[i_cur];
    if (lane < c0) { rw = A.srow[(int64_t)i_cur * cap + lane]; tv = A.sval[(int64_t)i_cur * cap + lane]; }
    if (lane < c0) cw = (double)__ldg(Cg + (int64_t)i_cur * ld + rw);
  }
  int done = 0;
#ifdef SRO_PHASE_TIMING
  PhaseState ph_state;
  for (int q = 0; q < 16; q++) ph_state.acc[q] = 0;
  ph_state.t = clock64();
  PhaseState* g_ph = &ph_state;
#endif
  for (int s = 0; s < A.steps; s++) {
    const long long kk = A.k0 + s;
    int i;
    // ---- refresh owned h registers touched by the previous step
    if (dirty[tid]) {
      dirty[tid] = 0;
      const int nu = misc[3];
      for (int e = 0; e < nu; e++) {
        const int k = upd_row[e];
        const double hv = upd_h[e];
#pragma unroll
        for (int u = 0; u < MAXV; u++)
#pragma unroll
          for (int t = 0; t < W; t++)
            if (k == W * (tid + u * BCFW_THREADS) + t) hd[u * W + t] = hv;
        if (k == kt) htail = hv;
      }
    }
    if (GA) {
      if (tid == 0) misc[0] = ga_draw_sh(fens, Gs, n, uniform53(rng_u64(A.seed, 1, (uint64_t)kk)));
      __syncthreads();
      i = misc[0];
      col.fetch(i);
      if (warp == 0) {            // slab of the drawn column, overlapping the column fetch
        c0 = sh_cnt[i];
        bi = A.b[i];
        rw = 0x7fffffff; tv = 0.0;
        if (lane < c0) { rw = A.srow[(int64_t)i * cap + lane]; tv = A.sval[(int64_t)i * cap + lane]; }
      }
      col.advance();
    } else {
      i = i_cur;
      col.advance();
      if (s + 1 < A.steps) col.fetch(i_nxt);                      // lands during this step
      if (warp == 0 && s + 1 < A.steps && i_nxt != i) {           // next slab, a step ahead
        c0n = sh_cnt[i_nxt];
        bin = A.b[i_nxt];
        rwn = 0x7fffffff; tvn = 0.0;
        if (lane < c0n) { rwn = A.srow[(int64_t)i_nxt * cap + lane]; tvn = A.sval[(int64_t)i_nxt * cap + lane]; }
      }
    }
    PHASE_MARK(0);
    // ---- LMO (Eq. 9) from registers: CTA argmin of c_i + h, lowest row on ties
    double best = dinf();
    int bj = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < MAXV; u++) {
      const int q = tid + u * BCFW_THREADS;
      if (q < col.nvec) vproc(col.cur[u], hd + u * W, W * q, best, bj);
    }
    if (kt < m) {
      const double x = d_add((double)col.ctail, htail);
      if (x < best) { best = x; bj = kt; }
    }
    PHASE_MARK(1);
    unsigned long long key = okey(best);
    warp_argmin_redux(key, bj);
    if (lane == 0) { wkey[warp] = key; wj[warp] = bj; }
    PHASE_MARK(2);
    __syncthreads();
    PHASE_MARK(3);
    if (warp == 0) {
      unsigned long long k2 = lane < BCFW_WARPS ? wkey[lane] : ~0ULL;
      int j = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
      warp_argmin_redux(k2, j);
      const double mv = okey_inv(k2);
      PHASE_MARK(4);
      if (GA && lane < c0) cw = (double)__ldg(Cg + (int64_t)i * ld + rw);
      const double gk = lane < c0 ? d_add(cw, sh_h[rw]) : 0.0;
      const StepOut o = serial_step<VAR>(A, kk, i, j, mv, bi, c0, rw, tv, gk, sh_r, sh_h, nullptr, sh_a, sh_cnt, slots,
                                         nullptr SP_ARG);
      PHASE_MARK(5);
      // publish the touched rows of h for their register owners
      if (o.ev) {
        upd_row[lane] = o.erow;
        upd_h[lane] = o.hnew;
        const int kr = o.erow;
        const int owner = kr < col.nvec * W ? (kr / W) % BCFW_THREADS : kr - col.nvec * W;
        dirty[owner] = 1;
      }
      const unsigned evm = __ballot_sync(FULL, o.ev);
      if (lane == 0) {
        misc[3] = __popc(evm);
        miscd[1] = o.gfw;
        if (o.abort) {
          misc[2] = 1;
          set_status(A.status, !(mv < 1.0e308 && mv > -1.0e308) ? 5 : 6);
        } else if (A.trace) {
          double* tr = A.trace + 9 * (int64_t)s;
          tr[0] = (double)kk; tr[1] = i; tr[2] = j; tr[3] = (VAR == VAR_PLAIN) ? -1 : o.vrow;
          tr[4] = o.dir; tr[5] = o.gamma; tr[6] = o.num; tr[7] = o.den; tr[8] = mv;
        }
      }
      if (!o.abort) {
        if (GA || i_nxt == i) {
          new_slab_entry(o, rw, tv);
          c0 = o.nk;
          if (!GA && lane < c0) cw = (double)__ldg(Cg + (int64_t)i * ld + rw);
        } else if (s + 1 < A.steps) {
          c0 = c0n; bi = bin; rw = rwn; tv = tvn;
          if (lane < c0) cw = (double)__ldg(Cg + (int64_t)i_nxt * ld + rw);   // consumed next step
        }
      }
    }
    if (!GA) { i_cur = i_nxt; i_nxt = (s + 2 < A.steps) ? vis[s + 2] : i_nxt; }
    PHASE_MARK(6);
    __syncthreads();
    PHASE_MARK(7);
    if (misc[2]) break;
    // ---- GA: refresh the visited column's stored gap (Alg. A.4 line 6)
    if (GA && A.ga_inner) {
      if (A.ga_post) {
        if (dirty[tid]) {
          dirty[tid] = 0;
          const int nu = misc[3];
          for (int e = 0; e < nu; e++) {
            const int k = upd_row[e];
            const double hv = upd_h[e];
#pragma unroll
            for (int u = 0; u < MAXV; u++)
#pragma unroll
              for (int t = 0; t < W; t++)
                if (k == W * (tid + u * BCFW_THREADS) + t) hd[u * W + t] = hv;
            if (k == kt) htail = hv;
          }
        }
        double b2 = dinf();
        int j2 = 0x7fffffff;
#pragma unroll
        for (int u = 0; u < MAXV; u++) {
          const int q = tid + u * BCFW_THREADS;
          if (q < col.nvec) vproc(col.cur[u], hd + u * W, W * q, b2, j2);
        }
        if (kt < m) {
          const double x = d_add((double)col.ctail, htail);
          if (x < b2) { b2 = x; j2 = kt; }
        }
        unsigned long long key2 = okey(b2);
        warp_argmin_redux(key2, j2);
        if (lane == 0) { wkey[warp] = key2; wj[warp] = j2; }
        __syncthreads();
        if (warp == 0) {
          unsigned long long k3 = lane < BCFW_WARPS ? wkey[lane] : ~0ULL;
          int jj2 = lane < BCFW_WARPS ? wj[lane] : 0x7fffffff;
          warp_argmin_redux(k3, jj2);
          const double mv2 = okey_inv(k3);
          const double c2 = lane < c0 ? (double)__ldg(Cg + (int64_t)i * ld + rw) : 0.0;
          const double term = lane < c0 ? d_mul(tv, d_add(c2, sh_h[rw])) : 0.0;
          const double dot2 = warp_seq_sum(term, c0);
          const double gnew = d_sub(dot2, d_mul(bi, mv2));
          const double delta = d_sub(wpos(gnew), wpos(Gs[i]));
          __syncwarp();
          ga_add_warp(fens, n, i, delta);
          if (lane == 0) { Gs[i] = gnew; misc[3] = 0; }
        }
      } else if (warp == 0) {
        const double gnew = miscd[1];
        const double delta = d_sub(wpos(gnew), wpos(Gs[i]));
        __syncwarp();
        ga_add_warp(fens, n, i, delta);
        if (lane == 0) Gs[i] = gnew;
      }
      __syncthreads();
    }
    done = s + 1;
  }
  __syncthreads();
  for (int k = tid; k < m; k += BCFW_THREADS) { A.h[k] = sh_h[k]; A.r[k] = sh_r[k]; }
  if (GA) {
    for (int c = tid; c < n; c += BCFW_THREADS) A.G[c] = Gs[c];
    for (int c = tid; c <= n; c += BCFW_THREADS) A.fen[c] = fens[c];
  }
  if (tid == 0) *A.steps_done = done;
#ifdef SRO_PHASE_TIMING
  if (tid == 0 && A.phase) for (int q = 0; q < 16; q++) A.phase[q] += ph_state.acc[q];
#endif
}

// Fenwick rebuild after a GA global refresh: fen[i] = max(G_{i-1}, 0), then
// the standard linear build (R14), in order, in shared memory when it fits.
__global__ void k_fen_build(const double* __restrict__ G, double* fen, int n, int use_smem, const int* stop) {
  if (stop && *stop) return;   // a failed segment: keep the tree as it is
  extern __shared__ double fs[];
  double* f = use_smem ? fs : fen;
  for (int i = threadIdx.x; i <= n; i += blockDim.x) f[i] = i == 0 ? 0.0 : wpos(G[i - 1]);
  __syncthreads();
  // The build `for i = 1..n: fen[i + lowbit(i)] += fen[i]` adds into node p its children
  // i = p - 2^(k-1), ..., p - 2, p - 1 (lowbit(p) = 2^k) in that (increasing) order, each
  // already complete: done level by level (nodes of one lowbit in parallel), the same sums.
  for (int k = 1; (1 << k) <= n; k++) {
    const int step = 1 << (k + 1), first = 1 << k;
    for (int p = first + threadIdx.x * step; p <= n; p += blockDim.x * step) {
      double v = f[p];
      for (int jb = k - 1; jb >= 0; jb--) v = d_add(v, f[p - (1 << jb)]);
      f[p] = v;
    }
    __syncthreads();
  }
  if (use_smem) for (int i = threadIdx.x; i <= n; i += blockDim.x) fen[i] = f[i];
}

}  // namespace sro
