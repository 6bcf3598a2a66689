// k_block_tail.cuh — the whole post-LMO part of a plain step over a small
// column set (|U| <= 1024: batched blocks, FW on small n) in ONE CTA with the
// step's pairs resident in shared memory (the global-memory tail of
// k_block.cuh spends its time on dependent L2 round trips between ~15
// barrier phases).
//
// Same arithmetic and summation shapes as every other block step (R19):
//   * the merged supports supp(t_i) U {j_i} become (row, pair) keys,
//     key = row << 12 | q with q the pair index (q ascends with the column
//     position), sorted in shared memory (bitonic);
//   * along a row the sorted keys are in ascending position, so one thread
//     per row sums each (row, chunk) run left to right from +0.0 and combines
//     the run partials — chunks ascending — with an O(runs) stack evaluation
//     of the 256-leaf adjacent-pair tree (zero leaves are identities);
//   * the denominator is the 256-chunk sum over the m rows of Delta_k^2 with the
//     touched rows (ascending) found per chunk by binary search.
// When the LMO sweep left per-slab partials, the tail merges them itself
// (thread per column, slab order) and evaluates the column gaps (Eq. 11) —
// the k_lmo_merge launch folded into this one.
// Steps whose pair count exceeds TS_PMAX run the global-memory tail instead.
// Host side: used for L <= 1024 and m < 2^20 (the row field of a key).
#pragma once
#include "k_block.cuh"
#include "k_sweep.cuh"

namespace sro {

// The sweep's slab partials and the cost source for the gap epilogue.
struct TailMerge {
  int nslabs;            // <= 1: the sweep wrote the final j / minval / g itself
  const int* pj;         // [nslabs * L] partial argmin rows
  const double* pmin;    // [nslabs * L] partial minima
  int* j;                // outputs over U (the arrays BlockArgs::j / minval / g read)
  double* minval;
  double* g;
  int kind;              // 0/1 dense f32/f64; 2/3 colour f32 sqeuclid/euclid; 4/5 colour f64 sqeuclid/euclid
  const void* C;
  int64_t ld;
  const void* x;
  const void* y;
  // the sweep's staged supports (nslabs > 1; k_sweep.cuh stage_support): size, first SW_KP
  // entries entry-major, b
  const int* st_cnt;
  const int* st_row;
  const double* st_val;
  const double* st_b;
  const double* st_term;   // the staged gap terms (k_sweep.cuh stage_terms), or nullptr
};
__device__ __forceinline__ double tm_cost(const TailMerge& M, int k, int i) {
  switch (M.kind) {
    case 0: return SrcDense<float>{(const float*)M.C, M.ld}.cost(k, i);
    case 1: return SrcDense<double>{(const double*)M.C, M.ld}.cost(k, i);
    case 2: return SrcColour<float, false>{(const float*)M.x, (const float*)M.y}.cost(k, i);
    case 3: return SrcColour<float, true>{(const float*)M.x, (const float*)M.y}.cost(k, i);
    case 4: return SrcColour<double, false>{(const double*)M.x, (const double*)M.y}.cost(k, i);
    default: return SrcColour<double, true>{(const double*)M.x, (const double*)M.y}.cost(k, i);
  }
}

constexpr int TS_PMAX = 4096;   // pairs held in shared memory
constexpr int TS_SORT = 8192;   // bitonic buffer (power of two >= TS_PMAX)
constexpr int TS_RADIX_HIST = 128 * 4 * 32;   // radix-sort histogram: 2^7 digits x 4 rounds x 32 warps

struct TailSmem {
  uint32_t key[TS_SORT];
  union {
    double pd[TS_PMAX];   // s - t, then t' - t
    double rX[TS_PMAX];   // Delta_k^2 of the touched rows (after the Delta run sums)
  };
  double ptold[TS_PMAX];
  int prow[TS_PMAX];
  uint8_t pchunk[TS_PMAX];  // 256-chunk of the pair's column position
  union {
    struct {
      double runv[TS_PMAX];   // (row, chunk) run sums, sorted order
      uint8_t runc[TS_PMAX];  // their chunks
      uint16_t runu[TS_PMAX + 1];  // their first sorted index
      int rowrun[TS_PMAX + 1];  // touched row -> its first run
      int rrow[TS_PMAX];      // touched rows, ascending
    };
    int rcnt[TS_RADIX_HIST];  // radix sort by row (before the runs exist): per-(digit, round, warp) counts
  };
  int hot[TS_PMAX / 8];   // touched rows with more than TS_SMALL (= 8) runs
  int mid[TS_PMAX / 3];   // touched rows with 3 .. TS_SMALL runs
  double gcol[1024];       // column gaps over U (G_U = psum256 of them)
  int wsum[32];
  int misc[8];            // [0] touched rows [1] runs [2] hot rows [3] abort flag [5] mid rows
  double red[8];
  double bc[4];           // broadcasts: [2] gamma
  long long tsacc[16];    // SRO_PHASE_TIMING builds: phase clocks (thread 0), added to A.phase at exit
};
static_assert(sizeof(TailSmem) + 1408 <= 232448, "k_block_tail_sm shared memory");
constexpr size_t TAIL_SM_BYTES = sizeof(TailSmem) > 32 * 256 * 8 ? sizeof(TailSmem) : 32 * 256 * 8;

// Ascending bitonic sort of the P keys in buf[0, P) (Pp = 1024 E >= P, buf holds 2 Pp
// with positions [P, Pp) of both halves set to the maximal key): every merge of
// block size k starts by comparing u with its mirror u ^ (k - 1), then halves
// with u ^ jj, always keeping the minimum at the lower index, so the padding
// stays at positions >= P.
// Thread t owns keys [t E, t E + E): exchanges inside a thread in registers,
// inside a warp by shuffles, across warps through alternating halves of buf
// (one barrier per stage). Result back in buf[0, Pp). (Skipping the compares of
// warps that hold only padding measured slower on B200: kept uniform.)
template <int E>
__device__ __forceinline__ void ts_sort(uint32_t* buf, int Pp, int P) {
  const int t = threadIdx.x;
  uint32_t x[E];
#pragma unroll
  for (int e = 0; e < E; e++) x[e] = buf[t * E + e];
  int half = 1;
  for (int k = 2; k <= Pp; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      const bool mirror = jj == (k >> 1);
      const int pm = mirror ? k - 1 : jj;   // partner of u: u ^ pm
      if (pm < E) {
#pragma unroll
        for (int c = 1; c < E; c++) {
          if (c != pm) continue;
#pragma unroll
          for (int e = 0; e < E; e++) {
            const int f = e ^ c;
            if (f <= e) continue;
            const uint32_t a = x[e], b = x[f];
            x[e] = min(a, b);
            x[f] = max(a, b);
          }
        }
      } else if (pm < 32 * E) {
        const int lx = pm / E;
        uint32_t y[E];
#pragma unroll
        for (int e = 0; e < E; e++) y[e] = __shfl_xor_sync(FULL, mirror ? x[E - 1 - e] : x[e], lx);
#pragma unroll
        for (int e = 0; e < E; e++) {
          const int u = t * E + e;
          const bool low = (u & jj) == 0;
          x[e] = low ? min(x[e], y[e]) : max(x[e], y[e]);
        }
      } else {
        uint32_t* hb = buf + half * Pp;
#pragma unroll
        for (int e = 0; e < E; e++) hb[t * E + e] = x[e];
        __syncthreads();
        uint32_t y[E];
#pragma unroll
        for (int e = 0; e < E; e++) y[e] = hb[(t * E + e) ^ pm];
#pragma unroll
        for (int e = 0; e < E; e++) {
          const int u = t * E + e;
          const bool low = (u & jj) == 0;
          x[e] = low ? min(x[e], y[e]) : max(x[e], y[e]);
        }
        half ^= 1;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; e++) buf[t * E + e] = x[e];
  __syncthreads();
}

// Block-wide exclusive scan of one int per thread (1024 threads); returns the
// thread's offset, *total the sum.
__device__ __forceinline__ int block_scan1024(int x, int* wsum, int* total) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int incl = x;
  for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(FULL, incl, o); if (lane >= o) incl += v; }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int s = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(FULL, s, o); if (lane >= o) s += v; }
    wsum[lane] = s;
  }
  __syncthreads();
  const int off = incl - x + (w ? wsum[w - 1] : 0);
  *total = wsum[31];
  __syncthreads();
  return off;
}

#ifdef SRO_PHASE_TIMING
#define TS_MARK(idx)                                                     \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long t_ = clock64();                                    \
      S.tsacc[idx] += t_ - ts_t;                                         \
      ts_t = t_;                                                         \
    }                                                                    \
  } while (0)
#else
#define TS_MARK(idx) do {} while (0)
#endif

// Keys (row << 12 | q), held at index q, sorted by row with a stable LSD radix sort (digits
// of at most 7 row bits, 2 passes for m <= 16384): key q lives in round e = q / 1024 of thread
// q % 1024; per pass every warp ranks its keys of a round by digit (match.any: lanes in order),
// the per-(digit, round, warp) counts are scanned in that order, and each key is scattered to
// its digit's base + its rank — stable, so the final order is (row, q): the order of the
// bitonic sort (the keys are unique). Histogram in S.rcnt (128 x E x 32 ints).
template <int E>
__device__ __forceinline__ void ts_radix_sort(TailSmem& S, int P, int m) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int nbits = m > 1 ? 32 - __clz(m - 1) : 1;
  const int passes = (nbits + 6) / 7;
  const int db = max(5, (nbits + passes - 1) / passes);   // >= 32 digits: every warp's scan segment is whole
  const int nd = 1 << db;
  const int NH = nd * E * 32;
  uint32_t* src = S.key;
  uint32_t* dst = S.key + TS_PMAX;
  int* hist = S.rcnt;
  for (int pass = 0, shift = 12; pass < passes; pass++, shift += db) {
    for (int q = t; q < NH; q += 1024) hist[q] = 0;
    __syncthreads();
    uint32_t k[E];
    int dg[E], rk[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int idx = e * 1024 + t;
      const bool valid = idx < P;
      k[e] = valid ? src[idx] : 0u;
      dg[e] = valid ? (int)((k[e] >> shift) & (unsigned)(nd - 1)) : -1;
      const unsigned mask = __match_any_sync(FULL, dg[e]);
      rk[e] = __popc(mask & lt_mask);
      if (valid && rk[e] == 0) hist[(dg[e] * E + e) * 32 + w] = __popc(mask);
    }
    __syncthreads();
    // exclusive scan of hist in index order: warp w owns NH / 32 consecutive entries
    {
      const int seg = NH >> 5, base = w * seg;
      int carry = 0;
      for (int it = 0; it < seg; it += 32) {
        const int v = hist[base + it + lane];
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, incl, o); if (lane >= o) incl += y; }
        hist[base + it + lane] = carry + incl - v;
        carry += __shfl_sync(FULL, incl, 31);
      }
      if (lane == 0) S.wsum[w] = carry;
      __syncthreads();
      if (w == 0) {
        int v = S.wsum[lane], incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, incl, o); if (lane >= o) incl += y; }
        S.wsum[lane] = incl - v;
      }
      __syncthreads();
      const int add = S.wsum[w];
      for (int it = 0; it < seg; it += 32) hist[base + it + lane] += add;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++)
      if (dg[e] >= 0) dst[hist[(dg[e] * E + e) * 32 + w] + rk[e]] = k[e];
    __syncthreads();
    uint32_t* tmp = src; src = dst; dst = tmp;
  }
  if (src != S.key) {
    for (int q = t; q < P; q += 1024) S.key[q] = src[q];
    __syncthreads();
  }
}

// Per-row sums over the sorted pairs (R19), in two parts. ts_structure (once
// per step; the pair set and its order are the same for Delta and Delta'):
// the (row, chunk) runs of the sorted keys (start index runu, chunk runc), the
// touched rows ascending (rrow) with their first run (rowrun), and the rows
// with more than TS_SMALL runs (hot), 3 .. TS_SMALL runs (mid). ts_sums<MODE>(vals): thread
// per run sums it left to right from +0.0; thread per touched row with one or two runs, or with
// 3 .. TS_SMALL runs (adjacent runs merged deepest common ancestor first);
// warp per hot row: lane l gathers chunks [8l, 8l+8), tree8 + butterfly (the
// dense tree with zero leaves). MODE 0: rX (Delta_k^2, for the denominator;
// rX aliases the pair values, dead by then); MODE 1: r_k += D,
// h_k = (r_k - a_k)/lambda.
constexpr int TS_SMALL = 8;   // TailSmem::hot holds P / (TS_SMALL + 1) rows
template <int E>
__device__ __forceinline__ void ts_structure(TailSmem& S, int P) {
  const int t = threadIdx.x;
  uint32_t key[E + 1];
#pragma unroll
  for (int e = 0; e <= E; e++) {
    const int u = t * E + e - 1;
    key[e] = (u >= 0 && u < P) ? S.key[u] : 0xffffffffu;
  }
  int runf = 0, rowf = 0, packed = 0;
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int u = t * E + e;
    if (u >= P) continue;
    const bool row_start = u == 0 || (key[e + 1] >> 12) != (key[e] >> 12);
    const bool run_start = row_start || S.pchunk[key[e + 1] & 4095u] != S.pchunk[key[e] & 4095u];
    runf |= (int)run_start << e;
    rowf |= (int)row_start << e;
    packed += (int)run_start + ((int)row_start << 16);
  }
  int total;
  const int off = block_scan1024(packed, S.wsum, &total);
  int ri = off & 0xffff, wi = off >> 16;
#pragma unroll
  for (int e = 0; e < E; e++) {
    if (!((runf >> e) & 1)) continue;
    S.runu[ri] = (uint16_t)(t * E + e);
    S.runc[ri] = S.pchunk[key[e + 1] & 4095u];
    if ((rowf >> e) & 1) { S.rowrun[wi] = ri; S.rrow[wi] = (int)(key[e + 1] >> 12); wi++; }
    ri++;
  }
  const int T = total >> 16, R = total & 0xffff;
  if (t == 0) { S.rowrun[T] = R; S.runu[R] = (uint16_t)P; S.misc[0] = T; S.misc[1] = R; S.misc[2] = 0; S.misc[5] = 0; }
  __syncthreads();
  for (int w = t; w < T; w += 1024) {
    const int nr = S.rowrun[w + 1] - S.rowrun[w];
    if (nr > TS_SMALL) S.hot[atomicAdd(&S.misc[2], 1)] = w;
    else if (nr > 2) S.mid[atomicAdd(&S.misc[5], 1)] = w;
  }
  __syncthreads();
}

template <int MODE>
__device__ __forceinline__ void ts_sums(const BlockArgs& A, TailSmem& S, const double* vals) {
#ifdef SRO_PHASE_TIMING
  const long long ts_t0 = clock64();
#endif
  const int t = threadIdx.x;
  const int T = S.misc[0], R = S.misc[1], NH = S.misc[2];
  for (int ri = t; ri < R; ri += 1024) {
    const int u1 = S.runu[ri + 1];
    int u = S.runu[ri];
    double run = d_add(0.0, vals[S.key[u] & 4095u]);
    for (u++; u < u1; u++) run = d_add(run, vals[S.key[u] & 4095u]);
    S.runv[ri] = run;
  }
  __syncthreads();
#ifdef SRO_PHASE_TIMING
  if (threadIdx.x == 0) S.tsacc[15] += clock64() - ts_t0;
#endif
  auto finish = [&](int w, double D, double rk, double ak) {
    if (MODE == 0) {
      S.rX[w] = d_mul(D, D);
    } else {
      const double rn = d_add(rk, D);
      A.r[S.rrow[w]] = rn;
      const double dd = d_sub(rn, ak);
      A.h[S.rrow[w]] = A.lambda == 1.0 ? dd : d_div(dd, A.lambda);
    }
  };
#ifdef SRO_PHASE_TIMING
  if (MODE == 0 && threadIdx.x == 0 && A.phase) {
    atomicAdd((unsigned long long*)&A.phase[20], (unsigned long long)T);
    atomicAdd((unsigned long long*)&A.phase[21], (unsigned long long)R);
    atomicAdd((unsigned long long*)&A.phase[22], (unsigned long long)S.misc[5]);
    atomicAdd((unsigned long long*)&A.phase[23], (unsigned long long)NH);
  }
  long long ts_t1 = clock64();
#endif
  // one or two runs: the tree's value is the run or the sum of the two (every other leaf is
  // +0.0, an identity; run sums start from +0.0 so are never -0.0), one thread per row
  for (int w = t; w < T; w += 1024) {
    const int r0 = S.rowrun[w], r1 = S.rowrun[w + 1];
    if (r1 - r0 > 2) continue;
    double rk = 0.0, ak = 0.0;
    if (MODE == 1) { const int row = S.rrow[w]; rk = A.r[row]; ak = A.a[row]; }
    const double D = r1 - r0 == 1 ? S.runv[r0] : d_add(S.runv[r0], S.runv[r0 + 1]);
    finish(w, D, rk, ak);
  }
  const int lane = t & 31;
#ifdef SRO_PHASE_TIMING
  if (MODE == 0 && A.phase) { const long long t2 = clock64(); atomicAdd((unsigned long long*)&A.phase[24], (unsigned long long)(t2 - ts_t1) / 1024); ts_t1 = t2; }
#endif
  // 3 .. TS_SMALL runs, one thread per row: the adjacent-pair tree over the row's runs (chunks
  // ascending; zero leaves are identities) is evaluated by merging, n - 1 times, the adjacent pair
  // whose lowest common ancestor is deepest (31 - clz(c_e ^ c_e+1) smallest; adjacent levels
  // differ, so the choice is unique): the merged pair's level to its right neighbour is the right
  // one's (the left neighbour's is unchanged) — the same additions in the same order as the tree.
  {
    const int NM = S.misc[5];
    for (int b = t; b < NM; b += 1024) {
      const int w = S.mid[b];
      const int r0 = S.rowrun[w], nr = S.rowrun[w + 1] - r0;
      double v[TS_SMALL];
      int lv[TS_SMALL];
      int cprev = 0;
#pragma unroll
      for (int e = 0; e < TS_SMALL; e++) {
        const bool in = e < nr;
        const int c = in ? (int)S.runc[r0 + e] : 0;
        v[e] = in ? S.runv[r0 + e] : 0.0;
        if (e > 0) lv[e - 1] = in ? 31 - __clz(c ^ cprev) : 99;
        cprev = c;
      }
      lv[TS_SMALL - 1] = 99;
#pragma unroll
      for (int it = 0; it < TS_SMALL - 1; it++) {
        if (it >= nr - 1) break;
        int best = 0, bl = lv[0];
#pragma unroll
        for (int e = 1; e < TS_SMALL - 1; e++)
          if (lv[e] < bl) { bl = lv[e]; best = e; }
        // merge best and best + 1, shift the tail left by one
#pragma unroll
        for (int e = 0; e < TS_SMALL - 1; e++) {
          if (e == best) { v[e] = d_add(v[e], v[e + 1]); lv[e] = lv[e + 1]; }
          else if (e > best) { v[e] = v[e + 1]; lv[e] = lv[e + 1]; }
        }
        lv[TS_SMALL - 1] = 99;
      }
      double rk = 0.0, ak = 0.0;
      if (MODE == 1) { const int row = S.rrow[w]; rk = A.r[row]; ak = A.a[row]; }
      finish(w, v[0], rk, ak);
    }
  }
#ifdef SRO_PHASE_TIMING
  if (MODE == 0 && A.phase) { const long long t2 = clock64(); atomicAdd((unsigned long long*)&A.phase[25], (unsigned long long)(t2 - ts_t1) / 1024); ts_t1 = t2; }
#endif
  for (int b = t >> 5; b < NH; b += 32) {
    const int w = S.hot[b];
    const int r0 = S.rowrun[w], r1 = S.rowrun[w + 1];
    double rk = 0.0, ak = 0.0;
    if (MODE == 1 && lane == 0) { const int row = S.rrow[w]; rk = A.r[row]; ak = A.a[row]; }
    int lo = r0, hi = r1;   // first run with chunk >= 8 lane
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (S.runc[mid] < 8 * lane) lo = mid + 1; else hi = mid; }
    double x[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const bool hit = lo < r1 && S.runc[lo] == 8 * lane + e;
      x[e] = hit ? S.runv[lo] : 0.0;
      lo += hit;
    }
    const double D = warp_pair_tree(tree8(x));
    if (lane == 0) finish(w, D, rk, ak);
  }
#ifdef SRO_PHASE_TIMING
  if (MODE == 0 && A.phase) { const long long t2 = clock64(); atomicAdd((unsigned long long*)&A.phase[26], (unsigned long long)(t2 - ts_t1) / 1024); }
#endif
  __syncthreads();
}

// Step size (ELS, Eq. 10 / A.1 / joint block search; or DEC 2n'/(k'+2n')) from
// G_U and the denominator; scal[1..3] and the trace as dev_gamma.
__device__ __forceinline__ double ts_gamma_value(const BlockArgs& A, double GU, double den) {
  const double num = d_mul(A.lambda, GU);
  double gamma;
  if (A.step_rule == 1) {
    if (!(num > 0.0) || den == 0.0) gamma = 0.0;
    else { gamma = d_div(num, den); if (gamma > 1.0) gamma = 1.0; }
  } else {
    gamma = d_div((double)(2LL * A.nprime), (double)(blk_kk(A) + 2LL * A.nprime));
  }
  return gamma;
}
__device__ __forceinline__ void ts_gamma_record(const BlockArgs& A, double GU, double den, double gamma) {
  const double num = d_mul(A.lambda, GU);
  A.scal[1] = den;
  A.scal[2] = gamma;
  A.scal[3] = num;
  if (A.trace) {
    double* tr = blk_trace(A);
    tr[0] = (double)blk_kk(A); tr[1] = A.col0_dev ? A.col0_dev[blk_cur(A)] * A.trace_col0_mul : 0; tr[2] = A.j[0]; tr[3] = -1;
    tr[4] = 0; tr[5] = gamma; tr[6] = num; tr[7] = den; tr[8] = A.minval[0];
  }
}

// Denominator: psum256 over the m rows of Delta_k^2 (zero off the touched
// rows; ascending touched rows found per chunk by binary search), then gamma
// for every thread. 1024 threads.
__device__ __forceinline__ double ts_den_gamma(const BlockArgs& A, TailSmem& S, double GU) {
#ifdef SRO_PHASE_TIMING
  long long ts_t = clock64();
#endif
  const int T = S.misc[0];
  const int c = threadIdx.x;
  double acc = 0.0;
  if (c < 256) {
    const int lo = (int)chunk_lo(c, A.m, 256), hi = (int)chunk_lo(c + 1, A.m, 256);
    int a = 0, b = T;   // first touched row >= lo
    while (a < b) { const int mid = (a + b) >> 1; if (S.rrow[mid] < lo) a = mid + 1; else b = mid; }
    for (int u = a; u < T && S.rrow[u] < hi; u++) acc = d_add(acc, S.rX[u]);
    acc = warp_pair_tree(acc);
    if ((c & 31) == 0) S.red[c >> 5] = acc;
  }
  __syncthreads();
  TS_MARK(13);
  // every warp combines the 8 warp partials and computes gamma itself (the
  // same operations, so the same value everywhere); thread 0 records it
  double v = ((c & 31) < 8) ? S.red[c & 31] : 0.0;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
  v = __shfl_sync(FULL, v, 0);
  const double gamma = ts_gamma_value(A, GU, v);
  if (c == 0) ts_gamma_record(A, GU, v, gamma);
  TS_MARK(14);
  return gamma;
}

// merged support supp(t_i) U {j} in ascending rows from a register copy of
// the first KP support entries (c <= KP): entry e -> (row, told)
template <int KP, class F>
__device__ __forceinline__ void for_merged_reg(int c, const int* crow, const double* cval, int j, F f) {
  int e_out = 0;
  bool ins = false;
#pragma unroll
  for (int e = 0; e < KP; e++) {
    if (e < c) {
      const int rw = crow[e];
      if (!ins && j < rw) { f(e_out++, j, 0.0); ins = true; }
      if (rw == j) ins = true;
      f(e_out++, rw, cval[e]);
    }
  }
  if (!ins) f(e_out++, j, 0.0);
}

__global__ void __launch_bounds__(1024, 1) k_block_tail_sm(BlockArgs A, TailMerge M) { pdl_entry();
  extern __shared__ __align__(16) unsigned char tail_raw[];
#ifdef SRO_PHASE_TIMING
  long long ts_t = clock64();
#endif
  TailSmem& S = *reinterpret_cast<TailSmem*>(tail_raw);
#ifdef SRO_PHASE_TIMING
  if (threadIdx.x == 0) for (int q = 0; q < 16; q++) S.tsacc[q] = 0;
  struct Flush {   // adds the phase clocks to A.phase on every exit path
    const BlockArgs& A; TailSmem& S;
    __device__ ~Flush() { if (threadIdx.x == 0 && A.phase) for (int q = 0; q < 16; q++) A.phase[q] += S.tsacc[q]; }
  } ts_flush{A, S};
#endif
  const int t = threadIdx.x, L = A.L, cap = A.cap;
  const bool own = t < L;
  constexpr int KP = 4;
  static_assert(KP == SW_KP, "staged support width");
  // Every load that does not depend on the step cursor is issued here, together: the cursor,
  // the status / stop words, the supports the sweep staged (all KP entries, used or not: the
  // buffers hold 1024 x KP) and the first round of slab partials. Before, each came after the
  // previous one's round trip (cursor -> status -> column index -> supports -> partials).
  const unsigned cur0 = A.cur ? *A.cur : 0u;
  const int status0 = *A.status;
  const int stop0 = A.stop ? *A.stop : 0;
  const bool staged = M.nslabs > 1 && M.st_cnt;
  int c = 0, j = 0;
  int crow[KP];
  double cval[KP];
  double bi = 0.0, gcol = 0.0;
#pragma unroll
  for (int e = 0; e < KP; e++) { crow[e] = 0; cval[e] = 0.0; }
  double stt[KP];
  if (own && staged) {   // staged by the sweep: coalesced reads, independent of the column index
    c = M.st_cnt[t];
    bi = M.st_b[t];
#pragma unroll
    for (int e = 0; e < KP; e++) {
      crow[e] = M.st_row[e * L + t];
      cval[e] = M.st_val[e * L + t];
      stt[e] = M.st_term ? M.st_term[e * L + t] : 0.0;
    }
  }
  const int R = M.nslabs > 1 ? 1024 / L : 1;
  const int mp = t % L, mr = t / L;
  double pv[8];
  int pjv[8];
  if (M.nslabs > 1 && t < R * L) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int q = mr + u * R;
      const bool in = q < M.nslabs;
      pv[u] = in ? M.pmin[(int64_t)q * L + mp] : __longlong_as_double(0x7ff0000000000000LL);
      pjv[u] = in ? M.pj[(int64_t)q * L + mp] : 0x7fffffff;
    }
  }
  // take the step cursor (blk_take_cursor with the value loaded above)
  if (A.cur) {
    A.kk += (long long)cur0;
    if (A.trace) A.trace += 9 * (int64_t)cur0;
    if (A.col0_dev) A.col0_dev += cur0;
  }
  __syncthreads();
  if (t == 0 && A.cur) *A.cur = cur0 + 1u;
  A.cur = nullptr;
  if (status0 || stop0) return;
  TS_MARK(12);
  const int col0 = block_col0(A);
  const int i = col0 + t;
  // Per-column state of column i = col0 + t not staged by the sweep: support size, its first KP
  // entries (read whether or not they are in use), b_i, and the sweep's j / g when it merged its
  // slabs itself.
  if (own && !staged) {
    c = A.cnt[i];
    bi = A.b[i];
    crow[0] = A.srow[(int64_t)i * cap];   // read even when c == 0 (b_i = 0): unused then
    cval[0] = A.sval[(int64_t)i * cap];
    if (M.nslabs <= 1) { j = A.j[t]; gcol = A.g[t]; }
#pragma unroll
    for (int e = 1; e < KP; e++)
      if (e < c) { crow[e] = A.srow[(int64_t)i * cap + e]; cval[e] = A.sval[(int64_t)i * cap + e]; }
  }
  if (t == 0) S.misc[3] = 0;
  if (M.nslabs > 1) {
    // LMO merge over the slabs (argmin, lowest row on ties: R1 — the result does
    // not depend on the merge order): R = 1024 / L threads per column each merge
    // a strided subset of the slabs (8 loads in flight), then one combines the R
    // results and evaluates the column gap (Eq. 11)
    // g_i = sum_{k in supp, ascending} t_ki (C_ki + h_k) - b_i min_k (C_ki + h_k).
    double* mv = S.pd;   // free until the pairs are generated
    int* mj = S.prow;
    if (t < R * L) {
      double best = __longlong_as_double(0x7ff0000000000000LL);
      int bj = 0x7fffffff;
#pragma unroll
      for (int u = 0; u < 8; u++) argmin_merge(best, bj, pv[u], pjv[u]);   // the round loaded at entry
      for (int q0 = mr + 8 * R; q0 < M.nslabs; q0 += 8 * R) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int q = q0 + u * R;
          const bool in = q < M.nslabs;
          pv[u] = in ? M.pmin[(int64_t)q * L + mp] : __longlong_as_double(0x7ff0000000000000LL);
          pjv[u] = in ? M.pj[(int64_t)q * L + mp] : 0x7fffffff;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) argmin_merge(best, bj, pv[u], pjv[u]);
      }
      mv[t] = best;
      mj[t] = bj;
    }
    __syncthreads();
    TS_MARK(11);
    if (own) {
      double best = mv[t];
      int bj = mj[t];
      for (int r = 1; r < R; r++) argmin_merge(best, bj, mv[r * L + t], mj[r * L + t]);
      if (!(best < 1.0e308 && best > -1.0e308)) { set_status(A.status, 5); S.misc[3] = 1; }
      double dot = 0.0;
      if (c <= KP && staged && M.st_term) {   // the sweep's slab warps staged t_ki (C_ki + h_k)
#pragma unroll
        for (int e = 0; e < KP; e++)
          if (e < c) dot = d_add(dot, stt[e]);
      } else if (c <= KP) {
        double term[KP];
#pragma unroll
        for (int e = 0; e < KP; e++)
          term[e] = e < c ? d_mul(cval[e], d_add(tm_cost(M, crow[e], i), A.h[crow[e]])) : 0.0;
#pragma unroll
        for (int e = 0; e < KP; e++)
          if (e < c) dot = d_add(dot, term[e]);
      } else {
        for (int e = 0; e < c; e++) {
          const int k = A.srow[(int64_t)i * cap + e];
          dot = d_add(dot, d_mul(A.sval[(int64_t)i * cap + e], d_add(tm_cost(M, k, i), A.h[k])));
        }
      }
      j = bj;
      gcol = d_sub(dot, d_mul(bi, best));
      M.j[t] = bj;
      M.minval[t] = best;
      M.g[t] = gcol;
    }
  }
  if (own) S.gcol[t] = gcol;
  __syncthreads();
  TS_MARK(10);
  if (S.misc[3]) return;
  const double GU = dev_psumW(S.gcol, L, 256, A.scal + 0, A.eps, A.stop);   // G_U (FW: stop check)
  TS_MARK(0);
  if (A.stop && GU <= *A.eps) return;
  // merged support sizes -> offsets
  int Mp = 0;
  if (own) {
    bool in = false;
    if (c <= KP) {
#pragma unroll
      for (int e = 0; e < KP; e++) in |= (e < c && crow[e] == j);
    } else {
      for (int e = 0; e < c; e++) in |= (A.srow[(int64_t)i * cap + e] == j);
    }
    Mp = c + (in ? 0 : 1);
  }
  int P;
  const int off = block_scan1024(Mp, S.wsum, &P);
  TS_MARK(1);
  if (P > TS_PMAX) {   // too many pairs for shared memory: the global-memory tail
    dev_tail_rest(A, reinterpret_cast<double*>(tail_raw));
    return;
  }
  if (own) {
    const int c_t = chunk_index(t, L, 256);
    auto put = [&](int e, int row, double told) {
      const int q = off + e;
      S.prow[q] = row;
      S.ptold[q] = told;
      S.pd[q] = d_sub(row == j ? bi : 0.0, told);
      S.pchunk[q] = (uint8_t)c_t;
      S.key[q] = ((uint32_t)row << 12) | (uint32_t)q;
    };
    if (c <= KP) for_merged_reg<KP>(c, crow, cval, j, put);
    else for_merged(A, i, j, put);
  }
  int Pp = 1024;
  while (Pp < P) Pp <<= 1;
  for (int u = P + t; u < Pp; u += 1024) { S.key[u] = 0xffffffffu; S.key[Pp + u] = 0xffffffffu; }
  __syncthreads();
  TS_MARK(2);
  // sort of the keys (unique: one pair per (row, column)): bitonic for up to 1024 keys, a
  // stable radix sort by row above (config [4], B = 1024: 21.4k -> 11.6k cycles)
  if (Pp == 1024) ts_sort<1>(S.key, Pp, P);
  else if (Pp == 2048) ts_radix_sort<2>(S, P, A.m);
  else ts_radix_sort<4>(S, P, A.m);
  TS_MARK(3);
  // Delta_k per touched row -> denominator -> gamma
  if (Pp == 1024) ts_structure<1>(S, P);
  else if (Pp == 2048) ts_structure<2>(S, P);
  else ts_structure<4>(S, P);
  TS_MARK(9);
  ts_sums<0>(A, S, S.pd);
  TS_MARK(4);
  const double gamma = ts_den_gamma(A, S, GU);
  TS_MARK(5);
  // capacity check before anything is mutated
  const double omg = d_sub(1.0, gamma);
  const double gb = d_mul(gamma, bi);
  if (own) {
    int keep = 0;
    for (int q = off; q < off + Mp; q++) {
      double tn = d_mul(omg, S.ptold[q]);
      if (S.prow[q] == j) tn = d_add(tn, gb);
      keep += (tn != 0.0);
    }
    if (keep > cap) { set_status(A.status, 6); S.misc[3] = 1; }
  }
  __syncthreads();
  TS_MARK(6);
  if (S.misc[3]) return;
  // t_i <- (1-gamma) t_i + gamma s_i; exact zeros dropped (R13); Delta' = t' - t
  if (own) {
    int keep = 0;
    for (int q = off; q < off + Mp; q++) {
      const double told = S.ptold[q];
      double tn = d_mul(omg, told);
      if (S.prow[q] == j) tn = d_add(tn, gb);
      S.pd[q] = d_sub(tn, told);
      if (tn != 0.0) {
        A.srow[(int64_t)i * cap + keep] = S.prow[q];
        A.sval[(int64_t)i * cap + keep] = tn;
        keep++;
      }
    }
    A.cnt[i] = keep;
  }
  __syncthreads();
  TS_MARK(7);
  ts_sums<1>(A, S, S.pd);
  TS_MARK(8);
  if (t == 0) atomicAdd(A.dsteps, 1ULL);
}

}  // namespace sro
