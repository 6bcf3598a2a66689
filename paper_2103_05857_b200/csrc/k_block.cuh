// k_block.cuh — the plain step over a contiguous column set U = [col0, col0+L)
// (R18): FW (Alg. A.1) is
// U = [n], batched BCFW is a B-column block. After the LMO sweep over U
// (k_sweep.cuh) the step needs two per-row sums over the block's columns:
//   Delta_k  = sum_{i in U} (s_ik - t_ik)     (direction, for the Eq. A.1 denominator)
//   Delta'_k = sum_{i in U} (t'_ik - t_ik)    (row-sum update r += Delta')
// Both follow R19: U's positions are split in 256 chunks, each (row, chunk)
// run is summed left to right (ascending column), and the 256 chunk partials
// of a row combine by adjacent pairs. No float atomics anywhere:
//   1. every column of U lists its merged support supp(t_i) U {j_i} as
//      (row, d) pairs, rows ascending (pairs_count / scan / pairs_gen);
//   2. the touched rows get contiguous run-list segments (a scan of their pair
//      counts); the first pair of each (row, chunk) run sums the run in column
//      order and appends (chunk, partial) to its row's list (dev_runs) — work
//      per pair is O(chunk length x |supp|), independent of how many columns
//      share a row;
//   3. a warp per touched row scatters its list into 256 shared-memory slots
//      (zero outside use) and combines them with the adjacent-pair tree
//      (dev_row_tree); only the few nonzero chunks of a row touch memory.
//
// Sharded mode: the G shards of U hold the contiguous position
// ranges [s L/G, (s+1) L/G), which are exactly the chunks [s 256/G, (s+1) 256/G)
// of U (G a power of two dividing L). A shard runs the same phases with
// W = 256/G chunks over its own positions, so its row tree yields the subtree
// of the global 256-leaf tree; the G subtree values (per row, plus the
// block's G_U subtree and status flags) are exchanged and every shard combines
// them with the same adjacent-pair tree — bitwise the unsharded result.
//
// Every phase is a __device__ function over grid-stride loops, so the same
// code runs either as one kernel per phase (large U, many CTAs) or inside a
// single CTA (small U: one launch for the whole post-LMO step).
#pragma once
#include <cooperative_groups.h>
#include "sro_device.cuh"

namespace sro {


struct BlockArgs {
  int m, n, cap;
  int runs_kmax;         // k_runs: chunks with more pairs search the supports instead (<= RUN_KMAX)
  double lambda;
  const double* a;
  const double* b;
  double* r;
  double* h;
  int* cnt;
  int* srow;
  double* sval;
  const int* col0_dev;   // block index pointer (batched) or nullptr
  unsigned* cur;         // device step cursor (nullptr: none): col0_dev, kk and trace advance by it
  int col0_mul;          // columns of U held here (B, or B/G for a shard)
  int L;
  int W;                 // chunks over the positions held here: 256, or 256/G for a shard
  // LMO outputs over U
  const int* j;
  const double* minval;
  const double* g;       // column gaps over U
  // pair workspace (P = L (cap+1))
  int* pcount;           // L
  int* poff;             // L+1
  int* ptotal;           // 1
  int* prow;             // P: row of the pair
  int* ppos;             // P: position of the pair's column in U
  double* pd;            // P: s_ik - t_ik
  double* ptold;         // P: t_ik (sharded mode: rollback after a remote capacity error)
  double* pdelta;        // P: t'_ik - t_ik
  int* rowcnt;           // m: pairs per row in this step, zero outside a step
  int* rowidx;           // m: touched-list index of a touched row
  int* trows;            // touched rows (unordered; every row's work is independent)
  int* ntouch;           // number of touched rows
  int* tstart;           // touched index -> start of its run-list segment (scan of its pair count)
  int* tcur;             // touched index -> runs appended so far (zero outside a step)
  int* runc;             // run lists: chunk index
  double* runv;          // run lists: partial sum
  int* bigw;             // touched indices of rows with more than ROW_SMALL runs
  int* nbig;             // [2]: their count in the first / second tree of a step
  double* X;             // m: Delta_k^2, zero outside a step
  double* scal;          // [0]=G_U [1]=den [2]=gamma [3]=num
  const double* eps;     // FW stop check (nullptr for batched)
  int* stop;             // FW stop flag (nullptr for batched)
  int* status;
  // step parameters
  int step_rule;
  long long kk, nprime;
  double* trace;
  int trace_col0_mul;    // global block size (trace records the global first column)
  unsigned long long* dsteps;   // completed steps (device counter; host reads at sync points)
  // sharded mode (G > 1)
  int G, shard, slot_len;
  double* x1;            // G slots of slot_len: Delta subtree per row, [m] = G_U subtree, [m+1] = status
  double* x2;            // G slots: Delta' subtree per row, [m] = capacity failure, [m+1] = status
  int* capfail;          // this shard's capacity check failed (nullptr when unsharded)
  long long* phase;      // SRO_PHASE_TIMING builds only: clock64 phase totals
};

__device__ __forceinline__ bool blk_skip(const BlockArgs& A) {
  return (A.stop && *A.stop) || *A.status || (A.capfail && *A.capfail);
}
__device__ __forceinline__ unsigned blk_cur(const BlockArgs& A) { return A.cur ? *A.cur : 0u; }
__device__ __forceinline__ int block_col0(const BlockArgs& A) { return A.col0_dev ? A.col0_dev[blk_cur(A)] * A.col0_mul : 0; }
__device__ __forceinline__ long long blk_kk(const BlockArgs& A) { return A.kk + (long long)blk_cur(A); }
__device__ __forceinline__ double* blk_trace(const BlockArgs& A) { return A.trace ? A.trace + 9 * (int64_t)blk_cur(A) : nullptr; }
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

// Adjacent-pair tree over G (a power of two) values get(0..G-1), evaluated
// left to right with a stack of completed subtrees.
template <class F>
__device__ __forceinline__ double pair_tree_pow2(int G, F get) {
  double st[10];
  int sz[10];
  int top = 0;
  for (int s = 0; s < G; s++) {
    double v = get(s);
    int w = 1;
    while (top > 0 && sz[top - 1] == w) { v = d_add(st[top - 1], v); w *= 2; top--; }
    st[top] = v; sz[top] = w; top++;
  }
  return st[0];
}

// ---------------------------------------------------------------------------
// Phases
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dev_zero_dbl(double* x, int N) {
  for (int q = gtid(); q < N; q += gstride()) x[q] = 0.0;
}

__device__ __forceinline__ void dev_pairs_count(const BlockArgs& A) {
  const int col0 = block_col0(A);
  for (int p = gtid(); p < A.L; p += gstride()) A.pcount[p] = merged_count(A, col0 + p, A.j[p]);
}

// Exclusive scan of get(0..N) (integers: order-free) -> put(q, prefix), returning the total.
// One CTA of exactly 1024 threads over tiles of 4096 values, four consecutive per thread (the
// CTA's loads coalesced; the next tile's values are requested while the current one is scanned).
// A thread-per-contiguous-range scan made each warp load touch 32 lines: ~80 us for 65536
// counts at config [3].
template <class Get, class Put>
__device__ __forceinline__ int block_scan_tiles(int N, Get get, Put put) {
  __shared__ int ws[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int carry = 0;
  int v[4];
#pragma unroll
  for (int u = 0; u < 4; u++) v[u] = 4 * t + u < N ? get(4 * t + u) : 0;
  for (int base = 0; base < N; base += 4096) {
    int nv[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = base + 4096 + 4 * t + u;
      nv[u] = q < N ? get(q) : 0;
    }
    const int s = (v[0] + v[1]) + (v[2] + v[3]);
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, incl, o); if (lane >= o) incl += y; }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
      int x = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, x, o); if (lane >= o) x += y; }
      ws[lane] = x;
    }
    __syncthreads();
    int run = carry + (w ? ws[w - 1] : 0) + incl - s;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = base + 4 * t + u;
      if (q < N) put(q, run);
      run += v[u];
    }
    carry += ws[31];
    __syncthreads();   // ws is rewritten by the next tile
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = nv[u];
  }
  return carry;
}

// Exclusive scan of x[0..N) into y[0..N], y[N] = total. One CTA of exactly 1024 threads.
__device__ __forceinline__ void dev_scan_excl(const int* __restrict__ x, int N, int* y, int* total) {
  const int tot = block_scan_tiles(N, [&](int q) { return x[q]; }, [&](int q, int e) { y[q] = e; });
  if (threadIdx.x == 0) { y[N] = tot; if (total) *total = tot; }
  __syncthreads();
}

// pairs of every merged support (rows ascending within a column): row, column
// position, d = s - t (and t itself in sharded mode); touched-row list.
__device__ __forceinline__ void dev_pairs_gen(const BlockArgs& A) {
  const int col0 = block_col0(A);
  for (int p = gtid(); p < A.L; p += gstride()) {
    const int i = col0 + p, j = A.j[p];
    const double bi = A.b[i];
    const int base = A.poff[p];
    for_merged(A, i, j, [&](int e, int row, double told) {
      const int q = base + e;
      A.prow[q] = row;
      A.ppos[q] = p;
      A.pd[q] = d_sub(row == j ? bi : 0.0, told);
      if (A.ptold) A.ptold[q] = told;
      // per-row pair counts, warp-aggregated (columns share their argmin rows: one atomic per
      // distinct row of the converged lanes instead of one per pair); the first to count a row
      // appends it to the order-free touched list
      const unsigned grp = __match_any_sync(__activemask(), row);
      if ((int)(threadIdx.x & 31) == __ffs(grp) - 1 && atomicAdd(&A.rowcnt[row], __popc(grp)) == 0) {
        const int w = atomicAdd(A.ntouch, 1);
        A.trows[w] = row;
        A.rowidx[row] = w;
      }
    });
  }
}

// pair index of row k in column position pp's merged support (rows ascending), or -1
__device__ __forceinline__ int find_pair(const BlockArgs& A, int pp, int k) {
  const int hi = A.poff[pp + 1];
  for (int q = A.poff[pp]; q < hi; q++) {
    const int r = A.prow[q];
    if (r >= k) return r == k ? q : -1;
  }
  return -1;
}

// Run-list segments of the touched rows: tstart = exclusive scan over the
// touched list of the rows' pair counts (one CTA of exactly 1024 threads).
__device__ __forceinline__ void dev_touched_scan(const BlockArgs& A) {
  const int N = *A.ntouch;
  block_scan_tiles(N, [&](int q) { return A.rowcnt[A.trows[q]]; }, [&](int q, int e) { A.tstart[q] = e; });
  __syncthreads();
}

// The (row k, chunk c) run of val summed in column order from +0.0 (R19) by
// the run's first pair, appended to row k's run list as (c, sum).
// the run that pair q starts, if it is the first pair of its row in its chunk (searching the
// earlier positions' supports)
__device__ __forceinline__ void run_of_pair(const BlockArgs& A, const double* __restrict__ val, int q) {
  {
    const int p = A.ppos[q], k = A.prow[q];
    const int c = chunk_index(p, A.L, A.W);
    const int lo = (int)chunk_lo(c, A.L, A.W), hi = (int)chunk_lo(c + 1, A.L, A.W);
    bool start = true;
    for (int pp = lo; pp < p && start; pp++) start = find_pair(A, pp, k) < 0;
    if (!start) return;
    double s = d_add(0.0, val[q]);
    for (int pp = p + 1; pp < hi; pp++) {
      const int qq = find_pair(A, pp, k);
      if (qq >= 0) s = d_add(s, val[qq]);
    }
    const int w = A.rowidx[k];
    const int slot = A.tstart[w] + atomicAdd(&A.tcur[w], 1);   // order-free: one entry per chunk
    A.runc[slot] = c;
    A.runv[slot] = s;
  }
}
__device__ __forceinline__ void dev_runs(const BlockArgs& A, const double* __restrict__ val) {
  const int P = *A.ptotal;
  for (int q = gtid(); q < P; q += gstride()) run_of_pair(A, val, q);
}

// Applies a touched row's combined sum D. MODE 0: X[k] = D^2; MODE 1: r_k += D,
// h_k = (r_k - a_k)/lambda; MODE 2: slot[k] = D (a shard's subtree). Resets the
// row's run counter, and its pair count when `clear` (last tree of a step).
template <int MODE>
__device__ __forceinline__ void row_finish(const BlockArgs& A, int w, int k, double D, double* slot, bool clear) {
  if (MODE == 0) {
    A.X[k] = d_mul(D, D);
  } else if (MODE == 1) {
    const double rn = d_add(A.r[k], D);
    A.r[k] = rn;
    const double d = d_sub(rn, A.a[k]);
    A.h[k] = A.lambda == 1.0 ? d : d_div(d, A.lambda);   // x / 1 == x exactly
    A.X[k] = 0.0;
  } else {
    slot[k] = D;
  }
  A.tcur[w] = 0;
  if (clear) A.rowcnt[k] = 0;
}

constexpr int ROW_SMALL = 8;   // rows with at most this many chunk runs: one thread per row

// The 256-leaf adjacent-pair tree over the K nonzero chunk partials of a row
// (zero leaves are additive identities): sort by chunk, then K-1 times merge
// (left + right) the adjacent pair whose lowest common ancestor is lowest —
// the dense tree's merges, in an order that only swaps independent ones.
__device__ __forceinline__ double sparse_tree256(int K, int* c, double* v) {
  for (int a = 1; a < K; a++) {
    const int cc = c[a];
    const double vv = v[a];
    int b = a - 1;
    while (b >= 0 && c[b] > cc) { c[b + 1] = c[b]; v[b + 1] = v[b]; b--; }
    c[b + 1] = cc; v[b + 1] = vv;
  }
  while (K > 1) {
    int t = 0, best = 99;
    for (int u = 0; u + 1 < K; u++) {
      const int hb = 31 - __clz(c[u] ^ c[u + 1]);
      if (hb < best) { best = hb; t = u; }
    }
    v[t] = d_add(v[t], v[t + 1]);
    for (int u = t + 1; u + 1 < K; u++) { c[u] = c[u + 1]; v[u] = v[u + 1]; }
    K--;
  }
  return v[0];
}

// Pass 1, thread per touched row: rows with <= ROW_SMALL runs are combined in
// registers / local memory; larger ones (hot rows) go to the big list.
template <int MODE>
__device__ __forceinline__ void dev_row_tree_small(const BlockArgs& A, double* slot, bool clear, int pass) {
  const int T = *A.ntouch;
  for (int w = gtid(); w < T; w += gstride()) {
    const int k = A.trows[w];
    const int st = A.tstart[w], K = A.tcur[w];
    if (K > ROW_SMALL) { A.bigw[atomicAdd(&A.nbig[pass], 1)] = w; continue; }
    int c[ROW_SMALL];
    double v[ROW_SMALL];
    for (int e = 0; e < K; e++) { c[e] = A.runc[st + e]; v[e] = A.runv[st + e]; }
    row_finish<MODE>(A, w, k, sparse_tree256(K, c, v), slot, clear);
  }
}

// Pass 2, warp per big row: scatter its runs into the warp's 256 shared slots
// (zero outside use), the dense 256-leaf tree, clear the slots.
template <int MODE>
__device__ __forceinline__ void dev_row_tree_big(const BlockArgs& A, double* slot, bool clear, int pass,
                                                 double* wslots_all, bool all_rows = false) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  double* sl = wslots_all + 256 * warp;
  const int NB = all_rows ? *A.ntouch : A.nbig[pass];
  for (int b = blockIdx.x * nwarps + warp; b < NB; b += gridDim.x * nwarps) {
    const int w = all_rows ? b : A.bigw[b];
    const int k = A.trows[w];
    const int st = A.tstart[w], K = A.tcur[w];
    for (int e = lane; e < K; e += 32) sl[A.runc[st + e]] = A.runv[st + e];
    __syncwarp();
    double x[8];
#pragma unroll
    for (int t = 0; t < 8; t++) x[t] = sl[8 * lane + t];
    const double D = warp_pair_tree(tree8(x));
    __syncwarp();
    for (int e = lane; e < K; e += 32) sl[A.runc[st + e]] = 0.0;
    __syncwarp();
    if (lane == 0) row_finish<MODE>(A, w, k, D, slot, clear);
  }
}

// Both passes inside one CTA (single-CTA tails).
template <int MODE>
__device__ __forceinline__ void dev_row_tree(const BlockArgs& A, double* slot, bool clear, int pass,
                                             double* wslots_all) {
  dev_row_tree_small<MODE>(A, slot, clear, pass);
  __syncthreads();
  dev_row_tree_big<MODE>(A, slot, clear, pass, wslots_all);
}

// Chunked pairwise sum (R19) of x[0..L) with W chunks (W = 256: psum256; W =
// 256/G: a shard's subtree) for a CTA of >= 256 threads (threads >= 256 idle
// but present at the barriers). Result in *out; optional FW stop check.
__device__ __forceinline__ double dev_psumW(const double* __restrict__ x, int64_t L, int W, double* out,
                                            const double* eps, int* stop_flag) {
  __shared__ double red[8];
  const int c = threadIdx.x;
  double acc = 0.0;
  if (c < 256) {
    if (c < W) {
      acc = chunk_seq_sum(x, chunk_lo(c, L, W), chunk_lo(c + 1, L, W));
    }
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
      if (out) *out = v;
      if (stop_flag && eps && v <= *eps) *stop_flag = 1;
    }
  }
  __syncthreads();
  const double v = red[0];
  __syncthreads();
  return v;
}

// dev_psumW for long chunks (one CTA of exactly 256 threads): the chunks are staged through
// shared memory 16 elements per chunk at a time, each half-warp loading 128 contiguous bytes of
// one chunk (the next slice requested while the current one is summed); thread c still adds
// chunk c left to right from +0.0. Reading 256 chunks of 256 doubles directly (thread c walking
// chunk c) touched 32 lines per warp load and took ~30 us at config [3].
constexpr int PSUM_K = 16;
__device__ __forceinline__ double dev_psumW_tiled(const double* __restrict__ x, int64_t L, int W, double* out,
                                                  const double* eps, int* stop_flag) {
  // threads 0..255 load and sum; a larger CTA's other threads only take part in the barriers
  __shared__ double tile[256][PSUM_K + 1];
  __shared__ int64_t rlo[257];
  __shared__ double red[8];
  const int c = threadIdx.x;
  const bool act = c < 256;
  if (act) rlo[c] = c < W ? chunk_lo(c, L, W) : L;
  if (c == 0) rlo[256] = L;
  __syncthreads();
  const int64_t maxlen = (L + W - 1) / W;
  const int u = c & 15, r0 = (c & 255) >> 4;
  double nv[16];
  auto load = [&](int64_t U) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int r = r0 + 16 * k;
      const int64_t q = rlo[r] + U + u;
      nv[k] = (act && r < W && q < rlo[r + 1]) ? x[q] : 0.0;
    }
  };
  load(0);
  double acc = 0.0;
  const int64_t len = c < W ? rlo[c + 1] - rlo[c] : 0;
  for (int64_t U = 0; U < maxlen; U += PSUM_K) {
    if (act) {
#pragma unroll
      for (int k = 0; k < 16; k++) tile[r0 + 16 * k][u] = nv[k];
    }
    __syncthreads();
    if (U + PSUM_K < maxlen) load(U + PSUM_K);
    const int64_t rem = len - U;
    const int kk = rem < PSUM_K ? (rem > 0 ? (int)rem : 0) : PSUM_K;
    for (int e = 0; e < kk; e++) acc = d_add(acc, tile[c][e]);
    __syncthreads();
  }
  if (act) {
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
      if (out) *out = v;
      if (stop_flag && eps && v <= *eps) *stop_flag = 1;
    }
  }
  __syncthreads();
  const double v = red[0];
  __syncthreads();
  return v;
}
__device__ __forceinline__ double dev_psumW_any(const double* __restrict__ x, int64_t L, int W, double* out,
                                                const double* eps, int* stop_flag) {
  return (L + W - 1) / W > 2 * PSUM_K ? dev_psumW_tiled(x, L, W, out, eps, stop_flag)
                                      : dev_psumW(x, L, W, out, eps, stop_flag);
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
    gamma = d_div((double)(2LL * A.nprime), (double)(blk_kk(A) + 2LL * A.nprime));
  }
  A.scal[2] = gamma;
  A.scal[3] = num;
  if (A.trace) {
    double* tr = blk_trace(A);
    tr[0] = (double)blk_kk(A); tr[1] = A.col0_dev ? A.col0_dev[blk_cur(A)] * A.trace_col0_mul : 0; tr[2] = A.j[0]; tr[3] = -1;
    tr[4] = 0; tr[5] = gamma; tr[6] = num; tr[7] = den; tr[8] = A.minval[0];
  }
}

// Capacity check for every column of U before anything is mutated: sets the
// status word (unsharded) or this shard's capfail flag (sharded).
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
    if (keep > A.cap) {
      if (A.capfail) atomicOr(A.capfail, 1);
      else set_status(A.status, 6);
    }
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

// Warp per column (the multi-CTA phase kernels): the merged support supp(t_i) U {j} held one
// entry per lane, rows ascending (lane < M) — the entries for_merged visits, in its order. Every
// load is issued at once (the support slab is read for lane < cap whatever its size), so a column
// costs one round trip instead of one per support entry.
struct WarpMerged {
  int M;         // merged support size (<= cap + 1 <= 32)
  int row;       // this lane's entry
  double told;
};
__device__ __forceinline__ WarpMerged warp_merged(const BlockArgs& A, int i, int j) {
  const int lane = threadIdx.x & 31;
  const int c0 = A.cnt[i];
  int rw = 0x7fffffff;
  double tv = 0.0;
  if (lane < A.cap) { rw = A.srow[(int64_t)i * A.cap + lane]; tv = A.sval[(int64_t)i * A.cap + lane]; }
  if (lane >= c0) { rw = 0x7fffffff; tv = 0.0; }
  const bool j_in = __ballot_sync(FULL, rw == j) != 0u;
  const int ins = __popc(__ballot_sync(FULL, rw < j));
  int src = (j_in || lane < ins) ? lane : lane - 1;
  if (src < 0) src = 0;
  WarpMerged w;
  w.row = __shfl_sync(FULL, rw, src);
  w.told = __shfl_sync(FULL, tv, src);
  if (!j_in && lane == ins) { w.row = j; w.told = 0.0; }
  w.M = c0 + (j_in ? 0 : 1);
  return w;
}
__device__ __forceinline__ int gwarp() { return (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); }
__device__ __forceinline__ int gwarps() { return (int)((gridDim.x * blockDim.x) >> 5); }

__device__ __forceinline__ void dev_pairs_count_w(const BlockArgs& A) {
  const int col0 = block_col0(A);
  for (int p = gwarp(); p < A.L; p += gwarps()) {
    const WarpMerged w = warp_merged(A, col0 + p, A.j[p]);
    if ((threadIdx.x & 31) == 0) A.pcount[p] = w.M;
  }
}
__device__ __forceinline__ void dev_pairs_gen_w(const BlockArgs& A) {
  const int col0 = block_col0(A);
  const int lane = threadIdx.x & 31;
  for (int p = gwarp(); p < A.L; p += gwarps()) {
    const int i = col0 + p, j = A.j[p];
    const double bi = A.b[i];
    const int base = A.poff[p];
    const WarpMerged w = warp_merged(A, i, j);
    if (lane < w.M) {
      const int q = base + lane;
      A.prow[q] = w.row;
      A.ppos[q] = p;
      A.pd[q] = d_sub(w.row == j ? bi : 0.0, w.told);
      if (A.ptold) A.ptold[q] = w.told;
      if (atomicAdd(&A.rowcnt[w.row], 1) == 0) {   // order-free touched list
        const int t = atomicAdd(A.ntouch, 1);
        A.trows[t] = w.row;
        A.rowidx[w.row] = t;
      }
    }
  }
}
__device__ __forceinline__ void dev_cap_check_w(const BlockArgs& A) {
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  for (int p = gwarp(); p < A.L; p += gwarps()) {
    const int i = col0 + p, j = A.j[p];
    const double gb = d_mul(gamma, A.b[i]);
    const WarpMerged w = warp_merged(A, i, j);
    bool kept = false;
    if ((int)(threadIdx.x & 31) < w.M) {
      double tn = d_mul(omg, w.told);
      if (w.row == j) tn = d_add(tn, gb);
      kept = tn != 0.0;
    }
    const int keep = __popc(__ballot_sync(FULL, kept));
    if ((threadIdx.x & 31) == 0 && keep > A.cap) {
      if (A.capfail) atomicOr(A.capfail, 1);
      else set_status(A.status, 6);
    }
  }
}
// t_i <- (1-gamma) t_i + gamma s_i; exact zeros dropped (R13), as dev_update_cols
__device__ __forceinline__ void dev_update_cols_w(const BlockArgs& A) {
  const int col0 = block_col0(A);
  const double gamma = A.scal[2];
  const double omg = d_sub(1.0, gamma);
  const int lane = threadIdx.x & 31;
  for (int p = gwarp(); p < A.L; p += gwarps()) {
    const int i = col0 + p, j = A.j[p];
    const double gb = d_mul(gamma, A.b[i]);
    const int base = A.poff[p];
    const WarpMerged w = warp_merged(A, i, j);
    double tn = 0.0;
    if (lane < w.M) {
      tn = d_mul(omg, w.told);
      if (w.row == j) tn = d_add(tn, gb);
      A.pdelta[base + lane] = d_sub(tn, w.told);
    }
    const bool kept = lane < w.M && tn != 0.0;
    const unsigned km = __ballot_sync(FULL, kept);
    const int e = __popc(km & ((1u << lane) - 1u));
    if (kept && e < A.cap) {
      A.srow[(int64_t)i * A.cap + e] = w.row;
      A.sval[(int64_t)i * A.cap + e] = tn;
    }
    if (lane == 0) A.cnt[i] = __popc(km);
  }
}

// ---------------------------------------------------------------------------
// Kernels: one per phase (multi-CTA path) ...
// ---------------------------------------------------------------------------
__global__ void k_pairs_count(BlockArgs A) { pdl_entry(); if (!blk_skip(A)) dev_pairs_count_w(A); }
// Step start and pair offsets in one launch (unsharded multi-CTA step, after k_pairs_count): G_U =
// psumW(g) with the FW stop check (Alg. A.1 line 4) and the counter resets of k_step_begin, then,
// unless the step stops, the exclusive scan of the merged-support sizes. One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_begin_scan(BlockArgs A, double* out) { pdl_entry();
  if (A.stop && *A.stop) return;
  if (*A.status) return;
  if (threadIdx.x == 0) { *A.ntouch = 0; A.nbig[0] = 0; A.nbig[1] = 0; if (A.capfail) *A.capfail = 0; }
  const double gu = dev_psumW_any(A.g, A.L, A.W, out, A.eps, A.stop);
  if (A.stop && A.eps && gu <= *A.eps) return;
  dev_scan_excl(A.pcount, A.L, A.poff, A.ptotal);
}
__global__ void __launch_bounds__(1024) k_scan_pairs(BlockArgs A) { pdl_entry();
  if (blk_skip(A)) return;
  dev_scan_excl(A.pcount, A.L, A.poff, A.ptotal);
}
__global__ void k_pairs_gen(BlockArgs A) { pdl_entry(); if (!blk_skip(A)) dev_pairs_gen_w(A); }
// The (row, chunk) runs of one step, a CTA per chunk (grid-stride over the W chunks): the chunk's
// pairs (contiguous: positions ascending, rows ascending within one) become (row << 12 | local
// index) keys in shared memory, sorted (bitonic), so each row's pairs are adjacent in column
// order; the first of each row sums them left to right from +0.0 — the sums dev_runs forms
// (R19), without its per-pair search through the earlier columns' supports in global memory
// (config [1] FW: 18.6 us per launch). Chunks with more than RUN_KMAX pairs, or m >= 2^20 - 1,
// take that search.
constexpr int RUN_KMAX = 4096;
__global__ void __launch_bounds__(256) k_runs(BlockArgs A, const double* __restrict__ val) { pdl_entry();
  if (blk_skip(A)) return;
  __shared__ uint32_t key[RUN_KMAX];
  __shared__ double sv[RUN_KMAX];
  const int t = threadIdx.x;
  for (int c = blockIdx.x; c < A.W; c += gridDim.x) {
    const int lo = (int)chunk_lo(c, A.L, A.W), hi = (int)chunk_lo(c + 1, A.L, A.W);
    const int q0 = A.poff[lo], N = A.poff[hi] - q0;
    if (N > A.runs_kmax || A.m >= (1 << 20) - 1) {
      for (int q = q0 + t; q < q0 + N; q += blockDim.x) run_of_pair(A, val, q);
      continue;
    }
    int NP = 1;
    while (NP < N) NP <<= 1;
    for (int u = t; u < NP; u += blockDim.x) {
      if (u < N) { key[u] = ((uint32_t)A.prow[q0 + u] << 12) | (uint32_t)u; sv[u] = val[q0 + u]; }
      else key[u] = 0xffffffffu;
    }
    __syncthreads();
    for (int k = 2; k <= NP; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = t; i < NP; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint32_t a = key[i], b = key[ixj];
            if ((a > b) == ((i & k) == 0)) { key[i] = b; key[ixj] = a; }
          }
        }
        __syncthreads();
      }
    for (int u = t; u < N; u += blockDim.x) {
      const uint32_t ku = key[u];
      const uint32_t row = ku >> 12;
      if (u > 0 && (key[u - 1] >> 12) == row) continue;
      double s = d_add(0.0, sv[ku & 4095u]);
      for (int v = u + 1; v < N && (key[v] >> 12) == row; v++) s = d_add(s, sv[key[v] & 4095u]);
      const int w = A.rowidx[row];
      const int slot = A.tstart[w] + atomicAdd(&A.tcur[w], 1);   // order-free: one entry per chunk
      A.runc[slot] = c;
      A.runv[slot] = s;
    }
    __syncthreads();
  }
}
__global__ void __launch_bounds__(1024) k_touched_scan(BlockArgs A) { pdl_entry(); if (!blk_skip(A)) dev_touched_scan(A); }
template <int MODE>
__global__ void __launch_bounds__(256) k_row_tree_small(BlockArgs A, double* slot, int clear, int pass) {
  if (!blk_skip(A)) dev_row_tree_small<MODE>(A, slot, clear != 0, pass);
}
// Warp per touched row over every touched row (the multi-CTA path: one launch).
// done_ticket (the unsharded step's last kernel): the last CTA to finish also ends the step — the
// step count and the cursor advance (every CTA has read the cursor by then) — behind a threadfence
// and an arrival counter it resets, one launch fewer per step.
template <int MODE>
__global__ void __launch_bounds__(256) k_row_tree_all(BlockArgs A, double* slot, int clear, unsigned* done_ticket) {
  pdl_entry();
  __shared__ double wsl[8 * 256];
  const bool skip = blk_skip(A);
  if (!skip) {
    for (int q = threadIdx.x; q < 8 * 256; q += blockDim.x) wsl[q] = 0.0;
    __syncthreads();
    dev_row_tree_big<MODE>(A, slot, clear != 0, 0, wsl, true);
  }
  if (done_ticket) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(done_ticket, 1u) == gridDim.x - 1;
      if (last) {
        *done_ticket = 0u;
        if (!skip) atomicAdd(A.dsteps, 1ULL);
        if (A.cur) *A.cur += 1u;
      }
    }
  }
}
template <int MODE>
__global__ void __launch_bounds__(256) k_row_tree_big(BlockArgs A, double* slot, int clear, int pass) {
  __shared__ double wsl[8 * 256];
  if (blk_skip(A) || A.nbig[pass] == 0) return;
  for (int q = threadIdx.x; q < 8 * 256; q += blockDim.x) wsl[q] = 0.0;
  __syncthreads();
  dev_row_tree_big<MODE>(A, slot, clear != 0, pass, wsl);
}
// The denominator psum256 of Delta_k^2 over the m rows and gamma in one launch (unsharded multi-CTA
// step; thread 0 writes scal[1] and reads it back for gamma). One CTA of 256 threads.
__global__ void __launch_bounds__(256) k_den_gamma(BlockArgs A) { pdl_entry();
  if (blk_skip(A)) return;
  dev_psumW_any(A.X, A.m, 256, A.scal + 1, nullptr, nullptr);
  dev_gamma(A);
}
__global__ void k_cap_check(BlockArgs A) { pdl_entry(); if (!blk_skip(A)) dev_cap_check_w(A); }
__global__ void k_update_cols(BlockArgs A) { pdl_entry(); if (!blk_skip(A)) dev_update_cols_w(A); }
__global__ void k_zero_slot(BlockArgs A, double* slot) { if (!blk_skip(A)) dev_zero_dbl(slot, A.m); }

// Step start: G_U = psumW(g) (FW: stop check, Alg. A.1 line 4) into *out,
// touched-row count and capacity flag reset. One CTA of 256 threads.
__global__ void __launch_bounds__(256) k_step_begin(BlockArgs A, double* out) { pdl_entry();
  if (A.stop && *A.stop) return;
  if (*A.status) return;
  if (threadIdx.x == 0) { *A.ntouch = 0; A.nbig[0] = 0; A.nbig[1] = 0; if (A.capfail) *A.capfail = 0; }
  dev_psumW_any(A.g, A.L, A.W, out, A.G > 1 ? nullptr : A.eps, A.G > 1 ? nullptr : A.stop);
}

// psum256 of x[0..L) -> *out (one CTA of 256 threads). If stop_flag is given,
// sets *stop_flag = (total <= *eps).
__global__ void __launch_bounds__(256) k_psum256(const double* __restrict__ x, int64_t L, double* out,
                                                 const double* __restrict__ eps, int* stop_flag,
                                                 const int* __restrict__ stop_in) { pdl_entry();
  if (stop_in && *stop_in) return;
  dev_psumW_any(x, L, 256, out, eps, stop_flag);
}


// Single-CTA kernels: take the cursor's values once, then advance it (every
// thread has read it before thread 0 writes).
__device__ __forceinline__ void blk_take_cursor(BlockArgs& A) {
  if (!A.cur) return;
  const unsigned c = *A.cur;
  A.kk += (long long)c;
  if (A.trace) A.trace += 9 * (int64_t)c;
  if (A.col0_dev) A.col0_dev += c;
  __syncthreads();
  if (threadIdx.x == 0) *A.cur = c + 1u;
  A.cur = nullptr;
}

// ... and the whole post-LMO step in one CTA of 1024 threads (small U).
// dev_tail_rest: everything after G_U (also the fallback of k_block_tail_sm).
__device__ __forceinline__ void dev_tail_rest(BlockArgs& A, double* tail_slots) {   // 32 warps x 256
  for (int q = threadIdx.x; q < 32 * 256; q += blockDim.x) tail_slots[q] = 0.0;
  if (threadIdx.x == 0) { *A.ntouch = 0; A.nbig[0] = 0; A.nbig[1] = 0; }
  dev_pairs_count(A);
  __syncthreads();
  dev_scan_excl(A.pcount, A.L, A.poff, A.ptotal);
  dev_pairs_gen(A);
  __syncthreads();
  dev_touched_scan(A);
  dev_runs(A, A.pd);
  __syncthreads();
  dev_row_tree<0>(A, nullptr, false, 0, tail_slots);
  __syncthreads();
  dev_psumW(A.X, A.m, 256, A.scal + 1, nullptr, nullptr);
  dev_gamma(A);
  __syncthreads();
  dev_cap_check(A);
  __syncthreads();
  if (*A.status) return;
  dev_update_cols(A);
  __syncthreads();
  dev_runs(A, A.pdelta);
  __syncthreads();
  dev_row_tree<1>(A, nullptr, true, 1, tail_slots);
  if (threadIdx.x == 0) atomicAdd(A.dsteps, 1ULL);
}

__global__ void __launch_bounds__(1024, 1) k_block_tail(BlockArgs A) { pdl_entry();
  extern __shared__ double tail_slots[];   // zero outside use
  blk_take_cursor(A);
  if (*A.status) return;
  dev_psumW(A.g, A.L, 256, A.scal + 0, A.eps, A.stop);        // G_U (FW: stop check)
  if (A.stop && *A.stop) return;
  dev_tail_rest(A, tail_slots);
}

// ... and for larger U the same phases in ONE cooperative launch (every CTA resident,
// grid-wide barriers between the phases instead of 14 dependent launches): the
// single-CTA phases (step begin, the scans, the denominator, gamma) run on CTA 0.
// 1024 threads per CTA; dynamic shared memory: 32 warps x 256 chunk slots. Opt-in
// (SRO_COOP=1): ten grid barriers cost more than the per-phase kernels' gaps inside
// a CUDA graph (FW at config [1]: 40 vs 34 ms).
__global__ void __launch_bounds__(1024) k_block_coop(BlockArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double wsl[];   // zero outside use
  const bool lead_cta = blockIdx.x == 0;
  if ((A.stop && *A.stop) || *A.status) {   // uniform: nothing changes during this check
    grid.sync();
    if (lead_cta && threadIdx.x == 0 && A.cur) *A.cur += 1u;
    return;
  }
  for (int q = threadIdx.x; q < 32 * 256; q += blockDim.x) wsl[q] = 0.0;
  if (lead_cta) {
    if (threadIdx.x == 0) { *A.ntouch = 0; A.nbig[0] = 0; A.nbig[1] = 0; }
    dev_psumW(A.g, A.L, 256, A.scal + 0, A.eps, A.stop);   // G_U (FW: stop check)
  }
  dev_pairs_count(A);
  grid.sync();
  const bool stopped = A.stop && *A.stop;
  if (!stopped) {
    if (lead_cta) dev_scan_excl(A.pcount, A.L, A.poff, A.ptotal);
    grid.sync();
    dev_pairs_gen(A);
    grid.sync();
    if (lead_cta) dev_touched_scan(A);
    grid.sync();
    dev_runs(A, A.pd);
    grid.sync();
    dev_row_tree_big<0>(A, nullptr, false, 0, wsl, true);
    grid.sync();
    if (lead_cta) {
      dev_psumW(A.X, A.m, 256, A.scal + 1, nullptr, nullptr);
      dev_gamma(A);
    }
    grid.sync();
    dev_cap_check(A);
    grid.sync();
    if (!*A.status) {
      dev_update_cols(A);
      grid.sync();
      dev_runs(A, A.pdelta);
      grid.sync();
      dev_row_tree_big<1>(A, nullptr, true, 1, wsl, true);
      if (lead_cta && threadIdx.x == 0) atomicAdd(A.dsteps, 1ULL);
    }
  }
  grid.sync();   // every read of the cursor done
  if (lead_cta && threadIdx.x == 0 && A.cur) *A.cur += 1u;
}

// ---------------------------------------------------------------------------
// Sharded step (G > 1): phase A (LMO partials) -> exchange x1 -> phase B
// (gamma, update, Delta' partials) -> exchange x2 -> apply (r, h).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double* slot_of(const BlockArgs& A, double* x, int s) {
  return x + (size_t)s * A.slot_len;
}

// After phase A: publish this shard's status (its G_U subtree and Delta
// subtrees are already in its x1 slot).
__global__ void k_publish_a(BlockArgs A) {
  if (threadIdx.x == 0) slot_of(A, A.x1, A.shard)[A.m + 1] = (double)*A.status;
}
// After phase B: publish this shard's capacity flag and status (its Delta'
// subtrees are already in its x2 slot).
__global__ void k_publish_b(BlockArgs A) {
  if (threadIdx.x != 0) return;
  double* s2 = slot_of(A, A.x2, A.shard);
  s2[A.m] = (A.stop && *A.stop) ? 0.0 : (double)*A.capfail;
  s2[A.m + 1] = (double)*A.status;
}

// Combine the G phase-A slots: first error in shard order -> local status;
// G_U = tree over the shards' subtrees (FW: stop check); den = psum256 over
// rows of (tree over the shards' Delta subtrees)^2; gamma. >= 256 threads.
__device__ __forceinline__ void dev_shard_gamma(const BlockArgs& A) {
  int st = 0;
  for (int s = 0; s < A.G && !st; s++) st = (int)slot_of(A, A.x1, s)[A.m + 1];
  __syncthreads();
  if (st) { if (threadIdx.x == 0) set_status(A.status, st); return; }
  const double GU = pair_tree_pow2(A.G, [&](int s) { return slot_of(A, A.x1, s)[A.m]; });
  if (A.eps && GU <= *A.eps) {   // FW stop (every shard takes the same decision)
    if (threadIdx.x == 0) { A.scal[0] = GU; *A.stop = 1; }
    return;
  }
  __shared__ double red[8];
  const int c = threadIdx.x;
  double acc = 0.0;
  if (c < 256) {
    const int lo = (int)chunk_lo(c, A.m, 256), hi = (int)chunk_lo(c + 1, A.m, 256);
    for (int k = lo; k < hi; k++) {
      const double D = pair_tree_pow2(A.G, [&](int s) { return slot_of(A, A.x1, s)[k]; });
      acc = d_add(acc, d_mul(D, D));
    }
    acc = warp_pair_tree(acc);
    if ((c & 31) == 0) red[c >> 5] = acc;
  }
  __syncthreads();
  if (c < 32) {
    double v = (c < 8) ? red[c] : 0.0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
    if (c == 0) { A.scal[0] = GU; A.scal[1] = v; }
  }
  __syncthreads();
  dev_gamma(A);
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_shard_gamma(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  dev_shard_gamma(A);
}

// Combine the G phase-B slots. Any capacity failure: every shard restores its
// columns of U (if it had updated them) and reports SRO_ERR_CAPACITY, leaving
// the state before the step. Otherwise r_k += tree over the shards' Delta'
// subtrees and h_k = (r_k - a_k)/lambda on every row (an untouched row adds
// +0.0, which leaves r and h bitwise unchanged).
__global__ void k_shard_apply(BlockArgs A) {
  if ((A.stop && *A.stop) || *A.status) return;
  int st = 0, cf = 0;
  for (int s = 0; s < A.G; s++) {
    const double* x = slot_of(A, A.x2, s);
    if (!st) st = (int)x[A.m + 1];
    cf |= (x[A.m] != 0.0);
  }
  if (st) { if (gtid() == 0) set_status(A.status, st); return; }
  if (cf) {
    const int col0 = block_col0(A);
    if (!*A.capfail) {
      for (int p = gtid(); p < A.L; p += gstride()) {
        const int i = col0 + p;
        int keep = 0;
        for (int q = A.poff[p]; q < A.poff[p + 1]; q++) {
          if (A.ptold[q] != 0.0) {
            A.srow[(int64_t)i * A.cap + keep] = A.prow[q];
            A.sval[(int64_t)i * A.cap + keep] = A.ptold[q];
            keep++;
          }
        }
        A.cnt[i] = keep;
      }
    }
    for (int w = gtid(); w < *A.ntouch; w += gstride()) { A.rowcnt[A.trows[w]] = 0; A.tcur[w] = 0; }
    if (gtid() == 0) set_status(A.status, 6);
    return;
  }
  for (int k = gtid(); k < A.m; k += gstride()) {
    const double D = pair_tree_pow2(A.G, [&](int s) { return slot_of(A, A.x2, s)[k]; });
    const double rn = d_add(A.r[k], D);
    A.r[k] = rn;
    A.h[k] = d_div(d_sub(rn, A.a[k]), A.lambda);
  }
  if (gtid() == 0) atomicAdd(A.dsteps, 1ULL);
}

// Phase A in one CTA of 1024 threads (small U).
__global__ void __launch_bounds__(1024, 1) k_shard_tail_a(BlockArgs A) {
  extern __shared__ double tail_slots[];
  double* s1 = slot_of(A, A.x1, A.shard);
  if (!(A.stop && *A.stop) && !*A.status) {
    for (int q = threadIdx.x; q < 32 * 256; q += blockDim.x) tail_slots[q] = 0.0;
    if (threadIdx.x == 0) { *A.ntouch = 0; *A.capfail = 0; A.nbig[0] = 0; A.nbig[1] = 0; }
    dev_psumW(A.g, A.L, A.W, s1 + A.m, nullptr, nullptr);
    dev_pairs_count(A);
    dev_zero_dbl(s1, A.m);
    __syncthreads();
    dev_scan_excl(A.pcount, A.L, A.poff, A.ptotal);
    dev_pairs_gen(A);
    __syncthreads();
    dev_touched_scan(A);
    dev_runs(A, A.pd);
    __syncthreads();
    dev_row_tree<2>(A, s1, false, 0, tail_slots);
  }
  __syncthreads();
  if (threadIdx.x == 0) s1[A.m + 1] = (double)*A.status;
}

// Phase B in one CTA of 1024 threads (small U).
__global__ void __launch_bounds__(1024, 1) k_shard_tail_b(BlockArgs A) {
  extern __shared__ double tail_slots[];
  double* s2 = slot_of(A, A.x2, A.shard);
  for (int q = threadIdx.x; q < 32 * 256; q += blockDim.x) tail_slots[q] = 0.0;
  bool run = !(A.stop && *A.stop) && !*A.status;
  if (run) {
    dev_shard_gamma(A);
    __syncthreads();
    run = !(A.stop && *A.stop) && !*A.status;
  }
  if (run) {
    dev_cap_check(A);
    dev_zero_dbl(s2, A.m);
    __syncthreads();
    if (*A.capfail == 0) {
      dev_update_cols(A);
      __syncthreads();
      dev_runs(A, A.pdelta);
      __syncthreads();
      dev_row_tree<2>(A, s2, true, 1, tail_slots);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s2[A.m] = run ? (double)*A.capfail : 0.0;
    s2[A.m + 1] = (double)*A.status;
  }
}

}  // namespace sro
