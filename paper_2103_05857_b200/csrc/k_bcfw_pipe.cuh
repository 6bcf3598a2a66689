// k_bcfw_pipe.cuh — pipelined, warp-specialised persistent loop for the
// sequential BCFW family (BCFW Alg. 1, BCAFW Alg. A.2, BCPFW Alg. A.3; U / P /
// explicit visits; DEC or ELS) on dense costs: the LMO of the NEXT visited
// column runs concurrently with the serial update of the current one.
//
// Why this is exact. Step s (column i_s) changes h only on its merged support
// T_s = supp(t_{i_s}) U {j_s} (r moves on those rows only). So the
// LMO of column i_{s+1} (Eq. 9) can be split:
//   * the LMO warps scan every row NOT in T_s against h before step s — the
//     same values as after it — while warp 0 runs the serial part of step s;
//   * then warp 0 evaluates the <= 32 rows of T_s exactly with the updated h
//     (C_{k,i_{s+1}} prefetched during step s) and merges them with the warp
//     partials. min / argmin with the lowest-row tie-break is order-free, so
//     j_{s+1} and its value are exactly those of a full scan.
//
// Roles (16 warps launched; warp w runs on SM sub-partition w % 4):
//   * warp 0: serial part (serial_step of k_bcfw.cuh — the same arithmetic as
//     every other BCFW kernel), the merge, and publishing the next mask. Warps
//     4, 8, 12 stay idle so warp 0 has its sub-partition to itself.
//   * the 12 warps with w % 4 != 0 (384 threads): LMO. Thread lt owns the
//     128-bit vectors q = lt + u*384 (u < MAXV) and tail row nvec*W + lt,
//     prefetches its part of the column one visit ahead into registers and
//     reads h from a planar shared-memory copy (plane p holds the pairs
//     (h[Wq+2p], h[Wq+2p+1]) at index q: conflict-free 128-bit loads) that warp 0
//     keeps current; the rows warp 0 writes during step s are exactly the masked
//     rows, so the concurrent reads never depend on them. Masks travel as one
//     bit word per owner thread.
// Warp 0 and the LMO warps run separate loops and hand off through two named
// barriers: BAR_PART (LMO partials ready: LMO warps arrive, warp 0 waits) and
// BAR_MASK (next mask published: warp 0 arrives, LMO warps wait).
#pragma once
#include <type_traits>
#include "k_bcfw.cuh"

namespace sro {

constexpr int PIPE_THREADS = 512;
constexpr int PIPE_LMO_WARPS = 12;
constexpr int PIPE_LMO = PIPE_LMO_WARPS * 32;
constexpr int PIPE_SYNC = PIPE_LMO + 32;   // threads taking part in the named barriers
constexpr int BAR_PART = 1, BAR_MASK = 2;

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <typename T, int MAXV, int NL = PIPE_LMO>
struct PipeCol {
  using V = typename Vec<T>::type;
  static constexpr int W = Vec<T>::W;
  const T* C;
  int64_t ld;
  int m, nvec;
  V cur[MAXV], nxt[MAXV];
  T ctail, ntail;
  __device__ __forceinline__ void fetch(int i, int lt) {
    const V* p = reinterpret_cast<const V*>(C + (int64_t)i * ld);
#pragma unroll
    for (int u = 0; u < MAXV; u++) {
      const int q = lt + u * NL;
      if (q < nvec) nxt[u] = __ldg(p + q);
    }
    const int kt = nvec * W + lt;
    if (kt < m) ntail = __ldg(C + (int64_t)i * ld + kt);
  }
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int u = 0; u < MAXV; u++) cur[u] = nxt[u];
    ctail = ntail;
  }
};

// h of the W rows of vector q from the planar copy
__device__ __forceinline__ void pipe_h(const double2* hp, int nvec, int q, float4*, double* hv) {
  const double2 a = hp[q], b = hp[nvec + q];
  hv[0] = a.x; hv[1] = a.y; hv[2] = b.x; hv[3] = b.y;
}
__device__ __forceinline__ void pipe_h(const double2* hp, int, int q, double2*, double* hv) {
  const double2 a = hp[q];
  hv[0] = a.x; hv[1] = a.y;
}
template <int W>
__device__ __forceinline__ int pipe_hidx(int k, int nvec) {   // double index of row k < nvec*W in the planar copy
  const int q = k / W, t = k % W;
  return (((t >> 1) * nvec + q) << 1) + (t & 1);
}

// Masked local argmin over one vector: rows whose bit is set in `mk` are skipped.
__device__ __forceinline__ void vproc_mask(const float4& v, const double* hd, int k, unsigned mk, double& best,
                                           int& bj) {
  const double x0 = d_add((double)v.x, hd[0]), x1 = d_add((double)v.y, hd[1]);
  const double x2 = d_add((double)v.z, hd[2]), x3 = d_add((double)v.w, hd[3]);
  if (!(mk & 1u) && x0 < best) { best = x0; bj = k; }
  if (!(mk & 2u) && x1 < best) { best = x1; bj = k + 1; }
  if (!(mk & 4u) && x2 < best) { best = x2; bj = k + 2; }
  if (!(mk & 8u) && x3 < best) { best = x3; bj = k + 3; }
}
__device__ __forceinline__ void vproc_mask(const double2& v, const double* hd, int k, unsigned mk, double& best,
                                           int& bj) {
  const double x0 = d_add(v.x, hd[0]), x1 = d_add(v.y, hd[1]);
  if (!(mk & 1u) && x0 < best) { best = x0; bj = k; }
  if (!(mk & 2u) && x1 < best) { best = x1; bj = k + 1; }
}

struct PipeLayout {
  __host__ __device__ static size_t fixed() {
    return 256 * 8 + 16 * 8 + 16 * 4 + 16 * 4 + 8 * 8      // slots, wkey, wj, misc, (spare)
           + PIPE_LMO * 4;                                   // mask words
  }
  __host__ __device__ static size_t bytes(int m, int n, int steps, bool visit_smem) {
    size_t b = fixed() + 4 * rup16((size_t)m * 8) + rup16((size_t)n * 4);
    if (visit_smem) b += rup16((size_t)steps * 4);
    return b;
  }
};

// LMO thread index and bit of row k (rows of full vectors, then the tail rows)
template <int W, int NL = PIPE_LMO>
__device__ __forceinline__ void pipe_owner(int k, int nvec, int& lt, unsigned& bit) {
  if (k < nvec * W) {
    const int q = k / W;
    lt = q % NL;
    bit = 1u << ((q / NL) * W + (k % W));
  } else {
    lt = k - nvec * W;
    bit = 1u << 31;
  }
}

#ifdef SRO_PHASE_TIMING
#define PW_MARK(idx)                          \
  do {                                        \
    const long long t_ = clock64();           \
    pw_acc[idx] += t_ - pw_t;                 \
    pw_t = t_;                                \
  } while (0)
#else
#define PW_MARK(idx) do {} while (0)
#endif

template <typename T, int MAXV, int VAR>
__global__ void __launch_bounds__(PIPE_THREADS, 1) k_bcfw_pipe(BcfwArgs A, const T* __restrict__ Cg, int64_t ld) {
  if (bcfw_halted(A)) return;
  constexpr int W = Vec<T>::W;
  extern __shared__ __align__(16) char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  const int nvec = m / W;
  const int steps = A.steps;
  char* p = smraw;
  double* slots = reinterpret_cast<double*>(p); p += 256 * 8;
  unsigned long long* wkey = reinterpret_cast<unsigned long long*>(p); p += 16 * 8;
  int* wj = reinterpret_cast<int*>(p); p += 16 * 4;
  volatile int* misc = reinterpret_cast<volatile int*>(p); p += 16 * 4;   // [2] = abort
  p += 8 * 8;
  unsigned* mflag = reinterpret_cast<unsigned*>(p); p += PIPE_LMO * 4;
  double* sh_h = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_r = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_a = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* hpd = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);   // planar h (rows < nvec*W)
  const double2* hp = reinterpret_cast<const double2*>(hpd);
  int* sh_cnt = reinterpret_cast<int*>(p); p += rup16((size_t)n * 4);
  const int* vis = A.visit;
  if (A.visit_smem) {
    int* sv = reinterpret_cast<int*>(p); p += rup16((size_t)steps * 4);
    for (int q = tid; q < steps; q += PIPE_THREADS) sv[q] = A.visit[q];
    vis = sv;
  }
  for (int c = tid; c < 256; c += PIPE_THREADS) slots[c] = 0.0;
  for (int k = tid; k < m; k += PIPE_THREADS) {
    const double hk = A.h[k];
    sh_h[k] = hk; sh_r[k] = A.r[k]; sh_a[k] = A.a[k];
    if (k < nvec * W) hpd[pipe_hidx<W>(k, nvec)] = hk;
  }
  for (int c = tid; c < n; c += PIPE_THREADS) sh_cnt[c] = A.cnt[c];
  for (int c = tid; c < PIPE_LMO; c += PIPE_THREADS) mflag[c] = 0;
  if (tid == 0) misc[2] = 0;
  if (tid < 16) { wkey[tid] = ~0ULL; wj[tid] = 0x7fffffff; }
  __syncthreads();

  if (steps > 0 && warp > 0 && (warp & 3) != 0) {
    // =================== LMO warps ===================
    const int lw = warp - 1 - (warp >> 2);   // 0..11
    const int lt = lw * 32 + lane;
    const int kt = nvec * W + lt;
    PipeCol<T, MAXV> col;
    col.C = Cg; col.ld = ld; col.m = m; col.nvec = nvec;
    col.fetch(vis[0], lt);
    for (int t = 0; t < steps; t++) {
      col.advance();
      if (t + 1 < steps) col.fetch(vis[t + 1], lt);   // lands during the next step
      nbar_sync(BAR_MASK, PIPE_SYNC);                  // mask T_{t-1} published (empty for t = 0)
      if (misc[2]) break;
      const unsigned mk = mflag[lt];
      mflag[lt] = 0;
      double hv[MAXV][W];
#pragma unroll
      for (int u = 0; u < MAXV; u++) {
        const int q = lt + u * PIPE_LMO;
        if (q < nvec) pipe_h(hp, nvec, q, col.cur, hv[u]);
      }
      const double ht = kt < m ? sh_h[kt] : 0.0;
      double best = dinf();
      int bj = 0x7fffffff;
      if (mk == 0u) {
#pragma unroll
        for (int u = 0; u < MAXV; u++) {
          const int q = lt + u * PIPE_LMO;
          if (q < nvec) vproc(col.cur[u], hv[u], W * q, best, bj);
        }
        if (kt < m) {
          const double x = d_add((double)col.ctail, ht);
          if (x < best) { best = x; bj = kt; }
        }
      } else {
#pragma unroll
        for (int u = 0; u < MAXV; u++) {
          const int q = lt + u * PIPE_LMO;
          if (q < nvec) vproc_mask(col.cur[u], hv[u], W * q, (mk >> (u * W)) & ((1u << W) - 1u), best, bj);
        }
        if (kt < m && !(mk >> 31)) {
          const double x = d_add((double)col.ctail, ht);
          if (x < best) { best = x; bj = kt; }
        }
      }
      unsigned long long key = okey(best);
      warp_argmin_redux(key, bj);
      if (lane == 0) { wkey[lw] = key; wj[lw] = bj; }
      nbar_arrive(BAR_PART, PIPE_SYNC);
    }
  } else if (steps > 0 && warp == 0) {
    // =================== serial warp ===================
    int i = vis[0];
    int rw = 0x7fffffff, c0 = 0;
    double tv = 0.0, bi = 0.0, cw = 0.0;
    c0 = sh_cnt[i];
    bi = A.b[i];
    if (lane < c0) { rw = A.srow[(int64_t)i * cap + lane]; tv = A.sval[(int64_t)i * cap + lane]; }
    if (lane < c0) cw = (double)__ldg(Cg + (int64_t)i * ld + rw);
    // the next visited column's slab (loaded a step ahead, C at its rows a step
    // later) and the slab after it: no dependent global load on a step's critical path
    int i1 = steps > 1 ? vis[1] : i, c01 = 0, rw1 = 0x7fffffff;
    double tv1 = 0.0, bi1 = 0.0;
    if (steps > 1) {
      c01 = sh_cnt[i1];
      bi1 = A.b[i1];
      if (lane < c01) { rw1 = A.srow[(int64_t)i1 * cap + lane]; tv1 = A.sval[(int64_t)i1 * cap + lane]; }
    }
    int iprev = -1;
    int j = 0, trow = 0x7fffffff, MT = 0;
    double mv = 0.0;
    // merged support of (slab, j) -> this lane's mask row; set the owners' mask bits
    auto publish_mask = [&]() {
      const bool j_in = __ballot_sync(FULL, lane < c0 && rw == j) != 0u;
      const int ins = __popc(__ballot_sync(FULL, lane < c0 && rw < j));
      MT = c0 + (j_in ? 0 : 1);
      int src = (j_in || lane < ins) ? lane : lane - 1;
      if (src < 0) src = 0;
      trow = __shfl_sync(FULL, rw, src);
      if (!j_in && lane == ins) trow = j;
      if (lane >= MT) trow = 0x7fffffff;
      if (lane < MT) {
        int ot;
        unsigned bit;
        pipe_owner<W>(trow, nvec, ot, bit);
        atomicOr(&mflag[ot], bit);
      }
    };
    // prologue: the full LMO of the first column
    nbar_arrive(BAR_MASK, PIPE_SYNC);
    nbar_sync(BAR_PART, PIPE_SYNC);
    {
      unsigned long long k2 = lane < PIPE_LMO_WARPS ? wkey[lane] : ~0ULL;
      int j2 = lane < PIPE_LMO_WARPS ? wj[lane] : 0x7fffffff;
      warp_argmin_redux(k2, j2);
      j = j2;
      mv = okey_inv(k2);
    }
    publish_mask();
    __syncwarp();
    if (steps > 1) nbar_arrive(BAR_MASK, PIPE_SYNC);
    int done = 0;
    int inext = steps > 1 ? vis[1] : i;   // the next visited column (carried in a register)
#ifdef SRO_PHASE_TIMING
    long long pw_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long pw_t = clock64();
    PhaseState sp_state;
    for (int q = 0; q < 16; q++) sp_state.acc[q] = 0;
#endif
    for (int s = 0; s < steps; s++) {
      const long long kk = A.k0 + s;
      const bool has_next = s + 1 < steps;
      const int i2 = s + 2 < steps ? vis[s + 2] : inext;
      // ---- prefetch what the merge and the next steps need
      double cn = 0.0, cwn = 0.0, tvn = 0.0, bin = 0.0;
      int c0n = 0, rwn = 0x7fffffff;
      if (has_next) {
        if (lane < MT) cn = (double)__ldg(Cg + (int64_t)inext * ld + trow);
        if (lane < c01) cwn = (double)__ldg(Cg + (int64_t)inext * ld + rw1);
      }
      PW_MARK(7);
      if (s + 2 < steps) {
        c0n = sh_cnt[i2];
        bin = A.b[i2];
        if (lane < c0n) { rwn = A.srow[(int64_t)i2 * cap + lane]; tvn = A.sval[(int64_t)i2 * cap + lane]; }
      }
      // ---- the serial part of step s
      PW_MARK(0);
      const double gk = lane < c0 ? d_add(cw, sh_h[rw]) : 0.0;
      PW_MARK(1);
#ifdef SRO_PHASE_TIMING
      sp_state.t = clock64();
      const StepOut o =
          serial_step<VAR>(A, kk, i, j, mv, bi, c0, rw, tv, gk, sh_r, sh_h, nullptr, sh_a, sh_cnt, slots, nullptr, &sp_state);
#else
      const StepOut o =
          serial_step<VAR>(A, kk, i, j, mv, bi, c0, rw, tv, gk, sh_r, sh_h, nullptr, sh_a, sh_cnt, slots, nullptr);
#endif
      PW_MARK(2);
      if (o.ev && o.erow < nvec * W) hpd[pipe_hidx<W>(o.erow, nvec)] = o.hnew;   // planar copy for the LMO warps
      if (o.abort) {
        if (lane == 0) {
          misc[2] = 1;
          set_status(A.status, !(mv < 1.0e308 && mv > -1.0e308) ? 5 : 6);
        }
        __syncwarp();
        if (has_next) nbar_arrive(BAR_MASK, PIPE_SYNC);   // release the LMO warps (they see the abort)
        break;
      }
      if (A.trace && lane == 0) {
        double* tr = A.trace + 9 * (int64_t)s;
        tr[0] = (double)kk; tr[1] = i; tr[2] = j; tr[3] = (VAR == VAR_PLAIN) ? -1 : o.vrow;
        tr[4] = o.dir; tr[5] = o.gamma; tr[6] = o.num; tr[7] = o.den; tr[8] = mv;
      }
      done = s + 1;
      if (!has_next) break;
      // ---- merge: the rows of T_s with the updated h, and the LMO warp partials
      PW_MARK(3);
      PW_MARK(2);
      nbar_sync(BAR_PART, PIPE_SYNC);
      PW_MARK(3);
      unsigned long long ka = ~0ULL;
      int ja = 0x7fffffff;
      if (lane < MT) { ka = okey(d_add(cn, sh_h[trow])); ja = trow; }
      if (lane < PIPE_LMO_WARPS) {
        const unsigned long long kb = wkey[lane];
        const int jb = wj[lane];
        if (kb < ka || (kb == ka && jb < ja)) { ka = kb; ja = jb; }
      }
      warp_argmin_redux(ka, ja);
      PW_MARK(4);
      // ---- the next column's slab: its own updated slab when the same column is
      // visited again; reloaded when the prefetch may predate an update of it
      // (it was read before step s-1 ran); else the prefetched one
      if (inext == i) {
        new_slab_entry(o, rw, tv);
        c0 = o.nk;
        cw = lane < c0 ? (double)__ldg(Cg + (int64_t)i * ld + rw) : 0.0;
      } else if (inext == iprev) {
        c0 = sh_cnt[inext];
        bi = bi1;
        rw = 0x7fffffff; tv = 0.0;
        if (lane < c0) { rw = A.srow[(int64_t)inext * cap + lane]; tv = A.sval[(int64_t)inext * cap + lane]; }
        cw = lane < c0 ? (double)__ldg(Cg + (int64_t)inext * ld + rw) : 0.0;
      } else {
        c0 = c01; bi = bi1; rw = rw1; tv = tv1; cw = cwn;
      }
      c01 = c0n; bi1 = bin; rw1 = rwn; tv1 = tvn;
      iprev = i;
      i = inext;
      inext = i2;
      j = ja;
      mv = okey_inv(ka);
      PW_MARK(5);
      publish_mask();
      __syncwarp();
      nbar_arrive(BAR_MASK, PIPE_SYNC);
      PW_MARK(6);
    }
    if (lane == 0) *A.steps_done = done;
#ifdef SRO_PHASE_TIMING
    if (lane == 0 && A.phase) {
      for (int q = 0; q < 8; q++) A.phase[q] += pw_acc[q];
      for (int q = 8; q < 16; q++) A.phase[q] += sp_state.acc[q];
    }
#endif
  }
  __syncthreads();
  for (int k = tid; k < m; k += PIPE_THREADS) { A.h[k] = sh_h[k]; A.r[k] = sh_r[k]; }
  if (steps == 0 && tid == 0) *A.steps_done = 0;
}

// ---------------------------------------------------------------------------
// Gap-adaptive sampling (BCFW-GA, Alg. A.4; with the away /
// pairwise directions as in Fig. 4(c,d)) on dense costs. The next column is
// drawn from the Fenwick tree only after the current step has refreshed its
// stored gap, so steps cannot overlap; what the pipelined layout removes is the
// second LMO pass of the post-update refresh G_i = g_i(T^{k+1}) (R15):
//   min_k (C_ki + h'_k) = min( min over k not in T of (C_ki + h_k),
//                              min over k in T of (C_ki + h'_k) ),
// T = supp(t_i) U {j} the rows the step may change. The LMO warps get the support
// as a mask before they scan, and return for each warp the overall (value,
// row) minimum with its C_ki, plus the two smallest (value, row) pairs among
// the rows outside the support; the minimum outside T is the second of those
// if j lies outside the support, else the first. So one scan serves the step
// and the refresh, with every value computed exactly as a full scan would.
// Per step: draw (warp 0) -> column index to the LMO warps (BAR_COL) -> the
// support mask (BAR_MASK) -> partials (BAR_PART) -> serial part, gap refresh,
// Fenwick update (warp 0).
// Speculation (A.spec): while warp 0 runs the merge, serial part, gap refresh
// and Fenwick update of step s, the LMO warps would idle. Instead one of them
// draws a candidate next column i' from the tree as it stands (before step s's
// refresh: the drawn column about two times in three on config [1]), reads its
// support S' (step s changes no column but i_s; i' = i_s is not pre-scanned)
// and prefetches its slab lines for warp 0 into L1; all LMO warps load column
// i' and, once warp 0 has published T_s = supp(t_{i_s}) U {j_s} (the only rows
// whose h step s changes), pre-scan it over the rows outside S' U T_s, whose h
// is already final. If the draw gives i', each thread only adds its rows of
// T_s \ S' with the updated h, ordered by (value, row), which is exactly the
// first minimum and the second smallest value the ascending scan would find;
// else the full scan runs as before. Every value is the one without speculation.
constexpr int BAR_COL = 3;
constexpr int BAR_SPEC = 4;   // LMO warps only: the speculative next column (misc[4]) and its support mask
constexpr int BAR_T = 5;      // T of the step published (warp 0 arrives, LMO warps wait; speculation only)
// The LMO warps are the 12 with w % 4 != 0, as in k_bcfw_pipe: warp 0 has its SM
// sub-partition to itself, so the speculative pre-scan that runs during its
// serial part takes none of its issue slots (15 scanning warps, three of them
// beside warp 0, measured 3.09 us per step against 2.96 without speculation).
constexpr int GA_LMO_WARPS = PIPE_LMO_WARPS;
constexpr int GA_LMO = GA_LMO_WARPS * 32;
constexpr int GA_SYNC = GA_LMO + 32;

struct GaPipeLayout {
  __host__ __device__ static size_t fixed() {
    return 256 * 8 + 16 * 4 * 8 + 16 * 4 * 4 + 16 * 4 + 3 * GA_LMO * 4;   // slots, key partials, row partials, misc, 3 masks
  }
  // a_smem / gs_smem: a and the stored gaps in shared memory (else read from / written to
  // global memory: a is read for the touched rows only, the stored gap once per step
  // while the scan runs, so larger m, n keep the fast kernel)
  __host__ __device__ static size_t bytes(int m, int n, bool a_smem = true, bool gs_smem = true) {
    return fixed() + (a_smem ? 4 : 3) * rup16((size_t)m * 8) + rup16((size_t)n * 4) +
           (gs_smem ? rup16((size_t)n * 8) : 0) + rup16((size_t)(n + 1) * 8);
  }
};

// (key, row) lexicographic minimum over the warp with 3 REDUX.MIN; returns the lane that held it
__device__ __forceinline__ int warp_argmin_key(unsigned long long& key, int& j) {
  const unsigned long long k0 = key;
  const int j0 = j;
  warp_argmin_redux(key, j);
  return __ffs(__ballot_sync(FULL, k0 == key && j0 == j)) - 1;
}

// GSM: a and the stored gaps in shared memory (else both in global memory)
template <typename T, int MAXV, int VAR, bool GSM>
__global__ void __launch_bounds__(PIPE_THREADS, 1) k_bcfw_ga_pipe(BcfwArgs A, const T* __restrict__ Cg, int64_t ld) {
  if (bcfw_halted(A)) return;
  constexpr int W = Vec<T>::W;
  extern __shared__ __align__(16) char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m, n = A.n, cap = A.cap;
  const int nvec = m / W;
  const int steps = A.steps;
  char* p = smraw;
  double* slots = reinterpret_cast<double*>(p); p += 256 * 8;
  unsigned long long* pk = reinterpret_cast<unsigned long long*>(p); p += 16 * 4 * 8;   // [4][16]: all, u1, u2, cval
  int* pj = reinterpret_cast<int*>(p); p += 16 * 4 * 4;                               // [4][16] rows
  volatile int* misc = reinterpret_cast<volatile int*>(p); p += 16 * 4;   // [0] = column, [2] = abort
  unsigned* mflag = reinterpret_cast<unsigned*>(p); p += GA_LMO * 4;
  unsigned* mflagT = reinterpret_cast<unsigned*>(p); p += GA_LMO * 4;   // T of the step (speculation)
  unsigned* mflagS = reinterpret_cast<unsigned*>(p); p += GA_LMO * 4;   // support of the speculative column
  double* sh_h = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_r = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  double* sh_a = GSM ? reinterpret_cast<double*>(p) : const_cast<double*>(A.a);
  if (GSM) p += rup16((size_t)m * 8);
  double* hpd = reinterpret_cast<double*>(p); p += rup16((size_t)m * 8);
  const double2* hp = reinterpret_cast<const double2*>(hpd);
  int* sh_cnt = reinterpret_cast<int*>(p); p += rup16((size_t)n * 4);
  double* Gs = GSM ? reinterpret_cast<double*>(p) : A.G;
  if (GSM) p += rup16((size_t)n * 8);
  double* fens = reinterpret_cast<double*>(p); p += rup16((size_t)(n + 1) * 8);
  for (int c = tid; c < 256; c += PIPE_THREADS) slots[c] = 0.0;
  for (int k = tid; k < m; k += PIPE_THREADS) {
    const double hk = A.h[k];
    sh_h[k] = hk; sh_r[k] = A.r[k];
    if (GSM) sh_a[k] = A.a[k];
    if (k < nvec * W) hpd[pipe_hidx<W>(k, nvec)] = hk;
  }
  for (int c = tid; c < n; c += PIPE_THREADS) { sh_cnt[c] = A.cnt[c]; if (GSM) Gs[c] = A.G[c]; }
  for (int c = tid; c <= n; c += PIPE_THREADS) fens[c] = A.fen[c];
  for (int c = tid; c < GA_LMO; c += PIPE_THREADS) { mflag[c] = 0; mflagT[c] = 0; mflagS[c] = 0; }
  if (tid == 0) { misc[0] = 0; misc[2] = 0; misc[4] = -1; }
  __syncthreads();

  if (steps > 0 && warp > 0 && (warp & 3) != 0) {
    // =================== LMO warps ===================
    const int lw = warp - 1 - (warp >> 2);   // 0..11; sub-partition lw % 3 + 1
    const int lt = lw * 32 + lane;
    const int kt = nvec * W + lt;
    PipeCol<T, MAXV, GA_LMO> col;
    col.C = Cg; col.ld = ld; col.m = m; col.nvec = nvec;
    int ispec = -1;     // the column held in col.cur from the speculative prefetch (-1: none)
    bool pre = false;   // (pu1, pj1, pc1, pu2) hold the pre-scan of column ispec
    double pu1 = 0.0, pu2 = 0.0;
    T pc1 = T(0);
    int pj1 = 0x7fffffff;
    // two smallest (value, row) of this thread's rows outside the mask, rows ascending;
    // the second as a value only
    auto scan = [&](unsigned mk, double& u1, int& j1, T& c1, double& u2) {
      u1 = dinf(); u2 = dinf(); c1 = T(0); j1 = 0x7fffffff;
      auto go = [&](auto masked_tag) {
        constexpr bool MASKED = decltype(masked_tag)::value;
        auto visit = [&](T c, double h, int k, bool masked) {
          const double x = d_add((double)c, h);
          const bool l1 = !(MASKED && masked) && x < u1;
          const bool l2 = !(MASKED && masked) && !l1 && x < u2;
          u2 = l1 ? u1 : (l2 ? x : u2);
          u1 = l1 ? x : u1; j1 = l1 ? k : j1; c1 = l1 ? c : c1;
        };
#pragma unroll
        for (int u = 0; u < MAXV; u++) {
          const int q = lt + u * GA_LMO;
          if (q < nvec) {
            double hv[W];
            pipe_h(hp, nvec, q, col.cur, hv);
            const unsigned mu = mk >> (u * W);
            if constexpr (W == 4) {
              visit(col.cur[u].x, hv[0], W * q, mu & 1u);
              visit(col.cur[u].y, hv[1], W * q + 1, mu & 2u);
              visit(col.cur[u].z, hv[2], W * q + 2, mu & 4u);
              visit(col.cur[u].w, hv[3], W * q + 3, mu & 8u);
            } else {
              visit(col.cur[u].x, hv[0], W * q, mu & 1u);
              visit(col.cur[u].y, hv[1], W * q + 1, mu & 2u);
            }
          }
        }
        if (kt < m) visit(col.ctail, sh_h[kt], kt, mk >> 31);
      };
      if (__any_sync(FULL, mk != 0u)) go(std::true_type{});
      else go(std::false_type{});
    };
#ifdef SRO_PHASE_TIMING
    long long sp_t = 0;
#endif
    for (int t = 0; t < steps; t++) {
      nbar_sync(BAR_COL, GA_SYNC);                   // the drawn column (or abort)
      if (misc[2]) break;
      const int i = misc[0];
      const bool hit = pre && i == ispec;
#ifdef SRO_PHASE_TIMING
      if (lane == 0 && lw == 0 && A.phase && t > 0) {
        atomicAdd((unsigned long long*)&A.phase[21], (unsigned long long)(clock64() - sp_t));
        atomicAdd((unsigned long long*)&A.phase[22], (unsigned long long)hit);
        atomicAdd((unsigned long long*)&A.phase[23], (unsigned long long)pre);
      }
#endif
      if (i != ispec) {
        col.fetch(i, lt);
        col.advance();
      }
      nbar_sync(BAR_MASK, GA_SYNC);                  // its support as a mask
      const unsigned mk = mflag[lt];
      mflag[lt] = 0;
      const unsigned mkT = mflagT[lt];               // T of the previous step (speculation only)
      mflagT[lt] = 0;
#ifdef SRO_PHASE_TIMING
      long long lt0 = clock64() + (long long)(mk & 0u);
#endif
      // rows outside the support only: smallest (value, row) with its C, and the
      // second smallest value (the support rows are warp 0's: it holds their C)
      // (only warps holding a support row run the variant with the mask tests)
      double u1, u2;
      T c1;
      int j1;
      if (hit) {
        // the pre-scan covered every row outside supp U T_prev with h as it is now;
        // the rows of T_prev outside the support, with their updated h, join by
        // (value, row) order, which is what the ascending scan's first minimum is
        u1 = pu1; u2 = pu2; c1 = pc1; j1 = pj1;
        const unsigned fx = mkT & ~mk;
        if (__any_sync(FULL, fx != 0u)) {
          auto visit = [&](T c, double h, int k, bool on) {
            if (!on) return;
            const double x = d_add((double)c, h);
            if (x < u1 || (x == u1 && k < j1)) { u2 = u1; u1 = x; j1 = k; c1 = c; }
            else if (x < u2) u2 = x;
          };
#pragma unroll
          for (int u = 0; u < MAXV; u++) {
            const int q = lt + u * GA_LMO;
            const unsigned mu = fx >> (u * W);
            if (q < nvec && (mu & ((1u << W) - 1u))) {
              double hv[W];
              pipe_h(hp, nvec, q, col.cur, hv);
              if constexpr (W == 4) {
                visit(col.cur[u].x, hv[0], W * q, mu & 1u);
                visit(col.cur[u].y, hv[1], W * q + 1, mu & 2u);
                visit(col.cur[u].z, hv[2], W * q + 2, mu & 4u);
                visit(col.cur[u].w, hv[3], W * q + 3, mu & 8u);
              } else {
                visit(col.cur[u].x, hv[0], W * q, mu & 1u);
                visit(col.cur[u].y, hv[1], W * q + 1, mu & 2u);
              }
            }
          }
          if (kt < m && (fx >> 31)) visit(col.ctail, sh_h[kt], kt, true);
        }
      } else {
        scan(mk, u1, j1, c1, u2);
      }
#ifdef SRO_PHASE_TIMING
      long long lt1 = clock64() + (long long)(j1 & 0);
#endif
      unsigned long long k1 = okey(u1);
      int r1 = j1;
      const int w1 = warp_argmin_key(k1, r1);
      const double cw1 = (double)__shfl_sync(FULL, c1, w1);
      const unsigned long long k2l = lane == w1 ? okey(u2) : okey(u1);
      const unsigned h2 = __reduce_min_sync(FULL, (unsigned)(k2l >> 32));
      const unsigned l2 = __reduce_min_sync(FULL, (unsigned)(k2l >> 32) == h2 ? (unsigned)k2l : 0xffffffffu);
      if (lane == 0) {
        pk[lw] = k1; pj[lw] = r1; pk[16 + lw] = ((unsigned long long)h2 << 32) | l2;
        pk[48 + lw] = (unsigned long long)__double_as_longlong(cw1);
      }
      nbar_arrive(BAR_PART, GA_SYNC);
#ifdef SRO_PHASE_TIMING
      const long long lt2 = clock64();
      if (lane == 0 && (lw == 0 || lw == GA_LMO_WARPS - 1) && A.phase) {
        atomicAdd((unsigned long long*)&A.phase[lw == 0 ? 16 : 18], (unsigned long long)(lt1 - lt0));
        atomicAdd((unsigned long long*)&A.phase[lw == 0 ? 17 : 19], (unsigned long long)(lt2 - lt1));
      }
#endif
      pre = false;
      ispec = -1;
#ifdef SRO_PHASE_TIMING
      sp_t = clock64();
#endif
      if (A.spec && t + 1 < steps) {
        // speculative next draw from the tree as it stands (warp 0 may be updating
        // it: any node value read is an old or a new one; the result only decides
        // what to prefetch and pre-scan)
        if (lw == 0) {
          int ic = 0;
          if (lane == 0) {
            ic = ga_draw_sh(fens, Gs, n, uniform53(rng_u64(A.seed, 1, (uint64_t)(A.k0 + t + 1))));
            misc[4] = ic;
          }
          ic = __shfl_sync(FULL, ic, 0);
          if (ic != i) {
            // its support (step t does not touch column ic) -> mflagS; its slab lines
            // (warp 0's first loads after the draw) into L1
            const int cs = sh_cnt[ic];
            for (int q = lane; q < cs; q += 32) {
              int ot;
              unsigned bit;
              pipe_owner<W, GA_LMO>(A.srow[(int64_t)ic * cap + q], nvec, ot, bit);
              atomicOr(&mflagS[ot], bit);
            }
            const char* pl = nullptr;
            if (lane == 0) pl = reinterpret_cast<const char*>(A.srow + (int64_t)ic * cap);
            else if (lane <= 2 && (lane - 1) * 16 < cs) pl = reinterpret_cast<const char*>(A.sval + (int64_t)ic * cap + (lane - 1) * 16);
            else if (lane == 3) pl = reinterpret_cast<const char*>(A.b + ic);
            if (pl) asm volatile("prefetch.global.L1 [%0];" ::"l"(pl));
          }
        }
        nbar_sync(BAR_SPEC, GA_LMO);
        ispec = misc[4];
        col.fetch(ispec, lt);
        const unsigned mkS = mflagS[lt];
        mflagS[lt] = 0;
        nbar_sync(BAR_T, GA_SYNC);                    // T_t = supp(t_i) U {j} published by warp 0
        col.advance();
        if (ispec != i) {
          // rows outside supp(t_ispec) U T_t: their h is final for step t+1
          scan(mkS | mflagT[lt], pu1, pj1, pc1, pu2);
          pre = true;
        }
      }
#ifdef SRO_PHASE_TIMING
      if (lane == 0 && lw == 0 && A.phase) {
        const long long t2 = clock64();
        atomicAdd((unsigned long long*)&A.phase[20], (unsigned long long)(t2 - sp_t));
        sp_t = t2;
      }
#endif
    }
  } else if (steps > 0 && warp == 0) {
    // =================== serial warp ===================
    int done = 0;
    auto draw = [&](double u53) {
      int ii = 0;
      if (lane == 0) ii = ga_draw_sh(fens, Gs, n, u53);
      return __shfl_sync(FULL, ii, 0);
    };
#ifdef SRO_PHASE_TIMING
    long long pw_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long pw_t = clock64();
#endif
    int i = draw(uniform53(rng_u64(A.seed, 1, (uint64_t)A.k0)));
    if (lane == 0) misc[0] = i;
    __syncwarp();
    nbar_arrive(BAR_COL, GA_SYNC);
    for (int s = 0; s < steps; s++) {
      const long long kk = A.k0 + s;
      PW_MARK(0);
      // the drawn column's slab -> support mask for the LMO warps
      const int c0 = sh_cnt[i];
      const double bi = A.b[i];
      int rw = 0x7fffffff;
      double tv = 0.0;
      if (lane < c0) { rw = A.srow[(int64_t)i * cap + lane]; tv = A.sval[(int64_t)i * cap + lane]; }
      if (lane < c0) {
        int ot;
        unsigned bit;
        pipe_owner<W, GA_LMO>(rw, nvec, ot, bit);
        atomicOr(&mflag[ot], bit);
      }
      __syncwarp();
      nbar_arrive(BAR_MASK, GA_SYNC);
      PW_MARK(1);
      const double cw = lane < c0 ? (double)__ldg(Cg + (int64_t)i * ld + rw) : 0.0;
      // ---- partials -> LMO result (j, mv), C_ji, and the minimum outside T = supp U {j}
      const double gk = lane < c0 ? d_add(cw, sh_h[rw]) : 0.0;   // support rows: C + h (old h)
      unsigned long long ks = lane < c0 ? okey(gk) : ~0ULL;
      int js = lane < c0 ? rw : 0x7fffffff;
      const int wsl = warp_argmin_key(ks, js);
      const double csup = __shfl_sync(FULL, cw, wsl);
      const double u_next = uniform53(rng_u64(A.seed, 1, (uint64_t)(kk + 1)));   // next draw's uniform (while the LMO warps scan)
      const long long fen_node = ga_path_node(n, i);   // this lane's Fenwick node for the refresh (idem)
      // its value and the stored gap of column i (nothing writes either before the refresh)
      const double fen_old = fen_node <= n ? fens[fen_node] : 0.0;
      const double gs_old = Gs[i];
      const double dot = slab_dot(d_mul(tv, gk), c0);   // <t_i, grad_i f> (idem)
      nbar_sync(BAR_PART, GA_SYNC);
      unsigned long long k1 = lane < GA_LMO_WARPS ? pk[lane] : ~0ULL;
      int r1 = lane < GA_LMO_WARPS ? pj[lane] : 0x7fffffff;
      const unsigned long long k2lane = lane < GA_LMO_WARPS ? pk[16 + lane] : ~0ULL;
      const double cwl = lane < GA_LMO_WARPS ? __longlong_as_double((long long)pk[48 + lane]) : 0.0;
      const unsigned long long k1lane = k1;
      const int w1 = warp_argmin_key(k1, r1);
      const double c1 = __shfl_sync(FULL, cwl, w1);
      const unsigned long long k2c = lane == w1 ? k2lane : k1lane;
      const unsigned h2 = __reduce_min_sync(FULL, (unsigned)(k2c >> 32));
      const unsigned l2 = __reduce_min_sync(FULL, (unsigned)(k2c >> 32) == h2 ? (unsigned)k2c : 0xffffffffu);
      const unsigned long long k2 = ((unsigned long long)h2 << 32) | l2;
      // overall minimum: the outside-the-support one or the support one (disjoint rows)
      const bool sup_wins = ks < k1 || (ks == k1 && js < r1);
      const int j = sup_wins ? js : r1;
      const double mv = okey_inv(sup_wins ? ks : k1);
      const double cj = sup_wins ? csup : c1;
      const unsigned long long kout = sup_wins ? k1 : k2;   // min over rows outside T (old h = new h there)
      const double m_out = kout == ~0ULL ? dinf() : okey_inv(kout);
      // T = supp U {j} in merged-support lane layout, with C at each row (C_ji from the LMO),
      // for the gap refresh after the serial part (formed now: it needs no updated state)
      const bool j_in = __ballot_sync(FULL, lane < c0 && rw == j) != 0u;
      const int ins = __popc(__ballot_sync(FULL, lane < c0 && rw < j));
      int src = (j_in || lane < ins) ? lane : lane - 1;
      if (src < 0) src = 0;
      int mrow = __shfl_sync(FULL, rw, src);
      double mC = __shfl_sync(FULL, cw, src);
      if (!j_in && lane == ins) { mrow = j; mC = cj; }
      const int M = c0 + (j_in ? 0 : 1);
      if (A.spec && s + 1 < steps) {
        // T to the LMO warps: their pre-scan of the speculative next column skips these rows
        if (lane < M) {
          int ot;
          unsigned bit;
          pipe_owner<W, GA_LMO>(mrow, nvec, ot, bit);
          atomicOr(&mflagT[ot], bit);
        }
        __syncwarp();
        nbar_arrive(BAR_T, GA_SYNC);
      }
      // ---- the serial part
      PW_MARK(4);
      const StepOut o = serial_step<VAR, true>(A, kk, i, j, mv, bi, c0, rw, tv, gk, sh_r, sh_h, nullptr, sh_a, sh_cnt,
                                               slots, nullptr SP_NULL, dot);
      if (o.ev && o.erow < nvec * W) hpd[pipe_hidx<W>(o.erow, nvec)] = o.hnew;
      if (o.abort) {
        if (lane == 0) {
          misc[2] = 1;
          set_status(A.status, !(mv < 1.0e308 && mv > -1.0e308) ? 5 : 6);
        }
        __syncwarp();
        if (s + 1 < steps) nbar_arrive(BAR_COL, GA_SYNC);
        break;
      }
      if (A.trace && lane == 0) {
        double* tr = A.trace + 9 * (int64_t)s;
        tr[0] = (double)kk; tr[1] = i; tr[2] = j; tr[3] = (VAR == VAR_PLAIN) ? -1 : o.vrow;
        tr[4] = o.dir; tr[5] = o.gamma; tr[6] = o.num; tr[7] = o.den; tr[8] = mv;
      }
      // ---- GA: refresh the visited column's stored gap (Alg. A.4 line 6)
      PW_MARK(5);
      if (A.ga_inner) {
        double gnew = o.gfw;
        if (A.ga_post) {
          // post-update minimum: outside T unchanged (m_out), on T with the updated h
          const unsigned long long kt2 = okey(lane < M ? d_add(mC, sh_h[mrow]) : dinf());
          const unsigned hi = __reduce_min_sync(FULL, (unsigned)(kt2 >> 32));
          const unsigned lo = __reduce_min_sync(FULL, (unsigned)(kt2 >> 32) == hi ? (unsigned)kt2 : 0xffffffffu);
          const double mT = okey_inv(((unsigned long long)hi << 32) | lo);
          const double mnew = mT < m_out ? mT : m_out;
          // <t', c_i + h'> over the new support, rows ascending (entries in o's lane layout)
          const double ce = o.merged ? mC : cw;
          const double term = o.keep ? d_mul(o.tnew, d_add(ce, sh_h[o.erow])) : 0.0;
          // same adds in the same order; the first three terms' shuffles are issued
          // together (supports mostly hold at most three entries)
          const unsigned km0 = o.kmask, km1 = km0 & (km0 - 1u), km2 = km1 & (km1 - 1u);
          const double s0 = __shfl_sync(FULL, term, km0 ? __ffs(km0) - 1 : 0);
          const double s1 = __shfl_sync(FULL, term, km1 ? __ffs(km1) - 1 : 0);
          const double s2 = __shfl_sync(FULL, term, km2 ? __ffs(km2) - 1 : 0);
          double acc = 0.0;
          if (km0) acc = d_add(acc, s0);
          if (km1) acc = d_add(acc, s1);
          if (km2) acc = d_add(acc, s2);
          unsigned km = km2 & (km2 - 1u);
          while (km) {
            const int q = __ffs(km) - 1;
            km &= km - 1;
            acc = d_add(acc, __shfl_sync(FULL, term, q));
          }
          gnew = d_sub(acc, d_mul(bi, mnew));
        }
        const double delta = d_sub(wpos(gnew), wpos(gs_old));
        if (fen_node <= n) fens[fen_node] = d_add(fen_old, delta);   // ga_add_node with the value loaded early
        __syncwarp();
        PW_MARK(6);
        if (lane == 0) Gs[i] = gnew;
        __syncwarp();
      }
      done = s + 1;
      if (s + 1 < steps) {
        i = draw(u_next);
        PW_MARK(7);
        if (lane == 0) misc[0] = i;
        __syncwarp();
        nbar_arrive(BAR_COL, GA_SYNC);
      }
    }
    if (lane == 0) *A.steps_done = done;
#ifdef SRO_PHASE_TIMING
    if (lane == 0 && A.phase) for (int q = 0; q < 8; q++) A.phase[q] += pw_acc[q];
#endif
  }
  __syncthreads();
  for (int k = tid; k < m; k += PIPE_THREADS) { A.h[k] = sh_h[k]; A.r[k] = sh_r[k]; }
  if (GSM) for (int c = tid; c < n; c += PIPE_THREADS) A.G[c] = Gs[c];
  for (int c = tid; c <= n; c += PIPE_THREADS) A.fen[c] = fens[c];
  if (steps == 0 && tid == 0) *A.steps_done = 0;
}

}  // namespace sro
