// sro_api.cu — C-ABI (include/sro.h) and host runtime of the B200 hot path.
//
// The host side only validates arguments, owns device memory, generates the
// column-visit order from the counter-based SplitMix64 stream (R21-R22) and
// sequences kernels on the solver stream; every step of the method runs in
// the kernels of k_sweep.cuh, k_bcfw.cuh and k_block.cuh.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sro.h"
#include "k_bcfw.cuh"
#include "k_block.cuh"
#include "k_sweep.cuh"
#include "sro_device.cuh"

using namespace sro;

namespace {

struct Solver {
  int m = 0, n = 0, cap = 31, device = 0;
  double lambda = 1.0;
  int kind = 0, prec = 0, borrowed = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  // problem
  double *a = nullptr, *b = nullptr;
  void* C = nullptr;     // dense (fp32 or fp64), ld elements
  int64_t ld = 0;
  void* x = nullptr;     // colours
  void* y = nullptr;
  bool owns_cost = false;
  // state
  double *r = nullptr, *h = nullptr;
  int *cnt = nullptr, *srow = nullptr;
  double* sval = nullptr;
  long long k = 0;
  bool configured = false;
  int variant = -1;
  sro_options opt{};
  uint64_t seed = 0;
  // GA
  double *G = nullptr, *fen = nullptr;
  // scratch
  int* status = nullptr;      // device status word
  int* steps_done = nullptr;
  int* stop = nullptr;
  double* scal = nullptr;     // 8 device scalars
  double* epsd = nullptr;
  int* visit = nullptr;
  int64_t visit_cap = 0;
  double* trace = nullptr;
  int64_t trace_cap = 0;
  int* sw_j = nullptr;        // sweep outputs, length n
  double* sw_min = nullptr;
  double* sw_g = nullptr;
  int* part_j = nullptr;      // slab partials
  double* part_min = nullptr;
  int64_t part_cap = 0;
  // block-step workspace
  int64_t blk_L = 0, blk_P = 0;
  int *pcount = nullptr, *poff = nullptr, *ptotal = nullptr, *prow = nullptr, *ppos = nullptr;
  double *pd = nullptr, *pt = nullptr, *pdelta = nullptr;
  int *rowcnt = nullptr, *rowstart = nullptr, *cursor = nullptr, *tmp = nullptr, *sorted = nullptr;
  double* X = nullptr;
  int* trows = nullptr;
  int* ntouch = nullptr;
  unsigned long long* dsteps = nullptr;   // device count of completed block steps
  long long k_pending = 0;                // block steps enqueued since the last sync
  int num_sms = 148;
  // accounting
  long long* phase = nullptr;   // device [8] clock64 totals (SRO_PHASE_TIMING builds)
  double cmax = -1.0;           // max cost, computed once (ensure_cmax)
  bool no_rf = getenv("SRO_NO_RF") != nullptr;      // debug: force the shared-memory kernel
  bool no_tail = getenv("SRO_NO_TAIL") != nullptr;  // debug: force the multi-kernel block step
  sro_stats stats{};
  bool timing = false;
  struct Pending { cudaEvent_t a, b; int cat; int64_t units; };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<Pending> pending;
};

enum { CAT_BCFW = 0, CAT_SWEEP = 1, CAT_BLOCK = 2 };

cudaEvent_t take_event(Solver* s) {
  if (s->ev_pool.empty()) { cudaEvent_t e; cudaEventCreate(&e); return e; }
  cudaEvent_t e = s->ev_pool.back();
  s->ev_pool.pop_back();
  return e;
}
// open a timed region on the solver stream (no-op unless timing is on)
int timed_begin(Solver* s) {
  if (!s->timing) return -1;
  Solver::Pending p{take_event(s), take_event(s), 0, 0};
  cudaEventRecord(p.a, s->stream);
  s->pending.push_back(p);
  return (int)s->pending.size() - 1;
}
void timed_end(Solver* s, int idx, int cat, int64_t units) {
  if (idx < 0) return;
  Solver::Pending& p = s->pending[idx];
  p.cat = cat; p.units = units;
  cudaEventRecord(p.b, s->stream);
}
// after a stream sync: fold every completed region into the stats
void resolve_timing(Solver* s) {
  for (auto& p : s->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      if (p.cat == CAT_BCFW) s->stats.bcfw_ms += ms;
      else if (p.cat == CAT_SWEEP) s->stats.sweep_ms += ms;
      else s->stats.block_ms += ms;
    }
    s->ev_pool.push_back(p.a);
    s->ev_pool.push_back(p.b);
  }
  s->pending.clear();
}

#define CUDA_TRY(s, call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (s)->err = std::string(#call) + ": " + cudaGetErrorString(e_);                       \
      return e_ == cudaErrorMemoryAllocation ? SRO_ERR_OOM : SRO_ERR_CUDA;                 \
    }                                                                                      \
  } while (0)

thread_local std::string g_create_err;

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
}

// ---------------------------------------------------------------------------
// Small kernels: init, validation, hash generator, objective pieces, max cost
// ---------------------------------------------------------------------------
__global__ void k_init_plan(const double* __restrict__ b, const double* __restrict__ a, double* r, double* h,
                            int* cnt, int* srow, double* sval, int m, int n, int cap, double lambda) {
  // T^(0) = (b_1 e_1, ..., b_n e_1); r_0 = sum_i b_i left to right.
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int i = tid; i < n; i += stride) {
    cnt[i] = 1;
    srow[(int64_t)i * cap] = 0;
    sval[(int64_t)i * cap] = b[i];
  }
  for (int k = tid; k < m; k += stride) {
    if (k == 0) {
      double r0 = 0.0;
      for (int i = 0; i < n; i++) r0 = d_add(r0, b[i]);
      r[0] = r0;
      h[0] = d_div(d_sub(r0, a[0]), lambda);
    } else {
      r[k] = 0.0;
      h[k] = d_div(d_sub(0.0, a[k]), lambda);
    }
  }
}

template <typename T>
__global__ void k_check_dense(const T* __restrict__ C, int64_t ld, int m, int n, int* status) {
  const int64_t total = (int64_t)m * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / m, k = q % m;
    const double v = (double)C[i * ld + k];
    if (!(v >= 0.0) || !(v < 1.0e308)) set_status(status, 5);
  }
}

template <typename T>
__global__ void k_check_finite(const T* __restrict__ x, int64_t count, int* status) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[q];
    if (!(v > -1.0e308 && v < 1.0e308)) set_status(status, 5);
  }
}

// SRO_COST_HASH_UNIFORM: C_ki = (splitmix64(seed + (i m + k + 1) GOLDEN) >> 40) 2^-24, fp32 exact.
__global__ void k_gen_hash(float* C, int64_t ld, int m, int n, uint64_t seed) {
  const int64_t total = (int64_t)m * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / m, k = q % m;
    const uint64_t z = mix64(seed + ((uint64_t)q + 1) * GOLDEN);
    C[i * ld + k] = (float)(z >> 40) * 0x1p-24f;
  }
}

// lin_i = sum_{k in supp(t_i)} t_ki C_ki (rows ascending), one thread per column.
template <class Src>
__global__ void k_lin(Src src, const int* cnt, const int* srow, const double* sval, int cap, int n, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int e = 0; e < cnt[i]; e++) {
      const int k = srow[(int64_t)i * cap + e];
      acc = d_add(acc, d_mul(sval[(int64_t)i * cap + e], src.cost(k, i)));
    }
    out[i] = acc;
  }
}
__global__ void k_pen(const double* r, const double* a, int m, double* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const double d = d_sub(r[k], a[k]);
    out[k] = d_mul(d, d);
  }
}
__global__ void k_objective_final(const double* L, const double* pen, double lambda, double* f) {
  *f = d_add(*L, d_div(*pen, d_mul(2.0, lambda)));
}

// max_{k,i} C_ki (order-free max): GA stored-gap initial constant (R14).
template <class Src>
__global__ void k_max_cost(Src src, int m, int n, unsigned long long* out) {
  double mx = 0.0;
  const int64_t total = (int64_t)m * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const double c = src.cost((int)(q % m), (int)(q / m));
    if (c > mx) mx = c;
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));  // mx >= 0
}
__global__ void k_ga_init(double* G, double* fen, int n, const unsigned long long* cmax_bits, double lambda) {
  const double cinit = d_add(__longlong_as_double((long long)*cmax_bits), d_div(2.0, lambda));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) G[i] = cinit;
}


// ---------------------------------------------------------------------------
// Host helpers: visit order (R21-R22), identical definition to the paper reading
// ---------------------------------------------------------------------------
int uniform_index(uint64_t x, int N) {
  unsigned __int128 p = (unsigned __int128)(x >> 11) * (unsigned __int128)(uint32_t)N;
  return (int)(uint64_t)(p >> 53);
}
void make_visits(int sampling, uint64_t seed, long long k0, int64_t count, int N, const int32_t* explicit_visit,
                 int64_t done_offset, std::vector<int>& out) {
  out.resize(count);
  if (explicit_visit) {
    for (int64_t s = 0; s < count; s++) out[s] = explicit_visit[done_offset + s];
    return;
  }
  if (sampling == SRO_SAMPLE_U) {
    for (int64_t s = 0; s < count; s++) out[s] = uniform_index(rng_u64(seed, 0, (uint64_t)(k0 + s)), N);
    return;
  }
  // P: fresh Fisher-Yates permutation per epoch
  std::vector<int> perm(N);
  long long cur_epoch = -1;
  for (int64_t s = 0; s < count; s++) {
    const long long kk = k0 + s, e = kk / N;
    if (e != cur_epoch) {
      for (int q = 0; q < N; q++) perm[q] = q;
      for (int q = N - 1; q >= 1; q--) {
        const uint64_t x = rng_u64(seed, 2, (uint64_t)e * (uint64_t)N + (uint64_t)(N - 1 - q));
        const int rr = uniform_index(x, q + 1);
        std::swap(perm[q], perm[rr]);
      }
      cur_epoch = e;
    }
    out[s] = perm[kk % N];
  }
}

// ---------------------------------------------------------------------------
// Kernel dispatch over the cost source
// ---------------------------------------------------------------------------
template <class F>
sro_status with_sweep_src(Solver* s, F f) {
  if (s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM) {
    if (s->prec == SRO_FP32) return f(SrcDense<float>{(const float*)s->C, s->ld});
    return f(SrcDense<double>{(const double*)s->C, s->ld});
  }
  const bool eu = s->kind == SRO_COST_EUCLID;
  if (s->prec == SRO_FP32) {
    if (eu) return f(SrcColour<float, true>{(const float*)s->x, (const float*)s->y});
    return f(SrcColour<float, false>{(const float*)s->x, (const float*)s->y});
  }
  if (eu) return f(SrcColour<double, true>{(const double*)s->x, (const double*)s->y});
  return f(SrcColour<double, false>{(const double*)s->x, (const double*)s->y});
}

sro_status check_status(Solver* s) {
  int st = 0;
  CUDA_TRY(s, cudaMemcpyAsync(&st, s->status, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  if (st) {
    s->err = st == 5 ? "non-finite value met in the LMO" : st == 6 ? "column support exceeds slab_cap" : "device error";
    CUDA_TRY(s, cudaMemsetAsync(s->status, 0, sizeof(int), s->stream));
    return (sro_status)st;
  }
  return SRO_OK;
}

// LMO sweep over [col0, col0+L) -> out_j, out_min, out_g (device arrays of length >= L).
sro_status sweep(Solver* s, const int* col0_dev, int col0_mul, int col0_host, int L, int* out_j, double* out_min,
                 double* out_g, const int* stop) {
  const int nslabs = (s->m + SLAB - 1) / SLAB;
  if (nslabs > 1 && (int64_t)nslabs * L > s->part_cap) {
    cudaFree(s->part_j); cudaFree(s->part_min);
    s->part_cap = (int64_t)nslabs * L;
    CUDA_TRY(s, dalloc(&s->part_j, s->part_cap));
    CUDA_TRY(s, dalloc(&s->part_min, s->part_cap));
  }
  return with_sweep_src(s, [&](auto src) -> sro_status {
    using Src = decltype(src);
    const int rows = s->m < SLAB ? s->m : SLAB;
    const size_t smem = sizeof(double) * (size_t)((rows + 1) & ~1) + (size_t)Src::SMEM_PER_ROW * rows;
    auto kern = k_lmo_sweep<Src>;
    CUDA_TRY(s, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SWEEP_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    int gx = s->num_sms * per_sm;
    const int need = (L + SWEEP_WARPS - 1) / SWEEP_WARPS;
    if (nslabs > 1) gx = (gx + nslabs - 1) / nslabs;
    if (gx > need) gx = need;
    if (gx < 1) gx = 1;
    SweepOut o;
    if (nslabs == 1) { o.j = out_j; o.minval = out_min; o.g = out_g; }
    else { o.j = s->part_j; o.minval = s->part_min; o.g = nullptr; }
    const int tr = timed_begin(s);
    s->stats.kernel_launches += nslabs > 1 ? 2 : 1;
    s->stats.sweep_launches += 1;
    s->stats.sweep_columns += L;
    kern<<<dim3(gx, nslabs), SWEEP_THREADS, smem, s->stream>>>(src, s->m, s->h, col0_dev, col0_mul, col0_host, L,
                                                             s->cnt, s->srow, s->sval, s->cap, s->b, o, stop,
                                                             s->status);
    CUDA_TRY(s, cudaGetLastError());
    if (nslabs > 1) {
      int gm = (L + SWEEP_WARPS - 1) / SWEEP_WARPS;
      if (gm > s->num_sms * 8) gm = s->num_sms * 8;
      k_lmo_merge<Src><<<gm, SWEEP_THREADS, 0, s->stream>>>(src, nslabs, s->h, col0_dev, col0_mul, col0_host, L,
                                                            s->cnt, s->srow, s->sval, s->cap, s->b, s->part_j,
                                                            s->part_min, out_j, out_min, out_g, stop, s->status);
      CUDA_TRY(s, cudaGetLastError());
    }
    timed_end(s, tr, CAT_SWEEP, L);
    return SRO_OK;
  });
}

// Full gap sweep: g(T) = psum256_i g_i (Thm 2 / Eq. 11) -> host.
sro_status gap_sweep(Solver* s, double* total) {
  sro_status st = sweep(s, nullptr, 0, 0, s->n, s->sw_j, s->sw_min, s->sw_g, nullptr);
  if (st) return st;
  k_psum256<<<1, 256, 0, s->stream>>>(s->sw_g, s->n, s->scal + 4, nullptr, nullptr, nullptr);
  s->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  CUDA_TRY(s, cudaMemcpyAsync(total, s->scal + 4, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  st = check_status(s);  // synchronises
  resolve_timing(s);
  return st;
}

sro_status ensure_visit(Solver* s, int64_t count) {
  if (count > s->visit_cap) {
    cudaFree(s->visit);
    s->visit_cap = count < 4096 ? 4096 : count;
    CUDA_TRY(s, dalloc(&s->visit, s->visit_cap));
  }
  return SRO_OK;
}
sro_status ensure_trace(Solver* s, int64_t count) {
  if (count > s->trace_cap) {
    cudaFree(s->trace);
    s->trace_cap = count;
    CUDA_TRY(s, dalloc(&s->trace, 9 * s->trace_cap));
  }
  return SRO_OK;
}

void copy_trace_out(const std::vector<double>& tr, int64_t count, sro_trace_rec* out) {
  for (int64_t s = 0; s < count; s++) {
    const double* t = &tr[9 * s];
    out[s].k = (int64_t)t[0];
    out[s].i = (int32_t)t[1];
    out[s].j = (int32_t)t[2];
    out[s].v = (int32_t)t[3];
    out[s].dir = (int32_t)t[4];
    out[s].gamma = t[5];
    out[s].num = t[6];
    out[s].den = t[7];
    out[s].minval = t[8];
  }
}

// ---------------------------------------------------------------------------
// Sequential BCFW family: persistent kernel segments
// ---------------------------------------------------------------------------
template <class Col, int VAR, bool GA, bool SMEM>
sro_status launch_bcfw(Solver* s, BcfwArgs& A, Col col, size_t smem) {
  auto kern = k_bcfw<Col, VAR, GA, SMEM>;
  CUDA_TRY(s, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, BCFW_THREADS, smem, s->stream>>>(A, col);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->stats.kernel_launches += 1;
  s->stats.bcfw_launches += 1;
  s->stats.bcfw_steps += A.steps;
  return SRO_OK;
}

// Layout choice: the fast layout keeps h, r, counts (and the staged column or
// the source colours) in shared memory when they fit; GA arrays go to shared
// memory when they still fit, else stay in global memory.
sro_status ensure_cmax(Solver* s);

template <int VAR, bool GA>
sro_status bcfw_dispatch(Solver* s, BcfwArgs& A) {
  const int m = s->m, n = s->n;
  const bool dense = s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM;
  const size_t elem = s->prec == SRO_FP32 ? 4 : 8;
  const size_t col_fast = dense ? 2 * rup16((size_t)m * elem) : rup16((size_t)3 * m * elem);
  const size_t limit = 226 * 1024;
  size_t total = BcfwLayout::fixed_bytes();
  const bool smem = total + BcfwLayout::state_bytes(m, n) + col_fast <= limit;
  if (smem) total += BcfwLayout::state_bytes(m, n) + col_fast;
  A.ga_smem = 0; A.a_smem = 0; A.visit_smem = 0;
  if (GA && total + BcfwLayout::ga_bytes(n) <= limit) { A.ga_smem = 1; total += BcfwLayout::ga_bytes(n); }
  if (smem && total + BcfwLayout::a_bytes(m) <= limit) { A.a_smem = 1; total += BcfwLayout::a_bytes(m); }
  if (!GA && total + BcfwLayout::visit_bytes(A.steps) <= limit) { A.visit_smem = 1; total += BcfwLayout::visit_bytes(A.steps); }
  if (dense) {
    if (s->prec == SRO_FP32) {
      if (smem) {
        ColStaged<float> c{}; c.C = (const float*)s->C; c.ld = s->ld; c.m = m;
        return launch_bcfw<ColStaged<float>, VAR, GA, true>(s, A, c, total);
      }
      ColDirect<float> c{}; c.C = (const float*)s->C; c.ld = s->ld; c.m = m;
      return launch_bcfw<ColDirect<float>, VAR, GA, false>(s, A, c, total);
    }
    if (smem) { ColStaged<double> c{}; c.C = (const double*)s->C; c.ld = s->ld; c.m = m;
                return launch_bcfw<ColStaged<double>, VAR, GA, true>(s, A, c, total); }
    ColDirect<double> c{}; c.C = (const double*)s->C; c.ld = s->ld; c.m = m;
    return launch_bcfw<ColDirect<double>, VAR, GA, false>(s, A, c, total);
  }
  const int eu = s->kind == SRO_COST_EUCLID;
  if (s->prec == SRO_FP32) {
    if (smem) { ColColour<float, true> c{}; c.x = (const float*)s->x; c.y = (const float*)s->y; c.m = m; c.euclid = eu;
                return launch_bcfw<ColColour<float, true>, VAR, GA, true>(s, A, c, total); }
    ColColour<float, false> c{}; c.x = (const float*)s->x; c.y = (const float*)s->y; c.m = m; c.euclid = eu;
    return launch_bcfw<ColColour<float, false>, VAR, GA, false>(s, A, c, total);
  }
  if (smem) { ColColour<double, true> c{}; c.x = (const double*)s->x; c.y = (const double*)s->y; c.m = m; c.euclid = eu;
              return launch_bcfw<ColColour<double, true>, VAR, GA, true>(s, A, c, total); }
  ColColour<double, false> c{}; c.x = (const double*)s->x; c.y = (const double*)s->y; c.m = m; c.euclid = eu;
  return launch_bcfw<ColColour<double, false>, VAR, GA, false>(s, A, c, total);
}

template <typename T, int MAXV, int VAR, bool GA>
sro_status launch_rf(Solver* s, BcfwArgs& A, size_t smem) {
  auto kern = k_bcfw_rf<T, MAXV, VAR, GA>;
  CUDA_TRY(s, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, BCFW_THREADS, smem, s->stream>>>(A, (const T*)s->C, s->ld);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->stats.kernel_launches += 1;
  s->stats.bcfw_launches += 1;
  s->stats.bcfw_steps += A.steps;
  return SRO_OK;
}

// Register-file kernel for dense costs when the owned rows fit in registers
// (<= 4 vectors per thread) and h, r, a, counts fit in shared memory.
// Returns SRO_ERR_DIMENSION (not an error to the caller) when it does not apply.
template <int VAR, bool GA>
sro_status bcfw_try_rf(Solver* s, BcfwArgs& A) {
  const bool dense = s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM;
  if (!dense) return SRO_ERR_DIMENSION;
  const int W = s->prec == SRO_FP32 ? 4 : 2;
  const int nvec = s->m / W;
  const int need = (nvec + BCFW_THREADS - 1) / BCFW_THREADS;
  if (need > 4) return SRO_ERR_DIMENSION;
  const size_t limit = 226 * 1024;
  A.ga_smem = GA;   // the register-file kernel keeps GA arrays in shared memory (else generic kernel)
  A.visit_smem = !GA && RfLayout::bytes(s->m, s->n, A.steps, false, true) <= limit;
  A.a_smem = 1;
  const size_t bytes = RfLayout::bytes(s->m, s->n, A.steps, A.ga_smem, A.visit_smem);
  if (bytes > limit) return SRO_ERR_DIMENSION;
  if (s->prec == SRO_FP32) {
    if (need <= 2) return launch_rf<float, 2, VAR, GA>(s, A, bytes);
    return launch_rf<float, 4, VAR, GA>(s, A, bytes);
  }
  if (need <= 2) return launch_rf<double, 2, VAR, GA>(s, A, bytes);
  return launch_rf<double, 4, VAR, GA>(s, A, bytes);
}

template <int VAR, bool GA>
sro_status bcfw_run(Solver* s, BcfwArgs& A) {
  if (!s->no_rf) {
    sro_status st = bcfw_try_rf<VAR, GA>(s, A);
    if (st != SRO_ERR_DIMENSION) return st;
  }
  return bcfw_dispatch<VAR, GA>(s, A);
}

sro_status bcfw_segment(Solver* s, int variant, const sro_options* o, int steps, const int* dvisit,
                        double* dtrace) {
  BcfwArgs A{};
  A.m = s->m; A.n = s->n; A.cap = s->cap; A.lambda = s->lambda;
  A.a = s->a; A.b = s->b; A.r = s->r; A.h = s->h; A.cnt = s->cnt; A.srow = s->srow; A.sval = s->sval;
  A.visit = dvisit; A.steps = steps; A.k0 = s->k; A.step_rule = o->step;
  A.G = s->G; A.fen = s->fen; A.ga_inner = o->ga_inner; A.ga_post = o->ga_post_update; A.seed = s->seed;
  A.status = s->status; A.steps_done = s->steps_done; A.trace = dtrace;
  A.phase = s->phase;
  const bool ga = o->sampling == SRO_SAMPLE_GA;
  { sro_status st = ensure_cmax(s); if (st) return st; }
  A.cmax = s->cmax;
  if (variant == SRO_BCFW) return ga ? bcfw_run<VAR_PLAIN, true>(s, A) : bcfw_run<VAR_PLAIN, false>(s, A);
  if (variant == SRO_BCAFW) return ga ? bcfw_run<VAR_AWAY, true>(s, A) : bcfw_run<VAR_AWAY, false>(s, A);
  return ga ? bcfw_run<VAR_PAIR, true>(s, A) : bcfw_run<VAR_PAIR, false>(s, A);
}

// max_{k,i} C_ki, once per handle (order-free max; the fp32 LMO filter window
// and the GA stored-gap constant use it).
sro_status ensure_cmax(Solver* s) {
  if (s->cmax >= 0.0) return SRO_OK;
  unsigned long long* d_cmax = reinterpret_cast<unsigned long long*>(s->scal + 6);
  CUDA_TRY(s, cudaMemsetAsync(d_cmax, 0, sizeof(unsigned long long), s->stream));
  sro_status st = with_sweep_src(s, [&](auto src) -> sro_status {
    k_max_cost<<<s->num_sms * 4, 256, 0, s->stream>>>(src, s->m, s->n, d_cmax);
    s->stats.kernel_launches += 1;
    CUDA_TRY(s, cudaGetLastError());
    return SRO_OK;
  });
  if (st) return st;
  unsigned long long bits = 0;
  CUDA_TRY(s, cudaMemcpyAsync(&bits, d_cmax, sizeof(bits), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  double v;
  memcpy(&v, &bits, sizeof(v));
  s->cmax = v;
  return SRO_OK;
}

sro_status fen_build(Solver* s) {
  const size_t bytes = sizeof(double) * ((size_t)s->n + 1);
  const int use_smem = bytes <= 200 * 1024;
  if (use_smem) CUDA_TRY(s, cudaFuncSetAttribute(k_fen_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  k_fen_build<<<1, 256, use_smem ? bytes : 0, s->stream>>>(s->G, s->fen, s->n, use_smem);
  s->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  return SRO_OK;
}

sro_status ga_global_refresh(Solver* s) {
  sro_status st = sweep(s, nullptr, 0, 0, s->n, s->sw_j, s->sw_min, s->G, nullptr);
  if (st) return st;
  return fen_build(s);
}

sro_status ga_initialise(Solver* s) {
  unsigned long long* d_cmax = reinterpret_cast<unsigned long long*>(s->scal + 6);
  CUDA_TRY(s, cudaMemsetAsync(d_cmax, 0, sizeof(unsigned long long), s->stream));
  sro_status st = with_sweep_src(s, [&](auto src) -> sro_status {
    k_max_cost<<<s->num_sms * 4, 256, 0, s->stream>>>(src, s->m, s->n, d_cmax);
    CUDA_TRY(s, cudaGetLastError());
    return SRO_OK;
  });
  if (st) return st;
  k_ga_init<<<64, 256, 0, s->stream>>>(s->G, s->fen, s->n, d_cmax, s->lambda);
  s->stats.kernel_launches += 2;
  CUDA_TRY(s, cudaGetLastError());
  return fen_build(s);
}

// ---------------------------------------------------------------------------
// Plain step over a contiguous column set (FW / batched)
// ---------------------------------------------------------------------------
sro_status ensure_block_ws(Solver* s, int64_t L) {
  const int64_t P = L * (s->cap + 1);
  if (L <= s->blk_L && P <= s->blk_P) return SRO_OK;
  cudaFree(s->pcount); cudaFree(s->poff); cudaFree(s->ptotal); cudaFree(s->prow); cudaFree(s->ppos);
  cudaFree(s->pd); cudaFree(s->pt); cudaFree(s->pdelta); cudaFree(s->tmp); cudaFree(s->sorted);
  if (!s->rowcnt) {
    CUDA_TRY(s, dalloc(&s->rowcnt, s->m)); CUDA_TRY(s, dalloc(&s->rowstart, s->m + 1));
    CUDA_TRY(s, dalloc(&s->cursor, s->m + 1)); CUDA_TRY(s, dalloc(&s->X, s->m));
    CUDA_TRY(s, dalloc(&s->trows, s->m)); CUDA_TRY(s, dalloc(&s->ntouch, 1));
  }
  s->blk_L = L; s->blk_P = P;
  CUDA_TRY(s, dalloc(&s->pcount, L)); CUDA_TRY(s, dalloc(&s->poff, L + 1)); CUDA_TRY(s, dalloc(&s->ptotal, 1));
  CUDA_TRY(s, dalloc(&s->prow, P)); CUDA_TRY(s, dalloc(&s->ppos, P)); CUDA_TRY(s, dalloc(&s->pd, P));
  CUDA_TRY(s, dalloc(&s->pt, P)); CUDA_TRY(s, dalloc(&s->pdelta, P)); CUDA_TRY(s, dalloc(&s->tmp, P));
  CUDA_TRY(s, dalloc(&s->sorted, P));
  return SRO_OK;
}

// One plain step over [col0, col0+L). For FW (stop_check) the gap G_[n] is
// checked against epsilon before the update (Alg. A.1 line 4). Small U: the
// LMO sweep plus one single-CTA launch for the rest of the step; large U: one
// kernel per phase.
sro_status plain_block_step(Solver* s, const int* col0_dev, int col0_mul, int L, int step_rule, long long nprime,
                            bool stop_check, double* trace_dev) {
  sro_status st = ensure_block_ws(s, L);
  if (st) return st;
  const int trb = timed_begin(s);
  int* stop = stop_check ? s->stop : nullptr;
  st = sweep(s, col0_dev, col0_mul, 0, L, s->sw_j, s->sw_min, s->sw_g, stop);
  if (st) return st;
  BlockArgs A{};
  A.m = s->m; A.n = s->n; A.cap = s->cap; A.lambda = s->lambda; A.a = s->a; A.b = s->b; A.r = s->r; A.h = s->h;
  A.cnt = s->cnt; A.srow = s->srow; A.sval = s->sval; A.col0_dev = col0_dev; A.col0_mul = col0_mul; A.L = L;
  A.j = s->sw_j; A.minval = s->sw_min; A.g = s->sw_g; A.pcount = s->pcount; A.poff = s->poff; A.ptotal = s->ptotal;
  A.prow = s->prow; A.ppos = s->ppos; A.pd = s->pd; A.gsum = s->pt; A.pdelta = s->pdelta; A.rowcnt = s->rowcnt;
  A.rowstart = s->rowstart; A.cursor = s->cursor; A.tmp = s->tmp; A.sorted = s->sorted; A.X = s->X;
  A.scal = s->scal; A.eps = stop_check ? s->epsd : nullptr; A.stop = stop; A.status = s->status;
  A.trows = s->trows; A.ntouch = s->ntouch;
  A.step_rule = step_rule; A.kk = s->k + s->k_pending; A.nprime = nprime; A.trace = trace_dev;
  A.dsteps = s->dsteps;
  if (L <= 1024 && !s->no_tail) {
    const size_t smem = sizeof(double) * 32 * 256;
    CUDA_TRY(s, cudaFuncSetAttribute(k_block_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_block_tail<<<1, 1024, smem, s->stream>>>(A);
    CUDA_TRY(s, cudaGetLastError());
    s->stats.kernel_launches += 1;
  } else {
    const int tpb = 256;
    int gL = (L + tpb - 1) / tpb; if (gL > s->num_sms * 8) gL = s->num_sms * 8;
    const int gP = s->num_sms * 8;
    const int gG = (s->m + 7) / 8 < s->num_sms * 8 ? (s->m + 7) / 8 : s->num_sms * 8;
    k_psum256<<<1, 256, 0, s->stream>>>(s->sw_g, L, s->scal + 0, A.eps, stop, nullptr);
    k_pairs_count<<<gL, tpb, 0, s->stream>>>(A);
    k_scan_excl<<<1, 1024, 0, s->stream>>>(s->pcount, L, s->poff, nullptr, s->ptotal, stop, s->status);
    CUDA_TRY(s, cudaMemsetAsync(s->rowcnt, 0, sizeof(int) * s->m, s->stream));
    CUDA_TRY(s, cudaMemsetAsync(s->ntouch, 0, sizeof(int), s->stream));
    k_pairs_gen<<<gL, tpb, 0, s->stream>>>(A);
    k_scan_excl<<<1, 1024, 0, s->stream>>>(s->rowcnt, s->m, s->rowstart, s->cursor, nullptr, stop, s->status);
    k_place<<<gP, tpb, 0, s->stream>>>(A);
    k_rank<<<gP, tpb, 0, s->stream>>>(A);
    CUDA_TRY(s, cudaMemsetAsync(s->X, 0, sizeof(double) * s->m, s->stream));
    k_row_groups<<<gP, tpb, 0, s->stream>>>(A, s->pd);
    k_row_tree<0><<<gG, 256, 0, s->stream>>>(A);
    k_psum256<<<1, 256, 0, s->stream>>>(s->X, s->m, s->scal + 1, nullptr, nullptr, stop);
    k_gamma<<<1, 32, 0, s->stream>>>(A);
    k_cap_check<<<gL, tpb, 0, s->stream>>>(A);
    k_update_cols<<<gL, tpb, 0, s->stream>>>(A);
    k_row_groups<<<gP, tpb, 0, s->stream>>>(A, s->pdelta);
    k_row_tree<1><<<gG, 256, 0, s->stream>>>(A);
    k_step_done<<<1, 32, 0, s->stream>>>(A);
    CUDA_TRY(s, cudaGetLastError());
    s->stats.kernel_launches += 16;
  }
  s->stats.block_steps += 1;
  s->k_pending += 1;
  timed_end(s, trb, CAT_BLOCK, L);
  return SRO_OK;
}

// Sync point for asynchronously enqueued block steps: read how many completed
// (a skipped step — FW stop or an error — does not count), advance k, and
// report a device error.
sro_status drain_block_steps(Solver* s, int64_t* done) {
  unsigned long long ds = 0;
  CUDA_TRY(s, cudaMemcpyAsync(&ds, s->dsteps, sizeof(ds), cudaMemcpyDeviceToHost, s->stream));
  sro_status st = check_status(s);   // synchronises
  resolve_timing(s);
  CUDA_TRY(s, cudaMemsetAsync(s->dsteps, 0, sizeof(unsigned long long), s->stream));
  s->k += (long long)ds;
  *done += (int64_t)ds;
  s->k_pending = 0;
  return st;
}

bool options_equal(const sro_options& x, const sro_options& y) {
  return x.step == y.step && x.sampling == y.sampling && x.epsilon == y.epsilon && x.gap_period == y.gap_period &&
         x.ga_M == y.ga_M && x.ga_inner == y.ga_inner && x.ga_post_update == y.ga_post_update &&
         x.block_size == y.block_size;
}

sro_status objective_dev(Solver* s, double* f_host) {
  sro_status st = with_sweep_src(s, [&](auto src) -> sro_status {
    k_lin<<<(s->n + 255) / 256, 256, 0, s->stream>>>(src, s->cnt, s->srow, s->sval, s->cap, s->n, s->sw_g);
    CUDA_TRY(s, cudaGetLastError());
    return SRO_OK;
  });
  if (st) return st;
  k_psum256<<<1, 256, 0, s->stream>>>(s->sw_g, s->n, s->scal + 4, nullptr, nullptr, nullptr);
  k_pen<<<(s->m + 255) / 256, 256, 0, s->stream>>>(s->r, s->a, s->m, s->sw_min);
  k_psum256<<<1, 256, 0, s->stream>>>(s->sw_min, s->m, s->scal + 5, nullptr, nullptr, nullptr);
  k_objective_final<<<1, 1, 0, s->stream>>>(s->scal + 4, s->scal + 5, s->lambda, s->scal + 7);
  s->stats.kernel_launches += 5;
  CUDA_TRY(s, cudaGetLastError());
  CUDA_TRY(s, cudaMemcpyAsync(f_host, s->scal + 7, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  return SRO_OK;
}

sro_status do_reset(Solver* s) {
  k_init_plan<<<s->num_sms, 256, 0, s->stream>>>(s->b, s->a, s->r, s->h, s->cnt, s->srow, s->sval, s->m, s->n, s->cap,
                                                s->lambda);
  s->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  CUDA_TRY(s, cudaMemsetAsync(s->stop, 0, sizeof(int), s->stream));
  s->k = 0;
  s->configured = false;
  return SRO_OK;
}

void free_solver(Solver* s) {
  if (!s) return;
  void* ptrs[] = {s->dsteps, s->phase, s->a, s->b, s->r, s->h, s->cnt, s->srow, s->sval, s->G, s->fen, s->status, s->steps_done,
                  s->stop, s->scal, s->epsd, s->visit, s->trace, s->sw_j, s->sw_min, s->sw_g, s->part_j,
                  s->part_min, s->pcount, s->poff, s->ptotal, s->prow, s->ppos, s->pd, s->pt, s->pdelta,
                  s->rowcnt, s->rowstart, s->cursor, s->tmp, s->sorted, s->X, s->trows, s->ntouch};
  for (void* p : ptrs) if (p) cudaFree(p);
  if (s->owns_cost) { if (s->C) cudaFree(s->C); if (s->x) cudaFree(s->x); if (s->y) cudaFree(s->y); }
  for (auto& p : s->pending) { s->ev_pool.push_back(p.a); s->ev_pool.push_back(p.b); }
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

}  // namespace

struct sro_solver : Solver {};

extern "C" {

const char* sro_version(void) { return "sro-b200 0.1 (sm_100a)"; }

const char* sro_last_error(sro_handle h) {
  if (!h) return g_create_err.c_str();
  return static_cast<Solver*>(h)->err.c_str();
}

sro_status sro_create(const double* a, const double* b, const sro_cost* cost, const sro_params* p, sro_handle* out) {
  g_create_err.clear();
  if (!out || !a || !b || !cost || !p) { g_create_err = "null argument"; return SRO_ERR_INVALID_ARG; }
  *out = nullptr;
  if (p->m < 1 || p->n < 1) { g_create_err = "m, n must be >= 1"; return SRO_ERR_DIMENSION; }
  if (!(p->lambda > 0.0) || !std::isfinite(p->lambda)) { g_create_err = "lambda must be finite and > 0"; return SRO_ERR_INVALID_ARG; }
  const int cap = p->slab_cap == 0 ? 31 : p->slab_cap;
  if (cap < 1 || cap > 31) { g_create_err = "slab_cap must be in [1, 31]"; return SRO_ERR_INVALID_ARG; }
  if (cost->kind < 0 || cost->kind > 3 || cost->prec < 0 || cost->prec > 1) { g_create_err = "bad cost kind/precision"; return SRO_ERR_INVALID_ARG; }
  // marginals: finite, a >= 0, b > 0, each summing to 1 within 1e-12
  double sa = 0.0, sb = 0.0;
  for (int k = 0; k < p->m; k++) { if (!(a[k] >= 0.0) || !std::isfinite(a[k])) { g_create_err = "a must be finite and >= 0"; return SRO_ERR_MARGINALS; } sa += a[k]; }
  for (int i = 0; i < p->n; i++) { if (!(b[i] > 0.0) || !std::isfinite(b[i])) { g_create_err = "b must be finite and > 0"; return SRO_ERR_MARGINALS; } sb += b[i]; }
  if (std::fabs(sa - 1.0) > 1e-12 || std::fabs(sb - 1.0) > 1e-12) { g_create_err = "marginals must sum to 1 within 1e-12"; return SRO_ERR_MARGINALS; }

  Solver* s = new Solver();
  s->m = p->m; s->n = p->n; s->cap = cap; s->lambda = p->lambda; s->device = p->device;
  s->kind = cost->kind; s->prec = cost->prec; s->borrowed = cost->data_on_device;
  if (s->kind == SRO_COST_HASH_UNIFORM) s->prec = SRO_FP32;
  auto fail = [&](sro_status st, const std::string& msg) { g_create_err = msg.empty() ? s->err : msg; free_solver(s); return st; };
  if (cudaSetDevice(p->device) != cudaSuccess) return fail(SRO_ERR_CUDA, "cudaSetDevice failed (no CUDA device?)");
  cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, p->device);
  if (p->cuda_stream) s->stream = (cudaStream_t)p->cuda_stream;
  else { if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(SRO_ERR_CUDA, "stream"); s->own_stream = true; }
  cudaEventCreate(&s->ev0); cudaEventCreate(&s->ev1);
  const int m = s->m, n = s->n;
#define ALLOC(ptr, cnt_)                                                              \
  if (dalloc(&(ptr), (cnt_)) != cudaSuccess) return fail(SRO_ERR_OOM, "device allocation failed");
  ALLOC(s->a, m); ALLOC(s->b, n); ALLOC(s->r, m); ALLOC(s->h, m);
  ALLOC(s->cnt, n); ALLOC(s->srow, (size_t)n * cap); ALLOC(s->sval, (size_t)n * cap);
  ALLOC(s->G, n); ALLOC(s->fen, (size_t)n + 1);
  ALLOC(s->phase, 16);
  ALLOC(s->dsteps, 1);
  cudaMemsetAsync(s->dsteps, 0, sizeof(unsigned long long), s->stream);
  cudaMemsetAsync(s->phase, 0, 16 * sizeof(long long), s->stream);
  ALLOC(s->status, 1); ALLOC(s->steps_done, 1); ALLOC(s->stop, 1); ALLOC(s->scal, 8); ALLOC(s->epsd, 1);
  ALLOC(s->sw_j, n); ALLOC(s->sw_min, (size_t)(m > n ? m : n)); ALLOC(s->sw_g, (size_t)(m > n ? m : n));
  cudaMemsetAsync(s->status, 0, sizeof(int), s->stream);
  cudaMemcpyAsync(s->a, a, sizeof(double) * m, cudaMemcpyHostToDevice, s->stream);
  cudaMemcpyAsync(s->b, b, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream);
  const size_t esz = s->prec == SRO_FP32 ? 4 : 8;
  const int vec = 16 / (int)esz;
  if (s->kind == SRO_COST_DENSE) {
    if (!cost->data || cost->ld < m) return fail(SRO_ERR_INVALID_ARG, "dense cost needs data and ld >= m");
    if (cost->data_on_device) {
      if (((uintptr_t)cost->data % 16) != 0 || (cost->ld * (int64_t)esz) % 16 != 0)
        return fail(SRO_ERR_INVALID_ARG, "borrowed dense cost must be 16-byte aligned with ld*elem % 16 == 0");
      s->C = const_cast<void*>(cost->data); s->ld = cost->ld;
    } else {
      s->ld = ((int64_t)m + vec - 1) / vec * vec;
      if (cudaMalloc(&s->C, esz * (size_t)s->ld * n) != cudaSuccess) return fail(SRO_ERR_OOM, "cost allocation failed");
      s->owns_cost = true;
      if (cudaMemcpy2DAsync(s->C, esz * s->ld, cost->data, esz * cost->ld, esz * m, n, cudaMemcpyHostToDevice, s->stream) != cudaSuccess)
        return fail(SRO_ERR_CUDA, "cost upload failed");
    }
    if (s->prec == SRO_FP32) k_check_dense<float><<<s->num_sms * 4, 256, 0, s->stream>>>((const float*)s->C, s->ld, m, n, s->status);
    else k_check_dense<double><<<s->num_sms * 4, 256, 0, s->stream>>>((const double*)s->C, s->ld, m, n, s->status);
  } else if (s->kind == SRO_COST_HASH_UNIFORM) {
    s->ld = ((int64_t)m + 3) / 4 * 4;
    if (cudaMalloc(&s->C, 4 * (size_t)s->ld * n) != cudaSuccess) return fail(SRO_ERR_OOM, "cost allocation failed");
    s->owns_cost = true;
    k_gen_hash<<<s->num_sms * 8, 256, 0, s->stream>>>((float*)s->C, s->ld, m, n, cost->hash_seed);
  } else {
    if (!cost->x || !cost->y) return fail(SRO_ERR_INVALID_ARG, "colour cost needs x and y");
    if (cost->data_on_device) { s->x = const_cast<void*>(cost->x); s->y = const_cast<void*>(cost->y); }
    else {
      if (cudaMalloc(&s->x, esz * 3 * (size_t)m) != cudaSuccess || cudaMalloc(&s->y, esz * 3 * (size_t)n) != cudaSuccess)
        return fail(SRO_ERR_OOM, "colour allocation failed");
      s->owns_cost = true;
      cudaMemcpyAsync(s->x, cost->x, esz * 3 * (size_t)m, cudaMemcpyHostToDevice, s->stream);
      cudaMemcpyAsync(s->y, cost->y, esz * 3 * (size_t)n, cudaMemcpyHostToDevice, s->stream);
    }
    if (s->prec == SRO_FP32) {
      k_check_finite<float><<<64, 256, 0, s->stream>>>((const float*)s->x, 3LL * m, s->status);
      k_check_finite<float><<<64, 256, 0, s->stream>>>((const float*)s->y, 3LL * n, s->status);
    } else {
      k_check_finite<double><<<64, 256, 0, s->stream>>>((const double*)s->x, 3LL * m, s->status);
      k_check_finite<double><<<64, 256, 0, s->stream>>>((const double*)s->y, 3LL * n, s->status);
    }
  }
  if (cudaGetLastError() != cudaSuccess) return fail(SRO_ERR_CUDA, "kernel launch failed at create");
  int st = 0;
  cudaMemcpyAsync(&st, s->status, sizeof(int), cudaMemcpyDeviceToHost, s->stream);
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) return fail(SRO_ERR_CUDA, "create failed");
  if (st) return fail(SRO_ERR_NONFINITE, "cost must be finite and >= 0");
  if (do_reset(s) != SRO_OK) return fail(SRO_ERR_CUDA, "");
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) return fail(SRO_ERR_CUDA, "init failed");
  *out = static_cast<sro_handle>(static_cast<sro_solver*>(s));
  return SRO_OK;
}

void sro_destroy(sro_handle h) {
  if (!h) return;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  free_solver(s);
}

sro_status sro_reset(sro_handle h) {
  if (!h) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  sro_status st = do_reset(s);
  if (st) return st;
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  return SRO_OK;
}

sro_status sro_solve(sro_handle h, int32_t variant, const sro_options* o, int64_t iters, uint64_t seed, sro_result* out) {
  if (!h || !o || !out || iters < 0) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  memset(out, 0, sizeof(*out));
  out->gap = NAN;
  out->objective = NAN;
  if (variant < SRO_FW || variant > SRO_BATCHED) { s->err = "bad variant"; return SRO_ERR_INVALID_ARG; }
  if (o->gap_period < 1) { s->err = "gap_period must be >= 1"; return SRO_ERR_INVALID_ARG; }
  if ((variant == SRO_BCAFW || variant == SRO_BCPFW) && o->step != SRO_STEP_ELS) { s->err = "away/pairwise need the line search (Alg. A.2/A.3)"; return SRO_ERR_INVALID_ARG; }
  if (o->sampling == SRO_SAMPLE_GA && !(variant == SRO_BCFW || variant == SRO_BCAFW || variant == SRO_BCPFW)) { s->err = "GA sampling needs a BCFW-family variant"; return SRO_ERR_INVALID_ARG; }
  if (o->sampling == SRO_SAMPLE_GA && o->ga_M < 1) { s->err = "ga_M must be >= 1"; return SRO_ERR_INVALID_ARG; }
  if (o->sampling < 0 || o->sampling > 2 || o->step < 0 || o->step > 1) { s->err = "bad sampling/step"; return SRO_ERR_INVALID_ARG; }
  long long nprime;
  if (variant == SRO_FW) nprime = 1;
  else if (variant == SRO_BATCHED) {
    if (o->block_size < 1 || s->n % o->block_size != 0) { s->err = "block_size must divide n"; return SRO_ERR_INVALID_ARG; }
    nprime = s->n / o->block_size;
  } else nprime = s->n;
  if (s->configured) {
    if (s->variant != variant || s->seed != seed || !options_equal(s->opt, *o)) { s->err = "solver configured differently; call sro_reset"; return SRO_ERR_STATE; }
  }
  const bool ga = o->sampling == SRO_SAMPLE_GA && variant != SRO_FW;
  sro_status st = SRO_OK;
  CUDA_TRY(s, cudaEventRecord(s->ev0, s->stream));
  if (!s->configured) {
    s->configured = true; s->variant = variant; s->opt = *o; s->seed = seed;
    s->opt.visit = nullptr; s->opt.trace = nullptr;
    if (ga) { st = ga_initialise(s); if (st) return st; }
  }
  CUDA_TRY(s, cudaMemcpyAsync(s->epsd, &o->epsilon, sizeof(double), cudaMemcpyHostToDevice, s->stream));
  const int m = s->m, n = s->n;
  int64_t done = 0;
  const long long period = (long long)o->gap_period * nprime;
  std::vector<int> hv;
  std::vector<double> htr;
  if (o->trace) { st = ensure_trace(s, iters > 0 ? iters : 1); if (st) return st; }

  if (variant == SRO_FW) {
    CUDA_TRY(s, cudaMemsetAsync(s->stop, 0, sizeof(int), s->stream));
    while (done < iters) {
      const int64_t chunk = (iters - done) < 8 ? (iters - done) : 8;
      for (int64_t q = 0; q < chunk; q++) {
        st = plain_block_step(s, nullptr, 0, n, o->step, 1, true, o->trace ? s->trace + 9 * (done + q) : nullptr);
        if (st) return st;
      }
      const int64_t before = done;
      double G = 0.0;
      int stopped = 0;
      CUDA_TRY(s, cudaMemcpyAsync(&G, s->scal + 0, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      CUDA_TRY(s, cudaMemcpyAsync(&stopped, s->stop, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
      st = drain_block_steps(s, &done);
      if (st) return st;
      out->gap = G;
      out->gap_checks += (int)(done - before) + (stopped ? 1 : 0);
      out->entries_scanned += (int64_t)m * n * ((done - before) + (stopped ? 1 : 0));
      if (stopped) { out->converged = 1; break; }
    }
    CUDA_TRY(s, cudaMemsetAsync(s->stop, 0, sizeof(int), s->stream));
  } else {
    // visit order for the whole call (U / P / explicit); GA draws on the device
    if (!ga) {
      make_visits(o->sampling, seed, s->k, iters, (int)nprime, o->visit, 0, hv);
      st = ensure_visit(s, iters > 0 ? iters : 1);
      if (st) return st;
      if (iters > 0) CUDA_TRY(s, cudaMemcpyAsync(s->visit, hv.data(), sizeof(int) * iters, cudaMemcpyHostToDevice, s->stream));
    }
    const long long gaMn = ga ? (long long)o->ga_M * n : 0;
    for (;;) {
      if (s->k % period == 0) {
        double g = 0.0;
        st = gap_sweep(s, &g);
        if (st) return st;
        out->gap = g; out->gap_checks++;
        out->entries_scanned += (int64_t)m * n;
        if (g <= o->epsilon) { out->converged = 1; break; }
      }
      if (done >= iters) break;
      if (variant == SRO_BATCHED) {
        // enqueue every block step up to the next gap check, then one sync
        long long seg = iters - done;
        const long long to_check = period - s->k % period;
        if (seg > to_check) seg = to_check;
        const int64_t before = done;
        for (long long q = 0; q < seg; q++) {
          st = plain_block_step(s, s->visit + done + q, o->block_size, o->block_size, o->step, nprime, false,
                                o->trace ? s->trace + 9 * (done + q) : nullptr);
          if (st) return st;
        }
        st = drain_block_steps(s, &done);
        out->entries_scanned += (int64_t)m * o->block_size * (done - before);
        if (st) break;
        continue;
      }
      long long seg = iters - done;
      const long long to_check = period - s->k % period;
      if (seg > to_check) seg = to_check;
      if (ga) { const long long to_ref = gaMn - s->k % gaMn; if (seg > to_ref) seg = to_ref; }
      st = bcfw_segment(s, variant, o, (int)seg, ga ? nullptr : s->visit + done, o->trace ? s->trace + 9 * done : nullptr);
      if (st) return st;
      int sd = 0;
      CUDA_TRY(s, cudaMemcpyAsync(&sd, s->steps_done, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
      st = check_status(s);
      resolve_timing(s);
      s->k += sd; done += sd;
      out->entries_scanned += (int64_t)m * sd * ((ga && o->ga_inner && o->ga_post_update) ? 2 : 1);
      if (st) break;
      if (ga && s->k % gaMn == 0) {
        st = ga_global_refresh(s);
        if (st) return st;
        out->entries_scanned += (int64_t)m * n;
      }
    }
  }
  out->iters_done = done;
  out->k = s->k;
  CUDA_TRY(s, cudaEventRecord(s->ev1, s->stream));
  if (o->trace && done > 0) {
    htr.resize(9 * (size_t)done);
    CUDA_TRY(s, cudaMemcpyAsync(htr.data(), s->trace, sizeof(double) * 9 * done, cudaMemcpyDeviceToHost, s->stream));
  }
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s->ev0, s->ev1);
  out->device_ms = ms;
  if (o->trace && done > 0) copy_trace_out(htr, done, o->trace);
  if (st) return st;
  double f = NAN;
  sro_status st2 = objective_dev(s, &f);
  if (st2) return st2;
  out->objective = f;
  return out->converged ? SRO_OK : SRO_NOT_CONVERGED;
}

sro_status sro_gap(sro_handle h, double* total, double* per_column, int32_t* argmin_rows) {
  if (!h || !total) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  sro_status st = gap_sweep(s, total);
  if (st) return st;
  if (per_column) CUDA_TRY(s, cudaMemcpyAsync(per_column, s->sw_g, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
  if (argmin_rows) CUDA_TRY(s, cudaMemcpyAsync(argmin_rows, s->sw_j, sizeof(int) * s->n, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  return SRO_OK;
}

sro_status sro_objective(sro_handle h, double* f) {
  if (!h || !f) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  return objective_dev(s, f);
}

sro_status sro_get_rowsums(sro_handle h, double* r) {
  if (!h || !r) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  CUDA_TRY(s, cudaMemcpyAsync(r, s->r, sizeof(double) * s->m, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  return SRO_OK;
}

sro_status sro_get_plan(sro_handle h, double* dense, int32_t* rows, int32_t* cols, double* vals, int64_t cap,
                        int64_t* nnz) {
  if (!h) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  std::vector<int> hc(s->n), hr((size_t)s->n * s->cap);
  std::vector<double> hv((size_t)s->n * s->cap);
  CUDA_TRY(s, cudaMemcpyAsync(hc.data(), s->cnt, sizeof(int) * s->n, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaMemcpyAsync(hr.data(), s->srow, sizeof(int) * hr.size(), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaMemcpyAsync(hv.data(), s->sval, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  if (dense) memset(dense, 0, sizeof(double) * (size_t)s->m * s->n);
  int64_t q = 0;
  for (int i = 0; i < s->n; i++)
    for (int e = 0; e < hc[i]; e++) {
      const int k = hr[(size_t)i * s->cap + e];
      const double v = hv[(size_t)i * s->cap + e];
      if (dense) dense[(size_t)i * s->m + k] = v;
      if (rows && cols && vals && q < cap) { rows[q] = k; cols[q] = i; vals[q] = v; }
      q++;
    }
  if (nnz) *nnz = q;
  if (rows && cols && vals && q > cap) { s->err = "COO capacity too small"; return SRO_ERR_CAPACITY; }
  return SRO_OK;
}

sro_status sro_get_stats(sro_handle h, sro_stats* out, int32_t reset) {
  if (!h || !out) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  resolve_timing(s);
  *out = s->stats;
  if (reset) s->stats = sro_stats{};
  return SRO_OK;
}

// Debug: copy the 8 accumulated clock64 phase totals of the persistent kernel
// (non-zero only in builds compiled with -DSRO_PHASE_TIMING). Not in sro.h.
sro_status sro_debug_phase(sro_handle h, long long* out8) {
  if (!h || !out8) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  CUDA_TRY(s, cudaMemcpyAsync(out8, s->phase, 16 * sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, cudaStreamSynchronize(s->stream));
  return SRO_OK;
}

sro_status sro_set_timing(sro_handle h, int32_t on) {
  if (!h) return SRO_ERR_INVALID_ARG;
  static_cast<Solver*>(h)->timing = on != 0;
  return SRO_OK;
}

}  // extern "C"
