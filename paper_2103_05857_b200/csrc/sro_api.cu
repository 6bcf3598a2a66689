// sro_api.cu — C-ABI (include/sro.h) and host runtime of the B200 hot path.
//
// The host side only validates arguments, owns device memory, generates the
// column-visit order from the counter-based SplitMix64 stream (R21-R22) and
// sequences kernels on the solver stream; every step of the method runs in
// the kernels of k_sweep.cuh, k_bcfw.cuh and k_block.cuh.
//
// Column sharding: a handle holds one or more shards (struct
// Solver each: its columns' cost, slabs and workspaces, plus replicas of r
// and h). The lead shard is the handle; with nranks == 1 it also owns the
// other G-1 shards ("peers") and runs every phase for each of them in turn on
// one stream, each shard writing its partials straight into its slot of the
// shared exchange buffers; with nranks == G each process holds one shard and
// the slots are filled by in-place NCCL all-gathers on the solver stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <thread>
#include <vector>

#include "../../include/sro.h"
#include "k_bcfw.cuh"
#include "k_bcfw_pipe.cuh"
#include "k_block.cuh"
#include "k_block_tail.cuh"
#include "k_plan.cuh"
#include "k_kmeans.cuh"
#include "k_ga_block.cuh"
#include "k_sweep.cuh"
#include "sro_device.cuh"

using namespace sro;

namespace {

// NCCL, loaded at run time (only sharded handles with nranks > 1 need it).
struct NcclApi {
  bool tried = false, ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  // the NCCL the process already uses (torch's), else SRO_NCCL_LIB (the Python binding points it at
  // the wheel torch ships), else the loader's default: loading an older system libnccl.so.2 first
  // would break a later `import torch` (its libtorch_cuda needs the newer NCCL's symbols)
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!lib && getenv("SRO_NCCL_LIB")) lib = dlopen(getenv("SRO_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) { api.err = std::string("cannot load libnccl.so.2: ") + dlerror(); return api; }
  api.get_id = (decltype(api.get_id))dlsym(lib, "ncclGetUniqueId");
  api.init = (decltype(api.init))dlsym(lib, "ncclCommInitRank");
  api.destroy = (decltype(api.destroy))dlsym(lib, "ncclCommDestroy");
  api.allgather = (decltype(api.allgather))dlsym(lib, "ncclAllGather");
  api.errstr = (decltype(api.errstr))dlsym(lib, "ncclGetErrorString");
  api.ok = api.get_id && api.init && api.destroy && api.allgather && api.errstr;
  if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  return api;
}

struct Solver {
  int m = 0, n = 0, cap = 31, device = 0;   // n: columns held by this shard
  double lambda = 1.0;
  int kind = 0, prec = 0, borrowed = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_sync = nullptr;   // marks the stream position a host wait (wait_event) polls for
  // Pinned mailbox for the solve loop's small device->host readbacks (rb()): a copy into
  // pageable memory would hold the calling thread inside cudaMemcpyAsync until the stream
  // reached it, busy on the CPU that other handles' threads need to launch their work.
  char* pin = nullptr;
  size_t pin_off = 0;
  struct PinDst { void* dst; size_t off, bytes; };
  std::vector<PinDst> pin_pending;
  // sequential-family epochs enqueued ahead of the host (seq_epochs): per slot, the
  // epoch's steps done, status and gap land in pinned memory; an event marks its end
  char* pin_ep = nullptr;
  cudaEvent_t ev_ep[2] = {nullptr, nullptr};
  std::string err;
  // problem
  double *a = nullptr, *b = nullptr;
  double* b_full = nullptr;   // all n_glob target weights (r_0 = sum_i b_i, global order)
  void* C = nullptr;     // dense (fp32 or fp64), ld elements
  int64_t ld = 0;
  void* x = nullptr;     // colours
  void* y = nullptr;
  bool owns_cost = false;
  // sharding: shard `shard` of G; global column of local p = (p / Bl) Bo + shard Bl + p % Bl
  int G = 1, shard = 0, nranks = 1, n_glob = 0, Bo = 0, Bl = 0;
  Solver* lead = this;                 // the handle (owns peers, exchange buffers, stats)
  std::vector<Solver*> peers;          // other shards held by this process (nranks == 1)
  ncclComm_t comm = nullptr;
  sro_exchange_fn xfn = nullptr;       // host all-gather (sro_params.exchange) instead of NCCL
  void* xuser = nullptr;
  double* xhost = nullptr;             // pinned staging buffer of the host exchange
  size_t xhost_cap = 0;
  int slot_len = 0;
  double *x1 = nullptr, *x2 = nullptr, *gx = nullptr;   // exchange buffers (lead-owned)
  int* capfail = nullptr;
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
  double *G_ga = nullptr, *fen = nullptr;
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
  bool defer_merge = false;   // the next sweep leaves its slab partials to the block tail
  int* st_cnt = nullptr;      // supports staged by a deferred-merge sweep for the block tail
  int* st_row = nullptr;
  double* st_val = nullptr;
  double* st_b = nullptr;
  double* st_term = nullptr;
  double* ga_blk = nullptr;   // sharded GA: the visited block's gathered column gaps (lead)
  int ga_blk_cap = 0;
  const unsigned* sweep_cur = nullptr;   // the next sweep's block index is col0_dev[*sweep_cur]
  unsigned* cur = nullptr;    // device step cursor of the current solve call (block steps enqueued)
  cudaGraphExec_t gexec = nullptr;       // captured block steps of the current solve call
  int gexec_steps = 0;
  int last_nslabs = 1;        // slabs of the last sweep
  unsigned* done_ticket = nullptr;   // k_row_tree_all<1>'s arrival counter (zeroed; its last CTA resets it)
  // block-step workspace
  int64_t blk_L = 0, blk_P = 0;
  int *pcount = nullptr, *poff = nullptr, *ptotal = nullptr, *prow = nullptr, *ppos = nullptr;
  double *pd = nullptr, *ptold = nullptr, *pdelta = nullptr;
  int* rowcnt = nullptr;       // m (zero outside a step)
  int *rowidx = nullptr, *tstart = nullptr, *tcur = nullptr;   // touched-row run-list bookkeeping (tcur zero outside a step)
  int* runc = nullptr;         // run lists (P entries)
  int *bigw = nullptr, *nbig = nullptr;   // hot rows of a step (m), their counts [2]
  double* runv = nullptr;
  double* X = nullptr;         // m (zero outside a step)
  int* trows = nullptr;
  int* ntouch = nullptr;
  unsigned long long* dsteps = nullptr;   // device count of completed block steps
  long long k_pending = 0;                // block steps enqueued since the last sync
  int num_sms = 148;
  // rows of h per sweep CTA (occupancy vs. merge work; SRO_SLAB overrides, multiple of 4, <= SLAB_MAX)
  int slab_rows = getenv("SRO_SLAB") ? std::max(4, std::min(SLAB_MAX, atoi(getenv("SRO_SLAB")) / 4 * 4)) : 4096;
  int slab_bulk = getenv("SRO_SLAB") ? std::max(4, std::min(SLAB_MAX, atoi(getenv("SRO_SLAB")) / 4 * 4)) : 4096;
  bool sweep_ldg = getenv("SRO_SWEEP_LDG") != nullptr;   // debug / A-B: dense sweeps without bulk copies
  // accounting
  long long* phase = nullptr;   // device [8] clock64 totals (SRO_PHASE_TIMING builds)
  double cmax = -1.0;           // max cost, computed once (ensure_cmax)
  bool no_rf = getenv("SRO_NO_RF") != nullptr;      // debug: force the shared-memory kernel
  bool no_tail = getenv("SRO_NO_TAIL") != nullptr;  // debug: force the multi-kernel block step
  bool no_smtail = getenv("SRO_NO_SMTAIL") != nullptr;  // debug: force the global-memory single-CTA tail
  // debug: chunks with more pairs than this take k_runs' support search instead of its sort (0: all)
  int runs_kmax = getenv("SRO_RUNS_KMAX") ? std::max(0, std::min(RUN_KMAX, atoi(getenv("SRO_RUNS_KMAX")))) : RUN_KMAX;
  // k_block_coop (one cooperative launch, grid barriers) measured slower than the per-phase
  // kernels replayed from a CUDA graph (FW config [1]: 40 vs 34 ms): opt-in only
  bool no_coop = getenv("SRO_COOP") == nullptr;
  // debug: no pipelined BCFW kernel (k_bcfw_pipe.cuh) -> register-file kernel k_bcfw_rf
  bool no_pipe = getenv("SRO_NO_PIPE") != nullptr || getenv("SRO_NO_RF") != nullptr;
  sro_stats stats{};
  bool timing = false;
  struct Pending { cudaEvent_t a, b; int cat; int64_t units; };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<Pending> pending;
};

// shards held by this process, lead first
std::vector<Solver*> held(Solver* s) {
  std::vector<Solver*> v{s};
  for (Solver* p : s->peers) v.push_back(p);
  return v;
}
int global_col(const Solver* s, int p) { return (p / s->Bl) * s->Bo + s->shard * s->Bl + p % s->Bl; }
// held columns in ascending global order: (global index, held-shard index, local column)
struct HeldCol { int global, hq, p; };
std::vector<HeldCol> held_order(Solver* s) {
  std::vector<HeldCol> v;
  auto H = held(s);
  for (size_t q = 0; q < H.size(); q++)
    for (int p = 0; p < H[q]->n; p++) v.push_back({H[q]->G == 1 ? p : global_col(H[q], p), (int)q, p});
  std::sort(v.begin(), v.end(), [](const HeldCol& x, const HeldCol& y) { return x.global < y.global; });
  return v;
}

constexpr int TAIL_SMEM = 32 * 256 * 8;   // warp-private chunk slots of the single-CTA block tails

enum { CAT_BCFW = 0, CAT_SWEEP = 1, CAT_BLOCK = 2 };

cudaEvent_t take_event(Solver* s) {
  if (s->ev_pool.empty()) { cudaEvent_t e; cudaEventCreate(&e); return e; }
  cudaEvent_t e = s->ev_pool.back();
  s->ev_pool.pop_back();
  return e;
}
// open a timed region on the solver stream (no-op unless timing is on)
int timed_begin(Solver* s) {
  s = s->lead;
  if (!s->timing) return -1;
  Solver::Pending p{take_event(s), take_event(s), 0, 0};
  cudaEventRecord(p.a, s->stream);
  s->pending.push_back(p);
  return (int)s->pending.size() - 1;
}
void timed_end(Solver* s, int idx, int cat, int64_t units) {
  s = s->lead;
  if (idx < 0) return;
  Solver::Pending& p = s->pending[idx];
  p.cat = cat; p.units = units;
  cudaEventRecord(p.b, s->stream);
}
// after a stream sync: fold every completed region into the stats
void resolve_timing(Solver* s) {
  std::vector<Solver::Pending> keep;   // pairs of work still in flight (enqueued ahead)
  for (auto& p : s->pending) {
    if (cudaEventQuery(p.b) == cudaErrorNotReady) { keep.push_back(p); continue; }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      if (p.cat == CAT_BCFW) s->stats.bcfw_ms += ms;
      else if (p.cat == CAT_SWEEP) s->stats.sweep_ms += ms;
      else s->stats.block_ms += ms;
    }
    s->ev_pool.push_back(p.a);
    s->ev_pool.push_back(p.b);
  }
  s->pending.swap(keep);
}

#define CUDA_TRY(s, call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (s)->err = std::string(#call) + ": " + cudaGetErrorString(e_);                       \
      if ((s)->lead) (s)->lead->pin_pending.clear(); /* no readback outlives a failure */ \
      return e_ == cudaErrorMemoryAllocation ? SRO_ERR_OOM : SRO_ERR_CUDA;                 \
    }                                                                                      \
  } while (0)

thread_local std::string g_create_err;

// Kernel launch with programmatic stream serialization (PDL, see pdl_entry in sro_device.cuh):
// the kernel's CTAs may be scheduled while the previous kernel on the stream drains; each opens
// with griddepcontrol.wait, so it still observes all of the previous kernel's writes. Inside CUDA
// graph capture this becomes a programmatic edge. Opt-in (SRO_PDL=1): alone it gains ~1% on FW /
// batched steps (launch latency is not what bounds them), and with several handles sharing the
// GPU the early-scheduled CTAs waiting at griddepcontrol.wait hold SM slots that the other
// handles' kernels need (bench step: FW 61 -> 70 ms, batched 35 -> 44 ms, BCFW-P 107 -> 119 ms).
bool pdl_enabled() {
  static const bool on = getenv("SRO_PDL") != nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Per-(device, kernel) cache of the dynamic shared-memory attribute and of the
// occupancy query: both are host API calls of several microseconds, and the
// batched / FW loops launch kernels back to back.
struct FuncAttrCache {
  struct E { int dev; const void* f; int smem_set; int threads; size_t smem; int per_sm; };
  std::vector<E> v;
  std::mutex mu;
};
FuncAttrCache& fcache() { static FuncAttrCache c; return c; }
cudaError_t set_dyn_smem(const void* f, int dev, int smem) {
  FuncAttrCache& c = fcache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto& e : c.v)
    if (e.dev == dev && e.f == f && e.threads == 0) {
      if (smem <= e.smem_set) return cudaSuccess;
      cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (r == cudaSuccess) e.smem_set = smem;
      return r;
    }
  cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (r == cudaSuccess) c.v.push_back({dev, f, smem, 0, 0, 0});
  return r;
}
cudaError_t occupancy(const void* f, int dev, int threads, size_t smem, int* per_sm) {
  FuncAttrCache& c = fcache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto& e : c.v)
    if (e.dev == dev && e.f == f && e.threads == threads && e.smem == smem) { *per_sm = e.per_sm; return cudaSuccess; }
  cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, f, threads, smem);
  if (r == cudaSuccess) c.v.push_back({dev, f, 0, threads, smem, *per_sm});
  return r;
}

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
}
// Host wait for an event: poll, yielding the core between polls. A blocking-sync
// wait sleeps until an interrupt wakes the thread (tens to hundreds of us per
// wait, paid on every gap check); a yielding poll returns within a poll of the
// event and still gives the core to other runnable threads (other handles'
// launch threads) when there are any.
cudaError_t wait_event(cudaEvent_t ev) {
  for (;;) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
    std::this_thread::yield();
  }
}

// Wait for the solver stream (record + wait_event).
cudaError_t stream_wait(Solver* s) {
  Solver* L = s->lead;
  if (!L->ev_sync) {
    cudaError_t e = cudaEventCreateWithFlags(&L->ev_sync, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaEventRecord(L->ev_sync, s->stream);
  if (e != cudaSuccess) return e;
  e = wait_event(L->ev_sync);
  if (e == cudaSuccess)
    for (const auto& q : L->pin_pending) memcpy(q.dst, L->pin + q.off, q.bytes);
  L->pin_pending.clear();
  L->pin_off = 0;
  return e;
}

// Device->host readback of a few bytes through the pinned mailbox: *dst holds the
// value after the next stream_wait (every caller synchronises before using it).
constexpr size_t PIN_BYTES = 4096;
cudaError_t rb(Solver* s, void* dst, const void* src, size_t bytes) {
  Solver* L = s->lead;
  if (!L->pin) {
    cudaError_t e = cudaHostAlloc((void**)&L->pin, PIN_BYTES, cudaHostAllocDefault);
    if (e != cudaSuccess) { L->pin = nullptr; return e; }
  }
  if (L->pin_off + bytes > PIN_BYTES) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyAsync(L->pin + L->pin_off, src, bytes, cudaMemcpyDeviceToHost, s->stream);
  if (e != cudaSuccess) return e;
  L->pin_pending.push_back({dst, L->pin_off, bytes});
  L->pin_off += (bytes + 15) & ~(size_t)15;
  return cudaSuccess;
}

// Stream-ordered (re)allocation of solve-time workspaces: no device-wide
// synchronisation, so handles running on other streams are not stalled.
template <typename T>
cudaError_t salloc(T** p, size_t count, cudaStream_t st) {
  static bool pool_set = false;   // keep freed blocks in the device's default pool (cheap reuse)
  if (!pool_set) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  return cudaMallocAsync((void**)p, sizeof(T) * (count ? count : 1), st);
}
inline void sfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// ---------------------------------------------------------------------------
// Small kernels: init, validation, hash generator, objective pieces, max cost
// ---------------------------------------------------------------------------
// r_0 = sum_i b_i over all n columns, left to right (every shard alike), into
// b_full[n_full]: once per handle, so a reset does not repeat the serial sum.
__global__ void k_r0(double* b_full, int n_full) {
  double r0 = 0.0;
  for (int i = 0; i < n_full; i++) r0 = d_add(r0, b_full[i]);
  b_full[n_full] = r0;
}

__global__ void k_init_plan(const double* __restrict__ b, const double* __restrict__ b_full, int n_full,
                            const double* __restrict__ a, double* r, double* h, int* cnt, int* srow, double* sval,
                            int m, int n, int cap, double lambda) {
  // T^(0) = (b_1 e_1, ..., b_n e_1) on the held columns;
  // r_0 = sum_i b_i over all n columns, left to right (every shard alike).
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int i = tid; i < n; i += stride) {
    cnt[i] = b[i] != 0.0 ? 1 : 0;   // a zero-mass column is the zero vector: empty support (R32)
    srow[(int64_t)i * cap] = 0;
    sval[(int64_t)i * cap] = b[i];
  }
  for (int k = tid; k < m; k += stride) {
    if (k == 0) {
      const double r0 = b_full[n_full];   // k_r0, once per handle
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

// SRO_COST_HASH_UNIFORM: C_ki = (splitmix64(seed + (i m + k + 1) GOLDEN) >> 40) 2^-24, fp32 exact,
// for the held local columns p (global column i = (p / Bl) Bo + shard Bl + p % Bl).
__global__ void k_gen_hash(float* C, int64_t ld, int m, int n, uint64_t seed, int Bo, int Bl, int shard) {
  const int64_t total = (int64_t)m * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = q / m, k = q % m;
    const int64_t i = (p / Bl) * Bo + (int64_t)shard * Bl + p % Bl;
    const uint64_t z = mix64(seed + ((uint64_t)(i * m + k) + 1) * GOLDEN);
    C[p * ld + k] = (float)(z >> 40) * 0x1p-24f;
  }
}

// psum256 (R19) over the n global columns of per-column values gathered from
// the G shards: x[s * nl + p] holds the value of local column p of shard s.
__global__ void __launch_bounds__(256) k_psum256_gathered(const double* __restrict__ x, int n, int Bo, int Bl, int nl,
                                                          double* out, const int* __restrict__ stop_in) {
  if (stop_in && *stop_in) return;
  __shared__ double red[8];
  const int c = threadIdx.x;
  const int lo = (int)chunk_lo(c, n, 256), hi = (int)chunk_lo(c + 1, n, 256);
  double acc = 0.0;
  for (int i = lo; i < hi; i++) {
    const int q = i / Bo, rem = i % Bo, s = rem / Bl;
    acc = d_add(acc, x[(size_t)s * nl + (size_t)q * Bl + rem % Bl]);
  }
  acc = warp_pair_tree(acc);
  if ((c & 31) == 0) red[c >> 5] = acc;
  __syncthreads();
  if (c < 32) {
    double v = (c < 8) ? red[c] : 0.0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
    if (c == 0) *out = v;
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

// After a failed step the row workspace (zero outside a step) may hold
// partials of the aborted step: clear it.
sro_status ws_clean(Solver* s) {
  if (s->rowcnt) CUDA_TRY(s, cudaMemsetAsync(s->rowcnt, 0, sizeof(int) * s->m, s->stream));
  if (s->X) CUDA_TRY(s, cudaMemsetAsync(s->X, 0, sizeof(double) * s->m, s->stream));
  if (s->tcur) CUDA_TRY(s, cudaMemsetAsync(s->tcur, 0, sizeof(int) * s->m, s->stream));
  return SRO_OK;
}

// A device status word read by the host: 0 -> SRO_OK; else the error, with the
// status words and workspaces cleared for the next call.
sro_status status_fail(Solver* s, int first) {
  if (!first) return SRO_OK;
  auto H = held(s->lead);
  s->lead->err = first == 5 ? "non-finite value met in the LMO" : first == 6 ? "column support exceeds slab_cap" : "device error";
  for (Solver* t : H) {
    CUDA_TRY(s, cudaMemsetAsync(t->status, 0, sizeof(int), s->stream));
    sro_status e = ws_clean(t);
    if (e) return e;
  }
  return (sro_status)first;
}

// Synchronise and read the status word of every held shard (they agree: the
// sharded phases propagate the first error of any shard to all of them).
sro_status check_status(Solver* s) {
  auto H = held(s->lead);
  std::vector<int> st(H.size(), 0);
  for (size_t q = 0; q < H.size(); q++)
    CUDA_TRY(s, rb(s, &st[q], H[q]->status, sizeof(int)));
  CUDA_TRY(s, stream_wait(s));
  int first = 0;
  for (int v : st) if (v && !first) first = v;
  return status_fail(s, first);
}

// Sharded exchange of `count` doubles per shard: buf holds G slots of `count`;
// every shard has written its own slot. nranks == 1: all slots are local
// already. nranks == G: in-place all-gather on the solver stream.
sro_status exchange(Solver* s, double* buf, size_t count) {
  if (s->nranks == 1) return SRO_OK;
  if (s->xfn) {   // host all-gather: device slots -> pinned host buffer -> callback -> device
    const size_t total = count * (size_t)s->nranks;
    if (total > s->xhost_cap) {
      if (s->xhost) cudaFreeHost(s->xhost);
      s->xhost = nullptr; s->xhost_cap = 0;
      CUDA_TRY(s, cudaHostAlloc((void**)&s->xhost, sizeof(double) * total, cudaHostAllocDefault));
      s->xhost_cap = total;
    }
    CUDA_TRY(s, cudaMemcpyAsync(s->xhost, buf, sizeof(double) * total, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, stream_wait(s));
    if (s->xfn(s->xuser, s->xhost, (int64_t)count, s->nranks, s->shard) != 0) { s->err = "host exchange failed"; return SRO_ERR_NCCL; }
    CUDA_TRY(s, cudaMemcpyAsync(buf, s->xhost, sizeof(double) * total, cudaMemcpyHostToDevice, s->stream));
    return SRO_OK;
  }
  NcclApi& api = nccl();
  ncclResult_t r = api.allgather(buf + (size_t)s->shard * count, buf, count, ncclFloat64, s->comm, s->stream);
  if (r != ncclSuccess) { s->err = std::string("ncclAllGather: ") + api.errstr(r); return SRO_ERR_NCCL; }
  return SRO_OK;
}

bool sweep_nt_wide() {
  static const bool wide = !(getenv("SRO_COLOUR_NT") && atoi(getenv("SRO_COLOUR_NT")) == 256);   // A-B
  return wide;
}
bool getenv_slab_fixed() {
  static const bool fixed = getenv("SRO_SLAB") != nullptr;   // debug / A-B: the slab the environment names
  return fixed;
}

sro_status ensure_partials(Solver* s, int nslabs, int L) {
  if (nslabs > 1 && (int64_t)nslabs * L > s->part_cap) {
    sfree(s->part_j, s->stream); sfree(s->part_min, s->stream);
    s->part_cap = (int64_t)nslabs * L;
    CUDA_TRY(s, salloc(&s->part_j, s->part_cap, s->stream));
    CUDA_TRY(s, salloc(&s->part_min, s->part_cap, s->stream));
  }
  return SRO_OK;
}

// Dense LMO sweep through the bulk-copy pipeline (k_lmo_sweep_bulk): one CTA
// per SM, (slab, column) items split evenly over the grid.
template <class Src>
sro_status sweep_bulk(Solver* s, Src src, const int* col0_dev, int col0_mul, int col0_host, int L, int* out_j,
                      double* out_min, double* out_g, const int* stop) {
  using T = std::remove_cv_t<std::remove_pointer_t<decltype(src.C)>>;
#ifndef SRO_BULK_S
#define SRO_BULK_S 4
#endif
  constexpr int S = SRO_BULK_S;
  // rows per (slab, column) item: the default slab, smaller when the sweep has few
  // columns (a batched block) so that every SM still gets several items
  int slab = s->slab_bulk;
  {
    // about twelve (slab, column) items per SM (batched config [1], B = 256, us per block step at
    // 4 / 8 / 12 / 16 / 24 items per SM: 33.0 / 31.3 / 30.7 / 32.7 / 33.4 with the round-2 tail, whose
    // slab merge is no longer the long pole; round 1 had 4 as best; SRO_BULK_ITEMS overrides for A/B)
    static const double items_per_sm = getenv("SRO_BULK_ITEMS") ? atof(getenv("SRO_BULK_ITEMS")) : 12.0;
    const int64_t target = (int64_t)((double)s->num_sms * items_per_sm);
    const int64_t want = ((int64_t)s->m * L + target - 1) / target;
    if (want < slab) slab = (int)std::max<int64_t>(256, (want + 3) / 4 * 4);
  }
  const int nslabs = (s->m + slab - 1) / slab;
  { sro_status st = ensure_partials(s, nslabs, L); if (st) return st; }
  const int rows = s->m < slab ? s->m : slab;
  const size_t smem = 1024 + (size_t)BULK_WARPS * S * BULK_CH + sizeof(double) * (size_t)rows;
  auto kern = k_lmo_sweep_bulk<T, S>;
  CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
  int per_sm = 0;
  CUDA_TRY(s, occupancy((const void*)kern, s->device, BULK_WARPS * 32, smem, &per_sm));
  if (per_sm < 1) per_sm = 1;
  const int64_t ntot = (int64_t)nslabs * L;
  int64_t nb = (int64_t)s->num_sms * per_sm;
  const int64_t need = (ntot + BULK_WARPS - 1) / BULK_WARPS;
  if (nb > need) nb = need;
  if (nb < 1) nb = 1;
  SweepOut o{};
  if (nslabs == 1) { o.j = out_j; o.minval = out_min; o.g = out_g; }
  else { o.j = s->part_j; o.minval = s->part_min; o.g = nullptr; }
  if (nslabs > 1 && s->defer_merge && s->st_cnt) { o.st_cnt = s->st_cnt; o.st_row = s->st_row; o.st_val = s->st_val; o.st_b = s->st_b; o.st_term = s->st_term; }
  const int tr = timed_begin(s);
  s->lead->stats.kernel_launches += (nslabs > 1 && !s->defer_merge) ? 2 : 1;
  s->lead->stats.sweep_launches += 1;
  s->lead->stats.sweep_columns += L;
  CUDA_TRY(s, launch_pdl(kern, dim3((int)nb), dim3(BULK_WARPS * 32), smem, s->stream, src, s->m, slab, nslabs, s->h, col0_dev, s->sweep_cur, col0_mul, col0_host, L,
                                                    s->cnt, s->srow, s->sval, s->cap, s->b, o, stop, s->status));
  CUDA_TRY(s, cudaGetLastError());
  s->last_nslabs = nslabs;
  if (nslabs > 1 && !s->defer_merge) {
    int gm = (L + SWEEP_WARPS - 1) / SWEEP_WARPS;
    if (gm > s->num_sms * 8) gm = s->num_sms * 8;
    CUDA_TRY(s, launch_pdl(k_lmo_merge<Src>, dim3(gm), dim3(SWEEP_THREADS), 0, s->stream, src, nslabs, s->h, col0_dev, s->sweep_cur, col0_mul, col0_host, L, s->cnt,
                                                          s->srow, s->sval, s->cap, s->b, s->part_j, s->part_min,
                                                          out_j, out_min, out_g, stop, s->status));
    CUDA_TRY(s, cudaGetLastError());
  }
  timed_end(s, tr, CAT_SWEEP, L);
  return SRO_OK;
}

// LMO sweep over [col0, col0+L) -> out_j, out_min, out_g (device arrays of length >= L).
sro_status sweep(Solver* s, const int* col0_dev, int col0_mul, int col0_host, int L, int* out_j, double* out_min,
                 double* out_g, const int* stop) {
  return with_sweep_src(s, [&](auto src) -> sro_status {
    using Src = decltype(src);
    if constexpr (Src::PLANAR) {
      if (!s->sweep_ldg) return sweep_bulk(s, src, col0_dev, col0_mul, col0_host, L, out_j, out_min, out_g, stop);
    }
    int slab = s->slab_rows;
    // several columns per warp when there are enough columns to fill the GPU that
    // way; a block with few columns (batched) keeps one column per warp and splits the rows
    // into shorter slabs instead, sized for about four CTAs per SM (measured against four
    // columns per warp over two-CTA-per-SM slabs: config [2] block step 35.4 -> 32.6 us, [4]
    // 43.8 -> 41.8 — fewer slab partials for the tail to read, more warps in flight)
    const bool multi = Src::COLS > 1 && (int64_t)L * ((s->m + slab - 1) / slab) >=
                                            (int64_t)s->num_sms * SWEEP_WARPS * Src::COLS * 2;
    if (Src::COLS > 1 && !multi && !getenv_slab_fixed()) {
      const int64_t per_slab = (L + SWEEP_WARPS - 1) / SWEEP_WARPS;
      const int64_t want = std::max<int64_t>(1, (int64_t)s->num_sms * 4 / per_slab);
      int64_t rows_want = (s->m + want - 1) / want;
      rows_want = (rows_want + 31) / 32 * 32;
      if (rows_want < 128) rows_want = 128;
      if (rows_want < slab) slab = (int)rows_want;
    }
    if (Src::WIDE && multi && sweep_nt_wide() && !getenv_slab_fixed()) {
      // a warp's work items are (slab, 4 columns); halve the slab (down to 1024 rows) while that
      // evens out the items per warp (config [2]: 4096-row slabs leave 3.46 items per warp,
      // 2048-row slabs 6.92)
      auto eff = [&](int sl) {
        const int64_t ns = (s->m + sl - 1) / sl, rw = s->m < sl ? s->m : sl;
        const int64_t sm = 8 * ((rw + 1) & ~1) + (int64_t)Src::SMEM_PER_ROW * rw;
        const int64_t per = std::max<int64_t>(1, std::min<int64_t>(2, (227 * 1024) / (sm + 1024)));
        const int64_t warps_slab = std::max<int64_t>(1, (s->num_sms * per + ns - 1) / ns) * (2 * SWEEP_WARPS);
        const int64_t items = (L + Src::COLS - 1) / Src::COLS;
        const int64_t rounds = (items + warps_slab - 1) / warps_slab;
        return (double)items / (double)(rounds * warps_slab);
      };
      double best = eff(slab);
      for (int sl = slab / 2; sl >= 1024 && sl % 32 == 0; sl /= 2) {
        const double e = eff(sl);
        if (e > best + 0.02) { best = e; slab = sl; }
      }
    }
    const int nslabs = (s->m + slab - 1) / slab;
    { sro_status st = ensure_partials(s, nslabs, L); if (st) return st; }
    const int rows = s->m < slab ? s->m : slab;
    // (+ 16 B: the binary32 colour planes start at even offsets, so one row takes 3 x 2 floats)
    const size_t smem = sizeof(double) * (size_t)((rows + 1) & ~1) + (size_t)Src::SMEM_PER_ROW * rows + 16;
    const int cols = multi ? Src::COLS : 1;
    // the multi-column colour sweep runs CTAs of 16 warps (twice the warps in flight per SM
    // for the same staged slab)
    constexpr bool wide_ok = Src::WIDE;   // the packed binary32 colour source
    const int nt = wide_ok && multi && sweep_nt_wide() ? 2 * SWEEP_THREADS : SWEEP_THREADS;
    auto kern = k_lmo_sweep<Src, 1>;
    if (multi) kern = k_lmo_sweep<Src, Src::COLS>;
    if constexpr (wide_ok) { if (nt > SWEEP_THREADS) kern = k_lmo_sweep<Src, Src::COLS, 2 * SWEEP_THREADS>; }
    CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
    int per_sm = 0;
    CUDA_TRY(s, occupancy((const void*)kern, s->device, nt, smem, &per_sm));
    if (per_sm < 1) per_sm = 1;
    int gx = s->num_sms * per_sm;
    const int warps = nt / 32;
    const int need = (L + warps * cols - 1) / (warps * cols);
    if (nslabs > 1) gx = (gx + nslabs - 1) / nslabs;
    if (gx > need) gx = need;
    if (gx < 1) gx = 1;
    SweepOut o{};
    if (nslabs == 1) { o.j = out_j; o.minval = out_min; o.g = out_g; }
    else { o.j = s->part_j; o.minval = s->part_min; o.g = nullptr; }
    if (nslabs > 1 && s->defer_merge && s->st_cnt) { o.st_cnt = s->st_cnt; o.st_row = s->st_row; o.st_val = s->st_val; o.st_b = s->st_b; o.st_term = s->st_term; }
    const int tr = timed_begin(s);
    s->lead->stats.kernel_launches += (nslabs > 1 && !s->defer_merge) ? 2 : 1;
    s->lead->stats.sweep_launches += 1;
    s->lead->stats.sweep_columns += L;
    CUDA_TRY(s, launch_pdl(kern, dim3(dim3(gx, nslabs)), dim3(nt), smem, s->stream, src, s->m, slab, s->h, col0_dev, s->sweep_cur, col0_mul, col0_host, L,
                                                             s->cnt, s->srow, s->sval, s->cap, s->b, o, stop,
                                                             s->status));
    CUDA_TRY(s, cudaGetLastError());
    s->last_nslabs = nslabs;
    if (nslabs > 1 && !s->defer_merge) {
      int gm = (L + SWEEP_WARPS - 1) / SWEEP_WARPS;
      if (gm > s->num_sms * 8) gm = s->num_sms * 8;
      CUDA_TRY(s, launch_pdl(k_lmo_merge<Src>, dim3(gm), dim3(SWEEP_THREADS), 0, s->stream, src, nslabs, s->h, col0_dev, s->sweep_cur, col0_mul, col0_host, L,
                                                            s->cnt, s->srow, s->sval, s->cap, s->b, s->part_j,
                                                            s->part_min, out_j, out_min, out_g, stop, s->status));
      CUDA_TRY(s, cudaGetLastError());
    }
    timed_end(s, tr, CAT_SWEEP, L);
    return SRO_OK;
  });
}

// Full gap sweep: g(T) = psum256_i g_i (Thm 2 / Eq. 11) -> host. Sharded:
// every held shard sweeps its columns into its slot of gx, the slots are
// exchanged and the total is the psum256 over the n global columns.
// The gap sweep without the synchronisation: *total is written when the stream
// reaches it (the caller synchronises; stop as in ga_global_refresh, unsharded only).
sro_status gap_sweep_kernels(Solver* s, const int* stop = nullptr) {
  sro_status st;
  if (s->G == 1) {
    st = sweep(s, nullptr, 0, 0, s->n, s->sw_j, s->sw_min, s->sw_g, stop);
    if (st) return st;
    k_psum256<<<1, 256, 0, s->stream>>>(s->sw_g, s->n, s->scal + 4, nullptr, nullptr, stop);
  } else {
    for (Solver* t : held(s)) {
      st = sweep(t, nullptr, 0, 0, t->n, t->sw_j, t->sw_min, s->gx + (size_t)t->shard * t->n, nullptr);
      if (st) return st;
    }
    st = exchange(s, s->gx, s->n);
    if (st) return st;
    k_psum256_gathered<<<1, 256, 0, s->stream>>>(s->gx, s->n_glob, s->Bo, s->Bl, s->n, s->scal + 4, nullptr);
  }
  s->lead->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  return SRO_OK;
}
sro_status gap_sweep_enqueue(Solver* s, double* total, const int* stop = nullptr) {
  sro_status st = gap_sweep_kernels(s, stop);
  if (st) return st;
  CUDA_TRY(s, rb(s, total, s->scal + 4, sizeof(double)));
  return SRO_OK;
}

sro_status gap_sweep(Solver* s, double* total) {
  sro_status st = gap_sweep_enqueue(s, total);
  if (st) return st;
  st = check_status(s);  // synchronises
  resolve_timing(s);
  return st;
}

sro_status ensure_visit(Solver* s, int64_t count) {
  if (count > s->visit_cap) {
    sfree(s->visit, s->stream);
    s->visit_cap = count < 4096 ? 4096 : count;
    CUDA_TRY(s, salloc(&s->visit, s->visit_cap, s->stream));
  }
  return SRO_OK;
}
sro_status ensure_trace(Solver* s, int64_t count) {
  if (count > s->trace_cap) {
    sfree(s->trace, s->stream);
    s->trace_cap = count;
    CUDA_TRY(s, salloc(&s->trace, 9 * s->trace_cap, s->stream));
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
  CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, BCFW_THREADS, smem, s->stream>>>(A, col);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->lead->stats.kernel_launches += 1;
  s->lead->stats.bcfw_launches += 1;
  s->lead->stats.bcfw_steps += A.steps;
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
  CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, BCFW_THREADS, smem, s->stream>>>(A, (const T*)s->C, s->ld);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->lead->stats.kernel_launches += 1;
  s->lead->stats.bcfw_launches += 1;
  s->lead->stats.bcfw_steps += A.steps;
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

template <typename T, int MAXV, int VAR>
sro_status launch_pipe(Solver* s, BcfwArgs& A, size_t smem) {
  auto kern = k_bcfw_pipe<T, MAXV, VAR>;
  CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, PIPE_THREADS, smem, s->stream>>>(A, (const T*)s->C, s->ld);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->lead->stats.kernel_launches += 1;
  s->lead->stats.bcfw_launches += 1;
  s->lead->stats.bcfw_steps += A.steps;
  return SRO_OK;
}

// Pipelined kernel (k_bcfw_pipe.cuh) for dense costs and U / P / explicit
// visits when the rows fit in the registers of 480 threads (<= 4 vectors each).
// Returns SRO_ERR_DIMENSION (not an error to the caller) when it does not apply.
template <int VAR>
sro_status bcfw_try_pipe(Solver* s, BcfwArgs& A) {
  const bool dense = s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM;
  if (!dense || s->no_pipe) return SRO_ERR_DIMENSION;
  const int W = s->prec == SRO_FP32 ? 4 : 2;
  const int nvec = s->m / W;
  const int need = (nvec + PIPE_LMO - 1) / PIPE_LMO;
  if (need > 4 || s->m - nvec * W > PIPE_LMO) return SRO_ERR_DIMENSION;
  const size_t limit = 226 * 1024;
  A.visit_smem = PipeLayout::bytes(s->m, s->n, A.steps, true) <= limit;
  A.ga_smem = 0;
  A.a_smem = 1;
  const size_t bytes = PipeLayout::bytes(s->m, s->n, A.steps, A.visit_smem);
  if (bytes > limit) return SRO_ERR_DIMENSION;
  if (s->prec == SRO_FP32) {
    if (need <= 1) return launch_pipe<float, 1, VAR>(s, A, bytes);
    if (need <= 2) return launch_pipe<float, 2, VAR>(s, A, bytes);
    if (need <= 3) return launch_pipe<float, 3, VAR>(s, A, bytes);
    return launch_pipe<float, 4, VAR>(s, A, bytes);
  }
  if (need <= 1) return launch_pipe<double, 1, VAR>(s, A, bytes);
  if (need <= 2) return launch_pipe<double, 2, VAR>(s, A, bytes);
  if (need <= 3) return launch_pipe<double, 3, VAR>(s, A, bytes);
  return launch_pipe<double, 4, VAR>(s, A, bytes);
}

template <typename T, int MAXV, int VAR>
sro_status launch_ga_pipe(Solver* s, BcfwArgs& A, size_t smem) {
  auto kern = A.ga_smem ? k_bcfw_ga_pipe<T, MAXV, VAR, true> : k_bcfw_ga_pipe<T, MAXV, VAR, false>;
  CUDA_TRY(s, set_dyn_smem((const void*)kern, s->device, (int)smem));
  const int tr = timed_begin(s);
  kern<<<1, PIPE_THREADS, smem, s->stream>>>(A, (const T*)s->C, s->ld);
  CUDA_TRY(s, cudaGetLastError());
  timed_end(s, tr, CAT_BCFW, A.steps);
  s->lead->stats.kernel_launches += 1;
  s->lead->stats.bcfw_launches += 1;
  s->lead->stats.bcfw_steps += A.steps;
  return SRO_OK;
}

// GA counterpart (k_bcfw_ga_pipe): dense costs, state + stored gaps + Fenwick
// tree in shared memory. SRO_ERR_DIMENSION when it does not apply.
template <int VAR>
sro_status bcfw_try_ga_pipe(Solver* s, BcfwArgs& A) {
  const bool dense = s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM;
  if (!dense || s->no_pipe) return SRO_ERR_DIMENSION;
  const int W = s->prec == SRO_FP32 ? 4 : 2;
  const int nvec = s->m / W;
  const int need = (nvec + GA_LMO - 1) / GA_LMO;
  if (need > 4 || s->m - nvec * W > GA_LMO) return SRO_ERR_DIMENSION;
  // a and the stored gaps in shared memory when they fit, else both in global memory
  const size_t lim = 226 * 1024;
  const bool gsm = GaPipeLayout::bytes(s->m, s->n, true, true) <= lim;
  const size_t bytes = GaPipeLayout::bytes(s->m, s->n, gsm, gsm);
  if (bytes > lim) return SRO_ERR_DIMENSION;
  A.ga_smem = gsm ? 1 : 0; A.a_smem = A.ga_smem; A.visit_smem = 0;
  if (s->prec == SRO_FP32) {
    if (need <= 1) return launch_ga_pipe<float, 1, VAR>(s, A, bytes);
    if (need <= 2) return launch_ga_pipe<float, 2, VAR>(s, A, bytes);
    if (need <= 3) return launch_ga_pipe<float, 3, VAR>(s, A, bytes);
    return launch_ga_pipe<float, 4, VAR>(s, A, bytes);
  }
  if (need <= 1) return launch_ga_pipe<double, 1, VAR>(s, A, bytes);
  if (need <= 2) return launch_ga_pipe<double, 2, VAR>(s, A, bytes);
  if (need <= 3) return launch_ga_pipe<double, 3, VAR>(s, A, bytes);
  return launch_ga_pipe<double, 4, VAR>(s, A, bytes);
}

template <int VAR, bool GA>
sro_status bcfw_run(Solver* s, BcfwArgs& A) {
  {
    sro_status st = GA ? bcfw_try_ga_pipe<VAR>(s, A) : bcfw_try_pipe<VAR>(s, A);
    if (st != SRO_ERR_DIMENSION) return st;
  }
  if (!s->no_rf) {
    sro_status st = bcfw_try_rf<VAR, GA>(s, A);
    if (st != SRO_ERR_DIMENSION) return st;
  }
  return bcfw_dispatch<VAR, GA>(s, A);
}

sro_status bcfw_segment(Solver* s, int variant, const sro_options* o, int steps, const int* dvisit,
                        double* dtrace, long long k0, const int* halt) {
  BcfwArgs A{};
  A.m = s->m; A.n = s->n; A.cap = s->cap; A.lambda = s->lambda;
  A.a = s->a; A.b = s->b; A.r = s->r; A.h = s->h; A.cnt = s->cnt; A.srow = s->srow; A.sval = s->sval;
  A.visit = dvisit; A.steps = steps; A.k0 = k0; A.step_rule = o->step; A.halt = halt;
  A.G = s->G_ga; A.fen = s->fen; A.ga_inner = o->ga_inner; A.ga_post = o->ga_post_update; A.seed = s->seed;
  A.status = s->status; A.steps_done = s->steps_done; A.trace = dtrace;
  A.phase = s->phase;
  A.dbg = getenv("SRO_DBG") ? atoi(getenv("SRO_DBG")) : 0;
  A.spec = getenv("SRO_NO_SPEC") ? 0 : 1;   // A/B: SRO_NO_SPEC turns the GA pipe's speculative pre-scan off
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
    s->lead->stats.kernel_launches += 1;
    CUDA_TRY(s, cudaGetLastError());
    return SRO_OK;
  });
  if (st) return st;
  unsigned long long bits = 0;
  CUDA_TRY(s, rb(s, &bits, d_cmax, sizeof(bits)));
  CUDA_TRY(s, stream_wait(s));
  double v;
  memcpy(&v, &bits, sizeof(v));
  s->cmax = v;
  return SRO_OK;
}

sro_status fen_build(Solver* s, int n_tree = -1, const int* stop = nullptr) {
  const int nt = n_tree < 0 ? s->n : n_tree;
  const size_t bytes = sizeof(double) * ((size_t)nt + 1);
  const int use_smem = bytes <= 200 * 1024;
  if (use_smem) CUDA_TRY(s, set_dyn_smem((const void*)k_fen_build, s->device, (int)bytes));
  k_fen_build<<<1, 256, use_smem ? bytes : 0, s->stream>>>(s->G_ga, s->fen, nt, use_smem, stop);
  s->lead->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  return SRO_OK;
}

// stop: device flag (the solver status) that turns the refresh into a no-op when
// the segment before it failed (enqueued before the host has seen that segment's status)
sro_status ga_global_refresh(Solver* s, const int* stop = nullptr) {
  sro_status st = sweep(s, nullptr, 0, 0, s->n, s->sw_j, s->sw_min, s->G_ga, stop);
  if (st) return st;
  return fen_build(s, -1, stop);
}

// GA global refresh that is also the epoch's gap check (M = 1 and the check falls on the same
// boundary, SURVEY c.7 / P:363): ONE sweep stores every g_i(T) as the new G_i and the gap total
// is the psum256 of those same values — bitwise what the separate refresh + gap sweep give.
sro_status ga_refresh_and_gap(Solver* s, const int* stop = nullptr) {
  sro_status st = sweep(s, nullptr, 0, 0, s->n, s->sw_j, s->sw_min, s->G_ga, stop);
  if (st) return st;
  st = fen_build(s, -1, stop);
  if (st) return st;
  k_psum256<<<1, 256, 0, s->stream>>>(s->G_ga, s->n, s->scal + 4, nullptr, nullptr, stop);
  s->lead->stats.kernel_launches += 1;
  CUDA_TRY(s, cudaGetLastError());
  return SRO_OK;
}

__global__ void k_halt_on_status(const int* status, int* halt) {
  if (*status) *halt = 1;
}
__global__ void k_halt_on_gap(const double* g, double eps, int* halt) {
  if (!*halt && *g <= eps) *halt = 1;
}

// The sequential BCFW family (Alg. 1, A.2-A.4) from s->k on, until the gap check
// meets epsilon, iters steps are done or a segment fails. One epoch = a persistent
// kernel segment up to the next gap check / GA global refresh (whichever is first),
// then that refresh and check. Epoch e+1 is enqueued before the host reads epoch
// e's outcome; its kernels test s->stop, which e's tail sets on failure or
// convergence, so a speculative epoch changes nothing. Same kernels, same order,
// same results as checking after every epoch.
sro_status seq_epochs(Solver* s, int variant, const sro_options* o, int64_t iters, long long period, long long gaMn,
                      bool ga, int64_t* done_io, sro_result* out) {
  Solver* L = s->lead;
  const int64_t m = s->m, n = s->n;
  if (!L->pin_ep) {
    if (cudaHostAlloc((void**)&L->pin_ep, 64, cudaHostAllocDefault) != cudaSuccess) {
      L->pin_ep = nullptr; s->err = "cudaHostAlloc"; return SRO_ERR_CUDA;
    }
    for (int q = 0; q < 2; q++)
      CUDA_TRY(s, cudaEventCreateWithFlags(&L->ev_ep[q], cudaEventDisableTiming));
  }
  struct Ep { long long k0; int64_t done0; long long seg; bool refresh, check; int slot; };
  auto plan = [&](long long k, int64_t dn, int slot) {
    Ep e;
    e.k0 = k; e.done0 = dn; e.slot = slot;
    long long sg = iters - dn;
    const long long tc = period - k % period;
    if (sg > tc) sg = tc;
    if (ga) { const long long tr = gaMn - k % gaMn; if (sg > tr) sg = tr; }
    e.seg = sg;
    e.refresh = ga && (k + sg) % gaMn == 0;
    e.check = (k + sg) % period == 0;
    return e;
  };
  auto enqueue = [&](const Ep& e) -> sro_status {
    sro_status st = bcfw_segment(s, variant, o, (int)e.seg, ga ? nullptr : s->visit + e.done0,
                                 o->trace ? s->trace + 9 * e.done0 : nullptr, e.k0, s->stop);
    if (st) return st;
    k_halt_on_status<<<1, 1, 0, s->stream>>>(s->status, s->stop);
    s->lead->stats.kernel_launches += 1;
    const bool fused = e.refresh && e.check && s->G == 1;
    if (e.refresh && !fused) { st = ga_global_refresh(s, s->stop); if (st) return st; }
    if (e.check) {
      st = fused ? ga_refresh_and_gap(s, s->stop) : gap_sweep_kernels(s, s->stop);
      if (st) return st;
      k_halt_on_gap<<<1, 1, 0, s->stream>>>(s->scal + 4, o->epsilon, s->stop);
      s->lead->stats.kernel_launches += 1;
    }
    CUDA_TRY(s, cudaGetLastError());
    char* slot = L->pin_ep + 32 * e.slot;
    CUDA_TRY(s, cudaMemcpyAsync(slot, s->steps_done, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, cudaMemcpyAsync(slot + 4, s->status, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    if (e.check) CUDA_TRY(s, cudaMemcpyAsync(slot + 8, s->scal + 4, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, cudaEventRecord(L->ev_ep[e.slot], s->stream));
    return SRO_OK;
  };
  CUDA_TRY(s, cudaMemsetAsync(s->stop, 0, sizeof(int), s->stream));
  int64_t done = *done_io;
  sro_status st = SRO_OK;
  Ep cur = plan(s->k, done, 0), nx{};
  bool spec = false;   // nx enqueued and not yet consumed
  st = enqueue(cur);
  while (!st) {
    const bool have_next = cur.done0 + cur.seg < iters;
    if (have_next) {
      nx = plan(cur.k0 + cur.seg, cur.done0 + cur.seg, cur.slot ^ 1);
      st = enqueue(nx);
      if (st) break;
      spec = true;
    }
    if (wait_event(L->ev_ep[cur.slot]) != cudaSuccess) { s->err = "epoch synchronisation"; st = SRO_ERR_CUDA; break; }
    const char* slot = L->pin_ep + 32 * cur.slot;
    int sd = 0, dst = 0;
    double g = 0.0;
    memcpy(&sd, slot, sizeof(int));
    memcpy(&dst, slot + 4, sizeof(int));
    if (cur.check) memcpy(&g, slot + 8, sizeof(double));
    resolve_timing(s);
    s->k += sd; done += sd;
    // LMO-call count as the method (and the oracle) defines it: a GAD post-update refresh is a
    // second LMO on the column; the kernels take it from the step's own column read (entries_read)
    out->entries_scanned += m * sd * ((ga && o->ga_inner && o->ga_post_update) ? 2 : 1);
    out->entries_read += m * sd;
    if (dst) { st = status_fail(s, dst); break; }
    if (sd != cur.seg) { s->err = "segment stopped early without a status"; st = SRO_ERR_CUDA; break; }
    if (cur.refresh) out->entries_scanned += m * n;
    if (cur.refresh && !(cur.check && s->G == 1)) out->entries_read += m * n;
    if (cur.check) {
      out->gap = g; out->gap_checks++;
      out->entries_scanned += m * n;
      out->entries_read += m * n;
      if (g <= o->epsilon) { out->converged = 1; break; }
    }
    if (!have_next) break;
    cur = nx;
    spec = false;
  }
  if (spec) {   // the epoch enqueued ahead was a no-op: its segment is not a launch of steps
    L->stats.bcfw_launches -= 1;
    L->stats.bcfw_steps -= nx.seg;
  }
  *done_io = done;
  // after any speculative epoch still in flight (a no-op)
  CUDA_TRY(s, cudaMemsetAsync(s->stop, 0, sizeof(int), s->stream));
  return st;
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
  k_ga_init<<<64, 256, 0, s->stream>>>(s->G_ga, s->fen, s->n, d_cmax, s->lambda);
  s->lead->stats.kernel_launches += 2;
  CUDA_TRY(s, cudaGetLastError());
  return fen_build(s);
}

// Sharded GA block sampling (R31): the lead keeps the tree over all n_glob columns (every
// process its own replica when nranks > 1); C_init from the largest cost over all shards.
sro_status ga_initialise_sharded(Solver* s) {
  unsigned long long* d_cmax = reinterpret_cast<unsigned long long*>(s->scal + 6);
  CUDA_TRY(s, cudaMemsetAsync(d_cmax, 0, sizeof(unsigned long long), s->stream));
  for (Solver* t : held(s)) {
    sro_status st = with_sweep_src(t, [&](auto src) -> sro_status {
      k_max_cost<<<s->num_sms * 4, 256, 0, s->stream>>>(src, t->m, t->n, d_cmax);
      CUDA_TRY(s, cudaGetLastError());
      return SRO_OK;
    });
    if (st) return st;
  }
  if (s->nranks > 1) {
    k_key_to_slot<<<1, 32, 0, s->stream>>>(d_cmax, s->x1 + (size_t)s->shard * s->slot_len);
    sro_status st = exchange(s, s->x1, s->slot_len);
    if (st) return st;
    k_max_slots<<<1, 32, 0, s->stream>>>(s->x1, s->G, s->slot_len, d_cmax);
  }
  k_ga_init<<<64, 256, 0, s->stream>>>(s->G_ga, s->fen, s->n_glob, d_cmax, s->lambda);
  CUDA_TRY(s, cudaGetLastError());
  return fen_build(s, s->n_glob);
}
sro_status ga_global_refresh_sharded(Solver* s, double* gap_out) {
  sro_status st = gap_sweep(s, gap_out);   // every shard's column gaps, exchanged, in gx
  if (st) return st;
  k_ga_gather_global<<<s->num_sms * 4, 256, 0, s->stream>>>(s->gx, s->G_ga, s->n, s->G, s->Bo, s->Bl);
  CUDA_TRY(s, cudaGetLastError());
  return fen_build(s, s->n_glob);
}

// ---------------------------------------------------------------------------
// Plain step over a contiguous column set (FW / batched)
// ---------------------------------------------------------------------------
sro_status ensure_block_ws(Solver* s, int64_t L) {
  const int64_t P = L * (s->cap + 1);
  if (!s->rowcnt) {   // row workspace: zero outside a step
    CUDA_TRY(s, salloc(&s->rowcnt, s->m, s->stream)); CUDA_TRY(s, salloc(&s->X, s->m, s->stream));
    CUDA_TRY(s, salloc(&s->trows, s->m, s->stream)); CUDA_TRY(s, salloc(&s->ntouch, 1, s->stream));
    CUDA_TRY(s, salloc(&s->rowidx, s->m, s->stream)); CUDA_TRY(s, salloc(&s->tstart, s->m, s->stream));
    CUDA_TRY(s, salloc(&s->tcur, s->m, s->stream)); CUDA_TRY(s, salloc(&s->capfail, 1, s->stream));
    CUDA_TRY(s, salloc(&s->bigw, s->m, s->stream)); CUDA_TRY(s, salloc(&s->nbig, 2, s->stream));
    { sro_status e = ws_clean(s); if (e) return e; }
    CUDA_TRY(s, cudaMemsetAsync(s->capfail, 0, sizeof(int), s->stream));
  }
  if (L <= s->blk_L && P <= s->blk_P) return SRO_OK;
  for (void* q : {(void*)s->pcount, (void*)s->poff, (void*)s->ptotal, (void*)s->prow, (void*)s->ppos, (void*)s->pd,
                  (void*)s->ptold, (void*)s->pdelta, (void*)s->runc, (void*)s->runv})
    sfree(q, s->stream);
  s->blk_L = L; s->blk_P = P;
  CUDA_TRY(s, salloc(&s->pcount, L, s->stream)); CUDA_TRY(s, salloc(&s->poff, L + 1, s->stream)); CUDA_TRY(s, salloc(&s->ptotal, 1, s->stream));
  CUDA_TRY(s, salloc(&s->prow, P, s->stream)); CUDA_TRY(s, salloc(&s->ppos, P, s->stream)); CUDA_TRY(s, salloc(&s->pd, P, s->stream));
  CUDA_TRY(s, salloc(&s->ptold, P, s->stream)); CUDA_TRY(s, salloc(&s->pdelta, P, s->stream));
  CUDA_TRY(s, salloc(&s->runc, P, s->stream)); CUDA_TRY(s, salloc(&s->runv, P, s->stream));
  return SRO_OK;
}

BlockArgs block_args(Solver* s, const int* col0_dev, int col0_mul, int L, int step_rule, long long nprime,
                     bool stop_check, double* trace_dev, unsigned* cur = nullptr, long long kbase = 0) {
  BlockArgs A{};
  A.m = s->m; A.n = s->n; A.cap = s->cap; A.lambda = s->lambda; A.a = s->a; A.b = s->b; A.r = s->r; A.h = s->h;
  A.cnt = s->cnt; A.srow = s->srow; A.sval = s->sval; A.col0_dev = col0_dev; A.col0_mul = col0_mul; A.L = L;
  A.W = 256 / s->G;
  A.runs_kmax = s->runs_kmax;
  A.j = s->sw_j; A.minval = s->sw_min; A.g = s->sw_g; A.pcount = s->pcount; A.poff = s->poff; A.ptotal = s->ptotal;
  A.prow = s->prow; A.ppos = s->ppos; A.pd = s->pd; A.ptold = s->G > 1 ? s->ptold : nullptr; A.pdelta = s->pdelta;
  A.rowcnt = s->rowcnt; A.rowidx = s->rowidx; A.trows = s->trows; A.ntouch = s->ntouch; A.X = s->X;
  A.tstart = s->tstart; A.tcur = s->tcur; A.runc = s->runc; A.runv = s->runv; A.bigw = s->bigw; A.nbig = s->nbig;
  A.scal = s->scal; A.eps = stop_check ? s->epsd : nullptr; A.stop = stop_check ? s->stop : nullptr;
  A.status = s->status;
  A.step_rule = step_rule; A.kk = cur ? kbase : s->lead->k + s->lead->k_pending; A.nprime = nprime; A.trace = trace_dev;
  A.cur = cur;
  A.trace_col0_mul = col0_mul * s->G;
  A.dsteps = s->dsteps;
  A.G = s->G; A.shard = s->shard; A.slot_len = s->lead->slot_len; A.x1 = s->lead->x1; A.x2 = s->lead->x2;
  A.capfail = s->G > 1 ? s->capfail : nullptr;
  A.phase = s->phase;
  return A;
}

// One plain step over [col0, col0+L). For FW (stop_check) the gap G_[n] is
// checked against epsilon before the update (Alg. A.1 line 4). Small U: the
// LMO sweep plus one single-CTA launch for the rest of the step; large U: one
// kernel per phase.
// Cursor mode (cur != nullptr): col0_dev, trace_dev and kbase are the solve call's bases and the
// step reads its block index, iteration and trace slot at *cur (advanced by the step's last
// kernel), so consecutive steps are identical launches (capturable in one CUDA graph).
sro_status plain_block_step(Solver* s, const int* col0_dev, int col0_mul, int L, int step_rule, long long nprime,
                            bool stop_check, double* trace_dev, unsigned* cur = nullptr, long long kbase = 0) {
  sro_status st = ensure_block_ws(s, L);
  if (st) return st;
  const int trb = timed_begin(s);
  int* stop = stop_check ? s->stop : nullptr;
  const bool smtail = L <= 1024 && !s->no_tail && !s->no_smtail && s->m < (1 << 20) - 1;
  if (smtail && !s->st_cnt) {
    CUDA_TRY(s, salloc(&s->st_cnt, 1024, s->stream));
    CUDA_TRY(s, salloc(&s->st_row, 1024 * SW_KP, s->stream));
    CUDA_TRY(s, salloc(&s->st_val, 1024 * SW_KP, s->stream));
    CUDA_TRY(s, salloc(&s->st_b, 1024, s->stream));
    CUDA_TRY(s, salloc(&s->st_term, 1024 * SW_KP, s->stream));
  }
  s->defer_merge = smtail;
  s->sweep_cur = cur;
  st = sweep(s, col0_dev, col0_mul, 0, L, s->sw_j, s->sw_min, s->sw_g, stop);
  s->defer_merge = false;
  s->sweep_cur = nullptr;
  if (st) return st;
  BlockArgs A = block_args(s, col0_dev, col0_mul, L, step_rule, nprime, stop_check, trace_dev, cur, kbase);
  if (smtail) {
    // pairs resident in shared memory (k_block_tail.cuh); the sweep's slab merge folded in
    TailMerge M{};
    M.nslabs = s->last_nslabs; M.pj = s->part_j; M.pmin = s->part_min;
    M.st_cnt = s->st_cnt; M.st_row = s->st_row; M.st_val = s->st_val; M.st_b = s->st_b; M.st_term = s->st_term;
    M.j = s->sw_j; M.minval = s->sw_min; M.g = s->sw_g;
    const bool dense = s->kind == SRO_COST_DENSE || s->kind == SRO_COST_HASH_UNIFORM;
    const bool f32 = s->prec == SRO_FP32, eu = s->kind == SRO_COST_EUCLID;
    M.kind = dense ? (f32 ? 0 : 1) : (f32 ? (eu ? 3 : 2) : (eu ? 5 : 4));
    M.C = s->C; M.ld = s->ld; M.x = s->x; M.y = s->y;
    CUDA_TRY(s, set_dyn_smem((const void*)k_block_tail_sm, s->device, (int)TAIL_SM_BYTES));
    CUDA_TRY(s, launch_pdl(k_block_tail_sm, dim3(1), dim3(1024), TAIL_SM_BYTES, s->stream, A, M));
    CUDA_TRY(s, cudaGetLastError());
    s->lead->stats.kernel_launches += 1;
  } else if (L <= 1024 && !s->no_tail) {
    CUDA_TRY(s, set_dyn_smem((const void*)k_block_tail, s->device, TAIL_SMEM));
    CUDA_TRY(s, launch_pdl(k_block_tail, dim3(1), dim3(1024), TAIL_SMEM, s->stream, A));
    CUDA_TRY(s, cudaGetLastError());
    s->lead->stats.kernel_launches += 1;
  } else if (!s->no_coop) {
    // all phases in one cooperative launch (k_block_coop): every CTA resident, grid barriers
    const size_t cs = (size_t)32 * 256 * sizeof(double);
    CUDA_TRY(s, set_dyn_smem((const void*)k_block_coop, s->device, (int)cs));
    int per_sm = 0;
    CUDA_TRY(s, occupancy((const void*)k_block_coop, s->device, 1024, cs, &per_sm));
    if (per_sm < 1) per_sm = 1;
    void* args[] = {(void*)&A};
    CUDA_TRY(s, cudaLaunchCooperativeKernel((const void*)k_block_coop, dim3(s->num_sms * per_sm), dim3(1024), args, cs,
                                            s->stream));
    s->lead->stats.kernel_launches += 1;
  } else {
    const int tpb = 256;
    int gL = (L + tpb / 32 - 1) / (tpb / 32); if (gL > s->num_sms * 8) gL = s->num_sms * 8;   // warp per column
    const int gP = s->num_sms * 8;
    const int gR = (s->m + 7) / 8 < s->num_sms * 8 ? (s->m + 7) / 8 : s->num_sms * 8;
    // k_pairs_count first (it needs nothing from the step start), then G_U / stop check / resets and
    // the pair scan in one single-CTA launch; the denominator and gamma in one launch
    CUDA_TRY(s, launch_pdl(k_pairs_count, dim3(gL), dim3(tpb), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_begin_scan, dim3(1), dim3(1024), 0, s->stream, A, s->scal + 0));
    CUDA_TRY(s, launch_pdl(k_pairs_gen, dim3(gL), dim3(tpb), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_touched_scan, dim3(1), dim3(1024), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_runs, dim3(A.W), dim3(tpb), 0, s->stream, A, s->pd));
    CUDA_TRY(s, launch_pdl(k_row_tree_all<0>, dim3(gR), dim3(256), 0, s->stream, A, nullptr, 0, (unsigned*)nullptr));
    CUDA_TRY(s, launch_pdl(k_den_gamma, dim3(1), dim3(256), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_cap_check, dim3(gL), dim3(tpb), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_update_cols, dim3(gL), dim3(tpb), 0, s->stream, A));
    CUDA_TRY(s, launch_pdl(k_runs, dim3(A.W), dim3(tpb), 0, s->stream, A, s->pdelta));
    if (!s->done_ticket) {
      CUDA_TRY(s, salloc(&s->done_ticket, 1, s->stream));
      CUDA_TRY(s, cudaMemsetAsync(s->done_ticket, 0, sizeof(unsigned), s->stream));
    }
    CUDA_TRY(s, launch_pdl(k_row_tree_all<1>, dim3(gR), dim3(256), 0, s->stream, A, nullptr, 1, s->done_ticket));   // + the step count and cursor advance
    CUDA_TRY(s, cudaGetLastError());
    s->lead->stats.kernel_launches += 11;
  }
  s->lead->stats.block_steps += 1;
  s->lead->k_pending += 1;
  timed_end(s, trb, CAT_BLOCK, L);
  return SRO_OK;
}

// The same step over G column shards: U's positions split in
// G contiguous ranges (local [col0, col0 + L) of every shard, L = |U| / G).
// Phase A per shard (LMO sweep, G_U subtree, Delta subtrees) -> exchange x1
// -> phase B per shard (combine, gamma, capacity check, update, Delta'
// subtrees) -> exchange x2 -> apply per shard (combine, r and h).
sro_status shard_block_step(Solver* s, const int* col0_dev, int col0_mul, int L, int step_rule, long long nprime,
                            bool stop_check, double* trace_dev) {
  auto H = held(s);
  for (Solver* t : H) { sro_status st = ensure_block_ws(t, L); if (st) return st; }
  const int trb = timed_begin(s);
  const bool tail = L <= 1024 && !s->no_tail;
  const int tpb = 256;
  int gL = (L + tpb / 32 - 1) / (tpb / 32); if (gL > s->num_sms * 8) gL = s->num_sms * 8;   // warp per column
  const int gP = s->num_sms * 8;
  const int gR = (s->m + 7) / 8 < s->num_sms * 8 ? (s->m + 7) / 8 : s->num_sms * 8;
  std::vector<BlockArgs> AA;
  for (Solver* t : H)
    AA.push_back(block_args(t, col0_dev, col0_mul, L, step_rule, nprime, stop_check,
                            t->shard == 0 ? trace_dev : nullptr));
  // phase A
  for (size_t q = 0; q < H.size(); q++) {
    Solver* t = H[q];
    BlockArgs& A = AA[q];
    sro_status st = sweep(t, col0_dev, col0_mul, 0, L, t->sw_j, t->sw_min, t->sw_g, stop_check ? t->stop : nullptr);
    if (st) return st;
    double* s1 = s->x1 + (size_t)t->shard * s->slot_len;
    if (tail) {
      CUDA_TRY(s, set_dyn_smem((const void*)k_shard_tail_a, s->device, TAIL_SMEM));
      k_shard_tail_a<<<1, 1024, TAIL_SMEM, s->stream>>>(A);
      s->stats.kernel_launches += 1;
    } else {
      k_step_begin<<<1, 256, 0, s->stream>>>(A, s1 + s->m);
      k_pairs_count<<<gL, tpb, 0, s->stream>>>(A);
      k_scan_pairs<<<1, 1024, 0, s->stream>>>(A);
      k_zero_slot<<<gR, 256, 0, s->stream>>>(A, s1);
      k_pairs_gen<<<gL, tpb, 0, s->stream>>>(A);
      k_touched_scan<<<1, 1024, 0, s->stream>>>(A);
      k_runs<<<A.W, tpb, 0, s->stream>>>(A, t->pd);
      k_row_tree_all<2><<<gR, 256, 0, s->stream>>>(A, s1, 0, nullptr);
      k_publish_a<<<1, 32, 0, s->stream>>>(A);
      s->stats.kernel_launches += 9;
    }
    CUDA_TRY(s, cudaGetLastError());
  }
  { sro_status st = exchange(s, s->x1, s->slot_len); if (st) return st; }
  // phase B
  for (size_t q = 0; q < H.size(); q++) {
    Solver* t = H[q];
    BlockArgs& A = AA[q];
    double* s2 = s->x2 + (size_t)t->shard * s->slot_len;
    if (tail) {
      CUDA_TRY(s, set_dyn_smem((const void*)k_shard_tail_b, s->device, TAIL_SMEM));
      k_shard_tail_b<<<1, 1024, TAIL_SMEM, s->stream>>>(A);
      s->stats.kernel_launches += 1;
    } else {
      k_shard_gamma<<<1, 256, 0, s->stream>>>(A);
      k_cap_check<<<gL, tpb, 0, s->stream>>>(A);
      k_zero_slot<<<gR, 256, 0, s->stream>>>(A, s2);
      k_update_cols<<<gL, tpb, 0, s->stream>>>(A);
      k_runs<<<A.W, tpb, 0, s->stream>>>(A, t->pdelta);
      k_row_tree_all<2><<<gR, 256, 0, s->stream>>>(A, s2, 1, nullptr);
      k_publish_b<<<1, 32, 0, s->stream>>>(A);
      s->stats.kernel_launches += 7;
    }
    CUDA_TRY(s, cudaGetLastError());
  }
  { sro_status st = exchange(s, s->x2, s->slot_len); if (st) return st; }
  // apply
  const int gA = std::max(gL, gR);
  for (size_t q = 0; q < H.size(); q++) {
    k_shard_apply<<<gA, tpb, 0, s->stream>>>(AA[q]);
    s->stats.kernel_launches += 1;
  }
  CUDA_TRY(s, cudaGetLastError());
  s->stats.block_steps += 1;
  s->k_pending += 1;
  timed_end(s, trb, CAT_BLOCK, L * (int64_t)H.size());
  return SRO_OK;
}

// Sync point for asynchronously enqueued block steps: read how many completed
// (a skipped step — FW stop or an error — does not count), advance k, and
// report a device error.
sro_status drain_block_steps(Solver* s, int64_t* done) {
  unsigned long long ds = 0;
  CUDA_TRY(s, rb(s, &ds, s->dsteps, sizeof(ds)));
  sro_status st = check_status(s);   // synchronises
  resolve_timing(s);
  for (Solver* t : held(s)) CUDA_TRY(s, cudaMemsetAsync(t->dsteps, 0, sizeof(unsigned long long), s->stream));
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

// f(T) = psum256_i lin_i + psum256_k (r_k - a_k)^2 / (2 lambda) (Eq. 7). Sharded:
// lin of the held columns goes to the shards' gx slots, which are exchanged.
sro_status objective_dev(Solver* s, double* f_host) {
  for (Solver* t : held(s)) {
    double* out = s->G == 1 ? t->sw_g : s->gx + (size_t)t->shard * t->n;
    sro_status st = with_sweep_src(t, [&](auto src) -> sro_status {
      k_lin<<<(t->n + 255) / 256, 256, 0, s->stream>>>(src, t->cnt, t->srow, t->sval, t->cap, t->n, out);
      CUDA_TRY(s, cudaGetLastError());
      return SRO_OK;
    });
    if (st) return st;
  }
  if (s->G == 1) {
    k_psum256<<<1, 256, 0, s->stream>>>(s->sw_g, s->n, s->scal + 4, nullptr, nullptr, nullptr);
  } else {
    sro_status st = exchange(s, s->gx, s->n);
    if (st) return st;
    k_psum256_gathered<<<1, 256, 0, s->stream>>>(s->gx, s->n_glob, s->Bo, s->Bl, s->n, s->scal + 4, nullptr);
  }
  k_pen<<<(s->m + 255) / 256, 256, 0, s->stream>>>(s->r, s->a, s->m, s->sw_min);
  k_psum256<<<1, 256, 0, s->stream>>>(s->sw_min, s->m, s->scal + 5, nullptr, nullptr, nullptr);
  k_objective_final<<<1, 1, 0, s->stream>>>(s->scal + 4, s->scal + 5, s->lambda, s->scal + 7);
  s->lead->stats.kernel_launches += 4 + (int64_t)held(s).size();
  CUDA_TRY(s, cudaGetLastError());
  CUDA_TRY(s, rb(s, f_host, s->scal + 7, sizeof(double)));
  CUDA_TRY(s, stream_wait(s));
  return SRO_OK;
}

sro_status do_reset(Solver* s) {
  for (Solver* t : held(s)) {
    { sro_status e = ws_clean(t); if (e) return e; }
    k_init_plan<<<s->num_sms, 256, 0, s->stream>>>(t->b, t->b_full, t->n_glob, t->a, t->r, t->h, t->cnt, t->srow,
                                                  t->sval, t->m, t->n, t->cap, t->lambda);
    s->lead->stats.kernel_launches += 1;
    CUDA_TRY(s, cudaGetLastError());
    CUDA_TRY(s, cudaMemsetAsync(t->stop, 0, sizeof(int), s->stream));
  }
  s->k = 0;
  s->configured = false;
  return SRO_OK;
}

void free_shard(Solver* s) {
  if (!s) return;
  // stream-ordered workspaces (salloc) go back to the pool on the stream; the rest with cudaFree
  // (the handle state too: stream-ordered from the retained pool, so creating and destroying
  // handles neither maps new memory nor synchronises the device)
  void* aptrs[] = {s->visit, s->trace, s->part_j, s->part_min, s->pcount, s->poff, s->ptotal, s->prow, s->ppos, s->pd,
                   s->ptold, s->pdelta, s->runc, s->runv, s->rowcnt, s->rowidx, s->tstart, s->tcur, s->X,
                   s->trows, s->ntouch, s->capfail, s->bigw, s->nbig, s->st_cnt, s->st_row, s->st_val, s->st_b, s->st_term,
                   s->done_ticket, s->ga_blk, s->dsteps, s->cur, s->phase, s->a, s->b, s->b_full, s->r, s->h, s->cnt, s->srow, s->sval, s->G_ga,
                   s->fen, s->status, s->steps_done, s->stop, s->scal, s->epsd, s->sw_j, s->sw_min, s->sw_g};
  if (s->stream) for (void* p : aptrs) sfree(p, s->stream);
  if (s->stream) stream_wait(s);
  if (s->gexec) cudaGraphExecDestroy(s->gexec);
  if (s->owns_cost) { if (s->C) cudaFree(s->C); if (s->x) cudaFree(s->x); if (s->y) cudaFree(s->y); }
  for (auto& p : s->pending) { s->ev_pool.push_back(p.a); s->ev_pool.push_back(p.b); }
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev_sync) cudaEventDestroy(s->ev_sync);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

void free_solver(Solver* s) {
  if (!s) return;
  if (s->pin) cudaFreeHost(s->pin);
  s->pin = nullptr;
  if (s->pin_ep) cudaFreeHost(s->pin_ep);
  s->pin_ep = nullptr;
  for (auto& e : s->ev_ep) if (e) { cudaEventDestroy(e); e = nullptr; }
  for (Solver* p : s->peers) free_shard(p);
  s->peers.clear();
  if (s->x1) cudaFree(s->x1);
  if (s->x2) cudaFree(s->x2);
  if (s->gx) cudaFree(s->gx);
  if (s->comm) nccl().destroy(s->comm);
  if (s->xhost) cudaFreeHost(s->xhost);
  free_shard(s);
}

// One shard's device state. b_loc: host fp64[n_loc] (its columns' weights);
// b_all: host fp64[n_glob]; the cost arguments describe its columns only.
// Cost pointers: dense `data` (column-major, cost_ld), colours x (m x 3) and
// y (n_loc x 3), each host (copied) or device (borrowed) per on_dev.
sro_status build_shard(Solver* s, const double* a, const double* b_loc, const double* b_all, const sro_cost* cost,
                       const void* data, int64_t cost_ld, const void* y, bool on_dev) {
  const int m = s->m, n = s->n;
  cudaEventCreate(&s->ev0); cudaEventCreate(&s->ev1);
#define ALLOC(ptr, cnt_)                                                              \
  if (salloc(&(ptr), (cnt_), s->stream) != cudaSuccess) { s->err = "device allocation failed"; return SRO_ERR_OOM; }
  ALLOC(s->a, m); ALLOC(s->b, n); ALLOC(s->b_full, s->n_glob + 1); ALLOC(s->r, m); ALLOC(s->h, m);
  ALLOC(s->cnt, n); ALLOC(s->srow, (size_t)n * s->cap); ALLOC(s->sval, (size_t)n * s->cap);
  if (s->G == 1) { ALLOC(s->G_ga, n); ALLOC(s->fen, (size_t)n + 1); }
  else if (s->lead == s) { ALLOC(s->G_ga, s->n_glob); ALLOC(s->fen, (size_t)s->n_glob + 1); }   // GA block sampling
  ALLOC(s->phase, 32);
  ALLOC(s->dsteps, 1);
  ALLOC(s->cur, 1);
  ALLOC(s->status, 1); ALLOC(s->steps_done, 1); ALLOC(s->stop, 1); ALLOC(s->scal, 8); ALLOC(s->epsd, 1);
  ALLOC(s->sw_j, n); ALLOC(s->sw_min, (size_t)(m > n ? m : n)); ALLOC(s->sw_g, (size_t)(m > n ? m : n));
#undef ALLOC
  cudaMemsetAsync(s->dsteps, 0, sizeof(unsigned long long), s->stream);
  cudaMemsetAsync(s->phase, 0, 32 * sizeof(long long), s->stream);
  cudaMemsetAsync(s->status, 0, sizeof(int), s->stream);
  cudaMemcpyAsync(s->a, a, sizeof(double) * m, cudaMemcpyHostToDevice, s->stream);
  cudaMemcpyAsync(s->b, b_loc, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream);
  cudaMemcpyAsync(s->b_full, b_all, sizeof(double) * s->n_glob, cudaMemcpyHostToDevice, s->stream);
  k_r0<<<1, 1, 0, s->stream>>>(s->b_full, s->n_glob);
  const size_t esz = s->prec == SRO_FP32 ? 4 : 8;
  const int vec = 16 / (int)esz;
  if (s->kind == SRO_COST_DENSE) {
    if (on_dev) {
      s->C = const_cast<void*>(data); s->ld = cost_ld;
    } else {
      s->ld = ((int64_t)m + vec - 1) / vec * vec;
      if (cudaMalloc(&s->C, esz * (size_t)s->ld * n) != cudaSuccess) { s->err = "cost allocation failed"; return SRO_ERR_OOM; }
      s->owns_cost = true;
      if (cudaMemcpy2DAsync(s->C, esz * s->ld, data, esz * cost_ld, esz * m, n, cudaMemcpyHostToDevice, s->stream) != cudaSuccess)
        { s->err = "cost upload failed"; return SRO_ERR_CUDA; }
    }
    if (s->prec == SRO_FP32) k_check_dense<float><<<s->num_sms * 4, 256, 0, s->stream>>>((const float*)s->C, s->ld, m, n, s->status);
    else k_check_dense<double><<<s->num_sms * 4, 256, 0, s->stream>>>((const double*)s->C, s->ld, m, n, s->status);
  } else if (s->kind == SRO_COST_HASH_UNIFORM) {
    s->ld = ((int64_t)m + 3) / 4 * 4;
    if (cudaMalloc(&s->C, 4 * (size_t)s->ld * n) != cudaSuccess) { s->err = "cost allocation failed"; return SRO_ERR_OOM; }
    s->owns_cost = true;
    k_gen_hash<<<s->num_sms * 8, 256, 0, s->stream>>>((float*)s->C, s->ld, m, n, cost->hash_seed, s->Bo, s->Bl, s->shard);
  } else {
    if (on_dev) { s->x = const_cast<void*>(cost->x); s->y = const_cast<void*>(y); }
    else {
      if (cudaMalloc(&s->x, esz * 3 * (size_t)m) != cudaSuccess || cudaMalloc(&s->y, esz * 3 * (size_t)n) != cudaSuccess)
        { s->err = "colour allocation failed"; return SRO_ERR_OOM; }
      s->owns_cost = true;
      cudaMemcpyAsync(s->x, cost->x, esz * 3 * (size_t)m, cudaMemcpyHostToDevice, s->stream);
      cudaMemcpyAsync(s->y, y, esz * 3 * (size_t)n, cudaMemcpyHostToDevice, s->stream);
    }
    if (s->prec == SRO_FP32) {
      k_check_finite<float><<<64, 256, 0, s->stream>>>((const float*)s->x, 3LL * m, s->status);
      k_check_finite<float><<<64, 256, 0, s->stream>>>((const float*)s->y, 3LL * n, s->status);
    } else {
      k_check_finite<double><<<64, 256, 0, s->stream>>>((const double*)s->x, 3LL * m, s->status);
      k_check_finite<double><<<64, 256, 0, s->stream>>>((const double*)s->y, 3LL * n, s->status);
    }
  }
  if (cudaGetLastError() != cudaSuccess) { s->err = "kernel launch failed at create"; return SRO_ERR_CUDA; }
  int st = 0;
  cudaMemcpyAsync(&st, s->status, sizeof(int), cudaMemcpyDeviceToHost, s->stream);
  if (stream_wait(s) != cudaSuccess) { s->err = "create failed"; return SRO_ERR_CUDA; }
  if (st) { s->err = "cost must be finite and >= 0"; return SRO_ERR_NONFINITE; }
  return SRO_OK;
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
  // marginals (Eq. 8): finite, a >= 0, b >= 0 (zero-mass columns: R32), each summing to 1 within 1e-12
  double sa = 0.0, sb = 0.0;
  for (int k = 0; k < p->m; k++) { if (!(a[k] >= 0.0) || !std::isfinite(a[k])) { g_create_err = "a must be finite and >= 0"; return SRO_ERR_MARGINALS; } sa += a[k]; }
  for (int i = 0; i < p->n; i++) { if (!(b[i] >= 0.0) || !std::isfinite(b[i])) { g_create_err = "b must be finite and >= 0"; return SRO_ERR_MARGINALS; } sb += b[i]; }
  if (std::fabs(sa - 1.0) > 1e-12 || std::fabs(sb - 1.0) > 1e-12) { g_create_err = "marginals must sum to 1 within 1e-12"; return SRO_ERR_MARGINALS; }
  // sharding
  const int G = p->shards <= 1 ? 1 : p->shards;
  const int Bo = (G == 1 || p->shard_block == 0) ? p->n : p->shard_block;
  const int nranks = p->nranks <= 1 ? 1 : p->nranks;
  if (G > 1) {
    if (G > 64 || (G & (G - 1))) { g_create_err = "shards must be a power of two <= 64"; return SRO_ERR_INVALID_ARG; }
    if (Bo < 1 || p->n % Bo != 0 || Bo % G != 0) { g_create_err = "shard_block must divide n and be a multiple of shards"; return SRO_ERR_INVALID_ARG; }
    if (nranks != 1 && nranks != G) { g_create_err = "nranks must be 1 or shards"; return SRO_ERR_INVALID_ARG; }
    if (nranks > 1 && (p->rank < 0 || p->rank >= G || (!p->nccl_id && !p->exchange))) { g_create_err = "nranks > 1 needs rank in [0, shards) and nccl_id or exchange"; return SRO_ERR_INVALID_ARG; }
    if (nranks == 1 && cost->data_on_device && cost->kind != SRO_COST_HASH_UNIFORM && Bo != p->n) {
      g_create_err = "borrowed device cost with nranks == 1 needs shard_block == n"; return SRO_ERR_INVALID_ARG;
    }
  } else if (nranks != 1) { g_create_err = "nranks > 1 needs shards > 1"; return SRO_ERR_INVALID_ARG; }
  const int nl = p->n / G, Bl = Bo / G;
  const int kind = cost->kind, prec = kind == SRO_COST_HASH_UNIFORM ? (int)SRO_FP32 : cost->prec;
  const size_t esz = prec == SRO_FP32 ? 4 : 8;
  if (kind == SRO_COST_DENSE) {
    if (!cost->data || cost->ld < p->m) { g_create_err = "dense cost needs data and ld >= m"; return SRO_ERR_INVALID_ARG; }
    if (cost->data_on_device && (((uintptr_t)cost->data % 16) != 0 || (cost->ld * (int64_t)esz) % 16 != 0)) {
      g_create_err = "borrowed dense cost must be 16-byte aligned with ld*elem % 16 == 0"; return SRO_ERR_INVALID_ARG;
    }
  } else if (kind != SRO_COST_HASH_UNIFORM && (!cost->x || !cost->y)) {
    g_create_err = "colour cost needs x and y"; return SRO_ERR_INVALID_ARG;
  }

  Solver* s = new Solver();
  auto fail = [&](sro_status st, const std::string& msg) { g_create_err = msg.empty() ? s->err : msg; free_solver(s); return st; };
  if (cudaSetDevice(p->device) != cudaSuccess) return fail(SRO_ERR_CUDA, "cudaSetDevice failed (no CUDA device?)");
  int num_sms = 148;
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, p->device);
  if (p->max_sms < 0) return fail(SRO_ERR_INVALID_ARG, "max_sms must be >= 0");
  if (p->max_sms > 0 && p->max_sms < num_sms) num_sms = p->max_sms;
  if (p->cuda_stream) s->stream = (cudaStream_t)p->cuda_stream;
  else { if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(SRO_ERR_CUDA, "stream"); s->own_stream = true; }
  std::vector<int> shards_held;
  if (nranks == 1) for (int q = 0; q < G; q++) shards_held.push_back(q);
  else shards_held.push_back(p->rank);
  for (size_t hq = 0; hq < shards_held.size(); hq++) {
    Solver* t = hq == 0 ? s : new Solver();
    if (hq > 0) { t->stream = s->stream; s->peers.push_back(t); }
    t->lead = s;
    t->m = p->m; t->n = nl; t->cap = cap; t->lambda = p->lambda; t->device = p->device; t->num_sms = num_sms;
    t->kind = kind; t->prec = prec; t->borrowed = cost->data_on_device;
    t->G = G; t->shard = shards_held[hq]; t->nranks = nranks; t->n_glob = p->n; t->Bo = Bo; t->Bl = Bl;
    // this shard's columns: weights, cost data
    std::vector<double> b_loc(nl);
    for (int q = 0; q < nl; q++) b_loc[q] = b[global_col(t, q)];
    const bool gather = G > 1 && nranks == 1;   // inputs cover all n columns: pick this shard's
    const void* data = cost->data;
    int64_t cld = cost->ld;
    const void* y = cost->y;
    std::vector<unsigned char> hdata, hy;
    if (gather && kind == SRO_COST_DENSE) {
      if (cost->data_on_device) data = (const char*)cost->data + esz * (size_t)cost->ld * (size_t)t->shard * Bl;
      else {
        hdata.resize(esz * (size_t)p->m * nl);
        for (int q = 0; q < nl; q++)
          memcpy(&hdata[esz * (size_t)p->m * q], (const char*)cost->data + esz * (size_t)cost->ld * global_col(t, q),
                 esz * p->m);
        data = hdata.data(); cld = p->m;
      }
    }
    if (gather && (kind == SRO_COST_SQEUCLID || kind == SRO_COST_EUCLID)) {
      if (cost->data_on_device) y = (const char*)cost->y + esz * 3 * (size_t)t->shard * Bl;
      else {
        hy.resize(esz * 3 * (size_t)nl);
        for (int q = 0; q < nl; q++) memcpy(&hy[esz * 3 * q], (const char*)cost->y + esz * 3 * (size_t)global_col(t, q), esz * 3);
        y = hy.data();
      }
    }
    sro_status st = build_shard(t, a, b_loc.data(), b, cost, data, cld, y, cost->data_on_device != 0);
    if (st) return fail(st, t->err);
  }
  if (G > 1) {
    s->slot_len = p->m + 8;
    if (dalloc(&s->x1, (size_t)G * s->slot_len) != cudaSuccess || dalloc(&s->x2, (size_t)G * s->slot_len) != cudaSuccess ||
        dalloc(&s->gx, (size_t)p->n) != cudaSuccess)
      return fail(SRO_ERR_OOM, "device allocation failed");
    cudaMemsetAsync(s->x1, 0, sizeof(double) * G * s->slot_len, s->stream);
    cudaMemsetAsync(s->x2, 0, sizeof(double) * G * s->slot_len, s->stream);
    if (nranks > 1 && p->exchange) {
      s->xfn = p->exchange;
      s->xuser = p->exchange_user;
    } else if (nranks > 1) {
      NcclApi& api = nccl();
      if (!api.ok) return fail(SRO_ERR_NCCL, api.err);
      ncclUniqueId id;
      memcpy(&id, p->nccl_id, sizeof(id));
      ncclResult_t r = api.init(&s->comm, nranks, id, p->rank);
      if (r != ncclSuccess) { s->comm = nullptr; return fail(SRO_ERR_NCCL, std::string("ncclCommInitRank: ") + api.errstr(r)); }
    }
  }
  if (do_reset(s) != SRO_OK) return fail(SRO_ERR_CUDA, "");
  if (stream_wait(s) != cudaSuccess) return fail(SRO_ERR_CUDA, "init failed");
  *out = static_cast<sro_handle>(static_cast<sro_solver*>(s));
  return SRO_OK;
}

void sro_destroy(sro_handle h) {
  if (!h) return;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  stream_wait(s);
  free_solver(s);
}

sro_status sro_reset(sro_handle h) {
  if (!h) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  sro_status st = do_reset(s);
  if (st) return st;
  CUDA_TRY(s, stream_wait(s));
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
  if (o->sampling == SRO_SAMPLE_GA && variant == SRO_FW) { s->err = "GA sampling needs a BCFW-family or batched variant"; return SRO_ERR_INVALID_ARG; }
  if (o->sampling == SRO_SAMPLE_GA && o->ga_M < 1) { s->err = "ga_M must be >= 1"; return SRO_ERR_INVALID_ARG; }
  if (o->sampling < 0 || o->sampling > 2 || o->step < 0 || o->step > 1) { s->err = "bad sampling/step"; return SRO_ERR_INVALID_ARG; }
  const int n = s->n_glob;                                   // all columns
  const int64_t n_held = (int64_t)s->n * (int64_t)held(s).size();   // columns this process sweeps
  if (s->G > 1) {
    if (variant != SRO_FW && variant != SRO_BATCHED) { s->err = "a sharded handle runs FW and BATCHED only (the sequential BCFW family does not shard)"; return SRO_ERR_INVALID_ARG; }
    if (variant == SRO_FW && s->Bo != n) { s->err = "sharded FW needs shard_block == n"; return SRO_ERR_INVALID_ARG; }
    if (variant == SRO_BATCHED && o->block_size != s->Bo) { s->err = "sharded BATCHED needs block_size == shard_block"; return SRO_ERR_INVALID_ARG; }
  }
  long long nprime;
  if (variant == SRO_FW) nprime = 1;
  else if (variant == SRO_BATCHED) {
    if (o->block_size < 1 || n % o->block_size != 0) { s->err = "block_size must divide n"; return SRO_ERR_INVALID_ARG; }
    nprime = n / o->block_size;
  } else nprime = n;
  auto block_step = [&](const int* col0_dev, int B, bool stop_check, double* tr) -> sro_status {
    if (s->G == 1) return plain_block_step(s, col0_dev, B, B, o->step, nprime, stop_check, tr);
    return shard_block_step(s, col0_dev, B / s->G, B / s->G, o->step, nprime, stop_check, tr);
  };
  // Unsharded FW / batched: cursor-mode steps (every step the same launches, reading its block
  // index, iteration and trace slot at the device cursor = steps enqueued in this call), replayed
  // from one CUDA graph of GRAPH_STEPS steps captured at the first segment (timing off).
  const long long kbase = s->k;
  const bool cursor_mode = s->G == 1 && (variant == SRO_FW || variant == SRO_BATCHED);
  if (cursor_mode) CUDA_TRY(s, cudaMemsetAsync(s->cur, 0, sizeof(unsigned), s->stream));
  if (s->gexec) { cudaGraphExecDestroy(s->gexec); s->gexec = nullptr; s->gexec_steps = 0; }
  const bool use_graph = cursor_mode && !s->timing && !getenv("SRO_NO_GRAPH");
  sro_stats gdelta{};
  long long gdelta_k = 0;
  auto run_steps = [&](int64_t count, int graph_steps, auto&& one) -> sro_status {
    int64_t q = 0;
    if (use_graph && count >= graph_steps + 1) {
      if (!s->gexec) {
        sro_status st1 = one();   // uncaptured: workspaces reach their size here
        if (st1) return st1;
        q++;
        const sro_stats st0 = s->stats;
        const long long kp0 = s->k_pending;
        cudaGraph_t g = nullptr;
        CUDA_TRY(s, cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
        sro_status cst = SRO_OK;
        for (int k = 0; k < graph_steps && cst == SRO_OK; k++) cst = one();
        const cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
        gdelta.kernel_launches = s->stats.kernel_launches - st0.kernel_launches;
        gdelta.sweep_launches = s->stats.sweep_launches - st0.sweep_launches;
        gdelta.sweep_columns = s->stats.sweep_columns - st0.sweep_columns;
        gdelta.block_steps = s->stats.block_steps - st0.block_steps;
        gdelta_k = s->k_pending - kp0;
        s->stats = st0;
        s->k_pending = kp0;
        if (cst != SRO_OK || ce != cudaSuccess) {
          if (g) cudaGraphDestroy(g);
          if (cst != SRO_OK) return cst;
          s->err = cudaGetErrorString(ce);
          return SRO_ERR_CUDA;
        }
        const cudaError_t ie = cudaGraphInstantiate(&s->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) { s->gexec = nullptr; s->err = cudaGetErrorString(ie); return SRO_ERR_CUDA; }
        s->gexec_steps = graph_steps;
      }
      while (count - q >= s->gexec_steps) {
        CUDA_TRY(s, cudaGraphLaunch(s->gexec, s->stream));
        s->stats.kernel_launches += gdelta.kernel_launches;
        s->stats.sweep_launches += gdelta.sweep_launches;
        s->stats.sweep_columns += gdelta.sweep_columns;
        s->stats.block_steps += gdelta.block_steps;
        s->k_pending += gdelta_k;
        q += s->gexec_steps;
      }
    }
    for (; q < count; q++) {
      sro_status st1 = one();
      if (st1) return st1;
    }
    return SRO_OK;
  };
  if (s->configured) {
    if (s->variant != variant || s->seed != seed || !options_equal(s->opt, *o)) { s->err = "solver configured differently; call sro_reset"; return SRO_ERR_STATE; }
  }
  const bool ga = o->sampling == SRO_SAMPLE_GA && variant != SRO_FW;
  sro_status st = SRO_OK;
  CUDA_TRY(s, cudaEventRecord(s->ev0, s->stream));
  if (!s->configured) {
    s->configured = true; s->variant = variant; s->opt = *o; s->seed = seed;
    s->opt.visit = nullptr; s->opt.trace = nullptr;
    if (ga) { st = s->G > 1 ? ga_initialise_sharded(s) : ga_initialise(s); if (st) return st; }
  }
  for (Solver* t : held(s)) CUDA_TRY(s, cudaMemcpyAsync(t->epsd, &o->epsilon, sizeof(double), cudaMemcpyHostToDevice, s->stream));
  const int m = s->m;
  int64_t done = 0;
  const long long period = (long long)o->gap_period * nprime;
  std::vector<int> hv;
  std::vector<double> htr;
  if (o->trace) { st = ensure_trace(s, iters > 0 ? iters : 1); if (st) return st; }

  if (variant == SRO_FW) {
    for (Solver* t : held(s)) CUDA_TRY(s, cudaMemsetAsync(t->stop, 0, sizeof(int), s->stream));
    while (done < iters) {
      const int64_t chunk = (iters - done) < 8 ? (iters - done) : 8;
      if (cursor_mode) {
        st = run_steps(chunk, 7, [&]() {
          return plain_block_step(s, nullptr, n, n, o->step, nprime, true, o->trace ? s->trace : nullptr, s->cur, kbase);
        });
        if (st) return st;
      } else {
        for (int64_t q = 0; q < chunk; q++) {
          st = block_step(nullptr, n, true, o->trace ? s->trace + 9 * (done + q) : nullptr);
          if (st) return st;
        }
      }
      const int64_t before = done;
      double G = 0.0;
      int stopped = 0;
      CUDA_TRY(s, rb(s, &G, s->scal + 0, sizeof(double)));
      CUDA_TRY(s, rb(s, &stopped, s->stop, sizeof(int)));
      st = drain_block_steps(s, &done);
      if (st) return st;
      out->gap = G;
      out->gap_checks += (int)(done - before) + (stopped ? 1 : 0);
      out->entries_scanned += (int64_t)m * n_held * ((done - before) + (stopped ? 1 : 0));
      out->entries_read += (int64_t)m * n_held * ((done - before) + (stopped ? 1 : 0));
      if (stopped) { out->converged = 1; break; }
    }
    for (Solver* t : held(s)) {
      CUDA_TRY(s, cudaMemsetAsync(t->stop, 0, sizeof(int), s->stream));
      // a sharded FW step decides to stop after its phase A (the G_U subtrees are exchanged
      // first), so that step's row workspace is left as phase A filled it: clear it
      if (s->G > 1) { sro_status e = ws_clean(t); if (e) return e; }
    }
  } else {
    // visit order for the whole call (U / P / explicit); GA draws on the device
    if (!ga) {
      if (o->visit)   // explicit visits index columns / blocks on the device: range-checked here
        for (int64_t q = 0; q < iters; q++)
          if (o->visit[q] < 0 || o->visit[q] >= nprime) { s->err = "visit entries must lie in [0, n') (n' = n, or n / block_size)"; return SRO_ERR_INVALID_ARG; }
      make_visits(o->sampling, seed, s->k, iters, (int)nprime, o->visit, 0, hv);
      st = ensure_visit(s, iters > 0 ? iters : 1);
      if (st) return st;
      if (iters > 0) CUDA_TRY(s, cudaMemcpyAsync(s->visit, hv.data(), sizeof(int) * iters, cudaMemcpyHostToDevice, s->stream));
    } else if (variant == SRO_BATCHED) {
      // the device draws write the blocks here; the refresh after a call's last step draws the
      // next block into slot iters (cursor mode), hence iters + 1 slots
      st = ensure_visit(s, iters + 1);
      if (st) return st;
    }
    const long long gaMn = ga ? (long long)o->ga_M * nprime : 0;   // global refresh period (R16, R31)
    bool refreshed_with_gap = false;   // batched GA: the refresh sweep that just ran was fused with this check
    for (;;) {
      if (s->k % period == 0) {
        double g = 0.0;
        if (refreshed_with_gap) {
          CUDA_TRY(s, rb(s, &g, s->scal + 4, sizeof(double)));
          st = check_status(s);
          resolve_timing(s);
        } else {
          st = gap_sweep(s, &g);
          out->entries_read += (int64_t)m * n_held;
        }
        if (st) return st;
        out->gap = g; out->gap_checks++;
        out->entries_scanned += (int64_t)m * n_held;
        if (g <= o->epsilon) { out->converged = 1; break; }
      }
      refreshed_with_gap = false;
      if (done >= iters) break;
      if (variant == SRO_BATCHED) {
        // enqueue every block step up to the next gap check, then one sync
        long long seg = iters - done;
        const long long to_check = period - s->k % period;
        if (seg > to_check) seg = to_check;
        if (ga) { const long long to_ref = gaMn - s->k % gaMn; if (seg > to_ref) seg = to_ref; }
        const int64_t before = done;
        if (cursor_mode) {
          const int gsteps = seg - 1 < 16 ? (int)(seg - 1 > 1 ? seg - 1 : 1) : 16;
          const int B = o->block_size;
          // GA: the segment's first block is drawn here, every later one by the previous
          // step's refresh kernel; without the inner refresh every step draws its own
          auto ga_draw_step = [&]() -> sro_status {
            k_ga_block_draw<<<1, 32, 0, s->stream>>>(s->fen, s->G_ga, n, B, seed, kbase, s->cur, s->visit, s->status);
            CUDA_TRY(s, cudaGetLastError());
            s->stats.kernel_launches += 1;
            return SRO_OK;
          };
          if (ga && o->ga_inner) { st = ga_draw_step(); if (st) return st; }
          st = run_steps(seg, gsteps, [&]() -> sro_status {
            if (ga && !o->ga_inner) { sro_status sd = ga_draw_step(); if (sd) return sd; }
            sro_status st1 = plain_block_step(s, s->visit, B, B, o->step, nprime, false,
                                              o->trace ? s->trace : nullptr, s->cur, kbase);
            if (st1 || !ga || !o->ga_inner) return st1;
            if (o->ga_post_update) {   // g_i(T^{k+1}) of the block's columns: a sweep at the new state
              s->sweep_cur = s->cur;
              st1 = sweep(s, s->visit - 1, B, 0, B, s->sw_j, s->sw_min, s->sw_g, nullptr);
              s->sweep_cur = nullptr;
              if (st1) return st1;
            }
            CUDA_TRY(s, set_dyn_smem((const void*)k_ga_block_refresh, s->device, (int)(sizeof(double) * B)));
            k_ga_block_refresh<<<1, 1024, sizeof(double) * B, s->stream>>>(s->G_ga, s->fen, n, B, s->visit, s->cur,
                                                                            s->sw_g, s->status, seed, kbase);
            CUDA_TRY(s, cudaGetLastError());
            s->stats.kernel_launches += 1;
            return SRO_OK;
          });
          if (st) return st;
        } else {
          const int B = o->block_size, Bs = B / s->G;
          if (ga && o->ga_inner && s->ga_blk_cap < B) {
            sfree(s->ga_blk, s->stream);
            CUDA_TRY(s, salloc(&s->ga_blk, (size_t)B, s->stream));
            s->ga_blk_cap = B;
          }
          for (long long q = 0; q < seg; q++) {
            int* slot = s->visit + done + q;
            if (ga) {   // sharded GA block sampling (R31): the lead's tree over all n_glob columns
              k_ga_block_draw_at<<<1, 32, 0, s->stream>>>(s->fen, s->G_ga, s->n_glob, B, seed, s->k + q, slot,
                                                          s->status);
              CUDA_TRY(s, cudaGetLastError());
            }
            st = block_step(slot, B, false, o->trace ? s->trace + 9 * (done + q) : nullptr);
            if (st) return st;
            if (ga && o->ga_inner) {
              // the block's column gaps, every shard's B/G in its slot (global position order)
              for (Solver* t : held(s)) {
                if (o->ga_post_update) {
                  st = sweep(t, slot, Bs, 0, Bs, t->sw_j, t->sw_min, t->sw_g, nullptr);
                  if (st) return st;
                }
                CUDA_TRY(s, cudaMemcpyAsync(s->ga_blk + (size_t)t->shard * Bs, t->sw_g, sizeof(double) * Bs,
                                            cudaMemcpyDeviceToDevice, s->stream));
              }
              st = exchange(s, s->ga_blk, (size_t)Bs);
              if (st) return st;
              CUDA_TRY(s, set_dyn_smem((const void*)k_ga_block_refresh_at, s->device, (int)(sizeof(double) * B)));
              k_ga_block_refresh_at<<<1, 1024, sizeof(double) * B, s->stream>>>(s->G_ga, s->fen, s->n_glob, B, slot,
                                                                                s->ga_blk, s->status);
              CUDA_TRY(s, cudaGetLastError());
            }
          }
        }
        st = drain_block_steps(s, &done);
        {
          const int64_t e = (int64_t)m * (o->block_size / s->G) * (int64_t)held(s).size() * (done - before) *
                            ((ga && o->ga_inner && o->ga_post_update) ? 2 : 1);   // post: a second sweep of the block
          out->entries_scanned += e;
          out->entries_read += e;
        }
        if (st) break;
        if (ga && s->k % gaMn == 0) {
          double gdummy = 0.0;
          if (s->G == 1 && s->k % period == 0) {   // the refresh sweep also gives the gap check due now
            st = ga_refresh_and_gap(s);
            refreshed_with_gap = true;
          } else {
            st = s->G > 1 ? ga_global_refresh_sharded(s, &gdummy) : ga_global_refresh(s);
          }
          if (st) return st;
          out->entries_scanned += (int64_t)m * n;
          out->entries_read += (int64_t)m * n;
        }
        continue;
      }
      // Sequential family: epochs (a persistent-kernel segment, then the GA global
      // refresh and the gap check due at its end) are enqueued one ahead of the host's
      // check, so the GPU never waits for the host between epochs. Every kernel of an
      // epoch is guarded by the device flag s->stop, which the epoch before sets when
      // its segment failed or its gap reached epsilon: a speculative epoch after it is
      // then a no-op and the state is exactly the checked one.
      st = seq_epochs(s, variant, o, iters, period, gaMn, ga, &done, out);
      break;
    }  }
  out->iters_done = done;
  out->k = s->k;
  CUDA_TRY(s, cudaEventRecord(s->ev1, s->stream));
  if (o->trace && done > 0) {
    htr.resize(9 * (size_t)done);
    CUDA_TRY(s, cudaMemcpyAsync(htr.data(), s->trace, sizeof(double) * 9 * done, cudaMemcpyDeviceToHost, s->stream));
  }
  CUDA_TRY(s, stream_wait(s));
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
  if (!per_column && !argmin_rows) return SRO_OK;
  auto cols = held_order(s);
  auto H = held(s);
  std::vector<std::vector<double>> g(H.size(), std::vector<double>(s->n));
  std::vector<std::vector<int>> j(H.size(), std::vector<int>(s->n));
  for (size_t q = 0; q < H.size(); q++) {
    const double* src = s->G == 1 ? s->sw_g : s->gx + (size_t)H[q]->shard * s->n;
    CUDA_TRY(s, cudaMemcpyAsync(g[q].data(), src, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, cudaMemcpyAsync(j[q].data(), H[q]->sw_j, sizeof(int) * s->n, cudaMemcpyDeviceToHost, s->stream));
  }
  CUDA_TRY(s, stream_wait(s));
  for (size_t c = 0; c < cols.size(); c++) {
    if (per_column) per_column[c] = g[cols[c].hq][cols[c].p];
    if (argmin_rows) argmin_rows[c] = j[cols[c].hq][cols[c].p];
  }
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
  CUDA_TRY(s, stream_wait(s));
  return SRO_OK;
}

sro_status sro_get_plan(sro_handle h, double* dense, int32_t* rows, int32_t* cols, double* vals, int64_t cap,
                        int64_t* nnz) {
  if (!h) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  auto H = held(s);
  std::vector<std::vector<int>> hc(H.size()), hr(H.size());
  std::vector<std::vector<double>> hv(H.size());
  for (size_t q = 0; q < H.size(); q++) {
    Solver* t = H[q];
    hc[q].resize(t->n); hr[q].resize((size_t)t->n * t->cap); hv[q].resize((size_t)t->n * t->cap);
    CUDA_TRY(s, cudaMemcpyAsync(hc[q].data(), t->cnt, sizeof(int) * t->n, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, cudaMemcpyAsync(hr[q].data(), t->srow, sizeof(int) * hr[q].size(), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(s, cudaMemcpyAsync(hv[q].data(), t->sval, sizeof(double) * hv[q].size(), cudaMemcpyDeviceToHost, s->stream));
  }
  CUDA_TRY(s, stream_wait(s));
  auto order = held_order(s);
  if (dense) memset(dense, 0, sizeof(double) * (size_t)s->m * order.size());
  int64_t q = 0;
  for (size_t c = 0; c < order.size(); c++) {
    const int hq = order[c].hq, p = order[c].p;
    for (int e = 0; e < hc[hq][p]; e++) {
      const int k = hr[hq][(size_t)p * s->cap + e];
      const double v = hv[hq][(size_t)p * s->cap + e];
      if (dense) dense[c * (size_t)s->m + k] = v;
      if (rows && cols && vals && q < cap) { rows[q] = k; cols[q] = order[c].global; vals[q] = v; }
      q++;
    }
  }
  if (nnz) *nnz = q;
  if (rows && cols && vals && q > cap) { s->err = "COO capacity too small"; return SRO_ERR_CAPACITY; }
  return SRO_OK;
}

}  // extern "C"

namespace {
// Per-row sums over the n columns of the plan (R19 shape), for channel d = -1
// (sum_i T_ki) and d = 0..2 (sum_i T_ki y_id); out[c] device arrays of length m.
sro_status plan_row_sums(Solver* s, const double* y_dev, const int* chans, int nch, double** out) {
  sro_status st = ensure_block_ws(s, s->n);
  if (st) return st;
  BlockArgs A = block_args(s, nullptr, 0, s->n, 0, 1, false, nullptr);
  const int tpb = 256;
  int gL = (s->n + tpb - 1) / tpb; if (gL > s->num_sms * 8) gL = s->num_sms * 8;
  const int gP = s->num_sms * 8;
  const int gR = (s->m + 7) / 8 < s->num_sms * 8 ? (s->m + 7) / 8 : s->num_sms * 8;
  k_plan_begin<<<1, 32, 0, s->stream>>>(A);
  k_plan_pairs_count<<<gL, tpb, 0, s->stream>>>(A);
  k_scan_pairs<<<1, 1024, 0, s->stream>>>(A);
  k_plan_pairs_gen<<<gL, tpb, 0, s->stream>>>(A);
  k_touched_scan<<<1, 1024, 0, s->stream>>>(A);
  for (int c = 0; c < nch; c++) {
    CUDA_TRY(s, cudaMemsetAsync(out[c], 0, sizeof(double) * s->m, s->stream));
    k_plan_channel<<<gP, tpb, 0, s->stream>>>(A, y_dev, chans[c], s->pdelta);
    k_runs<<<A.W, tpb, 0, s->stream>>>(A, s->pdelta);
    k_row_tree_all<2><<<gR, 256, 0, s->stream>>>(A, out[c], c == nch - 1 ? 1 : 0, nullptr);
  }
  s->lead->stats.kernel_launches += 5 + 3 * nch;
  CUDA_TRY(s, cudaGetLastError());
  return SRO_OK;
}
}  // namespace

extern "C" {

sro_status sro_barycentric(sro_handle h, const double* x, const double* y, double* xhat) {
  if (!h || !x || !y || !xhat) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  if (s->G > 1) { s->err = "sro_barycentric: unsharded handles only"; return SRO_ERR_INVALID_ARG; }
  const int m = s->m, n = s->n;
  double *buf = nullptr;
  CUDA_TRY(s, dalloc(&buf, (size_t)4 * m + 3 * (size_t)m + 3 * (size_t)n + 3 * (size_t)m));
  double* sums[4] = {buf, buf + m, buf + 2 * (size_t)m, buf + 3 * (size_t)m};
  double* xd = buf + 4 * (size_t)m;
  double* yd = xd + 3 * (size_t)m;
  double* xo = yd + 3 * (size_t)n;
  sro_status st = SRO_OK;
  do {
    if (cudaMemcpyAsync(xd, x, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s->stream) != cudaSuccess ||
        cudaMemcpyAsync(yd, y, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s->stream) != cudaSuccess) {
      s->err = "barycentric upload failed"; st = SRO_ERR_CUDA; break;
    }
    const int chans[4] = {-1, 0, 1, 2};
    st = plan_row_sums(s, yd, chans, 4, sums);
    if (st) break;
    k_plan_project<<<(m + 255) / 256, 256, 0, s->stream>>>(m, sums[0], sums[1], sums[2], sums[3], xd, xo);
    s->stats.kernel_launches += 1;
    if (cudaMemcpyAsync(xhat, xo, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
        stream_wait(s) != cudaSuccess) {
      s->err = "barycentric failed"; st = SRO_ERR_CUDA; break;
    }
  } while (0);
  cudaFree(buf);
  return st;
}

sro_status sro_metrics(sro_handle h, double* e_c, double* sparsity, double* lin) {
  if (!h || !e_c || !sparsity || !lin) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  if (s->G > 1) { s->err = "sro_metrics: unsharded handles only"; return SRO_ERR_INVALID_ARG; }
  const int m = s->m, n = s->n;
  double* buf = nullptr;
  CUDA_TRY(s, dalloc(&buf, (size_t)m + (size_t)(m > n ? m : n)));
  double* rs = buf;
  double* sq = buf + m;
  sro_status st = SRO_OK;
  double e1 = 0.0, e2 = 0.0;
  std::vector<int> hc(n);
  do {
    const int chans[1] = {-1};
    st = plan_row_sums(s, nullptr, chans, 1, &rs);
    if (st) break;
    k_plan_sq_rows<<<(m + 255) / 256, 256, 0, s->stream>>>(m, rs, s->a, sq);
    k_psum256<<<1, 256, 0, s->stream>>>(sq, m, s->scal + 4, nullptr, nullptr, nullptr);
    k_plan_sq_cols<<<(n + 255) / 256, 256, 0, s->stream>>>(n, s->cap, s->cnt, s->sval, s->b, sq);
    k_psum256<<<1, 256, 0, s->stream>>>(sq, n, s->scal + 5, nullptr, nullptr, nullptr);
    s->stats.kernel_launches += 4;
    if (cudaMemcpyAsync(&e1, s->scal + 4, sizeof(double), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
        cudaMemcpyAsync(&e2, s->scal + 5, sizeof(double), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
        cudaMemcpyAsync(hc.data(), s->cnt, sizeof(int) * n, cudaMemcpyDeviceToHost, s->stream) != cudaSuccess) {
      s->err = "metrics failed"; st = SRO_ERR_CUDA; break;
    }
    double f = 0.0;
    st = objective_dev(s, &f);   // leaves psum256_i <t_i, c_i> in scal[4] (synchronises)
    if (st) break;
    if (cudaMemcpy(lin, s->scal + 4, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
      s->err = "metrics failed"; st = SRO_ERR_CUDA; break;
    }
  } while (0);
  cudaFree(buf);
  if (st) return st;
  int64_t nnz = 0;
  for (int v : hc) nnz += v;
  *e_c = std::sqrt(e1) + std::sqrt(e2);
  *sparsity = 1.0 - (double)nnz / ((double)m * (double)n);
  return SRO_OK;
}

sro_status sro_lp_metrics(sro_handle h, const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz,
                          double* e_m, double* e_v) {
  if (!h || !e_m || !e_v || nnz < 0 || (nnz > 0 && (!rows || !cols || !vals))) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  if (s->G > 1) { s->err = "sro_lp_metrics: unsharded handles only"; return SRO_ERR_INVALID_ARG; }
  const int m = s->m, n = s->n;
  // T* in COO sorted by (column, row), entries within range: column pointers by counting
  std::vector<int64_t> colptr((size_t)n + 1, 0);
  for (int64_t q = 0; q < nnz; q++) {
    if (rows[q] < 0 || rows[q] >= m || cols[q] < 0 || cols[q] >= n || !std::isfinite(vals[q]) ||
        (q > 0 && (cols[q] < cols[q - 1] || (cols[q] == cols[q - 1] && rows[q] <= rows[q - 1])))) {
      s->err = "sro_lp_metrics: T* must be COO sorted by column then row (strictly), in range, finite";
      return SRO_ERR_INVALID_ARG;
    }
    colptr[(size_t)cols[q] + 1]++;
  }
  for (int i = 0; i < n; i++) colptr[(size_t)i + 1] += colptr[i];
  int64_t* dptr = nullptr;
  int* drow = nullptr;
  double *dval = nullptr, *buf = nullptr;
  sro_status st = SRO_OK;
  double D = 0.0, S2 = 0.0, SC = 0.0, lin = 0.0;
  do {
    if (dalloc(&dptr, (size_t)n + 1) != cudaSuccess || dalloc(&drow, (size_t)nnz) != cudaSuccess ||
        dalloc(&dval, (size_t)nnz) != cudaSuccess || dalloc(&buf, 3 * (size_t)n) != cudaSuccess) {
      s->err = "sro_lp_metrics: device allocation failed"; st = SRO_ERR_OOM; break;
    }
    if (cudaMemcpyAsync(dptr, colptr.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s->stream) != cudaSuccess ||
        (nnz > 0 && (cudaMemcpyAsync(drow, rows, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s->stream) != cudaSuccess ||
                     cudaMemcpyAsync(dval, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, s->stream) != cudaSuccess))) {
      s->err = "sro_lp_metrics: upload failed"; st = SRO_ERR_CUDA; break;
    }
    double *dd = buf, *ss = buf + n, *cc = buf + 2 * (size_t)n;
    st = with_sweep_src(s, [&](auto src) -> sro_status {
      k_lp_cols<<<(n + 255) / 256, 256, 0, s->stream>>>(src, n, s->cap, s->cnt, s->srow, s->sval, dptr, drow, dval, dd, ss, cc);
      CUDA_TRY(s, cudaGetLastError());
      return SRO_OK;
    });
    if (st) break;
    k_psum256<<<1, 256, 0, s->stream>>>(dd, n, s->scal + 1, nullptr, nullptr, nullptr);
    k_psum256<<<1, 256, 0, s->stream>>>(ss, n, s->scal + 2, nullptr, nullptr, nullptr);
    k_psum256<<<1, 256, 0, s->stream>>>(cc, n, s->scal + 3, nullptr, nullptr, nullptr);
    s->stats.kernel_launches += 4;
    CUDA_TRY(s, rb(s, &D, s->scal + 1, sizeof(double)));
    CUDA_TRY(s, rb(s, &S2, s->scal + 2, sizeof(double)));
    CUDA_TRY(s, rb(s, &SC, s->scal + 3, sizeof(double)));
    double f = 0.0;
    st = objective_dev(s, &f);   // psum256_i <t_i, c_i> in scal[4] (synchronises; the readbacks above land)
    if (st) break;
    CUDA_TRY(s, rb(s, &lin, s->scal + 4, sizeof(double)));
    CUDA_TRY(s, stream_wait(s));
  } while (0);
  for (void* q : {(void*)dptr, (void*)drow, (void*)dval, (void*)buf}) if (q) cudaFree(q);
  if (st) return st;
  *e_m = std::sqrt(D) / std::sqrt(S2);
  *e_v = std::fabs(lin - SC) / std::fabs(SC);
  return SRO_OK;
}

sro_status sro_held_columns(sro_handle h, int32_t* cols, int32_t* n_held) {
  if (!h || !n_held) return SRO_ERR_INVALID_ARG;
  auto order = held_order(static_cast<Solver*>(h));
  *n_held = (int32_t)order.size();
  if (cols) for (size_t c = 0; c < order.size(); c++) cols[c] = order[c].global;
  return SRO_OK;
}

sro_status sro_nccl_unique_id(uint8_t* out128) {
  if (!out128) return SRO_ERR_INVALID_ARG;
  NcclApi& api = nccl();
  if (!api.ok) { g_create_err = api.err; return SRO_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = api.get_id(&id);
  if (r != ncclSuccess) { g_create_err = std::string("ncclGetUniqueId: ") + api.errstr(r); return SRO_ERR_NCCL; }
  memcpy(out128, &id, sizeof(id));
  return SRO_OK;
}

sro_status sro_get_stats(sro_handle h, sro_stats* out, int32_t reset) {
  if (!h || !out) return SRO_ERR_INVALID_ARG;
  Solver* s = static_cast<Solver*>(h);
  cudaSetDevice(s->device);
  CUDA_TRY(s, stream_wait(s));
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
  CUDA_TRY(s, cudaMemcpyAsync(out8, s->phase, 32 * sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(s, stream_wait(s));
  return SRO_OK;
}

sro_status sro_set_timing(sro_handle h, int32_t on) {
  if (!h) return SRO_ERR_INVALID_ARG;
  static_cast<Solver*>(h)->timing = on != 0;
  return SRO_OK;
}


// ---------------------------------------------------------------------------
// Colour-transfer front end: k-means quantisation and
// recolouring (k_kmeans.cuh). Handle-free; scratch allocated per call.
// ---------------------------------------------------------------------------
static thread_local std::string g_km_err;

const char* sro_kmeans_error(void) { return g_km_err.c_str(); }

#define KM_TRY(call)                                                          \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) { g_km_err = cudaGetErrorString(e_); st = SRO_ERR_CUDA; goto done; } \
  } while (0)

// k-means++ seeding (R34): centre 0 = min(floor(u_0 N), N - 1) on the host, then per centre
// one k_kpp_update (D2 and its 4096-pixel block sums) and one k_kpp_pick (the D2-weighted draw).
sro_status sro_kmeanspp(const uint8_t* pixels, int64_t npix, int32_t k, const double* u, int32_t pixels_on_device,
                        void* cuda_stream, int32_t* init_idx) {
  g_km_err.clear();
  if (!pixels || !u || !init_idx || npix < 1 || k < 1 || k > npix) { g_km_err = "bad argument"; return SRO_ERR_INVALID_ARG; }
  if (npix > INT32_MAX) { g_km_err = "npix exceeds int32 pixel indices"; return SRO_ERR_DIMENSION; }
  for (int t = 0; t < k; t++)
    if (!(u[t] >= 0.0 && u[t] < 1.0)) { g_km_err = "u: k uniforms in [0, 1)"; return SRO_ERR_INVALID_ARG; }
  sro_status st = SRO_OK;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  const int64_t nb = (npix + KPP_BLOCK - 1) / KPP_BLOCK;
  uint8_t *dpx = nullptr, *dch = nullptr;
  int32_t *d2 = nullptr, *dcent = nullptr, *dcur = nullptr;
  long long* bsum = nullptr;
  double* du = nullptr;
  int64_t c0 = (int64_t)(u[0] * (double)npix);   // one rounded product, then floor
  if (c0 > npix - 1) c0 = npix - 1;
  const int32_t c0i = (int32_t)c0;
  const uint8_t one = 1;
  const uint8_t* px = pixels;
  if (!pixels_on_device) {
    KM_TRY(cudaMallocAsync(&dpx, (size_t)3 * npix, stream));
    KM_TRY(cudaMemcpyAsync(dpx, pixels, (size_t)3 * npix, cudaMemcpyHostToDevice, stream));
    px = dpx;
  }
  KM_TRY(cudaMallocAsync(&d2, sizeof(int32_t) * npix, stream));
  KM_TRY(cudaMallocAsync(&dch, (size_t)npix, stream));
  KM_TRY(cudaMallocAsync(&bsum, sizeof(long long) * nb, stream));
  KM_TRY(cudaMallocAsync(&du, sizeof(double) * k, stream));
  KM_TRY(cudaMallocAsync(&dcent, sizeof(int32_t) * k, stream));
  KM_TRY(cudaMallocAsync(&dcur, sizeof(int32_t), stream));
  KM_TRY(cudaMemsetAsync(dch, 0, (size_t)npix, stream));
  KM_TRY(cudaMemcpyAsync(du, u, sizeof(double) * k, cudaMemcpyHostToDevice, stream));
  KM_TRY(cudaMemcpyAsync(dcur, &c0i, sizeof(int32_t), cudaMemcpyHostToDevice, stream));
  KM_TRY(cudaMemcpyAsync(dcent, &c0i, sizeof(int32_t), cudaMemcpyHostToDevice, stream));
  KM_TRY(cudaMemcpyAsync(dch + c0, &one, 1, cudaMemcpyHostToDevice, stream));
  k_kpp_update<<<(unsigned)nb, 256, 0, stream>>>(px, npix, dcur, 1, d2, bsum);
  KM_TRY(cudaGetLastError());
  for (int t = 1; t < k; t++) {
    k_kpp_pick<<<1, 1024, 0, stream>>>(d2, npix, bsum, nb, du, t, dcent, dcur, dch);
    KM_TRY(cudaGetLastError());
    if (t + 1 < k) {
      k_kpp_update<<<(unsigned)nb, 256, 0, stream>>>(px, npix, dcur, 0, d2, bsum);
      KM_TRY(cudaGetLastError());
    }
  }
  KM_TRY(cudaMemcpyAsync(init_idx, dcent, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, stream));
  KM_TRY(cudaStreamSynchronize(stream));
done:
  for (void* q : {(void*)dpx, (void*)d2, (void*)dch, (void*)bsum, (void*)du, (void*)dcent, (void*)dcur})
    if (q) cudaFreeAsync(q, stream);
  cudaStreamSynchronize(stream);
  return st;
}

sro_status sro_kmeans(const uint8_t* pixels, int64_t npix, int32_t k, const int32_t* init_idx, int32_t max_iters,
                      int32_t pixels_on_device, void* cuda_stream, double* centroids, int32_t* labels,
                      int64_t* counts, int32_t* iters, int32_t* converged) {
  g_km_err.clear();
  if (!pixels || !init_idx || !centroids || !counts || !iters || !converged || npix < 1 || k < 1 || k > npix ||
      max_iters < 1) {
    g_km_err = "bad argument";
    return SRO_ERR_INVALID_ARG;
  }
  if (k > KM_KMAX) { g_km_err = "k exceeds the shared-memory centroid stage (8192)"; return SRO_ERR_DIMENSION; }
  {
    std::vector<int32_t> chk(init_idx, init_idx + k);
    std::sort(chk.begin(), chk.end());
    for (int c = 0; c < k; c++)
      if (chk[c] < 0 || chk[c] >= npix || (c && chk[c] == chk[c - 1])) { g_km_err = "init_idx: k distinct pixel indices"; return SRO_ERR_INVALID_ARG; }
  }
  sro_status st = SRO_OK;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  uint8_t* dpx = nullptr;
  int32_t *dinit = nullptr, *dlab = nullptr;
  double* dcen = nullptr;
  unsigned long long *dsums = nullptr, *dcnt = nullptr, *dsc = nullptr;   // dsc: changed, nempty, dmax, parg
  int* dmoved = nullptr;
  std::vector<double> hc;
  std::vector<unsigned long long> hcnt;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)3 * k * sizeof(float);
  int it = 0;
  bool conv = false, repaired = false;
  int gA = 0;
  if (!pixels_on_device) {
    KM_TRY(cudaMallocAsync(&dpx, (size_t)3 * npix, stream));
    KM_TRY(cudaMemcpyAsync(dpx, pixels, (size_t)3 * npix, cudaMemcpyHostToDevice, stream));
  }
  KM_TRY(cudaMallocAsync(&dinit, sizeof(int32_t) * k, stream));
  KM_TRY(cudaMallocAsync(&dlab, sizeof(int32_t) * npix, stream));
  KM_TRY(cudaMallocAsync(&dcen, sizeof(double) * 3 * k, stream));
  KM_TRY(cudaMallocAsync(&dsums, sizeof(unsigned long long) * 3 * k, stream));
  KM_TRY(cudaMallocAsync(&dcnt, sizeof(unsigned long long) * k, stream));
  KM_TRY(cudaMallocAsync(&dsc, sizeof(unsigned long long) * 4, stream));
  KM_TRY(cudaMallocAsync(&dmoved, sizeof(int), stream));
  KM_TRY(cudaMemcpyAsync(dinit, init_idx, sizeof(int32_t) * k, cudaMemcpyHostToDevice, stream));
  KM_TRY(cudaMemsetAsync(dlab, 0xff, sizeof(int32_t) * npix, stream));   // no class yet
  {
    const uint8_t* px = pixels_on_device ? pixels : dpx;
    k_km_init<<<(k + 255) / 256, 256, 0, stream>>>(px, dinit, k, dcen);
    KM_TRY(cudaGetLastError());
    KM_TRY(cudaFuncSetAttribute((const void*)k_km_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_km_assign, KM_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t need = (npix + (int64_t)KM_THREADS * KM_PIX - 1) / ((int64_t)KM_THREADS * KM_PIX);
    gA = (int)std::min<int64_t>(need, (int64_t)nsm * per_sm);
    const int gP = (int)std::min<int64_t>((npix + 255) / 256, (int64_t)nsm * 8);
    while (it < max_iters) {
      it++;
      KM_TRY(cudaMemsetAsync(dsums, 0, sizeof(unsigned long long) * 3 * k, stream));
      KM_TRY(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * k, stream));
      KM_TRY(cudaMemsetAsync(dsc, 0, sizeof(unsigned long long) * 2, stream));
      k_km_assign<<<gA, KM_THREADS, smem, stream>>>(px, npix, dcen, k, dlab, dsums, dcnt, dsc);
      KM_TRY(cudaGetLastError());
      unsigned long long chg = 0;
      KM_TRY(cudaMemcpyAsync(&chg, dsc, sizeof(chg), cudaMemcpyDeviceToHost, stream));
      KM_TRY(cudaStreamSynchronize(stream));
      if (it > 1 && !repaired && chg == 0) { conv = true; break; }
      repaired = false;
      k_km_update<<<(k + 255) / 256, 256, 0, stream>>>(dsums, dcnt, k, dcen, dsc + 1);
      KM_TRY(cudaGetLastError());
      unsigned long long nempty = 0;
      KM_TRY(cudaMemcpyAsync(&nempty, dsc + 1, sizeof(nempty), cudaMemcpyDeviceToHost, stream));
      KM_TRY(cudaStreamSynchronize(stream));
      if (nempty) {
        hcnt.resize(k);
        KM_TRY(cudaMemcpyAsync(hcnt.data(), dcnt, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost, stream));
        KM_TRY(cudaStreamSynchronize(stream));
        for (int c = 0; c < k; c++) {
          if (hcnt[c]) continue;
          const unsigned long long none = ~0ULL;
          KM_TRY(cudaMemsetAsync(dsc + 2, 0, sizeof(unsigned long long), stream));
          KM_TRY(cudaMemcpyAsync(dsc + 3, &none, sizeof(none), cudaMemcpyHostToDevice, stream));
          KM_TRY(cudaMemsetAsync(dmoved, 0, sizeof(int), stream));
          k_km_far_max<<<gP, 256, 0, stream>>>(px, npix, dcen, k, dlab, dcnt, dsc + 2);
          k_km_far_arg<<<gP, 256, 0, stream>>>(px, npix, dcen, k, dlab, dcnt, dsc + 2, dsc + 3);
          k_km_move<<<1, 1, 0, stream>>>(px, k, c, dsc + 3, dcen, dlab, dcnt, dmoved);
          KM_TRY(cudaGetLastError());
          int moved = 0;
          KM_TRY(cudaMemcpyAsync(&moved, dmoved, sizeof(int), cudaMemcpyDeviceToHost, stream));
          KM_TRY(cudaStreamSynchronize(stream));
          if (moved) repaired = true;
        }
      }
    }
    hc.resize((size_t)3 * k);
    hcnt.resize(k);
    KM_TRY(cudaMemcpyAsync(hc.data(), dcen, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost, stream));
    KM_TRY(cudaMemcpyAsync(hcnt.data(), dcnt, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost, stream));
    if (labels) KM_TRY(cudaMemcpyAsync(labels, dlab, sizeof(int32_t) * npix, cudaMemcpyDeviceToHost, stream));
    KM_TRY(cudaStreamSynchronize(stream));
    for (int c = 0; c < k; c++) {
      centroids[3 * c] = hc[c]; centroids[3 * c + 1] = hc[k + c]; centroids[3 * c + 2] = hc[2 * k + c];
      counts[c] = (int64_t)hcnt[c];
    }
    *iters = it;
    *converged = conv ? 1 : 0;
  }
done:
  for (void* q : {(void*)dpx, (void*)dinit, (void*)dlab, (void*)dcen, (void*)dsums, (void*)dcnt, (void*)dsc, (void*)dmoved})
    if (q) cudaFreeAsync(q, stream);
  cudaStreamSynchronize(stream);
  return st;
}

sro_status sro_recolour(const int32_t* labels, int64_t npix, const double* xhat, int32_t k, void* cuda_stream,
                        uint8_t* out_pixels) {
  g_km_err.clear();
  if (!labels || !xhat || !out_pixels || npix < 1 || k < 1) { g_km_err = "bad argument"; return SRO_ERR_INVALID_ARG; }
  for (int64_t p = 0; p < npix; p++)
    if (labels[p] < 0 || labels[p] >= k) { g_km_err = "label out of range"; return SRO_ERR_INVALID_ARG; }
  sro_status st = SRO_OK;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  int32_t* dl = nullptr;
  double* dx = nullptr;
  uint8_t* dout = nullptr;
  KM_TRY(cudaMallocAsync(&dl, sizeof(int32_t) * npix, stream));
  KM_TRY(cudaMallocAsync(&dx, sizeof(double) * 3 * k, stream));
  KM_TRY(cudaMallocAsync(&dout, (size_t)3 * npix, stream));
  KM_TRY(cudaMemcpyAsync(dl, labels, sizeof(int32_t) * npix, cudaMemcpyHostToDevice, stream));
  KM_TRY(cudaMemcpyAsync(dx, xhat, sizeof(double) * 3 * k, cudaMemcpyHostToDevice, stream));
  k_km_recolour<<<(int)std::min<int64_t>((3 * npix + 255) / 256, 148 * 16), 256, 0, stream>>>(dl, npix, dx, dout);
  KM_TRY(cudaGetLastError());
  KM_TRY(cudaMemcpyAsync(out_pixels, dout, (size_t)3 * npix, cudaMemcpyDeviceToHost, stream));
  KM_TRY(cudaStreamSynchronize(stream));
done:
  for (void* q : {(void*)dl, (void*)dx, (void*)dout}) if (q) cudaFreeAsync(q, stream);
  cudaStreamSynchronize(stream);
  return st;
}

sro_status sro_kmeans_features(const double* centroids, const int64_t* counts, int32_t k, double* colours,
                               double* weights) {
  g_km_err.clear();
  if (!centroids || !counts || !colours || !weights || k < 1) { g_km_err = "bad argument"; return SRO_ERR_INVALID_ARG; }
  int64_t total = 0;
  for (int c = 0; c < k; c++) {
    if (counts[c] < 0) { g_km_err = "negative count"; return SRO_ERR_INVALID_ARG; }
    total += counts[c];
  }
  if (total == 0) { g_km_err = "no pixels"; return SRO_ERR_INVALID_ARG; }
  // R29: colour x = centroid / 255 (one correctly rounded division per channel), histogram
  // a = count / N with N the total pixel count
  for (int c = 0; c < k; c++) {
    for (int d = 0; d < 3; d++) colours[3 * c + d] = centroids[3 * c + d] / 255.0;
    weights[c] = (double)counts[c] / (double)total;
  }
  return SRO_OK;
}

}  // extern "C"
