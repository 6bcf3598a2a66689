// k_ga_block.cuh — gap-adaptive sampling for batched BCFW (SURVEY §8(f) NEXT-4,
// DESIGN.md R31): the block of a column drawn with probability proportional to
// max(G_i, 0) (so a block with probability proportional to its columns' summed
// stored gaps) from the same Fenwick tree over the n stored column gaps as the
// BCFW-family GA (Alg. A.4), and after the block step the stored
// gaps of its B columns refreshed in ascending column order (Alg. A.4 line 6).
// Everything runs on the device between the steps, so a GA block step is as
// launch-invariant as a P / U one (device step cursor, one CUDA graph).
#pragma once
#include "k_bcfw.cuh"

namespace sro {

// visit[*cur] = the drawn block (the step's LMO sweep and tail read it there).
__global__ void k_ga_block_draw(const double* __restrict__ fen, const double* __restrict__ G, int n, int B,
                                uint64_t seed, long long kbase, const unsigned* __restrict__ cur, int* visit,
                                const int* __restrict__ status) {
  if (threadIdx.x != 0) return;
  const unsigned c = *cur;
  // after a failed step every later kernel of the call skips, but a slot must still hold a
  // valid block index for the kernels that read it before testing the status
  if (*status) { visit[c] = 0; return; }
  const double u53 = uniform53(rng_u64(seed, 1, (uint64_t)(kbase + (long long)c)));
  visit[c] = ga_draw(fen, G, n, u53) / B;
}

// Refresh of the block [c0, c0 + B): delta_i = max(g_i, 0) - max(G_i, 0) and G_i = g_i for
// the block's columns, then every Fenwick node covering some of them receives their deltas
// one by one in ascending column order — the additions ga_add performs column after column.
// One CTA; dl: B doubles of shared memory.
__device__ __forceinline__ void ga_block_refresh_body(double* G, double* fen, int n, int B, int c0,
                                                      const double* __restrict__ gnew, double* dl) {
  for (int t = threadIdx.x; t < B; t += blockDim.x) {
    const double gn = gnew[t];
    dl[t] = d_sub(wpos(gn), wpos(G[c0 + t]));
    G[c0 + t] = gn;
  }
  __syncthreads();
  // thread per (leaf t, level l): the node on leaf c0+t's update path that the
  // leaf is the first covered block column of
  const int levels = 32 - __clz(n);
  for (int w = threadIdx.x; w < B * levels; w += blockDim.x) {
    const int t = w / levels, l = w % levels;
    unsigned x = (unsigned)(c0 + t);
    for (int q = 0; q < l && x <= (unsigned)n; q++) x |= x + 1u;
    const long long p = (long long)x + 1;
    if (p > n) continue;
    const long long lo = p - (p & -p);                // covered leaves (0-based): [lo, p - 1]
    const long long first = lo > c0 ? lo : c0;
    if (c0 + t != first) continue;
    const long long last = (p - 1) < (long long)(c0 + B - 1) ? (p - 1) : (long long)(c0 + B - 1);
    double f = fen[p];
    for (long long i = first; i <= last; i++) f = d_add(f, dl[i - c0]);
    fen[p] = f;
  }
  __syncthreads();
}

// Cursor mode (unsharded): after the block step (the cursor already advanced), refresh
// the block just visited, then draw the next step's block (thread 0; the updated nodes
// are visible after the barrier), saving that step a launch; the first step of a
// segment (and one after a global refresh) draws with k_ga_block_draw instead.
__global__ void __launch_bounds__(1024) k_ga_block_refresh(double* G, double* fen, int n, int B, int* visit,
                                                           const unsigned* __restrict__ cur,
                                                           const double* __restrict__ gnew,
                                                           const int* __restrict__ status, uint64_t seed,
                                                           long long kbase) {
  extern __shared__ double dl[];
  if (*status) {   // the next slot still gets a valid block index (see k_ga_block_draw)
    if (threadIdx.x == 0) visit[*cur] = 0;
    return;
  }
  ga_block_refresh_body(G, fen, n, B, visit[*cur - 1u] * B, gnew, dl);
  if (threadIdx.x == 0) {
    const unsigned c = *cur;
    visit[c] = ga_draw(fen, G, n, uniform53(rng_u64(seed, 1, (uint64_t)(kbase + (long long)c)))) / B;
  }
}

// Explicit-slot forms (the sharded loop, which enqueues step by step from the host):
// draw step k's block into *slot; refresh the block *blk with the gathered gaps.
__global__ void k_ga_block_draw_at(const double* __restrict__ fen, const double* __restrict__ G, int n, int B,
                                   uint64_t seed, long long k, int* slot, const int* __restrict__ status) {
  if (threadIdx.x != 0) return;
  if (*status) { *slot = 0; return; }   // a valid index for the skipped step's kernels
  *slot = ga_draw(fen, G, n, uniform53(rng_u64(seed, 1, (uint64_t)k))) / B;
}
__global__ void __launch_bounds__(1024) k_ga_block_refresh_at(double* G, double* fen, int n, int B,
                                                              const int* __restrict__ blk,
                                                              const double* __restrict__ gnew,
                                                              const int* __restrict__ status) {
  extern __shared__ double dl[];
  if (*status) return;
  ga_block_refresh_body(G, fen, n, B, *blk * B, gnew, dl);
}

// Sharded GA helpers: the largest of the G exchanged cost maxima (bit patterns of
// nonnegative doubles) and the per-shard column gaps (gx, shard-major) put in global
// column order (shard s holds, in every group of Bo columns, the s-th Bl of them).
__global__ void k_max_slots(const double* __restrict__ slots, int G, size_t stride, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned long long m = 0ULL;
  for (int s = 0; s < G; s++) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(slots[(size_t)s * stride]);
    m = v > m ? v : m;
  }
  *out = m;
}
__global__ void k_key_to_slot(const unsigned long long* __restrict__ key, double* slot) {
  if (threadIdx.x == 0) *slot = __longlong_as_double((long long)*key);
}
__global__ void k_ga_gather_global(const double* __restrict__ gx, double* Gg, int n_loc, int G, int Bo, int Bl) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)G * n_loc;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(idx / n_loc), q = (int)(idx % n_loc);
    Gg[(int64_t)(q / Bl) * Bo + (int64_t)s * Bl + (q % Bl)] = gx[idx];
  }
}

}  // namespace sro
