// sro_device.cuh — device-side building blocks of the B200 hot path.
//
// Every binary64 operation that feeds r, h, gamma or T is written as an
// explicit round-to-nearest intrinsic (__dadd_rn, __dmul_rn, ...) and the
// library is compiled with --fmad=false, so no multiply-add is ever fused:
// the arithmetic is the one DESIGN.md §3 fixes operation by operation
// (readings R1-R22), which is what makes argmin indices bit-exact.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sro {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream serialization
// may start while its predecessor finishes; griddepcontrol.wait blocks until the predecessor
// grid has completed and its memory is visible (a no-op without PDL), and launch_dependents
// lets the next kernel's CTAs be scheduled early (they in turn wait). Every kernel of the block
// step / sweep chain opens with both, so only launch latency overlaps, never data.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double d_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double d_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double d_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double d_div(double a, double b) { return __ddiv_rn(a, b); }

// (value, row) lexicographic minimum: lowest value, then lowest row (R1, Eq. 9).
__device__ __forceinline__ void argmin_merge(double& v, int& j, double ov, int oj) {
  if (ov < v || (ov == v && oj < j)) { v = ov; j = oj; }
}
// (value, row) maximum with the lowest row on ties (away atom, Eq. 13, R1).
__device__ __forceinline__ void argmax_merge(double& v, int& j, double ov, int oj) {
  if (ov > v || (ov == v && oj < j)) { v = ov; j = oj; }
}
__device__ __forceinline__ void warp_argmin(double& v, int& j) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(FULL, v, o);
    int oj = __shfl_xor_sync(FULL, j, o);
    argmin_merge(v, j, ov, oj);
  }
}
__device__ __forceinline__ void warp_argmax(double& v, int& j) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(FULL, v, o);
    int oj = __shfl_xor_sync(FULL, j, o);
    argmax_merge(v, j, ov, oj);
  }
}

// Chunk c of W covers positions [floor(c L / W), floor((c+1) L / W)) (R19).
// Position p lies in chunk c = max{c : floor(c L / W) <= p} = floor((W (p+1) - 1) / L).
__device__ __forceinline__ int64_t chunk_lo(int c, int64_t L, int W) { return ((int64_t)c * L) / W; }
__device__ __forceinline__ int chunk_index(int64_t p, int64_t L, int W) {
  if (L < (1LL << 23)) return (int)(((unsigned)W * (unsigned)(p + 1) - 1u) / (unsigned)L);
  return (int)(((int64_t)W * (p + 1) - 1) / L);
}

// Order-preserving 64-bit key of a double: keys compare as unsigned integers
// exactly like the values (after -0 -> +0, so equal values share a key).
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d_add(v, 0.0));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)u);
}
// Warp argmin of (value, row), lowest row on ties, with three REDUX.MIN
// instructions on (key high word, key low word, row). Result in every lane.
__device__ __forceinline__ void warp_argmin_redux(unsigned long long& key, int& j) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned m1 = __reduce_min_sync(FULL, hi);
  const unsigned m2 = __reduce_min_sync(FULL, hi == m1 ? lo : 0xffffffffu);
  const unsigned m3 = __reduce_min_sync(FULL, (hi == m1 && lo == m2) ? (unsigned)j : 0x7fffffffu);
  key = ((unsigned long long)m1 << 32) | m2;
  j = (int)m3;
}

// Adjacent-pair tree over 8 values: ((x0+x1)+(x2+x3)) + ((x4+x5)+(x6+x7)).
__device__ __forceinline__ double tree8(const double* x) {
  return d_add(d_add(d_add(x[0], x[1]), d_add(x[2], x[3])), d_add(d_add(x[4], x[5]), d_add(x[6], x[7])));
}

// Butterfly over the 32 lanes with offsets 1, 2, 4, 8, 16: after it every lane
// holds the adjacent-pair tree of the 32 lane values (fp addition commutes).
__device__ __forceinline__ double warp_pair_tree(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// x[lo] + x[lo+1] + ... + x[hi-1] left to right from +0.0 (a chunk of R19's 256-chunk tree),
// with 16 loads in flight per batch: a thread's chunk is latency-bound, not bandwidth-bound
// (config [3]: 256 doubles per chunk, the one-at-a-time loop took ~30 us per psum256)
__device__ __forceinline__ double chunk_seq_sum(const double* __restrict__ x, int64_t lo, int64_t hi) {
  double acc = 0.0;
  int64_t p = lo;
  for (; p + 16 <= hi; p += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; u++) v[u] = x[p + u];
#pragma unroll
    for (int u = 0; u < 16; u++) acc = d_add(acc, v[u]);
  }
  for (; p < hi; p++) acc = d_add(acc, x[p]);
  return acc;
}

// psum256 (R19) of x[0..L) for a CTA of exactly 256 threads: thread c sums
// chunk c left to right from +0.0, then the 256 partials combine by adjacent
// pairs. Returns the total to every thread. `red` is __shared__ double[8].
__device__ __forceinline__ double block_psum256(const double* __restrict__ x, int64_t L, double* red) {
  const int c = threadIdx.x;
  double acc = chunk_seq_sum(x, chunk_lo(c, L, 256), chunk_lo(c + 1, L, 256));
  acc = warp_pair_tree(acc);
  if ((c & 31) == 0) red[c >> 5] = acc;
  __syncthreads();
  double v = 0.0;
  if (c < 32) {
    v = (c < 8) ? red[c] : 0.0;
    // lanes 0..7: butterfly with offsets 1, 2, 4 (adjacent-pair tree over 8 warps)
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) v = d_add(v, __shfl_xor_sync(FULL, v, o));
    if (c == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// psum256 over m rows of a vector that is zero except at up to 32 rows held
// one per lane (rows strictly ascending with the lane index; lanes >= cnt
// hold nothing). Emulates exactly the dense chunk_tree_sum(x, m, 256):
// chunk partials are left-to-right sums from +0.0, untouched chunks are +0.0.
// `slots` is warp-private __shared__ double[256], all +0.0 on entry and exit.
__device__ __forceinline__ double warp_sparse_psum256(int m, int cnt, int row, double x, double* slots) {
  const int lane = threadIdx.x & 31;
  const int c = (lane < cnt) ? chunk_index(row, m, 256) : 0;
  for (int q = 0; q < cnt; q++) {
    int cq = __shfl_sync(FULL, c, q);
    double xq = __shfl_sync(FULL, x, q);
    if (lane == 0) slots[cq] = d_add(slots[cq], xq);
    __syncwarp();
  }
  double s[8];
#pragma unroll
  for (int t = 0; t < 8; t++) s[t] = slots[8 * lane + t];
  double v = tree8(s);
  v = warp_pair_tree(v);
  __syncwarp();
  if (lane < cnt) slots[c] = 0.0;
  __syncwarp();
  return v;
}

// Sequential left-to-right sum (from +0.0) of the lane values of lanes
// 0..cnt-1 — the order a single column's sparse dot uses (R19). Result in
// every lane.
__device__ __forceinline__ double warp_seq_sum(double x, int cnt) {
  double acc = 0.0;
  for (int q = 0; q < cnt; q++) acc = d_add(acc, __shfl_sync(FULL, x, q));
  return acc;
}

// ----------------------------------------------------------------------------
// SplitMix64, counter-based (R21). Device copy used by the GA draw and the
// HASH_UNIFORM cost generator.
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t rng_u64(uint64_t seed, uint32_t stream, uint64_t t) {
  uint64_t key = mix64(seed ^ (0x5851F42D4C957F2DULL * (uint64_t)(stream + 1)));
  return mix64(key + (t + 1) * GOLDEN);
}
__host__ __device__ __forceinline__ double uniform53(uint64_t x) { return (double)(x >> 11) * 0x1p-53; }

// ----------------------------------------------------------------------------
// Cost of a colour pair (SRO_COST_SQEUCLID / EUCLID): ((dx*dx + dy*dy) + dz*dz)
// evaluated in the storage precision with no contraction; binary32 results
// are promoted exactly to binary64.
// ----------------------------------------------------------------------------
template <bool EUCLID>
__device__ __forceinline__ double colour_cost(double x0, double x1, double x2, double y0, double y1, double y2) {
  double dx = d_sub(x0, y0), dy = d_sub(x1, y1), dz = d_sub(x2, y2);
  double d2 = d_add(d_add(d_mul(dx, dx), d_mul(dy, dy)), d_mul(dz, dz));
  return EUCLID ? __dsqrt_rn(d2) : d2;
}
template <bool EUCLID>
__device__ __forceinline__ double colour_cost(float x0, float x1, float x2, float y0, float y1, float y2) {
  float dx = __fsub_rn(x0, y0), dy = __fsub_rn(x1, y1), dz = __fsub_rn(x2, y2);
  float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
  return EUCLID ? (double)__fsqrt_rn(d2) : (double)d2;
}

// Device status word: first error wins.
__device__ __forceinline__ void set_status(int* st, int code) { atomicCAS(st, 0, code); }

}  // namespace sro
