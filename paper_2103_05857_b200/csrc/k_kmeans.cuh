// k_kmeans.cuh — the colour-transfer front end: k-means
// quantisation of an 8-bit RGB image into k colours with their pixel histogram
// (readings R28-R30 in DESIGN.md).
//
// Lloyd iterations, every quantity exact or correctly rounded so the result is
// bit-identical to the oracle whatever the thread order:
//   * assignment: ((d0^2 + d1^2) + d2^2) in fp64 against every centroid (staged
//     in shared memory, broadcast reads), first minimum; four pixels per thread;
//   * update: integer channel sums and counts (64-bit integer atomics: order-free),
//     centroid = sum / count (one correctly rounded division);
//   * empty-cluster repair: the pixel farthest from its own centroid (first
//     maximum: an atomicMax over the fp64 bit pattern, then an atomicMin over the
//     indices attaining it), one empty cluster at a time in ascending order.
#pragma once
#include "sro_device.cuh"

namespace sro {

constexpr int KM_THREADS = 256;
constexpr int KM_PIX = 4;          // pixels per thread in the assignment
constexpr int KM_KMAX = 8192;      // centroids staged in shared memory (3 x 4 B each)

__global__ void k_km_init(const uint8_t* __restrict__ px, const int32_t* __restrict__ init, int k, double* cen) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    const int64_t p = init[c];
    cen[c] = (double)px[3 * p];
    cen[k + c] = (double)px[3 * p + 1];
    cen[2 * k + c] = (double)px[3 * p + 2];
  }
}

// Nearest centroid of every pixel; labels, changed count, integer sums and counts.
// An fp32 distance d_f is within M = 0.085 of the binary64 distance d for pixels and
// centroids in [0, 255] (|fl32(c) - c| <= 2^-24 256, then the subtractions, squares and
// sums of the fp32 formula), so a centroid can only match or beat the exact minimum
// if its d_f is at most the running fp32 minimum + 2M: only those (centroids in index
// order, margin 0.5) are evaluated exactly, with the same first-minimum rule, and the
// result is the exhaustive binary64 argmin. The fp32 centroid copy is in shared
// memory, the binary64 one is read (L1) only for candidates.
__global__ void __launch_bounds__(KM_THREADS) k_km_assign(const uint8_t* __restrict__ px, int64_t N,
                                                         const double* __restrict__ cen, int k, int32_t* labels,
                                                         unsigned long long* sums, unsigned long long* counts,
                                                         unsigned long long* changed) {
  extern __shared__ float kcf[];   // planar fp32: c0[k], c1[k], c2[k]
  for (int c = threadIdx.x; c < 3 * k; c += blockDim.x) kcf[c] = __double2float_rn(cen[c]);
  __syncthreads();
  constexpr float MARGIN = 0.5f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * KM_PIX;
  unsigned long long nchg = 0;
  for (int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * KM_PIX; p0 - (int64_t)(threadIdx.x & 31) * KM_PIX < N;
       p0 += stride) {
    // (the loop runs while any lane of the warp has pixels: the warp votes below)
    float f0[KM_PIX], f1[KM_PIX], f2[KM_PIX], bf[KM_PIX];
    double best[KM_PIX];
    int bj[KM_PIX];
#pragma unroll
    for (int q = 0; q < KM_PIX; q++) {
      const int64_t p = p0 + q < N ? p0 + q : N - 1;
      f0[q] = (float)px[3 * p]; f1[q] = (float)px[3 * p + 1]; f2[q] = (float)px[3 * p + 2];
      bf[q] = __int_as_float(0x7f800000);
      best[q] = __longlong_as_double(0x7ff0000000000000LL);
      bj[q] = 0;
    }
    for (int c = 0; c < k; c++) {
      const float c0 = kcf[c], c1 = kcf[k + c], c2 = kcf[2 * k + c];
      float df[KM_PIX];
      bool cand[KM_PIX];
      bool any = false;
#pragma unroll
      for (int q = 0; q < KM_PIX; q++) {
        const float e0 = __fsub_rn(f0[q], c0), e1 = __fsub_rn(f1[q], c1), e2 = __fsub_rn(f2[q], c2);
        df[q] = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
        cand[q] = df[q] <= __fadd_ru(bf[q], MARGIN);
        any |= cand[q];
      }
      if (__any_sync(FULL, any)) {
        const double c0d = cen[c], c1d = cen[k + c], c2d = cen[2 * k + c];
#pragma unroll
        for (int q = 0; q < KM_PIX; q++) {
          if (!cand[q]) continue;
          const double d0 = d_sub((double)f0[q], c0d), d1 = d_sub((double)f1[q], c1d), d2 = d_sub((double)f2[q], c2d);
          const double d = d_add(d_add(d_mul(d0, d0), d_mul(d1, d1)), d_mul(d2, d2));
          if (d < best[q]) { best[q] = d; bj[q] = c; }
        }
      }
#pragma unroll
      for (int q = 0; q < KM_PIX; q++) bf[q] = fminf(bf[q], df[q]);
    }
#pragma unroll
    for (int q = 0; q < KM_PIX; q++) {
      const int64_t p = p0 + q;
      if (p >= N) break;
      const int j = bj[q];
      nchg += labels[p] != j;
      labels[p] = j;
      atomicAdd(&counts[j], 1ULL);
      atomicAdd(&sums[3 * j], (unsigned long long)px[3 * p]);
      atomicAdd(&sums[3 * j + 1], (unsigned long long)px[3 * p + 1]);
      atomicAdd(&sums[3 * j + 2], (unsigned long long)px[3 * p + 2]);
    }
  }
  for (int o = 16; o; o >>= 1) nchg += __shfl_xor_sync(FULL, nchg, o);
  if ((threadIdx.x & 31) == 0 && nchg) atomicAdd(changed, nchg);
}

// centroid = sum / count for every non-empty class; empties counted.
__global__ void k_km_update(const unsigned long long* __restrict__ sums, const unsigned long long* __restrict__ counts,
                            int k, double* cen, unsigned long long* nempty) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    const unsigned long long n = counts[c];
    if (n == 0) { atomicAdd(nempty, 1ULL); continue; }
    const double dn = (double)n;
    cen[c] = d_div((double)sums[3 * c], dn);
    cen[k + c] = d_div((double)sums[3 * c + 1], dn);
    cen[2 * k + c] = d_div((double)sums[3 * c + 2], dn);
  }
}

__device__ __forceinline__ double km_own_dist(const uint8_t* px, const double* cen, int k, int64_t p, int j) {
  const double d0 = d_sub((double)px[3 * p], cen[j]), d1 = d_sub((double)px[3 * p + 1], cen[k + j]);
  const double d2 = d_sub((double)px[3 * p + 2], cen[2 * k + j]);
  return d_add(d_add(d_mul(d0, d0), d_mul(d1, d1)), d_mul(d2, d2));
}
// pass 1: the largest distance to the own centroid among pixels whose class keeps a member
__global__ void k_km_far_max(const uint8_t* __restrict__ px, int64_t N, const double* __restrict__ cen, int k,
                             const int32_t* __restrict__ labels, const unsigned long long* __restrict__ counts,
                             unsigned long long* dmax) {
  unsigned long long best = 0ULL;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
    const int j = labels[p];
    if (counts[j] <= 1) continue;
    // d >= 0: its bit pattern orders as the value; +1 so that 0 means "no candidate"
    const unsigned long long key = (unsigned long long)__double_as_longlong(km_own_dist(px, cen, k, p, j)) + 1ULL;
    if (key > best) best = key;
  }
  if (best) atomicMax(dmax, best);
}
// pass 2: the lowest index attaining it
__global__ void k_km_far_arg(const uint8_t* __restrict__ px, int64_t N, const double* __restrict__ cen, int k,
                             const int32_t* __restrict__ labels, const unsigned long long* __restrict__ counts,
                             const unsigned long long* __restrict__ dmax, unsigned long long* parg) {
  const unsigned long long want = *dmax;
  if (want == 0ULL) return;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
    const int j = labels[p];
    if (counts[j] <= 1) continue;
    const unsigned long long key = (unsigned long long)__double_as_longlong(km_own_dist(px, cen, k, p, j)) + 1ULL;
    if (key == want) { atomicMin(parg, (unsigned long long)p); break; }
  }
}
// class c takes pixel *parg (if any)
__global__ void k_km_move(const uint8_t* __restrict__ px, int k, int c, const unsigned long long* __restrict__ parg,
                          double* cen, int32_t* labels, unsigned long long* counts, int* moved) {
  const unsigned long long p = *parg;
  if (p == ~0ULL) return;
  cen[c] = (double)px[3 * p];
  cen[k + c] = (double)px[3 * p + 1];
  cen[2 * k + c] = (double)px[3 * p + 2];
  counts[labels[p]] -= 1ULL;
  labels[p] = c;
  counts[c] = 1ULL;
  *moved = 1;
}

// every pixel takes its class's projected colour, rint(255 x_hat) clipped to 0..255.
__global__ void k_km_recolour(const int32_t* __restrict__ labels, int64_t N, const double* __restrict__ xhat,
                              uint8_t* out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 3 * N; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = q / 3;
    const int t = (int)(q - 3 * p);
    double v = rint(d_mul(255.0, xhat[3 * (int64_t)labels[p] + t]));
    v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
    out[q] = (uint8_t)v;
  }
}

// ---------------------------------------------------------------------------
// k-means++ seeding (R34): D2(p) = min over the chosen centres of the
// squared RGB distance (8-bit pixels: exact integers <= 3 x 255^2), the next centre the first pixel
// whose inclusive prefix of D2 exceeds min(floor(u_t * total), total - 1). Integer sums: the
// parallel order cannot change them.
// ---------------------------------------------------------------------------
constexpr int KPP_BLOCK = 4096;   // pixels per partial sum (and per k_kpp_update CTA)

// D2 <- min(D2, d2(., centre)) (first: D2 = d2) over one 4096-pixel block per CTA; block sums.
__global__ void __launch_bounds__(256) k_kpp_update(const uint8_t* __restrict__ px, int64_t N,
                                                     const int32_t* __restrict__ centre, int first,
                                                     int32_t* d2, long long* bsum) {
  __shared__ long long red[8];
  const int64_t b0 = (int64_t)blockIdx.x * KPP_BLOCK;
  const int64_t c = *centre;
  const int c0 = px[3 * c], c1 = px[3 * c + 1], c2 = px[3 * c + 2];
  long long acc = 0;
  for (int64_t p = b0 + threadIdx.x; p < N && p < b0 + KPP_BLOCK; p += 256) {
    const int e0 = (int)px[3 * p] - c0, e1 = (int)px[3 * p + 1] - c1, e2 = (int)px[3 * p + 2] - c2;
    int v = (e0 * e0 + e1 * e1) + e2 * e2;
    if (!first) v = min(v, d2[p]);
    d2[p] = v;
    acc += v;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < 8; w++) t += red[w];
    bsum[blockIdx.x] = t;
  }
}

// Exclusive prefix over x[0..n) by one CTA of 1024 threads: returns the index q of the element
// whose [prefix, prefix + x_q) holds target (0 <= target < total), and that prefix in *base.
__device__ __forceinline__ long long kpp_find(const long long* x, int64_t n, long long target, long long* base,
                                              long long* sh) {
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t lo = min(n, t * per), hi = min(n, lo + per);
  long long s = 0;
  for (int64_t q = lo; q < hi; q++) s += x[q];
  // inclusive scan of the 1024 thread sums
  long long incl = s;
  for (int o = 1; o < 32; o <<= 1) { const long long y = __shfl_up_sync(FULL, incl, o); if ((t & 31) >= o) incl += y; }
  if ((t & 31) == 31) sh[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    long long w = sh[t];
    for (int o = 1; o < 32; o <<= 1) { const long long y = __shfl_up_sync(FULL, w, o); if (t >= o) w += y; }
    sh[t] = w;
  }
  __syncthreads();
  const long long start = incl - s + ((t >> 5) ? sh[(t >> 5) - 1] : 0);
  __shared__ long long res[2];
  if (s > 0 && start <= target && target < start + s) {   // exactly one thread: its range holds target
    long long run = start;
    int64_t q = lo;
    while (run + x[q] <= target) { run += x[q]; q++; }
    res[0] = q;
    res[1] = run;
  }
  __syncthreads();
  *base = res[1];
  const long long q = res[0];
  __syncthreads();
  return q;
}

// Centre t: from the block sums and D2 (one CTA of 1024 threads); the total-0 case takes the lowest
// pixel not yet chosen.
__global__ void __launch_bounds__(1024) k_kpp_pick(const int32_t* __restrict__ d2, int64_t N,
                                                    const long long* __restrict__ bsum, int64_t nb,
                                                    const double* __restrict__ u, int t, int32_t* centres,
                                                    int32_t* centre, uint8_t* chosen) {
  __shared__ long long sh[32];
  __shared__ long long stot[1];
  __shared__ int64_t sfirst;
  const int tid = threadIdx.x;
  long long s = 0;
  for (int64_t q = tid; q < nb; q += 1024) s += bsum[q];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if ((tid & 31) == 0) sh[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    long long tot = 0;
    for (int w = 0; w < 32; w++) tot += sh[w];
    stot[0] = tot;
    sfirst = N;
  }
  __syncthreads();
  const long long total = stot[0];
  int64_t pick;
  if (total == 0) {
    for (int64_t p = tid; p < N; p += 1024)
      if (!chosen[p]) { atomicMin((unsigned long long*)&sfirst, (unsigned long long)p); break; }
    __syncthreads();
    pick = sfirst;
  } else {
    long long target = (long long)d_mul(u[t], (double)total);   // one rounded product, then floor
    if (target > total - 1) target = total - 1;
    long long base = 0;
    const long long b = kpp_find(bsum, nb, target, &base, sh);
    // within block b: the D2 values as long long, found the same way
    __shared__ long long vals[KPP_BLOCK];
    const int64_t p0 = b * KPP_BLOCK;
    const int64_t cnt = min((int64_t)KPP_BLOCK, N - p0);
    for (int64_t q = tid; q < cnt; q += 1024) vals[q] = d2[p0 + q];
    __syncthreads();
    long long base2 = 0;
    const long long q = kpp_find(vals, cnt, target - base, &base2, sh);
    pick = p0 + q;
  }
  if (tid == 0) {
    centres[t] = (int32_t)pick;
    *centre = (int32_t)pick;
    chosen[pick] = 1;
  }
}

}  // namespace sro
