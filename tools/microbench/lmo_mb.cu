// Single-CTA LMO microbenchmark (design evidence for k_bcfw, not product code):
// cycles per dependent LMO step over a 4096-row fp32 column for
//   v0: exact fp64 from smem column + smem fp64 h       (current generic)
//   v1: fp32 filter from smem column + smem fp32 h32    (k_bcfw v3)
//   v2: fp32 filter, column + h32 in registers           (register-resident)
//   v3: exact fp64, column in registers, h fp64 in regs
// each followed by the same REDUX CTA argmin and one __syncthreads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 512, M = 4096, NV = M / 4 / NT;  // 2 float4 per thread
__device__ __forceinline__ unsigned long long okey(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v + 0.0);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ void redux(unsigned long long& key, int& j) {
  unsigned hi = key >> 32, lo = (unsigned)key;
  unsigned m1 = __reduce_min_sync(0xffffffff, hi);
  unsigned m2 = __reduce_min_sync(0xffffffff, hi == m1 ? lo : 0xffffffffu);
  unsigned m3 = __reduce_min_sync(0xffffffff, (hi == m1 && lo == m2) ? (unsigned)j : 0x7fffffffu);
  key = ((unsigned long long)m1 << 32) | m2; j = m3;
}

template <int V>
__global__ void __launch_bounds__(NT, 1) lmo(const float* __restrict__ C, int iters, long long* out, int* jout) {
  extern __shared__ __align__(16) char dyn[];
  double* h = reinterpret_cast<double*>(dyn);
  float* col = reinterpret_cast<float*>(dyn + M * 8);
  float* h32 = reinterpret_cast<float*>(dyn + M * 12);
  __shared__ unsigned long long wk[16];
  __shared__ int wj[16];
  for (int k = threadIdx.x; k < M; k += NT) { col[k] = C[k]; h[k] = (k % 97) * 1e-3 - 0.05; h32[k] = (float)h[k]; }
  __syncthreads();
  float4 creg[NV], hreg[NV];
  double hd[NV * 4];
  for (int u = 0; u < NV; u++) {
    int q = threadIdx.x + u * NT;
    creg[u] = reinterpret_cast<float4*>(col)[q];
    hreg[u] = reinterpret_cast<float4*>(h32)[q];
    for (int t = 0; t < 4; t++) hd[u * 4 + t] = h[4 * q + t];
  }
  long long t0 = clock64();
  int jsum = 0;
  for (int it = 0; it < iters; it++) {
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bj = 0x7fffffff;
    if (V == 0) {
      for (int u = 0; u < NV; u++) {
        int q = threadIdx.x + u * NT;
        float4 c = reinterpret_cast<float4*>(col)[q];
        double2 h01 = reinterpret_cast<double2*>(h)[2 * q], h23 = reinterpret_cast<double2*>(h)[2 * q + 1];
        double x0 = (double)c.x + h01.x, x1 = (double)c.y + h01.y, x2 = (double)c.z + h23.x, x3 = (double)c.w + h23.y;
        int k = 4 * q;
        if (x0 < best) { best = x0; bj = k; }
        if (x1 < best) { best = x1; bj = k + 1; }
        if (x2 < best) { best = x2; bj = k + 2; }
        if (x3 < best) { best = x3; bj = k + 3; }
      }
    } else if (V == 1 || V == 2) {
      float4 cq[NV], fq[NV];
      float fmin = __int_as_float(0x7f800000);
      for (int u = 0; u < NV; u++) {
        int q = threadIdx.x + u * NT;
        float4 c = V == 1 ? reinterpret_cast<float4*>(col)[q] : creg[u];
        float4 hh = V == 1 ? reinterpret_cast<float4*>(h32)[q] : hreg[u];
        cq[u] = c;
        fq[u] = make_float4(c.x + hh.x, c.y + hh.y, c.z + hh.z, c.w + hh.w);
        fmin = fminf(fmin, fminf(fminf(fq[u].x, fq[u].y), fminf(fq[u].z, fq[u].w)));
      }
      float thr = __fadd_ru(fmin, 1e-6f);
      for (int u = 0; u < NV; u++) {
        int k = 4 * (threadIdx.x + u * NT);
        if (fq[u].x <= thr) { double v = (double)cq[u].x + h[k]; if (v < best) { best = v; bj = k; } }
        if (fq[u].y <= thr) { double v = (double)cq[u].y + h[k + 1]; if (v < best) { best = v; bj = k + 1; } }
        if (fq[u].z <= thr) { double v = (double)cq[u].z + h[k + 2]; if (v < best) { best = v; bj = k + 2; } }
        if (fq[u].w <= thr) { double v = (double)cq[u].w + h[k + 3]; if (v < best) { best = v; bj = k + 3; } }
      }
    } else {
      for (int u = 0; u < NV; u++) {
        int k = 4 * (threadIdx.x + u * NT);
        double x0 = (double)creg[u].x + hd[4 * u], x1 = (double)creg[u].y + hd[4 * u + 1];
        double x2 = (double)creg[u].z + hd[4 * u + 2], x3 = (double)creg[u].w + hd[4 * u + 3];
        if (x0 < best) { best = x0; bj = k; }
        if (x1 < best) { best = x1; bj = k + 1; }
        if (x2 < best) { best = x2; bj = k + 2; }
        if (x3 < best) { best = x3; bj = k + 3; }
      }
    }
    unsigned long long key = okey(best);
    redux(key, bj);
    if ((threadIdx.x & 31) == 0) { wk[threadIdx.x >> 5] = key; wj[threadIdx.x >> 5] = bj; }
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long k2 = threadIdx.x < 16 ? wk[threadIdx.x] : ~0ULL;
      int j2 = threadIdx.x < 16 ? wj[threadIdx.x] : 0x7fffffff;
      redux(k2, j2);
      if (threadIdx.x == 0) { jsum += j2; h[j2] += 1e-9; h32[j2] = (float)h[j2]; }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = t1 - t0; *jout = jsum; }
}

int main() {
  float* C; cudaMalloc(&C, M * 4);
  float hC[M]; uint64_t s = 7;
  for (int k = 0; k < M; k++) { s = s * 6364136223846793005ULL + 1; hC[k] = (float)((s >> 40) & 0xffffff) / 16777216.0f; }
  cudaMemcpy(C, hC, M * 4, cudaMemcpyHostToDevice);
  long long* o; int* j; cudaMallocManaged(&o, 8); cudaMallocManaged(&j, 4);
  const int iters = 20000;
  const int sm = M * 16;
  cudaFuncSetAttribute(lmo<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(lmo<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(lmo<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(lmo<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  lmo<0><<<1, NT, sm>>>(C, iters, o, j); cudaDeviceSynchronize(); printf("v0 exact smem  : %.1f cyc/step\n", *o / (double)iters);
  lmo<1><<<1, NT, sm>>>(C, iters, o, j); cudaDeviceSynchronize(); printf("v1 filter smem : %.1f cyc/step\n", *o / (double)iters);
  lmo<2><<<1, NT, sm>>>(C, iters, o, j); cudaDeviceSynchronize(); printf("v2 filter regs : %.1f cyc/step\n", *o / (double)iters);
  lmo<3><<<1, NT, sm>>>(C, iters, o, j); cudaDeviceSynchronize(); printf("v3 exact regs  : %.1f cyc/step\n", *o / (double)iters);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
