// Issue cost of the LMO scan's fp64 operations on one SM (16 warps, independent
// streams): cycles per warp-instruction for F2F.F64.F32, DADD, DSETP, FSEL.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f2f f2f.cu
#include <cstdio>
#define N 4096
__global__ void k(const float* in, double* out, long long* cyc) {
  float f[8];
  for (int q = 0; q < 8; q++) f[q] = in[threadIdx.x * 8 + q];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; it++) {
#pragma unroll
    for (int q = 0; q < 8; q++) acc[q] += (double)f[q];   // F2F + DADD
#pragma unroll
    for (int q = 0; q < 8; q++) f[q] = __int_as_float(__float_as_int(f[q]) ^ 1);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int q = 0; q < 8; q++) s += acc[q];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DADD only
  double a2[8];
  for (int q = 0; q < 8; q++) a2[q] = (double)f[q];
  __syncthreads();
  t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; it++) {
#pragma unroll
    for (int q = 0; q < 8; q++) a2[q] = __dadd_rn(a2[q], 1.0);
  }
  __syncthreads();
  t1 = clock64();
  s = 0;
  for (int q = 0; q < 8; q++) s += a2[q];
  out[threadIdx.x] += s;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 512 * 8 * 4); cudaMalloc(&out, 512 * 8); cudaMalloc(&cyc, 16);
  cudaMemset(in, 0, 512 * 8 * 4);
  k<<<1, 512>>>(in, out, cyc);
  long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps x 8 ops x N iterations
  printf("{\"f2f_plus_dadd_cycles_per_warp_op\": %.2f, \"dadd_cycles_per_warp_op\": %.2f}\n",
         (double)h[0] / (4.0 * 8 * N), (double)h[1] / (4.0 * 8 * N));
}
