// Cycles per Fenwick draw (ga_draw of k_bcfw.cuh) on a 4096-column tree in shared memory.
#include <cstdio>
#include "../../paper_2103_05857_b200/csrc/k_bcfw.cuh"
using namespace sro;
__global__ void k(double* out, int n, int iters) {
  __shared__ double fen[2049];
  __shared__ double G[2048];
  for (int i = threadIdx.x; i <= n; i += blockDim.x) fen[i] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) G[i] = 1.0 + (i % 7);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i <= n; i++) fen[i] += G[i - 1];
    for (int i = 1; i <= n; i++) { int p = i + (i & -i); if (p <= n) fen[p] += fen[i]; }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      int ii = 0;
      const double u = uniform53(rng_u64(12345, 1, (uint64_t)(it + acc)));
      if (threadIdx.x == 0) ii = ga_draw_sh(fen, G, n, u);
      acc += __shfl_sync(0xffffffffu, ii, 0) & 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = acc; }
    // closed-form update path
    t0 = clock64();
    for (int it = 0; it < iters; it++) ga_add_warp(fen, n, (it * 2654435761u) % n, 1e-9);
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = (double)(t1 - t0) / iters;
    // rng only
    t0 = clock64();
    double s = 0;
    for (int it = 0; it < iters; it++) s += uniform53(rng_u64(12345, 1, (uint64_t)it + (s > 2 ? 1 : 0)));
    t1 = clock64();
    if (threadIdx.x == 0) { out[3] = (double)(t1 - t0) / iters; out[4] = s; }
  }
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int n = 2048;
  k<<<1, 256>>>(d, n, 4096);
  double h[5];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"draw_cycles\": %.1f, \"add_warp_cycles\": %.1f, \"rng_cycles\": %.1f, \"err\": \"%s\"}\n", h[0], h[2], h[3],
         cudaGetErrorString(cudaGetLastError()));
}
