// Column fetch latency (the GA LMO critical path): one CTA of 512 threads, 384 of
// them load a random column of an m x n fp32 matrix (3 float4 + tail per thread)
// and block-reduce; clock64 per iteration. Sizes: 16 MB (L2-resident) vs 64 MB.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o colfetch colfetch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fetch(const float4* __restrict__ C, int m, int n, int iters, long long* out, float* sink) {
  __shared__ float red[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nvec = m / 4;
  unsigned x = 12345u;
  float acc = 0.f;
  long long tsum = 0, tload = 0;
  for (int it = 0; it < iters; it++) {
    x = x * 1664525u + 1013904223u;
    const int col = (int)(x % (unsigned)n);
    __syncthreads();
    const long long t0 = clock64();
    float v = 0.f;
    if (tid < 384) {
      const float4* p = C + (size_t)col * nvec;
      float4 a[3];
#pragma unroll
      for (int u = 0; u < 3; u++) { const int q = tid + u * 384; a[u] = q < nvec ? __ldg(p + q) : make_float4(0, 0, 0, 0); }
#pragma unroll
      for (int u = 0; u < 3; u++) v += a[u].x + a[u].y + a[u].z + a[u].w;
    }
    const long long t1 = clock64();
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    const long long t2 = clock64();
    if (tid == 0) { float s = 0; for (int w = 0; w < 16; w++) s += red[w]; acc += s; }
    tsum += t2 - t0; tload += t1 - t0;
  }
  if (tid == 0) { out[0] = tsum / iters; out[1] = tload / iters; *sink = acc; }
}

int main() {
  const int m = 4096;
  for (int n : {1024, 4096, 8192}) {
    float4* C; long long* out; float* sink;
    cudaMalloc(&C, (size_t)m * n * 4); cudaMalloc(&out, 16); cudaMalloc(&sink, 4);
    cudaMemset(C, 0, (size_t)m * n * 4);
    for (int rep = 0; rep < 3; rep++) {
      k_fetch<<<1, 512>>>(C, m, n, 20000, out, sink);
      long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("{\"matrix_MB\": %d, \"rep\": %d, \"cycles_per_iter\": %lld, \"load_cycles_thread0\": %lld}\n", (int)((size_t)m * n * 4 >> 20), rep, h[0], h[1]);
    }
    cudaFree(C); cudaFree(out); cudaFree(sink);
  }
  return 0;
}
