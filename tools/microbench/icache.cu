// Is the instruction cache warm at kernel launch? One CTA runs a ~48 KB straight-line code block
// twice (clock64 around each pass); the kernel is launched 5 times back to back, with and without
// a different kernel in between. First pass >> second pass on every launch => code fetched cold
// at each launch (the block tail's "no_instruction" stalls, profiles/r02_ncu_tail.md).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu
#include <cstdio>
__device__ __noinline__ float body(float x, float y) {
#pragma unroll
  for (int q = 0; q < 3000; q++) x = __fmaf_rn(x, y, (float)q * 0.37f);
  return x;
}
__global__ void k(float* out, long long* cyc, float y) {
  float x = threadIdx.x;
  long long t0 = clock64();
  x = body(x, y);
  __syncthreads();
  long long t1 = clock64();
  x = body(x, y);
  __syncthreads();
  long long t2 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
__global__ void other(float* out) { out[threadIdx.x + 1024] += 1.0f; }
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 8192 * 4); cudaMalloc(&cyc, 16);
  for (int mode = 0; mode < 2; mode++) {
    for (int l = 0; l < 5; l++) {
      k<<<1, 1024>>>(out, cyc, 1.0001f);
      if (mode) other<<<148, 256>>>(out);
      long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
      printf("{\"mode\": \"%s\", \"launch\": %d, \"pass1_cycles\": %lld, \"pass2_cycles\": %lld}\n",
             mode ? "with_other_kernel_between" : "back_to_back", l, h[0], h[1]);
    }
  }
}
