// Column fetch latency, LDG against bulk asynchronous copies (cp.async.bulk, TMA engine):
// one CTA of 512 threads; each iteration picks a random column of an m x n fp32 matrix
// (m = 4096: 16 KB) and 384 threads reduce it. clock64 cycles per iteration.
//   mode 0: 3 x LDG.128 + tail per thread (the GA kernel's pattern)
//   mode 1: one 16 KB bulk copy by thread 0 onto one mbarrier, then LDS.128
//   mode 2: 16 x 1 KB bulk copies by 16 lanes of warp 0 onto one mbarrier
//   mode 3: per warp: lane 0 copies the warp's three 512 B pieces onto the warp's own mbarrier
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o colfetch_tma colfetch_tma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  }
}

__global__ void k_fetch(const float4* __restrict__ C, int m, int n, int iters, int mode, long long* out, float* sink) {
  __shared__ __align__(128) float4 buf[1024];
  __shared__ uint64_t bars[16];
  __shared__ float red[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nvec = m / 4;
  if (tid < 16) mbar_init(&bars[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned x = 12345u;
  float acc = 0.f;
  long long tsum = 0;
  for (int it = 0; it < iters; it++) {
    x = x * 1664525u + 1013904223u;
    const int col = (int)(x % (unsigned)n);
    const float4* p = C + (size_t)col * nvec;
    __syncthreads();
    const long long t0 = clock64();
    float v = 0.f;
    if (mode == 0) {
      if (tid < 384) {
        float4 a[3];
#pragma unroll
        for (int u = 0; u < 3; u++) { const int q = tid + u * 384; a[u] = q < nvec ? __ldg(p + q) : make_float4(0, 0, 0, 0); }
#pragma unroll
        for (int u = 0; u < 3; u++) v += a[u].x + a[u].y + a[u].z + a[u].w;
      }
    } else if (mode == 1 || mode == 2) {
      if (mode == 1 && tid == 0) { mbar_expect_tx(&bars[0], 16384); bulk_g2s(buf, p, 16384, &bars[0]); }
      if (mode == 2 && warp == 0) {
        if (lane == 0) mbar_expect_tx(&bars[0], 16384);
        __syncwarp();
        if (lane < 16) bulk_g2s(buf + lane * 64, p + lane * 64, 1024, &bars[0]);
      }
      mbar_wait(&bars[0], it & 1);
      if (tid < 384) {
#pragma unroll
        for (int u = 0; u < 3; u++) { const int q = tid + u * 384; if (q < nvec) { const float4 a = buf[q]; v += a.x + a.y + a.z + a.w; } }
      }
    } else {
      if (warp < 12) {
        if (lane == 0) {
          mbar_expect_tx(&bars[warp], 3 * 512 - (warp * 32 + 768 >= nvec ? 512 : 0));
#pragma unroll
          for (int u = 0; u < 3; u++) {
            const int q = warp * 32 + u * 384;
            if (q < nvec) bulk_g2s(buf + q, p + q, 512, &bars[warp]);
          }
        }
        mbar_wait(&bars[warp], it & 1);
#pragma unroll
        for (int u = 0; u < 3; u++) { const int q = tid + u * 384; if (q < nvec) { const float4 a = buf[q]; v += a.x + a.y + a.z + a.w; } }
      }
    }
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    const long long t2 = clock64();
    if (tid == 0) { float s = 0; for (int w = 0; w < 16; w++) s += red[w]; acc += s; }
    tsum += t2 - t0;
  }
  if (tid == 0) { out[0] = tsum / iters; *sink = acc; }
}

int main() {
  const int m = 4096;
  for (int n : {1024, 4096}) {
    float4* C; long long* out; float* sink;
    cudaMalloc(&C, (size_t)m * n * 4); cudaMalloc(&out, 16); cudaMalloc(&sink, 4);
    cudaMemset(C, 0, (size_t)m * n * 4);
    for (int mode = 0; mode < 4; mode++)
      for (int rep = 0; rep < 2; rep++) {
        k_fetch<<<1, 512>>>(C, m, n, 20000, mode, out, sink);
        long long h[2] = {0, 0};
        cudaError_t e = cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("{\"matrix_MB\": %d, \"mode\": %d, \"rep\": %d, \"cycles_per_iter\": %lld, \"err\": \"%s\"}\n",
               (int)((size_t)m * n * 4 >> 20), mode, rep, h[0], cudaGetErrorString(e));
      }
    cudaFree(C); cudaFree(out); cudaFree(sink);
  }
  return 0;
}
