// Microbenchmarks that fix the roofline denominators SURVEY.md §8(d.4) asks for
// before any hot-path kernel is tuned: device properties, read-only stream
// ceiling (fp32 column sweep with an fp64 add+argmin per entry), FP64 / FP32
// issue rates, single-CTA dependent-step latency and grid-barrier latency.
// Not part of the product; run once per box image via gpurun.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void fill(float* p, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) p[i] = (float)((i * 2654435761u) & 0xffffff) * (1.0f / 16777216.0f);
}

// plain read: sum of floats, float4 loads, unroll 4
__global__ void read_sum(const float4* __restrict__ p, size_t n4, float* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t s = (size_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (; i + 3 * s < n4; i += 4 * s) {
    float4 a = __ldcs(p + i), b = __ldcs(p + i + s), c = __ldcs(p + i + 2 * s), d = __ldcs(p + i + 3 * s);
    acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + c.x + c.y + c.z + c.w + d.x + d.y + d.z + d.w;
  }
  for (; i < n4; i += s) { float4 a = p[i]; acc += a.x + a.y + a.z + a.w; }
  if (acc == 12345.f) *out = acc;
}

// column argmin: column-major m x n fp32, fp64 h in smem, one CTA handles a
// column slab of `cols_per_cta` columns; block = 256, each warp one column at a time
template <int M>
__global__ void col_argmin(const float* __restrict__ C, const double* __restrict__ h, int n,
                           int* __restrict__ jout, double* __restrict__ vout) {
  __shared__ double sh[M];
  for (int k = threadIdx.x; k < M; k += blockDim.x) sh[k] = h[k];
  __syncthreads();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nw = blockDim.x >> 5;
  for (int col = blockIdx.x * nw + warp; col < n; col += gridDim.x * nw) {
    const float4* c4 = reinterpret_cast<const float4*>(C + (size_t)col * M);
    double best = 1e300; int bj = 0;
#pragma unroll 4
    for (int q = lane; q < M / 4; q += 32) {
      float4 v = __ldcs(c4 + q);
      int k = q * 4;
      double x0 = (double)v.x + sh[k], x1 = (double)v.y + sh[k + 1], x2 = (double)v.z + sh[k + 2], x3 = (double)v.w + sh[k + 3];
      if (x0 < best) { best = x0; bj = k; }
      if (x1 < best) { best = x1; bj = k + 1; }
      if (x2 < best) { best = x2; bj = k + 2; }
      if (x3 < best) { best = x3; bj = k + 3; }
    }
    for (int o = 16; o; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffff, best, o); int oj = __shfl_xor_sync(0xffffffff, bj, o);
      if (ob < best || (ob == best && oj < bj)) { best = ob; bj = oj; }
    }
    if (lane == 0) { jout[col] = bj; vout[col] = best; }
  }
}

__global__ void fp64_rate(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001;
  for (int i = 0; i < iters; i++) {
    a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 0.123) *out = s;
}
__global__ void fp32_rate(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 1.0000001f, c = 0.999f;
  for (int i = 0; i < iters; i++) {
    a0 = fmaf(a0, c, b); a1 = fmaf(a1, c, b); a2 = fmaf(a2, c, b); a3 = fmaf(a3, c, b);
    a4 = fmaf(a4, c, b); a5 = fmaf(a5, c, b); a6 = fmaf(a6, c, b); a7 = fmaf(a7, c, b);
  }
  float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 0.123f) *out = s;
}
__global__ void dadd_latency(double* out, int iters, long long* cyc) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) a = __dadd_rn(a, 1.0000001);
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; *out = a; }
}
__global__ void ddiv_latency(double* out, int iters, long long* cyc) {
  double a = threadIdx.x + 3.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) a = __ddiv_rn(a, 1.0000001) + 0.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; *out = a; }
}

// single-CTA dependent step loop: column load (fp32 from L2/HBM) + 1024-thread argmin + tiny update of h
template <int M>
__global__ void step_loop(const float* __restrict__ C, double* h_g, const int* visit, int steps, int n, long long* cyc, int* out) {
  __shared__ double sh[M];
  __shared__ double wb[32]; __shared__ int wj[32]; __shared__ int jsel;
  for (int k = threadIdx.x; k < M; k += blockDim.x) sh[k] = h_g[k];
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int s = 0; s < steps; s++) {
    int col = visit[s];
    const float* c = C + (size_t)col * M;
    double best = 1e300; int bj = 0;
    for (int k = threadIdx.x * 4; k < M; k += blockDim.x * 4) {
      float4 v = *reinterpret_cast<const float4*>(c + k);
      double x0 = (double)v.x + sh[k], x1 = (double)v.y + sh[k + 1], x2 = (double)v.z + sh[k + 2], x3 = (double)v.w + sh[k + 3];
      if (x0 < best) { best = x0; bj = k; }
      if (x1 < best) { best = x1; bj = k + 1; }
      if (x2 < best) { best = x2; bj = k + 2; }
      if (x3 < best) { best = x3; bj = k + 3; }
    }
    for (int o = 16; o; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffff, best, o); int oj = __shfl_xor_sync(0xffffffff, bj, o);
      if (ob < best || (ob == best && oj < bj)) { best = ob; bj = oj; }
    }
    if (lane == 0) { wb[warp] = best; wj[warp] = bj; }
    __syncthreads();
    if (warp == 0) {
      int nw = blockDim.x >> 5;
      best = lane < nw ? wb[lane] : 1e300; bj = lane < nw ? wj[lane] : 0x7fffffff;
      for (int o = 16; o; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffff, best, o); int oj = __shfl_xor_sync(0xffffffff, bj, o);
        if (ob < best || (ob == best && oj < bj)) { best = ob; bj = oj; }
      }
      if (lane == 0) { jsel = bj; sh[bj] = __dadd_rn(sh[bj], 1e-3); }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; *out = jsel; }
}

__global__ void grid_sync_loop(int iters, long long* cyc) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d,\"mem_bytes\":%zu,\"cc\":\"%d.%d\"}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.regsPerMultiprocessor, clk, p.totalGlobalMem, p.major, p.minor);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // stream read ceiling over 16 GiB fp32 (the [3] matrix size)
  size_t n = (size_t)1 << 32;  // 2^32 floats = 16 GiB
  float* C; CK(cudaMalloc(&C, n * sizeof(float)));
  fill<<<sms * 8, 1024>>>(C, n); CK(cudaDeviceSynchronize());
  float* dout; CK(cudaMalloc(&dout, 64));
  for (int bpsm : {4, 8, 16}) {
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(e0); read_sum<<<sms * bpsm, 256>>>((const float4*)C, n / 4, dout); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"bench\":\"read_sum\",\"blocks_per_sm\":%d,\"ms\":%.4f,\"GBps\":%.1f}\n", bpsm, best, n * 4.0 / best / 1e6);
  }
  // column argmin over 65536 x 65536 fp32 with fp64 add
  {
    const int M = 65536; int ncol = (int)(n / M);
    // M=65536 doubles do not fit smem; use M=4096 view: columns of 4096 rows
  }
  {
    const int M = 4096; int ncol = (int)(n / M);
    double* h; CK(cudaMalloc(&h, M * 8)); CK(cudaMemset(h, 0, M * 8));
    int* j; double* v; CK(cudaMalloc(&j, ncol * 4)); CK(cudaMalloc(&v, ncol * 8));
    for (int bpsm : {2, 4, 6}) {
      float best = 1e30f;
      for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0); col_argmin<M><<<sms * bpsm, 256>>>(C, h, ncol, j, v); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"bench\":\"col_argmin_f32_f64add\",\"m\":%d,\"blocks_per_sm\":%d,\"ms\":%.4f,\"GBps\":%.1f,\"entries_per_s\":%.3e}\n",
             M, bpsm, best, n * 4.0 / best / 1e6, n / (best * 1e-3));
    }
    CK(cudaFree(h)); CK(cudaFree(j)); CK(cudaFree(v));
  }
  // fp64 / fp32 rates
  {
    int iters = 1 << 16;
    cudaEventRecord(e0); fp64_rate<<<sms * 8, 256>>>((double*)dout, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 8 * 256 * iters * 8;
    printf("{\"bench\":\"dadd_rate\",\"Gops\":%.1f,\"per_sm_per_clk_at_1965\":%.2f}\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); fp32_rate<<<sms * 8, 256>>>((float*)dout, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\":\"ffma_rate\",\"Gops\":%.1f,\"per_sm_per_clk_at_1965\":%.2f}\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    long long* cyc; CK(cudaMallocManaged(&cyc, 8));
    dadd_latency<<<1, 32>>>((double*)dout, 4096, cyc); CK(cudaDeviceSynchronize());
    printf("{\"bench\":\"dadd_latency_cyc\",\"value\":%.2f}\n", *cyc / 4096.0);
    ddiv_latency<<<1, 32>>>((double*)dout, 1024, cyc); CK(cudaDeviceSynchronize());
    printf("{\"bench\":\"ddiv_plus_dadd_latency_cyc\",\"value\":%.2f}\n", *cyc / 1024.0);
    // single-CTA step loop at m=4096 (C region 64 MiB -> L2 resident after first touch)
    {
      const int M = 4096, ncol = 4096, steps = 20000;
      int* visit; CK(cudaMallocManaged(&visit, steps * 4));
      uint64_t s = 1; for (int i = 0; i < steps; i++) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; visit[i] = (int)((s >> 33) % ncol); }
      double* h; CK(cudaMalloc(&h, M * 8)); CK(cudaMemset(h, 0, M * 8));
      int* o; CK(cudaMalloc(&o, 4));
      for (int threads : {256, 512, 1024}) {
        step_loop<M><<<1, threads>>>(C, h, visit, steps, ncol, cyc, o); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); step_loop<M><<<1, threads>>>(C, h, visit, steps, ncol, cyc, o); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"single_cta_step\",\"m\":%d,\"threads\":%d,\"us_per_step\":%.3f,\"cyc_per_step\":%.1f}\n", M, threads, ms * 1e3 / steps, *cyc / (double)steps);
      }
    }
    // grid sync latency
    {
      int iters = 10000; void* args[] = {&iters, &cyc};
      for (int bpsm : {1, 2}) {
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((void*)grid_sync_loop, sms * bpsm, 256, args, 0, 0));
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"grid_sync\",\"blocks\":%d,\"us_per_sync\":%.3f}\n", sms * bpsm, ms * 1e3 / iters);
      }
    }
  }
  // kernel launch overhead (empty kernel back-to-back) and graph replay
  CK(cudaFree(C));
  printf("{\"done\":1}\n");
  return 0;
}
