// Latency microbenchmarks of the primitives on the sequential-BCFW critical path
// (one CTA; dependent chains timed with clock64). Output: JSON lines.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 4096

__global__ void k_lat(const double* __restrict__ gbuf, const int* __restrict__ gidx, long long* out, double* sink) {
  __shared__ double sd[1024];
  __shared__ int si[1024];
  __shared__ unsigned su[512];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int k = tid; k < 1024; k += blockDim.x) { sd[k] = 1.0 + k * 1e-9; si[k] = (k * 7 + 1) & 1023; }
  if (tid < 512) su[tid] = 0;
  __syncthreads();
  double acc = 1.0;
  int idx = tid & 1023;
  unsigned uv = tid;
  long long t0, t1;
  // 1. two CTA barriers per iteration (all warps)
  t0 = clock64();
  for (int it = 0; it < N_ITER; it++) { __syncthreads(); __syncthreads(); }
  t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / N_ITER;
  __syncthreads();
  if (tid < 32) {
    // 2. dependent LDS chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) idx = si[idx];
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0) / N_ITER;
    // 3. dependent SHFL chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) uv = __shfl_sync(0xffffffffu, uv, (uv + 1) & 31);
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0) / N_ITER;
    // 4. dependent REDUX chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) uv = __reduce_min_sync(0xffffffffu, uv + lane);
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0) / N_ITER;
    // 5. dependent BALLOT chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) uv = __ballot_sync(0xffffffffu, ((uv >> lane) & 1u) ^ (lane & 1));
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0) / N_ITER;
    // 6. dependent DADD chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) acc = __dadd_rn(acc, 1e-12);
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0) / N_ITER;
    // 7. dependent DDIV chain
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) acc = __ddiv_rn(acc, 1.0000001);
    t1 = clock64();
    if (tid == 0) out[6] = (t1 - t0) / N_ITER;
    // 8. dependent global (L2-resident) load chain
    int g = tid;
    t0 = clock64();
    for (int it = 0; it < N_ITER / 8; it++) g = __ldcg(gidx + g);
    t1 = clock64();
    if (tid == 0) out[7] = (t1 - t0) / (N_ITER / 8);
    // 9. shared atomicOr chain (dependent through the returned value)
    unsigned a = 1;
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) a = atomicOr(&su[(a + lane) & 511], a) | 1u;
    t1 = clock64();
    if (tid == 0) out[8] = (t1 - t0) / N_ITER;
    // 10. F2F.F64.F32 + DADD chain
    float f = 1.0f;
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) { acc = __dadd_rn((double)f, acc); f = (float)acc; }
    t1 = clock64();
    if (tid == 0) out[9] = (t1 - t0) / N_ITER;
    // 11. dependent DSETP/select chain (min tracking)
    double b = 1e300;
    t0 = clock64();
    for (int it = 0; it < N_ITER; it++) { const double x = sd[it & 1023] + acc; if (x < b) b = x; acc = b * 1e-30; }
    t1 = clock64();
    if (tid == 0) out[10] = (t1 - t0) / N_ITER;
    uv += g + a;
  }
  __syncthreads();
  // 12. barrier where warp 0 arrives late by a dependent LDS chain of 16 (handoff cost)
  t0 = clock64();
  for (int it = 0; it < N_ITER / 8; it++) {
    if (tid < 32) for (int q = 0; q < 16; q++) idx = si[idx];
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) out[11] = (t1 - t0) / (N_ITER / 8);
  // 13. named-barrier handoff: warp 0 arrives (bar.arrive), warps 1..15 sync; then reverse
  t0 = clock64();
  for (int it = 0; it < N_ITER; it++) {
    if (tid < 32) {
      asm volatile("bar.arrive 1, %0;" ::"r"(blockDim.x));
      asm volatile("bar.sync 2, %0;" ::"r"(blockDim.x));
    } else {
      asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x));
      asm volatile("bar.arrive 2, %0;" ::"r"(blockDim.x));
    }
  }
  t1 = clock64();
  if (tid == 0) out[12] = (t1 - t0) / N_ITER;
  if (acc == 0.123 || uv == 7u || idx == -5) *sink = acc + uv + idx;
}

int main() {
  double* gbuf; int* gidx; long long* out; double* sink;
  cudaMalloc(&gbuf, 1 << 20); cudaMalloc(&gidx, sizeof(int) * (1 << 22)); cudaMalloc(&out, 64 * 8); cudaMalloc(&sink, 8);
  // random-ish pointer chase over 16 MB (L2 resident after warm-up)
  int* h = (int*)malloc(sizeof(int) * (1 << 22));
  for (int q = 0; q < (1 << 22); q++) h[q] = (int)(((long long)q * 2654435761LL + 12345) & ((1 << 22) - 1));
  cudaMemcpy(gidx, h, sizeof(int) * (1 << 22), cudaMemcpyHostToDevice);
  const char* names[] = {"2xbar_512thr", "lds_dep", "shfl_dep", "redux_dep", "ballot_dep", "dadd_dep", "ddiv_dep",
                         "ldg_l2_dep", "atomicor_smem_dep", "f2f_dadd_dep", "dadd_min_dep", "bar_late16lds",
                         "named_bar_handoff_pair"};
  for (int rep = 0; rep < 2; rep++) {
    k_lat<<<1, 512>>>(gbuf, gidx, out, sink);
    cudaDeviceSynchronize();
  }
  long long r[13];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  for (int q = 0; q < 13; q++) printf("{\"bench\":\"%s\",\"cycles\":%lld}\n", names[q], r[q]);
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
