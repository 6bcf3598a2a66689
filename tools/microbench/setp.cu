// Dependent-chain latency of a Fenwick-descent level: compare f <= u, then select the next u
// (fp64 DSETP + FSEL, vs the same decision on the int64 bit patterns of nonnegative doubles).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o setp setp.cu
#include <cstdio>
#define N 4096
__global__ void k(const double* in, double* out, long long* cyc) {
  double u = in[0], f0 = in[1], f1 = in[2];
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; it++) {
    const bool t = f0 <= u;                 // DSETP
    const double un = __dsub_rn(u, f0);
    u = t ? un : u;                          // FSEL x2
    f0 = t ? f1 : f0;
  }
  long long t1 = clock64();
  out[0] = u + f0;
  cyc[0] = t1 - t0;
  long long ub = __double_as_longlong(u), fb = __double_as_longlong(f1);
  double ud = u;
  t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; it++) {
    const bool t = fb <= ub;                // 64-bit integer compare on the bit patterns
    const double un = __dsub_rn(ud, __longlong_as_double(fb));
    ud = t ? un : ud;
    ub = __double_as_longlong(ud);
    fb = t ? fb + 1 : fb;
  }
  t1 = clock64();
  out[1] = ud;
  cyc[1] = t1 - t0;
}
int main() {
  double h[3] = {1e300, 1e-300, 2e-300}; double* d; double* o; long long* c;
  cudaMalloc(&d, 24); cudaMalloc(&o, 16); cudaMalloc(&c, 16);
  cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o, c);
  long long hc[2]; cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("{\"dsetp_fsel_chain_cycles\": %.1f, \"isetp64_sel_chain_cycles\": %.1f}\n", (double)hc[0] / N, (double)hc[1] / N);
}
