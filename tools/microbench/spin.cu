// Keep-alive kernel for the single-CTA issue-throttle experiment (tools/throttle_probe.py):
// nblocks CTAs of 32 threads spin for `cycles` SM clocks, issuing (mode 0) or in __nanosleep (mode 1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libspin.so spin.cu
#include <cuda_runtime.h>
__global__ void k_spin(long long cycles, int mode, int* sink) {
  const long long t0 = clock64();
  int acc = 0;
  while (clock64() - t0 < cycles) {
    if (mode) __nanosleep(1000);
    else acc += (int)clock64() & 1;
  }
  if (acc == 0x7fffffff) *sink = acc;
}
extern "C" int spin(int nblocks, long long cycles, int mode, void* stream, int* sink) {
  k_spin<<<nblocks, 32, 0, (cudaStream_t)stream>>>(cycles, mode, sink);
  return (int)cudaGetLastError();
}
