// ptxas contraction of packed binary32 operations on sm_100a (round 2):
//   nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -cubin -o f32x2.cubin f32x2_contract.cu
//   cuobjdump -sass f32x2.cubin | grep -E "Function|FADD|FMUL|FFMA"
// k_packed_add: mul.rn.f32x2 feeding add.rn.f32x2 -> one FFMA2 (contracted despite .rn / --fmad=false)
// k_fma_m0:     fma.rn.f32x2(d, d, -0) feeding add.rn.f32x2 -> one FFMA2 as well
// k_scalar_add: mul.rn.f32x2, then the halves summed with scalar __fadd_rn -> FMUL2 + FADD (exact)
// k_bcast:      a broadcast scalar operand {x, x} folds into FADD2's .F32 operand form (no MOV)
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__global__ void k_packed_add(const float2* a, const float2* b, float2* c) {
  const int i = threadIdx.x;
  unsigned long long x = *(const unsigned long long*)&a[i], y = *(const unsigned long long*)&b[i], d, e;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(e) : "l"(d), "l"(d));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(e), "l"(x));
  *(unsigned long long*)&c[i] = d;
}
__global__ void k_fma_m0(const float2* a, const float2* b, float2* c) {
  const int i = threadIdx.x;
  unsigned long long x = *(const unsigned long long*)&a[i], y = *(const unsigned long long*)&b[i], d, e;
  const unsigned long long nz = 0x8000000080000000ULL;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(d), "l"(d), "l"(nz));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(e), "l"(x));
  *(unsigned long long*)&c[i] = d;
}
__global__ void k_scalar_add(const float2* a, const float2* b, float2* c) {
  const int i = threadIdx.x;
  unsigned long long x = *(const unsigned long long*)&a[i], y = *(const unsigned long long*)&b[i], d, e, f;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(e) : "l"(d), "l"(d));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(x), "l"(x));
  const float2 E = *(float2*)&e, F = *(float2*)&f;
  c[i] = make_float2(__fadd_rn(E.x, F.x), __fadd_rn(E.y, F.y));
}
__global__ void k_bcast(const float* a, const float2* b, float2* c) {
  const int i = threadIdx.x;
  const float x = a[i];
  unsigned long long y = *(const unsigned long long*)&b[i], d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(x, x)), "l"(y));
  *(unsigned long long*)&c[i] = d;
}
