// Dependent-chain latency of FFMA, FFMA2, FMUL2, FADD2 and MUFU.RSQ on sm_100a (one warp).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k(float* out, long long* cyc, float s0, float s1, int n) {
  float a = threadIdx.x * 1e-3f;
  u64 p, b, c;
  asm("mov.b64 %0, {%1, %1};" : "=l"(p) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s0));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(s1));
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(s0), "f"(s1));
  }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p) : "l"(b), "l"(c));
  }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) asm volatile("mul.f32x2 %0, %0, %1;" : "+l"(p) : "l"(b));
  }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) asm volatile("add.f32x2 %0, %0, %1;" : "+l"(p) : "l"(c));
  }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a));
  }
  long long t5 = clock64();
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p));
  out[threadIdx.x] = a + x + y;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 32 * sizeof(float));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const int n = 256;
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(out, cyc, 0.999f, 1e-3f, n); cudaDeviceSynchronize(); }
  const char* nm[5] = {"FFMA", "FFMA2", "FMUL2", "FADD2", "MUFU.RSQ"};
  for (int i = 0; i < 5; ++i) printf("%-9s latency %.2f cycles\n", nm[i], (double)cyc[i] / (n * 32));
  return 0;
}
