// Microbenchmark: does FFMA2 (packed fma.rn.f32x2, sm_100a) save issue slots?
// Per iteration each thread runs 16 FP32 FMAs (as 16 FFMA or 8 FFMA2) plus
// 8 independent integer ops; all warps resident.  Prints ns per launch.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s0, float s1) {
  float a[16];
  unsigned q[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = threadIdx.x + i;
  for (int t = 0; t < iters; ++t) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s0, s1);
    } else {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        u64 v = fma2(pk(a[i], a[i + 1]), pk(s0, s0), pk(s1, s1));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[i + 1]) : "l"(v));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = (q[i] ^ (q[i] >> 3)) + 0x9e37u;
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) r += (float)q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, 0.999f, 1e-3f);
      else k<1><<<148 * 8, 256>>>(out, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) {
        double fma = 148.0 * 8 * 256 * iters * 16, iop = 148.0 * 8 * 256 * iters * 8 * 2;
        printf("mode %s: %.3f ms  %.1f TFMA/s  (int ops %.1f T/s)\n", mode ? "FFMA2" : "FFMA ", ms, fma / ms / 1e9,
               iop / ms / 1e9);
      }
    }
  }
  return 0;
}
