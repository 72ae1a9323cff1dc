// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) throughput on sm_100a, pure
// FP32 FMA chains (16 independent chains per thread, 64 warps per SM).
// Reports warp-instructions per cycle per SM sub-partition (SMSP) and FMAs
// per clock per SM, from clock64() deltas inside the kernel.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, long long* cyc, int iters, float s0, float s1) {
  float a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = threadIdx.x * 1e-3f + i;
  u64 p[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
  u64 bs, cs;
  asm("mov.b64 %0, {%1, %1};" : "=l"(bs) : "f"(s0));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cs) : "f"(s1));
  __syncthreads();
  long long t0 = clock64();
  for (int t = 0; t < iters; ++t) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s0), "f"(s1));
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = fma2(p[i], bs, cs);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) p[i] = fma2(p[i], bs, cs);
    }
  }
  long long t1 = clock64();
  float r = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) r += a[i];
#pragma unroll
  for (int i = 0; i < 16; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); r += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int blocks = 148 * 8, iters = 8192;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 256 * sizeof(float));
  cudaMallocManaged(&cyc, blocks * sizeof(long long));
  const char* names[3] = {"16 FFMA /iter ", "8 FFMA2 /iter ", "16 FFMA2 /iter"};
  const int inst[3] = {16, 8, 16}, fmas[3] = {16, 16, 32};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<blocks, 256>>>(out, cyc, iters, 0.999f, 1e-3f);
      if (mode == 1) k<1><<<blocks, 256>>>(out, cyc, iters, 0.999f, 1e-3f);
      if (mode == 2) k<2><<<blocks, 256>>>(out, cyc, iters, 0.999f, 1e-3f);
      cudaDeviceSynchronize();
    }
    double c = 0;
    for (int b = 0; b < blocks; ++b) c += cyc[b];
    c /= blocks;  // cycles per block (all 8 blocks of an SM run concurrently)
    // per SM: 64 warps x iters x inst warp-instructions over c cycles, 4 SMSPs
    const double wi_per_cyc_smsp = 64.0 * iters * inst[mode] / c / 4.0;
    printf("%s: %.0f cycles, %.3f warp-inst/cycle/SMSP, %.1f FMA/clk/SM\n", names[mode], c, wi_per_cyc_smsp,
           64.0 * 32 * iters * fmas[mode] / c);
  }
  return 0;
}
