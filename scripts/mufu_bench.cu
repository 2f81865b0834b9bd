// MUFU throughput micro-benchmark (sm_100a): warp-instructions per SM per clock for
// sqrt.approx / rsqrt.approx / ex2.approx / sqrt+ex2 mixes (8 independent chains per thread).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, float seed) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      if (OP == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      if (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      if (OP == 3) {
        if (i & 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
        else asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      }
      v[i] = y + 1.0f;
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  const char* names[] = {"sqrt", "rsqrt", "ex2", "sqrt/ex2 mix"};
  for (int op = 0; op < 4; ++op) {
    for (int warps = 8; warps <= 32; warps *= 2) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto run = [&]() {
        if (op == 0) k<0><<<sms * 2, warps * 16>>>(d, iters, 0.5f);
        if (op == 1) k<1><<<sms * 2, warps * 16>>>(d, iters, 0.5f);
        if (op == 2) k<2><<<sms * 2, warps * 16>>>(d, iters, 0.5f);
        if (op == 3) k<3><<<sms * 2, warps * 16>>>(d, iters, 0.5f);
      };
      run(); cudaEventRecord(a); run(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * 2 * warps * 16 * iters * 8;
      printf("%-14s warps/SM=%2d  %.3f ms  %.2f Tops/s  %.2f lanes/clk/SM at %d MHz\n", names[op], warps, ms,
             ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
