// kernels_peak.cu — live ALU peak measurement for the bench's roofline denominators (cakf_alu_peaks):
// the MUFU (XU pipe) rate of the sqrt.approx / ex2.approx mix that bounds K1 (two MUFU ops per kernel
// pair) and the FP64 tensor-core (DMMA) rate of the fp64-accumulating low-rank GEMM.  Eight independent dependency chains per
// thread, 32 warps per SM, so the pipes, not the latencies, bound the loops.
#include <cuda_runtime.h>

#include "../../include/cakf.h"
#include "common.cuh"
#include "internal.h"

namespace cakf {
namespace {

__global__ void mufu_peak_kernel(float* out, int iters, float seed, long long* cycles) {
  const long long t0 = clock64();
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (i & 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      else asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      v[i] = y + 1.0f;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = clock64() - t0;
}

__global__ void dmma_peak_kernel(double* out, int iters) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 1234.5) out[0] = s;
}

}  // namespace
}  // namespace cakf

using namespace cakf;

extern "C" int cakf_alu_peaks(double* out3, void* stream) {
  if (!out3) return CAKF_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int sms = num_sms();
  float* f = nullptr;
  long long* cyc = nullptr;
  cudaEvent_t e0, e1;
  if (cudaMalloc(&f, 64) != cudaSuccess) return CAKF_E_CUDA;
  cyc = reinterpret_cast<long long*>(f + 8);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192, blocks = sms * 2, threads = 512;   // 32 warps per SM
  mufu_peak_kernel<<<blocks, threads, 0, st>>>(f, 256, 0.5f, cyc);   // warm-up (clocks ramp)
  cudaEventRecord(e0, st);
  mufu_peak_kernel<<<blocks, threads, 0, st>>>(f, iters, 0.5f, cyc);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  long long hc = 0;
  cudaMemcpy(&hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  const double mufu_ops = (double)blocks * threads * iters * 8;
  out3[0] = mufu_ops / (ms * 1e-3);                 // MUFU ops/s (sqrt / ex2 mix)
  out3[2] = (double)hc;                             // SM cycles of CTA 0 in the timed MUFU kernel (diagnostic)
  const int diters = 4096;
  dmma_peak_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<double*>(f), 64);
  cudaEventRecord(e0, st);
  dmma_peak_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<double*>(f), diters);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  out3[1] = (double)blocks * 8 * diters * 8 * 256 * 2 / (ms * 1e-3);   // fp64 flop/s (8 warps x 8 chains x 512 flop)
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(f);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? CAKF_OK : CAKF_E_CUDA;
}
