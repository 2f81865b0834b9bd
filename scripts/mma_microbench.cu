// mma_microbench.cu — tcgen05.mma.kind::f16 issue-rate microbenchmark on one SM per CTA.
// Measures clocks per 128 x N x 16 bf16 MMA for shared-memory operands with SWIZZLE_64B or
// SWIZZLE_128B K-major layouts (SS), and A from TMEM (TS).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mb scripts/mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, int layout, int sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) mb(int N, int layout, int ts, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const int sbo = layout == 2 ? 1024 : 512;
  const uint32_t a_addr = base, b_addr = base + 32768;
  const uint32_t idesc = idesc_bf16(128, N);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t bd = sdesc(b_addr + 32 * (i & 1), layout, sbo);
      if (ts) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 256 + 8 * (i & 1)),
                     "l"(bd), "r"(idesc), "r"(i > 0 ? 1 : 0));
      } else {
        const uint64_t ad = sdesc(a_addr + 32 * (i & 1), layout, sbo);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd),
                     "r"(idesc), "r"(i > 0 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    }
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(mb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  struct Cfg { int N, layout, ts; const char* name; } cfgs[] = {
      {208, 4, 0, "SS sw64  N=208"}, {256, 4, 0, "SS sw64  N=256"}, {128, 4, 0, "SS sw64  N=128"},
      {208, 2, 0, "SS sw128 N=208"}, {256, 2, 0, "SS sw128 N=256"}, {208, 4, 1, "TS sw64  N=208"},
      {256, 2, 1, "TS sw128 N=256"}};
  for (auto& c : cfgs) {
    for (int grid : {1, 148}) {
      mb<<<grid, 128, smem>>>(c.N, c.layout, c.ts, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double clk = (double)mx / iters;
      const double macs = 128.0 * c.N * 16;
      printf("%-16s grid %3d: %7.1f clk/MMA  %7.0f MAC/clk/SM\n", c.name, grid, clk, macs / clk);
    }
  }
  return 0;
}
