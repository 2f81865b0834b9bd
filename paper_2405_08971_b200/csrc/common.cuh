// common.cuh — shared device helpers of libcakf (sm_100a).
//
// Spatial Matérn kernels evaluated from PRESCALED coordinates: the handle stores
// x * sqrt(2 nu) / ell_x, so a = sqrt(|x - x'|^2) = sqrt(2 nu) rho / ell and
//   nu = 1/2: k = exp(-a)
//   nu = 3/2: k = (1 + a) exp(-a)                      (the paper's kernel)
//   nu = 5/2: k = (1 + a + a^2/3) exp(-a)
// fp32 uses the MUFU approximations sqrt.approx / ex2.approx (max rel. error ~2^-22);
// fp64 uses IEEE sqrt / exp.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <utility>

namespace cakf {

// Count of libcakf kernel launches (host side, all handles and host threads); read by
// cakf_kernel_launches().
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}

// One-time setup per (call site, CUDA device), thread-safe: handles on different host threads (serving
// mode) may make their first calls concurrently, and function attributes are per device context.
struct PerDeviceOnce {
  static constexpr int kMaxDev = 64;
  std::once_flag flag[kMaxDev];
  cudaError_t result[kMaxDev] = {};
};
template <typename F>
inline cudaError_t once_per_device(PerDeviceOnce& o, F&& f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PerDeviceOnce::kMaxDev) dev = 0;
  std::call_once(o.flag[dev], [&] { o.result[dev] = f(); });
  return o.result[dev];
}
// SM count of the first device queried (one GPU model per process), thread-safe
inline int num_sms() {
  static const int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}
// Environment switch read once (thread-safe magic static at each call site): true iff the variable is set
// and its first character equals `on`.
inline bool env_is(const char* name, char on) {
  const char* e = std::getenv(name);
  return e && e[0] == on;
}
inline cudaError_t note_launch_err() {
  ++launch_counter();
  return cudaGetLastError();
}

// Programmatic dependent launch (PDL): the inner-loop kernels are launched with programmatic stream
// serialisation so that a kernel's CTAs are scheduled while its predecessor drains; each such kernel
// calls griddep_wait() before touching memory (it returns once the predecessor grid has completed and
// its writes are visible; a no-op without a programmatic dependency).  CAKF_PDL=0 launches them plainly.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  ++launch_counter();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T> struct V4t;
template <> struct V4t<float> { using type = float4; };
template <> struct V4t<double> { using type = double4; };
template <typename T> using V4 = typename V4t<T>::type;

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kLog2e = 1.4426950408889634f;

template <int NU2> __device__ __forceinline__ float matern_from_d2(float d2) {
  const float a = sqrt_approx(d2);
  const float e = ex2_approx(-kLog2e * a);
  if constexpr (NU2 == 1) return e;
  else if constexpr (NU2 == 3) return fmaf(a, e, e);
  else return e * fmaf(a, fmaf(a, 1.0f / 3.0f, 1.0f), 1.0f);
}
// packed pair version (sm_100 f32x2 FMA-pipe ops; the two MUFU ops per value stay scalar).  Same
// arithmetic as matern_from_d2<NU2>(float) value by value.
template <int NU2> __device__ __forceinline__ float2 matern2_from_d2(float2 d2) {
  float2 a, e;
  a.x = sqrt_approx(d2.x);
  a.y = sqrt_approx(d2.y);
  const float2 t = __fmul2_rn(a, make_float2(-kLog2e, -kLog2e));
  e.x = ex2_approx(t.x);
  e.y = ex2_approx(t.y);
  if constexpr (NU2 == 1) return e;
  else if constexpr (NU2 == 3) return __ffma2_rn(a, e, e);
  else {
    const float2 p = __ffma2_rn(a, __ffma2_rn(a, make_float2(1.0f / 3.0f, 1.0f / 3.0f), make_float2(1.f, 1.f)),
                                make_float2(1.f, 1.f));
    return __fmul2_rn(e, p);
  }
}
template <int NU2> __device__ __forceinline__ double matern_from_d2(double d2) {
  const double a = sqrt(d2);
  const double e = exp(-a);
  if constexpr (NU2 == 1) return e;
  else if constexpr (NU2 == 3) return fma(a, e, e);
  else return e * fma(a, fma(a, 1.0 / 3.0, 1.0), 1.0);
}

template <typename T, typename P, typename Q>
__device__ __forceinline__ T dist2(const P& p, const Q& q) {
  const T dx = p.x - q.x, dy = p.y - q.y, dz = p.z - q.z;
  return fma(dz, dz, fma(dy, dy, dx * dx));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV doubles (blockDim.x multiple of 32, <= 1024); result valid in
// every thread.  Uses `scratch` (>= 32 * NV doubles of shared memory).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) scratch[q * 32 + warp] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = (lane < nw) ? scratch[q * 32 + lane] : 0.0;
    v[q] = warp_sum(t);
  }
  __syncthreads();
}

// "Last block finalises" pattern: every block calls this after writing its partials;
// exactly one block (the last to arrive) gets true and must reset *cnt to 0.
__device__ __forceinline__ bool arrive_last(unsigned* cnt) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// Philox4x32-10 (Salmon et al. 2011); R16 counter layout (j, i, k, 0), key = seed.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
__device__ __forceinline__ double philox_normal(uint64_t seed, uint32_t k, uint32_t i, uint32_t j) {
  uint32_t c[4] = {j, i, k, 0u};
  philox4x32_10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  const double u1 = ((double)(c[0] >> 8) + 1.0) * 0x1p-24;
  const double u2 = (double)(c[1] >> 8) * 0x1p-24;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

}  // namespace cakf
