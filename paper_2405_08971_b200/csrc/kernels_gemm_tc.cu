// kernels_gemm_tc.cu — the low-rank contractions of CAKF/CAKS on the tcgen05 tensor cores (sm_100a).
//
//   C = alpha * op(A) op(B) + beta * C        (fp32 storage; P:1532-1541 post-loop, alg:mfks smoother,
//                                              Sec. 3.2 truncation Gram F^T F and F Q_r)
//
// These are plain dense GEMMs of tall-skinny fp32 factors (D = 231,360 rows x a few hundred columns).
// fp32 accuracy from bf16 tensor cores exactly as K2 (kernels_gram_tc.cu): both operands are split
// exactly into three bf16 planes, a = a1 + a2 + a3, and each product is accumulated as
// a1b1 (TMEM accumulator D_big) + a1b2 + a2b1 + a2b2 + a1b3 + a3b1 (accumulator D_small), the dropped
// terms being ~2^-24 relative.  Long contractions are split over K (grid.z) and the fp32 partial
// tiles are summed in fp64 in a fixed order (deterministic), so no accumulator sees more than
// K / splits terms.
//
// Operands enter as K-major bf16 planes [3][rows][Kp] (split_planes_kernel: a coalesced pass that
// also transposes when the source is M-major, i.e. op = N for A / T for B).
// Per CTA: 128 x ntile (<= 256) output tile; warp 0 = TMA loader (A and B planes, 64B swizzle, zero
// fill out of bounds), warp 1 = MMA issuer (one elected lane, 12 MMAs per 32-deep K block),
// warps 2-5 = epilogue (tcgen05.ld 32x32b, lane quarter = warp % 4).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace cakf {

namespace {

constexpr int G_BM = 128;
constexpr int G_BK = 32;                 // 32 bf16 = one 64-byte swizzle atom row
constexpr int G_THREADS = 192;           // loader, MMA, 4 epilogue warps
constexpr int G_APLANE = G_BM * G_BK * 2;   // 8 KB
constexpr int G_SMEM_BUDGET = 220 * 1024;

int sm_count() { return num_sms(); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void split3(float a, uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  const uint32_t u = __float_as_uint(a);
  const uint32_t h1 = u & 0xFFFF0000u;
  const float r1 = a - __uint_as_float(h1);
  const uint32_t h2 = __float_as_uint(r1) & 0xFFFF0000u;
  const float r2 = r1 - __uint_as_float(h2);
  p1 = h1 >> 16;
  p2 = h2 >> 16;
  p3 = __float_as_uint(r2) >> 16;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// K-major, SWIZZLE_64B smem descriptor (8-row groups 512 B apart, sm_100 version 1)
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// grid (m tiles, n tiles, K splits).  work == nullptr: C = alpha acc + beta C directly (fp32, ldc);
// else the fp32 partial tile goes to work[(z N + n) M + m] for the fixed-order fp64 reduction.
__global__ void __launch_bounds__(G_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
               int nkb, int ntile, int stages, float alpha, float beta, float* __restrict__ C, size_t ldc,
               float* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  const uint32_t b_plane = (uint32_t)ntile * G_BK * 2;
  const uint32_t stage_bytes = ((3u * G_APLANE + 3u * b_plane) + 1023u) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(sbase + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * G_BM, n0 = blockIdx.y * ntile, z = blockIdx.z, S = gridDim.z;
  const int kb0 = (int)((long long)z * nkb / S), kb1 = (int)((long long)(z + 1) * nkb / S);
  const int nk = kb1 - kb0;
  const uint32_t acc_cols = ntile <= 32 ? 32 : ntile <= 64 ? 64 : ntile <= 128 ? 128 : 256;
  const uint32_t tmem_cols = 2 * acc_cols;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(sbase);

  if (warp == 0) {
    if (lane == 0) {   // ===== TMA loader
      const uint32_t bytes = 3u * (uint32_t)G_APLANE + 3u * b_plane;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % stages;
        if (kb >= stages) mbar_wait(smem_u32(&empty[s]), ((kb / stages) - 1) & 1);
        const uint32_t bar = smem_u32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        const uint32_t st0 = sm0 + s * stage_bytes;
        const int k0 = (kb0 + kb) * G_BK;
#pragma unroll
        for (int pl = 0; pl < 3; ++pl) tma3(st0 + pl * G_APLANE, &tmA, k0, m0, pl, bar);
#pragma unroll
        for (int pl = 0; pl < 3; ++pl) tma3(st0 + 3 * G_APLANE + pl * b_plane, &tmB, k0, n0, pl, bar);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer
    const uint32_t idesc = idesc_bf16(G_BM, ntile);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % stages;
      mbar_wait(smem_u32(&full[s]), (kb / stages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a0 = sm0 + s * stage_bytes, b0 = a0 + 3 * G_APLANE;
#pragma unroll
        for (int j = 0; j < G_BK / 16; ++j) {
          const uint64_t A1 = sdesc_sw64(a0 + 32 * j), A2 = sdesc_sw64(a0 + G_APLANE + 32 * j),
                         A3 = sdesc_sw64(a0 + 2 * G_APLANE + 32 * j);
          const uint64_t B1 = sdesc_sw64(b0 + 32 * j), B2 = sdesc_sw64(b0 + b_plane + 32 * j),
                         B3 = sdesc_sw64(b0 + 2 * b_plane + 32 * j);
          const uint32_t first = (kb | j) ? 1u : 0u;
          mma_bf16(tmem, A1, B1, idesc, first);
          mma_bf16(tmem + acc_cols, A1, B2, idesc, first);
          mma_bf16(tmem + acc_cols, A2, B1, idesc, 1u);
          mma_bf16(tmem + acc_cols, A2, B2, idesc, 1u);
          mma_bf16(tmem + acc_cols, A1, B3, idesc, 1u);
          mma_bf16(tmem + acc_cols, A3, B1, idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[s]))
                     : "memory");
        if (kb == nk - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(done))
                       : "memory");
      }
      __syncwarp();
    }
  } else {
    // ===== epilogue (warps 2-5): D_big + D_small
    if (nk > 0) mbar_wait(smem_u32(done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    for (int cb = 0; cb < ntile; cb += 16) {
      uint32_t r[16], q[16];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)cb;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15}, [%16];"
          : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
            "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
          : "r"(taddr + acc_cols));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int n = n0 + cb + t;
          if (cb + t < ntile && n < N) {
            const float v = nk > 0 ? __uint_as_float(r[t]) + __uint_as_float(q[t]) : 0.f;
            if (work) {
              work[((size_t)z * N + n) * M + row] = v;
            } else {
              float* c = C + row + (size_t)n * ldc;
              *c = beta != 0.f ? fmaf(alpha, v, beta * *c) : alpha * v;
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
  }
}

// Persistent variant for the un-split case (the truncation's M~ = F Q_r: D x r x c): one CTA per SM walks the
// 128 x ntile (<= 128) output tiles (n fastest, so the CTAs sharing an A tile run together); the two TMEM
// accumulators of a tile (2 x 128 columns) are double-buffered, so the epilogue of tile i overlaps the MMAs
// of tile i + 1 and the loader streams straight across tile boundaries.
constexpr int G_PN = 128;   // max ntile of the persistent kernel
__global__ void __launch_bounds__(G_THREADS, 1)
gemm_tc_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                       int nkb, int ntile, int ntiles, int nwork, int stages, float alpha, float beta,
                       float* __restrict__ C, size_t ldc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  const uint32_t b_plane = (uint32_t)ntile * G_BK * 2;
  const uint32_t stage_bytes = ((3u * G_APLANE + 3u * b_plane) + 1023u) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(sbase + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;   // [2] MMA -> epilogue, per accumulator buffer
  uint64_t* tfree = done + 2;        // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t acc_cols = G_PN;   // per accumulator; buffer b: big at 2b*128, small at (2b+1)*128

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&done[b]), 1);
      mbar_init(smem_u32(&tfree[b]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(sbase);

  if (warp == 0) {
    if (lane == 0) {   // ===== TMA loader: every K block of every tile of this CTA, in order
      const uint32_t bytes = 3u * (uint32_t)G_APLANE + 3u * b_plane;
      int it = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int m0 = (w / ntiles) * G_BM, n0 = (w % ntiles) * ntile;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          if (it >= stages) mbar_wait(smem_u32(&empty[s]), ((it / stages) - 1) & 1);
          const uint32_t bar = smem_u32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
          const uint32_t st0 = sm0 + s * stage_bytes;
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) tma3(st0 + pl * G_APLANE, &tmA, kb * G_BK, m0, pl, bar);
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) tma3(st0 + 3 * G_APLANE + pl * b_plane, &tmB, kb * G_BK, n0, pl, bar);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {   // ===== MMA issuer
    const uint32_t idesc = idesc_bf16(G_BM, ntile);
    int it = 0, i = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++i) {
      const int b = i & 1;
      if (i >= 2) mbar_wait(smem_u32(&tfree[b]), ((i >> 1) - 1) & 1);   // buffer b drained (tile i - 2)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dbig = tmem + (uint32_t)(2 * b) * acc_cols, dsmall = dbig + acc_cols;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(smem_u32(&full[s]), (it / stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = sm0 + s * stage_bytes, b0 = a0 + 3 * G_APLANE;
#pragma unroll
          for (int j = 0; j < G_BK / 16; ++j) {
            const uint64_t A1 = sdesc_sw64(a0 + 32 * j), A2 = sdesc_sw64(a0 + G_APLANE + 32 * j),
                           A3 = sdesc_sw64(a0 + 2 * G_APLANE + 32 * j);
            const uint64_t B1 = sdesc_sw64(b0 + 32 * j), B2 = sdesc_sw64(b0 + b_plane + 32 * j),
                           B3 = sdesc_sw64(b0 + 2 * b_plane + 32 * j);
            const uint32_t first = (kb | j) ? 1u : 0u;
            mma_bf16(dbig, A1, B1, idesc, first);
            mma_bf16(dsmall, A1, B2, idesc, first);
            mma_bf16(dsmall, A2, B1, idesc, 1u);
            mma_bf16(dsmall, A2, B2, idesc, 1u);
            mma_bf16(dsmall, A1, B3, idesc, 1u);
            mma_bf16(dsmall, A3, B1, idesc, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[s]))
                       : "memory");
          if (kb == nkb - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&done[b]))
                         : "memory");
        }
        __syncwarp();
      }
    }
  } else {   // ===== epilogue (warps 2-5): D_big + D_small of tile i from buffer i & 1
    const int quarter = warp & 3;
    int i = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++i) {
      const int b = i & 1;
      const int m0 = (w / ntiles) * G_BM, n0 = (w % ntiles) * ntile;
      const int row = m0 + quarter * 32 + lane;
      mbar_wait(smem_u32(&done[b]), (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int cb = 0; cb < ntile; cb += 16) {
        float old[16];
        if (beta != 0.f) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int n = n0 + cb + t;
            old[t] = (row < M && cb + t < ntile && n < N) ? C[row + (size_t)n * ldc] : 0.f;
          }
        }
        uint32_t r[16], q[16];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(2 * b) * acc_cols + (uint32_t)cb;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
              "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
            : "r"(taddr + acc_cols));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int n = n0 + cb + t;
            if (cb + t < ntile && n < N) {
              const float v = nkb > 0 ? __uint_as_float(r[t]) + __uint_as_float(q[t]) : 0.f;
              C[row + (size_t)n * ldc] = beta != 0.f ? fmaf(alpha, v, beta * old[t]) : alpha * v;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tfree[b]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// planes[p][r][k] (r < R, k < Kp, zero for k >= K) from src element (r, k) at
// KC ? src[k + r ld] (K contiguous) : src[r + k ld] (R contiguous; transposed through smem)
template <bool KC>
__global__ void split_planes_kernel(const float* __restrict__ src, int R, int K, int Kp, size_t ld,
                                    uint16_t* __restrict__ planes, size_t plane) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: 8 x 32
  if (!KC) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = k0 + ty + 8 * i, r = r0 + tx;
      tile[ty + 8 * i][tx] = (k < K && r < R) ? src[r + (size_t)k * ld] : 0.f;
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i, k = k0 + tx;
    if (r >= R || k >= Kp) continue;
    float v;
    if (KC) v = k < K ? src[k + (size_t)r * ld] : 0.f;
    else v = tile[tx][ty + 8 * i];
    uint32_t p1, p2, p3;
    split3(v, p1, p2, p3);
    const size_t e = (size_t)r * Kp + k;
    planes[e] = (uint16_t)p1;
    planes[plane + e] = (uint16_t)p2;
    planes[2 * plane + e] = (uint16_t)p3;
  }
}

// Rows-contiguous source (the truncation's F = [M^- | B], D x c): 64 k x 32 rows per block, transposed
// through shared memory; every thread splits 8 consecutive k of one row and writes one 16-byte chunk per
// plane (the generic version above writes 2-byte elements).  Same exact split, same planes.
__global__ void __launch_bounds__(256) split_planes_rc8_kernel(const float* __restrict__ src, int R, int K, int Kp,
                                                               size_t ld, uint16_t* __restrict__ planes,
                                                               size_t plane) {
  __shared__ float tile[64][33];
  const int k0 = blockIdx.x * 64, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // loads: 8 x 32
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = k0 + ty + 8 * i, r = r0 + tx;
    tile[ty + 8 * i][tx] = (k < K && r < R) ? src[r + (size_t)k * ld] : 0.f;
  }
  __syncthreads();
  const int rl = threadIdx.x >> 3, kq = threadIdx.x & 7, r = r0 + rl, k = k0 + 8 * kq;
  if (r >= R || k >= Kp) return;
  uint32_t w1[4], w2[4], w3[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t a1, a2, a3, b1, b2, b3;
    split3(tile[8 * kq + 2 * j][rl], a1, a2, a3);
    split3(tile[8 * kq + 2 * j + 1][rl], b1, b2, b3);
    w1[j] = a1 | (b1 << 16);
    w2[j] = a2 | (b2 << 16);
    w3[j] = a3 | (b3 << 16);
  }
  const size_t e = (size_t)r * Kp + k;   // Kp % 8 == 0, k % 8 == 0: 16-byte aligned
  *reinterpret_cast<uint4*>(planes + e) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  *reinterpret_cast<uint4*>(planes + plane + e) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
  *reinterpret_cast<uint4*>(planes + 2 * plane + e) = make_uint4(w3[0], w3[1], w3[2], w3[3]);
}

template <typename O>
__global__ void splitk_reduce_kernel(int M, int N, int S, const float* __restrict__ work, double alpha, double beta,
                                     O* __restrict__ C, size_t ldc) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)M * N) return;
  const int m = (int)(e % M), n = (int)(e / M);
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += (double)work[((size_t)z * N + n) * M + m];
  O* c = C + m + (size_t)n * ldc;
  *c = (O)(beta != 0.0 ? alpha * s + beta * (double)*c : alpha * s);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

bool make_plane_map(CUtensorMap* tm, const uint16_t* planes, int rows, int Kp, int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t gd[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, 3};
  const cuuint64_t gs[2] = {(cuuint64_t)Kp * 2, (cuuint64_t)Kp * rows * 2};
  const cuuint32_t box[3] = {G_BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, (void*)planes, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int gemm_tc_kp(int K) { return (K + 7) / 8 * 8; }

size_t gemm_tc_plane_bytes(int rows, int K) { return (size_t)3 * rows * gemm_tc_kp(K) * sizeof(uint16_t); }

cudaError_t gemm_tc_split(const float* src, int R, int K, size_t ld, bool k_contig, uint16_t* planes,
                          cudaStream_t st) {
  if (R <= 0 || K <= 0) return cudaSuccess;
  const int Kp = gemm_tc_kp(K);
  dim3 grid((Kp + 31) / 32, (R + 31) / 32);
  const size_t plane = (size_t)R * Kp;
  if (k_contig) {
    split_planes_kernel<true><<<grid, 256, 0, st>>>(src, R, K, Kp, ld, planes, plane);
  } else if (reinterpret_cast<uintptr_t>(planes) % 16 == 0 && plane % 8 == 0 && use_split_rc8()) {
    split_planes_rc8_kernel<<<dim3((Kp + 63) / 64, (R + 31) / 32), 256, 0, st>>>(src, R, K, Kp, ld, planes, plane);
  } else {
    split_planes_kernel<false><<<grid, 256, 0, st>>>(src, R, K, Kp, ld, planes, plane);
  }
  return note_launch_err();
}

cudaError_t gemm_tc_run(const uint16_t* Ap, int M, const uint16_t* Bp, int N, int K, double alpha, double beta,
                        float* C, double* Cd, size_t ldc, float* work, size_t work_floats, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int Kp = gemm_tc_kp(K);
  const int nkb = (Kp + G_BK - 1) / G_BK;
  const int ntiles = (N + 255) / 256;
  int ntile = (N + ntiles - 1) / ntiles;
  ntile = std::max(16, (ntile + 15) / 16 * 16);
  const int mt = (M + G_BM - 1) / G_BM;
  const uint32_t stage_bytes = ((3u * G_APLANE + 3u * (uint32_t)ntile * G_BK * 2) + 1023u) & ~1023u;
  const int stages = std::max(2, std::min(6, (int)((G_SMEM_BUDGET - 1024 - 256) / stage_bytes)));
  const size_t smem = (size_t)stages * stage_bytes + 1024 + 256;
  static PerDeviceOnce once;
  {
    const cudaError_t e = once_per_device(once, [] {
      return cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, G_SMEM_BUDGET);
    });
    if (e != cudaSuccess) return e;
  }
  // split K until the grid covers the SMs (each split keeps >= 8 K blocks), fp64 output always reduces
  const int tiles = mt * ntiles;
  int S = 1;
  if (nkb > 0) {
    const int want = (2 * sm_count() + tiles - 1) / tiles;
    S = std::max(1, std::min(want, nkb / 8));
    while (S > 1 && (size_t)S * M * N > work_floats) --S;
  }
  const bool reduce = Cd != nullptr || S > 1;
  if (reduce && (size_t)S * M * N > work_floats) return cudaErrorInvalidValue;
  if (!reduce && nkb > 0 && use_tc_persist()) {   // tall output (the truncation's F Q_r): persistent kernel
    const int pnt = (N + G_PN - 1) / G_PN;
    int pn = (N + pnt - 1) / pnt;
    pn = std::max(16, (pn + 15) / 16 * 16);
    const uint32_t pstage = ((3u * G_APLANE + 3u * (uint32_t)pn * G_BK * 2) + 1023u) & ~1023u;
    const int pstages = std::max(2, std::min(8, (int)((G_SMEM_BUDGET - 1024 - 256) / pstage)));
    const size_t psmem = (size_t)pstages * pstage + 1024 + 256;
    static PerDeviceOnce once_p;
    {
      const cudaError_t e = once_per_device(once_p, [] {
        return cudaFuncSetAttribute(gemm_tc_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    G_SMEM_BUDGET);
      });
      if (e != cudaSuccess) return e;
    }
    CUtensorMap pA, pB;
    if (!make_plane_map(&pA, Ap, M, Kp, G_BM) || !make_plane_map(&pB, Bp, N, Kp, pn)) return cudaErrorInvalidValue;
    const int nwork = mt * pnt;
    gemm_tc_persist_kernel<<<std::min(nwork, sm_count()), G_THREADS, psmem, st>>>(
        pA, pB, M, N, nkb, pn, pnt, nwork, pstages, (float)alpha, (float)beta, C, ldc);
    return note_launch_err();
  }
  CUtensorMap tmA, tmB;
  if (!make_plane_map(&tmA, Ap, M, Kp, G_BM) || !make_plane_map(&tmB, Bp, N, Kp, ntile)) return cudaErrorInvalidValue;
  dim3 grid(mt, ntiles, S);
  gemm_tc_kernel<<<grid, G_THREADS, smem, st>>>(tmA, tmB, M, N, nkb, ntile, stages, (float)alpha, (float)beta, C, ldc,
                                                reduce ? work : nullptr);
  cudaError_t e = note_launch_err();
  if (e != cudaSuccess || !reduce) return e;
  const size_t tot = (size_t)M * N;
  if (Cd) splitk_reduce_kernel<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, S, work, alpha, beta, Cd, ldc);
  else splitk_reduce_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, S, work, alpha, beta, C, ldc);
  return note_launch_err();
}

bool use_split_rc8() {
  static const bool v = !env_is("CAKF_SPLIT_RC8", '0');
  return v;
}

bool use_tc_persist() {
  static const bool v = !env_is("CAKF_TC_PERSIST", '0');
  return v;
}

bool use_tc_gemm() {
  static const bool v = !env_is("CAKF_GEMM_F64", '1');
  return v;
}

}  // namespace cakf
