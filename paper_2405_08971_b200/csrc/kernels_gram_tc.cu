// kernels_gram_tc.cu — K2 on the 5th-generation tensor cores (tcgen05, sm_100a).
//
//   Y[i, c] = alpha * sum_j k(x_i, x_j) B[j, c]        (the "Gramian x matrix" of P:644-647)
//
// The smoother's Sigma_k x (N_X x N_X x 2(r+1)) and the post-loop
// Sigma_k H^T [v V] (a7) are dense contractions whose A operand (kernel values) is
// generated on the fly.  fp32 accuracy from bf16 tensor cores ("3 x BF16"):
//   every fp32 value is split EXACTLY into three bf16 pieces by bit masking,
//   a = a1 + a2 + a3 (8 + 8 + 8 significand bits), and the product is accumulated as
//   a1b1 + a1b2 + a2b1 + a2b2 + a1b3 + a3b1 (dropped terms ~2^-24 relative) in fp32 TMEM.
// Six kind::f16 MMAs cost the same tensor time as three kind::tf32 MMAs, and the B planes
// take 6 bytes per element instead of 8.
//
// Per CTA: a 128-row x N_TILE (<= 256) output tile in TMEM.  Per K-block of 32:
//   * warp-specialised: 8 producer warps evaluate the 128 x 32 Matérn block (FP32 pipe +
//     MUFU), split it and store the three planes in the K-major SWIZZLE_64B canonical layout;
//     a 9th warp issues the MMAs; the two sides meet only at full / empty mbarriers;
//   * a loader warp brings the three B planes (precomputed, K-major) and the block's column
//     coordinates with TMA (cp.async.bulk.tensor, 64B swizzle = the UMMA canonical layout,
//     zero fill out of bounds), up to three blocks ahead;
//   (Tried: A as the TMEM operand written with tcgen05.st ("TS" mode) — correct but 2.5x slower
//    on B200, the stores serialise against the in-flight MMAs.)
//   * the MMA warp issues 2 k-steps x 6 tcgen05.mma.kind::f16 per block and commits to the
//     stage's empty barrier; with three stages the producers run up to two blocks ahead.
// Epilogue: tcgen05.ld (32x32b) -> registers -> coalesced column-major stores.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include <cuda_fp16.h>

#include "internal.h"

namespace cakf {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;                        // 32 bf16 = one 64-byte swizzle atom row
constexpr int TC_THREADS = 256;                  // producer warps (8): 2 column groups of 16 per tile row
constexpr int TC_NG = TC_THREADS / 128;          // column groups per 32-column K-block
constexpr int TC_KPT = 32 / TC_NG;               // columns (points) generated per producer thread and block
constexpr int TC_MMA_WARP = TC_THREADS / 32, TC_LOAD_WARP = TC_MMA_WARP + 1;
static_assert(TC_KPT % 8 == 0, "each producer thread writes whole 16-byte chunks of the swizzled rows");
constexpr int TC_MAXN = 208;
constexpr int A_STAGES = 3;                      // generated operand ring
constexpr int B_STAGES = 3;                      // TMA operand ring (loads run 2 blocks ahead)
constexpr int TC_STAGES = B_STAGES;
constexpr int A_PLANE = TC_BM * TC_BK * 2;       // 8 KB
constexpr int B_PLANE = TC_MAXN * TC_BK * 2;     // 13 KB (multiple of the 512 B SW64 atom)
constexpr int XC_BYTES = TC_BK * 16;             // the K-block's 32 column coordinates
constexpr int A_STAGE_BYTES = 3 * A_PLANE;                                   // 24 KB
constexpr int B_STAGE_BYTES = (3 * B_PLANE + XC_BYTES + 1023) / 1024 * 1024;  // 40 KB
constexpr int TC_SMEM = A_STAGES * A_STAGE_BYTES + B_STAGES * B_STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// exact 3-way bf16 split by truncation: returns the three bf16 bit patterns (low 16 bits)
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

// two-way fp16 split (round to nearest): a = h1 + h2 + O(2^-22 a) for a in the fp16 normal range
__device__ __forceinline__ void split2h(float a, uint32_t& p1, uint32_t& p2) {
  const __half h1 = __float2half_rn(a);
  const __half h2 = __float2half_rn(a - __half2float(h1));
  p1 = (uint32_t)__half_as_ushort(h1);
  p2 = (uint32_t)__half_as_ushort(h2);
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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_64B, 8-row groups 512 B apart (sm_100 version 1).
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);        // start address  [0, 14)
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;               // SBO = 512 B
  d |= (uint64_t)1 << 46;                        // version = 1
  d |= (uint64_t)4 << 61;                        // layout = SWIZZLE_64B
  return d;
}

// Instruction descriptor: kind::f16, D = f32, A = B = bf16, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Instruction descriptor: kind::f16, D = f32, A = B = f16, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// byte offset of 16-byte chunk c (0..3) of row r in a K-major SWIZZLE_64B tile
__device__ __forceinline__ uint32_t sw64_off(int r, int c) {
  return (uint32_t)((r >> 3) * 512 + (r & 7) * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

// F16 = false: 3 x BF16 planes, 6 MMAs per k-step (products to ~2^-24).
// F16 = true : 2 x FP16 planes (kernel values scaled by 2^14, B columns by powers of two into
//              [2^13, 2^14)), 3 MMAs per k-step (a1b1 | a1b2 + a2b1; products to ~2^-21), half
//              the tensor work; colinv[n] undoes both scalings in the epilogue.
template <int NU2, bool F16>
__global__ void __launch_bounds__(TC_THREADS + 64, 1)
gram_gemm_tc_kernel(const float4* __restrict__ xr, int M, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmX, int K, int C, int ntile,
                    float* __restrict__ Y, size_t ldy, float alpha, int diag_nogen,
                    const int* __restrict__ act_cnt, const int* __restrict__ act_list, int act_stride,
                    const float* __restrict__ colinv, int oneacc, int stack) {
  constexpr int NPL = F16 ? 2 : 3;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  unsigned char* a_base = sbase;                                   // A ring
  unsigned char* b_base = sbase + A_STAGES * A_STAGE_BYTES;        // B ring (+ coordinates)
  uint64_t* fullA = reinterpret_cast<uint64_t*>(b_base + B_STAGES * B_STAGE_BYTES);   // producers -> MMA
  uint64_t* emptyA = fullA + A_STAGES;                                                 // MMA -> producers
  uint64_t* fullB = emptyA + A_STAGES;                                                 // TMA -> producers
  uint64_t* emptyB = fullB + B_STAGES;                                                 // MMA -> loader
  uint64_t* done = emptyB + B_STAGES;                                                  // last MMA -> epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * TC_BM, n0 = blockIdx.y * ntile;
  // two accumulators: D_big = sum a1 b1 (the exact leading products) and D_small = the five
  // correction products; summed in fp32 round-to-nearest in the epilogue (tensor-core
  // accumulation truncates, so keeping the small terms apart cuts the biased error ~6x)
  // stack (3 x BF16, 3 ntile <= 256): the three B planes sit contiguously, so A1 x [B1|B2|B3] (N = 3 ntile),
  // A2 x [B1|B2] at column offset ntile and A3 x B1 at ntile give D_big = [0, ntile) and the five correction
  // products in [ntile, 3 ntile): 3 MMAs per k-step instead of 6 (each A plane read once)
  const uint32_t acc_cols = stack ? (uint32_t)ntile : ntile <= 32 ? 32 : ntile <= 64 ? 64 : ntile <= 128 ? 128 : 256;
  const uint32_t tmem_cols = stack ? 256u : 2 * acc_cols;
  const uint32_t b_pl = stack ? (uint32_t)ntile * 64u : (uint32_t)B_PLANE;   // B plane stride in a stage
  // exact-zero culling: only this tile's active K-blocks (ascending), else all of them
  const int nk = act_cnt ? act_cnt[blockIdx.x] : (K + TC_BK - 1) / TC_BK;
  const int* my_list = act_cnt ? act_list + (size_t)blockIdx.x * act_stride : nullptr;

  if (warp == TC_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(smem_u32(&fullA[s]), TC_THREADS / 32);   // one arrive per producer warp
      mbar_init(smem_u32(&emptyA[s]), 1);
    }
    for (int s = 0; s < B_STAGES; ++s) {
      mbar_init(smem_u32(&fullB[s]), 1);
      mbar_init(smem_u32(&emptyB[s]), 1);
    }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  auto a_addr = [&](int s) { return smem_u32(a_base + s * A_STAGE_BYTES); };
  auto b_addr = [&](int s) { return smem_u32(b_base + s * B_STAGE_BYTES); };

  if (warp == TC_MMA_WARP) {
    // ===== MMA issuer: one elected lane, back-to-back over the stage ring
    const uint32_t idesc = F16 ? idesc_f16(TC_BM, ntile) : idesc_bf16(TC_BM, ntile);
    for (int kb = 0; kb < nk; ++kb) {
      const int sa = kb % A_STAGES, sb = kb % B_STAGES;
      mbar_wait(smem_u32(&fullA[sa]), (kb / A_STAGES) & 1);
      mbar_wait(smem_u32(&fullB[sb]), (kb / B_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a0 = a_addr(sa), bb = b_addr(sb);
#pragma unroll
        for (int j = 0; j < TC_BK / 16; ++j) {
          const uint64_t A1 = sdesc_sw64(a0 + 32 * j), A2 = sdesc_sw64(a0 + A_PLANE + 32 * j),
                         A3 = sdesc_sw64(a0 + 2 * A_PLANE + 32 * j);
          const uint64_t B1 = sdesc_sw64(bb + 32 * j), B2 = sdesc_sw64(bb + b_pl + 32 * j),
                         B3 = sdesc_sw64(bb + 2 * b_pl + 32 * j);
          const uint32_t first = (kb | j) ? 1u : 0u;
          if (!F16 && stack) {
            mma_bf16(tmem, A1, B1, idesc_bf16(TC_BM, 3 * ntile), first);
            mma_bf16(tmem + acc_cols, A2, B1, idesc_bf16(TC_BM, 2 * ntile), 1u);
            mma_bf16(tmem + acc_cols, A3, B1, idesc, 1u);
          } else {
            mma_bf16(tmem, A1, B1, idesc, first);
            mma_bf16(tmem + (oneacc ? 0u : acc_cols), A1, B2, idesc, oneacc ? 1u : first);
            mma_bf16(tmem + (oneacc ? 0u : acc_cols), A2, B1, idesc, 1u);
            if (!F16) {
              mma_bf16(tmem + acc_cols, A2, B2, idesc, 1u);
              mma_bf16(tmem + acc_cols, A1, B3, idesc, 1u);
              mma_bf16(tmem + acc_cols, A3, B1, idesc, 1u);
            }
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&emptyA[sa]))
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&emptyB[sb]))
                     : "memory");
        if (kb == nk - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(done))
                       : "memory");
      }
      __syncwarp();
    }
  } else if (warp == TC_LOAD_WARP) {
    // ===== TMA loader: the three B planes (64B-swizzled boxes, zero-filled beyond C / K) and the
    // block's 32 column coordinates, up to TC_STAGES blocks ahead of the MMAs
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)NPL * (uint32_t)ntile * 64u + (uint32_t)XC_BYTES;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % B_STAGES;
        if (kb >= B_STAGES) mbar_wait(smem_u32(&emptyB[s]), ((kb / B_STAGES) - 1) & 1);
        const uint32_t bar = smem_u32(&fullB[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        const uint32_t b0 = b_addr(s);
        const int k0 = (my_list ? my_list[kb] : kb) * TC_BK;
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl) {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
              "[%5];" ::"r"(b0 + pl * b_pl),
              "l"(&tmB), "r"(k0), "r"(n0), "r"(pl), "r"(bar)
              : "memory");
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                b0 + 3 * B_PLANE),
            "l"(&tmX), "r"(0), "r"(k0), "r"(bar)
            : "memory");
      }
    }
    __syncwarp();
  } else {
    // ===== producers (warps 0-7): A generation from the staged column coordinates; thread = (tile row,
    // group of TC_KPT consecutive columns of the K-block)
    const int arow = tid & (TC_BM - 1), kq = tid >> 7;
    float4 xa = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m0 + arow < M) xa = xr[m0 + arow];
    for (int kb = 0; kb < nk; ++kb) {
      const int sa = kb % A_STAGES, sb = kb % B_STAGES;
      mbar_wait(smem_u32(&fullB[sb]), (kb / B_STAGES) & 1);                       // coords(kb) landed
      if (kb >= A_STAGES) mbar_wait(smem_u32(&emptyA[sa]), ((kb / A_STAGES) - 1) & 1);   // MMA(kb - 2) done
      const uint32_t a0 = a_addr(sa);
      const float4* sxc = reinterpret_cast<const float4*>(b_base + sb * B_STAGE_BYTES + 3 * B_PLANE) + TC_KPT * kq;
      uint32_t p1[TC_KPT / 2], p2[TC_KPT / 2], p3[TC_KPT / 2];   // bf16x2 packed
      if (!F16 && !diag_nogen) {
        // two columns per step on the packed f32x2 FMA-pipe ops (MUFU sqrt / ex2 stay scalar), then the
        // exact truncation split of both values at once: h1 = top 16 bits, r1 = v - h1, h2 = top of r1,
        // r2 = r1 - h2 (both subtractions exact); each plane's bf16x2 word is one byte permute of the
        // two values' high halves — the same planes as split3 + pack, in about half the instructions
#pragma unroll
        for (int q = 0; q < TC_KPT; q += 2) {
          const float4 c0 = sxc[q], c1 = sxc[q + 1];   // {x, x', y, y'}, {z, z', w, w'} of points k, k+1
          const float2 dx = __fadd2_rn(make_float2(c0.x, c0.y), make_float2(-xa.x, -xa.x));
          const float2 dy = __fadd2_rn(make_float2(c0.z, c0.w), make_float2(-xa.y, -xa.y));
          const float2 dz = __fadd2_rn(make_float2(c1.x, c1.y), make_float2(-xa.z, -xa.z));
          const float2 kv = matern2_from_d2<NU2>(__ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx))));
          const uint32_t ua = __float_as_uint(kv.x), ub = __float_as_uint(kv.y);
          const float2 h1 = make_float2(__uint_as_float(ua & 0xFFFF0000u), __uint_as_float(ub & 0xFFFF0000u));
          const float2 r1 = __fadd2_rn(kv, make_float2(-h1.x, -h1.y));
          const uint32_t va = __float_as_uint(r1.x), vb = __float_as_uint(r1.y);
          const float2 h2 = make_float2(__uint_as_float(va & 0xFFFF0000u), __uint_as_float(vb & 0xFFFF0000u));
          const float2 r2 = __fadd2_rn(r1, make_float2(-h2.x, -h2.y));
          p1[q >> 1] = __byte_perm(ua, ub, 0x7632);
          p2[q >> 1] = __byte_perm(va, vb, 0x7632);
          p3[q >> 1] = __byte_perm(__float_as_uint(r2.x), __float_as_uint(r2.y), 0x7632);
        }
      } else {
#pragma unroll
      for (int q = 0; q < TC_KPT; q += 2) {
        float kv[2];
        const float4 cA = sxc[q], cB = sxc[q + 1];   // pair-packed {x, x', y, y'}, {z, z', w, w'}
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float4 c = t == 0 ? make_float4(cA.x, cA.z, cB.x, 0.f) : make_float4(cA.y, cA.w, cB.y, 0.f);
          const float dx = xa.x - c.x, dy = xa.y - c.y, dz = xa.z - c.z;
          const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          kv[t] = diag_nogen ? d2 : matern_from_d2<NU2>(d2);   // diag_nogen: timing experiment only
        }
        uint32_t a1, a2, a3 = 0, b1, b2, b3 = 0;
        if (F16) {
          split2h(kv[0] * 16384.f, a1, a2);
          split2h(kv[1] * 16384.f, b1, b2);
        } else {
          split3(kv[0], a1, a2, a3);
          split3(kv[1], b1, b2, b3);
        }
        p1[q >> 1] = a1 | (b1 << 16);
        p2[q >> 1] = a2 | (b2 << 16);
        p3[q >> 1] = a3 | (b3 << 16);
      }
      }
#pragma unroll
      for (int h = 0; h < TC_KPT / 8; ++h) {
        const uint32_t off = sw64_off(arow, (TC_KPT / 8) * kq + h);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0 + off), "r"(p1[4 * h]), "r"(p1[4 * h + 1]),
                     "r"(p1[4 * h + 2]), "r"(p1[4 * h + 3])
                     : "memory");
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0 + A_PLANE + off), "r"(p2[4 * h]),
                     "r"(p2[4 * h + 1]), "r"(p2[4 * h + 2]), "r"(p2[4 * h + 3])
                     : "memory");
        if (!F16)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0 + 2 * A_PLANE + off), "r"(p3[4 * h]),
                       "r"(p3[4 * h + 1]), "r"(p3[4 * h + 2]), "r"(p3[4 * h + 3])
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> tensor core
      __syncwarp();   // every lane's writes (each fenced) before lane 0's release: one arrive per warp
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fullA[sa])) : "memory");
    }
    // ===== epilogue: D = D_big + D_small (fp32 round-to-nearest)
    if (nk > 0) mbar_wait(smem_u32(done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    // epilogue by the producer warps: lane quarter = warp % 4, the columns split into TC_NG parts
    const int part_cols = ((ntile + TC_NG - 1) / TC_NG + 15) / 16 * 16;
    const int c_begin = min(ntile, (warp >> 2) * part_cols);
    const int c_end = min(ntile, c_begin + part_cols);
    for (int cb = c_begin; cb < c_end; cb += 16) {
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
      uint32_t q2[16];
      if (stack) {   // the second correction block [2 ntile, 3 ntile)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(q2[0]), "=r"(q2[1]), "=r"(q2[2]), "=r"(q2[3]), "=r"(q2[4]), "=r"(q2[5]), "=r"(q2[6]),
              "=r"(q2[7]), "=r"(q2[8]), "=r"(q2[9]), "=r"(q2[10]), "=r"(q2[11]), "=r"(q2[12]), "=r"(q2[13]),
              "=r"(q2[14]), "=r"(q2[15])
            : "r"(taddr + 2 * acc_cols));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int n = n0 + cb + t;
          const float small = stack ? __uint_as_float(q[t]) + __uint_as_float(q2[t]) : __uint_as_float(q[t]);
          const float v = __uint_as_float(r[t]) + (oneacc ? 0.f : small);
          if (cb + t < c_end && n < C) Y[row + (size_t)n * ldy] = nk > 0 ? (F16 ? alpha * colinv[n] * v : alpha * v) : 0.f;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == TC_MMA_WARP) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
  }
}

// B (K x C column-major, ldb) -> three bf16 planes, each C x Kp K-major (row n = column n of B),
// zero-padded for k >= K.  Exact split (see split3).
__global__ void split_bf16x3_kernel(int K, int C, int Kp, const float* __restrict__ B, size_t ldb,
                                    uint16_t* __restrict__ planes, size_t plane) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)Kp * C) return;
  const int k = (int)(e % Kp), n = (int)(e / Kp);
  const float v = k < K ? B[k + (size_t)n * ldb] : 0.f;
  uint32_t p1, p2, p3;
  split3(v, p1, p2, p3);
  planes[e] = (uint16_t)p1;
  planes[plane + e] = (uint16_t)p2;
  planes[2 * plane + e] = (uint16_t)p3;
}

// per-column power-of-two scaling of B into [2^13, 2^14): scale[n] = 2^(14 - e), e = exponent with
// max|B[:, n]| < 2^e; colinv[n] = 2^-14 / scale[n] (also undoes the 2^14 kernel-value scaling)
__global__ void colscale_kernel(int K, const float* __restrict__ B, size_t ldb, float* __restrict__ scale,
                                float* __restrict__ colinv) {
  __shared__ float red[32];
  const int n = blockIdx.x;
  float m = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmaxf(m, fabsf(B[k + (size_t)n * ldb]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t = fmaxf(t, red[q]);
    int e = 0;
    if (t > 0.f && isfinite(t)) frexpf(t, &e);   // t in [2^(e-1), 2^e)
    scale[n] = ldexpf(1.f, 14 - e);
    colinv[n] = ldexpf(1.f, e - 28);
  }
}

// B (K x C column-major) -> two fp16 planes (C x Kp, K-major) of B[:, n] * scale[n], zero for k >= K
__global__ void split_f16x2_kernel(int K, int C, int Kp, const float* __restrict__ B, size_t ldb,
                                   const float* __restrict__ scale, uint16_t* __restrict__ planes, size_t plane) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)Kp * C) return;
  const int k = (int)(e % Kp), n = (int)(e / Kp);
  const float v = k < K ? B[k + (size_t)n * ldb] * scale[n] : 0.f;
  uint32_t p1, p2;
  split2h(v, p1, p2);
  planes[e] = (uint16_t)p1;
  planes[plane + e] = (uint16_t)p2;
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

// column coordinates as point pairs: out[2j] = {x_2j, x_2j+1, y_2j, y_2j+1}, out[2j+1] = {z.., w..}
// (zero partner for an odd count), so the producers' packed f32x2 operands load ready-paired
__global__ void pack_pairs_kernel(int K, const float4* __restrict__ xc, float4* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * j >= K) return;
  const float4 a = xc[2 * j], b = 2 * j + 1 < K ? xc[2 * j + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
  out[2 * j] = make_float4(a.x, b.x, a.y, b.y);
  out[2 * j + 1] = make_float4(a.z, b.z, a.w, b.w);
}

template <int NU2>
cudaError_t launch_tc_nu(const float4* xr, int M, const float4* xc, int K, const uint16_t* planes, int Kp, int C,
                         int ntile, float* Y, size_t ldy, float alpha, cudaStream_t st, const int* act_cnt,
                         const int* act_list, int act_stride, const float* colinv) {
  static PerDeviceOnce once;
  {
    const cudaError_t e = once_per_device(once, [] {
      cudaError_t r = cudaFuncSetAttribute(gram_gemm_tc_kernel<NU2, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(gram_gemm_tc_kernel<NU2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
      return r;
    });
    if (e != cudaSuccess) return e;
  }
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // B planes: 3 x [C rows] x [Kp bf16], K innermost; boxes of 32 K x ntile rows, 64B swizzle
  CUtensorMap tmB, tmX;
  const cuuint64_t gdB[3] = {(cuuint64_t)Kp, (cuuint64_t)C, 3};
  const cuuint64_t gsB[2] = {(cuuint64_t)Kp * 2, (cuuint64_t)Kp * C * 2};
  const cuuint32_t boxB[3] = {TC_BK, (cuuint32_t)ntile, 1};
  const cuuint32_t es3[3] = {1, 1, 1};
  if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, (void*)planes, gdB, gsB, boxB, es3, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // column coordinates, pair-packed (pack_pairs_kernel): [K2 rows] x [4 floats]; boxes of 32 rows, zero beyond
  const cuuint64_t gdX[2] = {4, (cuuint64_t)((K + 1) / 2 * 2)};
  const cuuint64_t gsX[1] = {16};
  const cuuint32_t boxX[2] = {4, TC_BK};
  const cuuint32_t es2[2] = {1, 1};
  if (enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)xc, gdX, gsX, boxX, es2, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static const int oneacc = [] { const char* e = getenv("CAKF_K2_ONEACC"); return (e && e[0] == '1') ? 1 : 0; }();
  static const int nogen = [] { const char* e = getenv("CAKF_TC_DIAG_NOGEN"); return (e && e[0] == '1') ? 1 : 0; }();
  dim3 grid((M + TC_BM - 1) / TC_BM, (C + ntile - 1) / ntile);
  if (colinv)
    gram_gemm_tc_kernel<NU2, true><<<grid, TC_THREADS + 64, TC_SMEM, st>>>(xr, M, tmB, tmX, K, C, ntile, Y, ldy, alpha,
                                                                           nogen, act_cnt, act_list, act_stride, colinv,
                                                                           oneacc, 0);
  else
    gram_gemm_tc_kernel<NU2, false><<<grid, TC_THREADS + 64, TC_SMEM, st>>>(
        xr, M, tmB, tmX, K, C, ntile, Y, ldy, alpha, nogen, act_cnt, act_list, act_stride, nullptr, 0,
        (3 * ntile <= 256 && use_k2_stack()) ? 1 : 0);
  return note_launch_err();
}

}  // namespace

// one block per 128-row output tile: ascending list of the 32-column K-blocks within the cut
__global__ void k2_active_kernel(const float4* __restrict__ sphM, const float4* __restrict__ sphK, int nkb, float cut,
                                 int* __restrict__ act_cnt, int* __restrict__ act_list, int act_stride,
                                 unsigned long long* __restrict__ total) {
  __shared__ int wcount[8];
  __shared__ int base;
  const float4 A = sphM[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int k0 = 0; k0 < nkb; k0 += 256) {
    const int kb = k0 + threadIdx.x;
    bool on = false;
    if (kb < nkb) {
      const float4 B = sphK[kb];
      const float ex = A.x - B.x, ey = A.y - B.y, ez = A.z - B.z;
      on = !(sqrtf(ex * ex + ey * ey + ez * ez) - A.w - B.w > cut);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wcount[w] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int q = 0; q < w; ++q) off += wcount[q];
    if (on) act_list[(size_t)blockIdx.x * act_stride + off + __popc(bal & ((1u << lane) - 1u))] = kb;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int q = 0; q < 8; ++q) t += wcount[q];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    act_cnt[blockIdx.x] = base;
    if (total) atomicAdd(total, (unsigned long long)base);
  }
}

bool use_tc_k2() {
  static const bool v = !env_is("CAKF_K2_SIMT", '1');
  return v;
}

cudaError_t launch_k2_active(const float4* sphM, int nmt, const float4* sphK, int nkb, float cut, int* act_cnt,
                             int* act_list, int act_stride, unsigned long long* total, cudaStream_t st) {
  if (nmt <= 0) return cudaSuccess;
  k2_active_kernel<<<nmt, 256, 0, st>>>(sphM, sphK, nkb, cut, act_cnt, act_list, act_stride, total);
  return note_launch_err();
}

size_t gram_gemm_tc_workspace(int K, int C) {
  const size_t Kp = ((size_t)K + TC_BK - 1) / TC_BK * TC_BK;
  // planes, column scales, and the pair-packed column coordinates (K rounded up to even) + alignment
  return 3 * Kp * (size_t)C * sizeof(uint16_t) + 2 * (size_t)C * sizeof(float) + ((size_t)K + 2) * 16 + 2048;
}

bool use_k2_stack() {
  static const bool v = !env_is("CAKF_K2_STACK", '0');
  return v;
}

bool use_f16_k2() {
  static const bool v = env_is("CAKF_K2_PREC", 'f') || env_is("CAKF_K2_PREC", 'F');   // "f16x2"; default 3 x BF16
  return v;
}

cudaError_t launch_gram_gemm_tc(int nu2, const float4* xr, int M, const float4* xc, int K, const float* B, size_t ldb,
                                int C, float* Y, size_t ldy, double alpha, float* work, cudaStream_t st,
                                const int* act_cnt, const int* act_list, int act_stride) {
  if (M <= 0 || C <= 0) return cudaSuccess;
  const int Kp = (K + TC_BK - 1) / TC_BK * TC_BK;
  uint16_t* planes = reinterpret_cast<uint16_t*>(work);
  const size_t plane = (size_t)Kp * C;
  const bool f16 = use_f16_k2();
  float* colscale = reinterpret_cast<float*>(planes + 3 * plane + 256);   // 512 B past the planes
  float* colinv = colscale + C;
  float4* xpair = reinterpret_cast<float4*>(((uintptr_t)(colinv + C) + 255) & ~(uintptr_t)255);
  if (K > 0) {
    pack_pairs_kernel<<<(unsigned)(((K + 1) / 2 + 255) / 256), 256, 0, st>>>(K, xc, xpair);
    const cudaError_t e = note_launch_err();
    if (e != cudaSuccess) return e;
  }
  xc = xpair;
  if (plane > 0) {
    if (f16) {
      colscale_kernel<<<C, 256, 0, st>>>(K, B, ldb, colscale, colinv);
      cudaError_t e = note_launch_err();
      if (e != cudaSuccess) return e;
      split_f16x2_kernel<<<(unsigned)((plane + 255) / 256), 256, 0, st>>>(K, C, Kp, B, ldb, colscale, planes, plane);
    } else {
      split_bf16x3_kernel<<<(unsigned)((plane + 255) / 256), 256, 0, st>>>(K, C, Kp, B, ldb, planes, plane);
    }
    cudaError_t e = note_launch_err();
    if (e != cudaSuccess) return e;
  }
  // N tile: fewest tiles of <= 256 columns, balanced, multiple of 16 (kind::f16, M = 128)
  const int ntiles = (C + TC_MAXN - 1) / TC_MAXN;
  int ntile = (C + ntiles - 1) / ntiles;
  ntile = ((ntile + 15) / 16) * 16;
  switch (nu2) {
    case 1: return launch_tc_nu<1>(xr, M, xc, K, planes, Kp, C, ntile, Y, ldy, (float)alpha, st, act_cnt, act_list,
                                   act_stride, f16 ? colinv : nullptr);
    case 3: return launch_tc_nu<3>(xr, M, xc, K, planes, Kp, C, ntile, Y, ldy, (float)alpha, st, act_cnt, act_list,
                                   act_stride, f16 ? colinv : nullptr);
    case 5: return launch_tc_nu<5>(xr, M, xc, K, planes, Kp, C, ntile, Y, ldy, (float)alpha, st, act_cnt, act_list,
                                   act_stride, f16 ? colinv : nullptr);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cakf
