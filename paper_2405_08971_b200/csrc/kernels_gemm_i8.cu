// kernels_gemm_i8.cu — fp64-accurate contractions of fp32 factors on the INT8 tensor cores (sm_100a).
//
//   C = alpha * op(A) op(B) + beta * C        (the fp32 path's low-rank contractions: post-loop
//                                              P:1532-1541, smoother alg:mfks P:388-409, truncation
//                                              Gram M^T M and M Q_r, Sec. 3.2)
//
// These contractions feed the downdate forms P = Sigma - M M^T, whose cancellation amplifies any
// accumulation error (fp32-accumulating tensor-core GEMMs fail the cfg1 fp32 bound).
// Products of fp32 numbers are made exact on integer tensor cores (the Ozaki splitting):
//   * every row r of op(A) (and of op(B)^T) is scaled per K chunk c of I_KC elements by a power of
//     two 2^e[r][c] > max |a| over the chunk, and the scaled value a 2^-e in (-1, 1) is cut into
//     I_S signed 7-bit slices: a = 2^e sum_s alpha_s 2^{-7(s+1)}, alpha_s in [-127, 127]
//     (exact for fp32 inputs within 2^{7 I_S - 24} of the chunk maximum; below that the absolute
//     error is < 2^{e - 7 I_S});
//   * the slice products with s + t < I_S are accumulated by tcgen05.mma.kind::i8 into one int32
//     TMEM accumulator per level L = s + t — exact, because I_S * 127^2 * I_KC < 2^31;
//   * the epilogue forms 2^{e_r + e_n} sum_L acc_L 2^{-7(L+2)} in fp64 per chunk and accumulates the
//     chunks of a K split in fp64; the splits are summed in a fixed order (deterministic).
// The dropped levels L >= I_S are < I_S 2^{-7 I_S + 1} relative to 2^{e_r + e_n} per product.
//
// Operands enter as K-major int8 planes [I_S][rows][Kp] (i8_planes_kernel, which also transposes
// when the source is M-major).  Persistent CTAs (one per SM) over 128 x ntile (<= 96) output tiles;
// warp 0 = TMA loader, warp 1 = MMA issuer (one elected lane, 2 x 15 MMAs per 64-deep K block),
// warps 2-9 = epilogue (tcgen05.ld 32x32b, lane quarter = warp % 4, two warps per quarter splitting the
// columns), which drains TMEM after each K chunk while the loader already streams the next one.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace cakf {

namespace {

constexpr int I_BM = 128;
constexpr int I_BK = 64;                      // int8 per K block: one 64-byte swizzle row
constexpr int I_S = 5;                        // 7-bit slices per operand (35 bits)
constexpr int I_KC = 8192;                    // K elements per exact int32 chunk (and per work item)
constexpr int I_KBC = I_KC / I_BK;            // K blocks per chunk
constexpr int I_MAXN = 96;                    // I_S accumulators of <= 96 columns in 512 TMEM columns
constexpr int I_STACK_MAXN = 48;              // stacked, one chunk: I_S levels x 48 <= 256 columns, two buffers
constexpr int I_EPI_WARPS = 8;               // two per TMEM lane quarter, each draining half the columns
constexpr int I_THREADS = 64 + 32 * I_EPI_WARPS;   // loader, MMA, epilogue warps
constexpr int I_APLANE = I_BM * I_BK;         // 8 KB
constexpr int I_SMEM_BUDGET = 220 * 1024;
static_assert((long long)I_S * 127 * 127 * I_KC < (1ll << 31), "int32 accumulators must stay exact");

int sm_count() { return num_sms(); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Chunk exponents, stored offset by kExpBias (0 = all-zero chunk): e = ilogb(max |src(r, k)|) + 1 over
// chunk c, so 2^e > max.  Blocks reduce a tile and atomicMax the encoded value (order-independent).
// A chunk holding a NaN or an Inf gets the reserved code kExpNaN (the largest, so atomicMax keeps it): its
// slices are written as zeros and every output that reads the chunk is NaN, so non-finite factors
// propagate instead of being sliced into finite garbage.
constexpr int kExpBias = 512;
constexpr int kExpNaN = 2 * kExpBias + 1;
__device__ __forceinline__ int enc_exp(float m) {
  if (!(m <= 3.402823466e38f)) return kExpNaN;   // Inf (NaN was mapped to Inf by nonfinite_abs)
  return m > 0.f ? min(max(ilogbf(m) + 1 + kExpBias, 1), 2 * kExpBias) : 0;
}
__device__ __forceinline__ int enc_exp(double m) {
  if (!(m <= 1.7976931348623157e308)) return kExpNaN;
  return m > 0.0 ? min(max(ilogb(m) + 1 + kExpBias, 1), 2 * kExpBias) : 0;
}
__device__ __forceinline__ int dec_exp(int v) { return v ? v - kExpBias : 0; }
// |x| with NaN mapped to +Inf (fmax would drop a NaN)
template <typename Src>
__device__ __forceinline__ Src nonfinite_abs(Src x) {
  const Src a = fabs(x);
  return a == a ? a : Src(INFINITY);
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

// kind::i8 instruction descriptor: D = S32 (2), A = B = signed 8-bit (1), both K-major
__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_s8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
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

__device__ __forceinline__ void tma3_mc(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t bar,
                                        uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// Persistent: CTA b takes work items w = b, b + grid, ... with w -> (n tile fastest, m tile, split z),
// so the CTAs sharing an A tile run together (L2 reuse).  Split z covers K chunks
// [z cps, min((z+1) cps, nchunk)).  work == nullptr (one chunk): C / Cd = alpha v + beta C directly;
// else split z's fp64 tile goes to work[(z N + n) M + m] (its chunks accumulated in place) for
// i8_reduce.  lower: skip tiles strictly above the diagonal (symmetric Gram, lower triangle wanted).
// The loader streams the K blocks of all the CTA's chunks back to back; the MMA warp waits for the
// epilogue to drain TMEM (tfree) before the first MMA of every chunk after the CTA's first.
__device__ __forceinline__ bool i8_item(int w, int ntiles, int mt, int ntile, int lower, int& m0, int& n0, int& z) {
  const int nt = w % ntiles, r = w / ntiles;
  m0 = (r % mt) * I_BM;
  n0 = nt * ntile;
  z = r / mt;
  return !(lower && n0 >= m0 + I_BM);
}

__global__ void __launch_bounds__(I_THREADS, 1)
gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const int* __restrict__ expA, const int* __restrict__ expB, int M, int N, int nkb, int nchunk, int cps,
               int ntile, int ntiles, int mt, int nwork, int stages, int lower, int stack, int mc, double alpha,
               double beta, float* __restrict__ C, double* __restrict__ Cd, size_t ldc, double* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  const uint32_t b_plane = (uint32_t)ntile * I_BK;
  const uint32_t stage_bytes = ((uint32_t)I_S * I_APLANE + (uint32_t)I_S * b_plane + 1023u) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(sbase + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;    // [2] MMA -> epilogue: chunk accumulated (per accumulator buffer)
  uint64_t* tfree = done + 2;         // [2] epilogue -> MMA: TMEM buffer drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // mc = 2 (CTA pair, one cluster): both CTAs walk the same items (m tile, pair of n tiles) in lockstep, each
  // computing its own n tile; every A plane of a K block is loaded once for the pair and multicast into both
  // CTAs' shared memory (each CTA issues its share of the planes), halving the L2 -> SM traffic of A, the
  // operand re-read by every n tile.  A stage is refilled only after both CTAs' MMAs released it.
  const int crank = mc > 1 ? (int)(blockIdx.x % mc) : 0;
  const int wfirst = blockIdx.x / mc, wstride = gridDim.x / mc;
  auto item = [&](int w, int& m0, int& n0, int& z) {
    if (!i8_item(w, ntiles, mt, ntile * mc, lower, m0, n0, z)) return false;
    n0 += crank * ntile;
    return true;
  };
  // stack: the B slices sit contiguously in shared memory, so one MMA A_s x [B_0 | ... | B_{4-s}] (N = (5-s)
  // ntile) at TMEM column offset s ntile lands every product A_s B_t on level s + t's columns: 5 MMAs per
  // 32-deep k-step instead of 15 (each A slice read once), levels ntile columns apart, and with ntile <= 48
  // the 5 levels fit in 256 columns: two accumulator buffers, so the drain of chunk g overlaps the MMAs of
  // chunk g + 1.  Otherwise: one accumulator per level (32-column aligned), one buffer.
  const uint32_t acc_stride = stack ? (uint32_t)ntile : (uint32_t)((ntile + 31) / 32 * 32);
  const int nbuf = (stack && I_S * ntile <= 256) ? 2 : 1;   // stacked ntile <= 48: two buffers; <= 96: one

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), mc);   // released by the MMAs of every CTA of the pair
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&done[b]), 1);
      mbar_init(smem_u32(&tfree[b]), I_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (mc > 1) {   // the peer's barriers exist before any multicast lands on them
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(sbase);

  if (warp == 0) {
    if (lane == 0) {   // ===== TMA loader: the K blocks of every item's chunks, in order
      const uint32_t bytes = (uint32_t)I_S * I_APLANE + (uint32_t)I_S * b_plane;
      int it = 0;
      for (int w = wfirst; w < nwork; w += wstride) {
        int m0, n0, z;
        if (!item(w, m0, n0, z)) continue;
        const int kb_begin = z * cps * I_KBC, kb_end = min(nkb, min(nchunk, (z + 1) * cps) * I_KBC);
        for (int kb = kb_begin; kb < kb_end; ++kb, ++it) {
          const int s = it % stages;
          if (it >= stages) mbar_wait(smem_u32(&empty[s]), ((it / stages) - 1) & 1);
          const uint32_t bar = smem_u32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
          const uint32_t st0 = sm0 + s * stage_bytes;
          const int k0 = kb * I_BK;
          if (mc > 1) {   // this CTA's share of the A planes, to both CTAs of the pair
#pragma unroll
            for (int pl = 0; pl < I_S; ++pl)
              if (pl % mc == crank) tma3_mc(st0 + pl * I_APLANE, &tmA, k0, m0, pl, bar, (uint16_t)((1u << mc) - 1u));
          } else {
#pragma unroll
            for (int pl = 0; pl < I_S; ++pl) tma3(st0 + pl * I_APLANE, &tmA, k0, m0, pl, bar);
          }
#pragma unroll
          for (int pl = 0; pl < I_S; ++pl) tma3(st0 + I_S * I_APLANE + pl * b_plane, &tmB, k0, n0, pl, bar);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer: per chunk, level L = s + t accumulates alpha_s beta_t into accumulator L
    const uint32_t idesc = idesc_s8(I_BM, ntile);
    int it = 0, gc = 0;   // K block / chunk counters of this CTA
    for (int w = wfirst; w < nwork; w += wstride) {
      int m0, n0, z;
      if (!item(w, m0, n0, z)) continue;
      const int c0 = z * cps, c1 = min(nchunk, c0 + cps);
      for (int c = c0; c < c1; ++c, ++gc) {
        const int b = gc % nbuf;
        if (gc >= nbuf) mbar_wait(smem_u32(&tfree[b]), ((gc / nbuf) - 1) & 1);   // buffer b drained
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tb = tmem + (uint32_t)b * 256u;
        const int kbe = min(nkb, (c + 1) * I_KBC);
        for (int kb = c * I_KBC; kb < kbe; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(smem_u32(&full[s]), (it / stages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (lane == 0) {
            const uint32_t a0 = sm0 + s * stage_bytes, b0 = a0 + I_S * I_APLANE;
            const bool first_kb = kb == c * I_KBC;
#pragma unroll
            for (int j = 0; j < I_BK / 32; ++j) {
              if (stack) {   // N per MMA <= 256: B rows [off, off + 256) start off * 64 bytes in (8-row aligned)
#pragma unroll
                for (int sa = 0; sa < I_S; ++sa) {
                  const int ntot = (I_S - sa) * ntile;
                  for (int off = 0; off < ntot; off += 256) {
                    const uint32_t acc = (first_kb && j == 0 && sa == 0) ? 0u : 1u;
                    mma_s8(tb + (uint32_t)(sa * ntile + off), sdesc_sw64(a0 + sa * I_APLANE + 32 * j),
                           sdesc_sw64(b0 + (uint32_t)off * I_BK + 32 * j), idesc_s8(I_BM, min(256, ntot - off)),
                           acc);
                  }
                }
              } else {
#pragma unroll
                for (int L = 0; L < I_S; ++L) {
#pragma unroll
                  for (int sa = 0; sa <= L; ++sa) {
                    const int sb = L - sa;
                    const uint32_t acc = (first_kb && j == 0 && sa == 0) ? 0u : 1u;
                    mma_s8(tb + (uint32_t)L * acc_stride, sdesc_sw64(a0 + sa * I_APLANE + 32 * j),
                           sdesc_sw64(b0 + sb * b_plane + 32 * j), idesc, acc);
                  }
                }
              }
            }
            if (mc > 1)   // release the stage in both CTAs (the peer may refill its A share into ours)
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                      smem_u32(&empty[s])),
                  "h"((uint16_t)((1u << mc) - 1u))
                  : "memory");
            else
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&empty[s]))
                           : "memory");
            if (kb == kbe - 1)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&done[b]))
                           : "memory");
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ===== epilogue (warps 2-9): one output row per thread, 8 columns per TMEM load
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;   // warps 2-5: columns [0, ntile/2), warps 6-9: [ntile/2, ntile)
    const bool direct = work == nullptr;
    int gc = 0;
    for (int w = wfirst; w < nwork; w += wstride) {
      int m0, n0, z;
      if (!item(w, m0, n0, z)) continue;
      const int c0 = z * cps, c1 = min(nchunk, c0 + cps);
      const int row = m0 + quarter * 32 + lane;
      const int cb0 = half * (ntile >> 1), cb1 = cb0 + (ntile >> 1);   // this warp's columns (ntile % 16 == 0)
      for (int c = c0; c < c1; ++c, ++gc) {
        const int lc = c - c0;
        // while the MMAs of this chunk run: pull the tile's old C (or split partial) lines into L2 so the
        // drain below reads them at L2 latency (the epilogue is on the critical path between chunks)
        if ((direct ? beta != 0.0 : lc != 0) && row < M) {
          const size_t esz = (direct && !Cd) ? 4 : 8;
          const char* base = !direct ? reinterpret_cast<const char*>(work + (size_t)z * N * M + row)
                             : Cd      ? reinterpret_cast<const char*>(Cd + row)
                                       : reinterpret_cast<const char*>(C + row);
          const size_t ldb = (direct ? ldc : (size_t)M) * esz;
          for (int t = cb0; t < cb1 && n0 + t < N; ++t)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)(n0 + t) * ldb));
        }
        const bool readold = direct ? beta != 0.0 : lc != 0;
        // the 8 columns' global operands (B exponents, the old C or the split partial) of batch cb, all
        // loads issued before any use (predicated); software-pipelined one batch ahead of the TMEM drain
        auto fetch = [&](int cb, int (&codeB)[8], double (&old)[8]) {
          bool ok[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int n = n0 + cb + t;
            ok[t] = row < M && cb + t < ntile && n < N;
            codeB[t] = ok[t] ? __ldg(expB + (size_t)n * nchunk + c) : 0;
          }
          if (readold && (!direct || Cd)) {
            const double* src = direct ? Cd + row : work + (size_t)z * N * M + row;
            const size_t ld = direct ? ldc : (size_t)M;
#pragma unroll
            for (int t = 0; t < 8; ++t) old[t] = ok[t] ? src[(size_t)(n0 + cb + t) * ld] : 0.0;
          } else if (readold) {
            float of[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) of[t] = ok[t] ? C[row + (size_t)(n0 + cb + t) * ldc] : 0.f;
#pragma unroll
            for (int t = 0; t < 8; ++t) old[t] = (double)of[t];
          } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) old[t] = 0.0;
          }
        };
        int codeN[8];
        double oldN[8];
        fetch(cb0, codeN, oldN);   // the first batch's loads overlap the chunk's MMAs
        const int b = gc % nbuf;
        mbar_wait(smem_u32(&done[b]), (gc / nbuf) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int codeA = row < M ? expA[(size_t)row * nchunk + c] : 0;
        const int ea = dec_exp(codeA);
        for (int cb = cb0; cb < cb1; cb += 8) {
          int codeB[8];
          double old[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            codeB[t] = codeN[t];
            old[t] = oldN[t];
          }
          if (cb + 8 < cb1) fetch(cb + 8, codeN, oldN);
          uint32_t r[I_S][8];
          const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)b * 256u + (uint32_t)cb;
#pragma unroll
          for (int L = 0; L < I_S; ++L) tmem_ld8(taddr + (uint32_t)L * acc_stride, r[L]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (row < M) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const int n = n0 + cb + t;
              if (cb + t < ntile && n < N) {
                // V = sum_L acc_L 2^{7(I_S-1-L)} exactly in int64 (|V| < 2^{31 + 7(I_S-1) + 1} <= 2^60),
                // one rounding to fp64, times the exact power of two 2^{e_a + e_b - 7(I_S+1)}
                long long V = (int)r[0][t];
#pragma unroll
                for (int L = 1; L < I_S; ++L) V = (V << 7) + (long long)(int)r[L][t];
                const int ex2 = ea + dec_exp(codeB[t]) - 7 * (I_S + 1);
                double v = (double)V * __longlong_as_double((long long)(ex2 + 1023) << 52);
                if (codeA == kExpNaN || codeB[t] == kExpNaN) v = __longlong_as_double(0x7ff8000000000000ll);
                if (direct) {
                  const double o = beta != 0.0 ? alpha * v + beta * old[t] : alpha * v;
                  if (Cd) Cd[row + (size_t)n * ldc] = o;
                  else C[row + (size_t)n * ldc] = (float)o;
                } else {
                  work[((size_t)z * N + n) * M + row] = lc == 0 ? v : old[t] + v;
                }
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tfree[b]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (mc > 1) {   // no CTA leaves while its peer may still multicast into it or arrive on its barriers
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

template <typename O>
__global__ void i8_reduce_kernel(int M, int N, int S, int lower, const double* __restrict__ work, double alpha,
                                 double beta, O* __restrict__ C, size_t ldc) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)M * N) return;
  const int m = (int)(e % M), n = (int)(e / M);
  if (lower && n > m) return;
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += work[((size_t)z * N + n) * M + m];
  O* c = C + m + (size_t)n * ldc;
  *c = (O)(beta != 0.0 ? alpha * s + beta * (double)*c : alpha * s);
}

// (r, k) at src[k + r ld]: block = one row, 2048 consecutive k (inside one chunk)
template <typename Src>
__global__ void i8_exps_kc_kernel(const Src* __restrict__ src, int R, int K, size_t ld, int nchunk,
                                  int* __restrict__ ex) {
  __shared__ Src red[8];
  const int r = blockIdx.x, k0 = blockIdx.y * 2048;
  Src m = 0;
  for (int k = k0 + threadIdx.x; k < min(K, k0 + 2048); k += 256) m = fmax(m, nonfinite_abs(src[k + (size_t)r * ld]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
    const int e = enc_exp(m);
    if (e) atomicMax(&ex[(size_t)r * nchunk + k0 / I_KC], e);
  }
}

// (r, k) at src[r + k ld]: thread = one row, 64 consecutive k (inside one chunk)
template <typename Src>
__global__ void i8_exps_rc_kernel(const Src* __restrict__ src, int R, int K, size_t ld, int nchunk,
                                  int* __restrict__ ex) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x, k0 = blockIdx.y * 64;
  if (r >= R) return;
  Src m = 0;
  for (int k = k0; k < min(K, k0 + 64); ++k) m = fmax(m, nonfinite_abs(src[r + (size_t)k * ld]));
  const int e = enc_exp(m);
  if (e) atomicMax(&ex[(size_t)r * nchunk + k0 / I_KC], e);
}

// planes[s][r][k] (r < R, k < Kp; zero for k >= K): the 7-bit slices of src(r, k) 2^-e[r][k / I_KC]
// at KC ? src[k + r ld] : src[r + k ld].  Tile 32 rows x 128 k; each thread slices 4 consecutive k of
// one row and stores them as one 4-byte word per plane (the M-major source goes through smem).
template <typename Src, bool KC>
__global__ void i8_planes_kernel(const Src* __restrict__ src, int R, int K, int Kp, size_t ld, int nchunk,
                                 const int* __restrict__ ex, int8_t* __restrict__ planes, size_t plane) {
  __shared__ Src tile[KC ? 1 : 128][33];
  const int k0 = blockIdx.x * 128, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: 8 x 32
  if (!KC) {
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int k = k0 + ty + 8 * i, r = r0 + tx;
      tile[ty + 8 * i][tx] = (k < K && r < R) ? src[r + (size_t)k * ld] : Src(0);
    }
    __syncthreads();
  }
  const int k = k0 + 4 * tx;
  if (k >= Kp) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i;
    if (r >= R) continue;
    const int code = ex[(size_t)r * nchunk + min(k, K - 1) / I_KC];   // 4 k never straddle a chunk
    const int e = dec_exp(code);
    uint32_t word[I_S] = {};
    if (code == kExpNaN) {   // non-finite chunk: zero slices, the epilogue writes NaN
      const size_t o = (size_t)r * Kp + k;
#pragma unroll
      for (int s_ = 0; s_ < I_S; ++s_) *reinterpret_cast<uint32_t*>(planes + s_ * plane + o) = 0u;
      continue;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      Src v;
      if (KC) v = k + j < K ? src[k + j + (size_t)r * ld] : Src(0);
      else v = tile[4 * tx + j][ty + 8 * i];
      // |t| < 1; each step t*128 and t - trunc(t) is exact in the source precision
      Src t = (Src)ldexp((double)v, -e);
#pragma unroll
      for (int s_ = 0; s_ < I_S; ++s_) {
        t *= Src(128);
        const Src a = trunc(t);
        word[s_] |= ((uint32_t)(int)a & 0xFFu) << (8 * j);
        t -= a;
      }
    }
    const size_t o = (size_t)r * Kp + k;
#pragma unroll
    for (int s_ = 0; s_ < I_S; ++s_) *reinterpret_cast<uint32_t*>(planes + s_ * plane + o) = word[s_];
  }
}

// One pass for the K-contiguous case: block (chunk c, row r) holds the chunk's <= I_KC values in registers,
// reduces their max to the chunk exponent (written, no atomics: the block owns the chunk) and writes the
// slices — the source is read once instead of twice (i8_exps_kc_kernel + i8_planes_kernel<KC>).  Same
// exponent code and the same slicing arithmetic, so the planes are bit-identical to the two-pass path.
constexpr int I_SPLIT_T = 256;
constexpr int I_SPLIT_G = I_KC / (4 * I_SPLIT_T);   // groups of 4 consecutive k per thread (8)
template <typename Src>
__global__ void __launch_bounds__(I_SPLIT_T) i8_split_kc_kernel(const Src* __restrict__ src, int K, int Kp, size_t ld,
                                                                int nchunk, int* __restrict__ ex,
                                                                int8_t* __restrict__ planes, size_t plane) {
  __shared__ Src red[I_SPLIT_T / 32];
  const int c = blockIdx.x, r = blockIdx.y;
  const int k0 = c * I_KC, kend = min(Kp, k0 + I_KC);
  const Src* row = src + (size_t)r * ld;
  Src v[I_SPLIT_G][4];
  Src m = Src(0);
  // fp32 rows with 16-byte alignment (ld % 4 == 0, aligned base): one float4 load per group of 4
  const bool vec = sizeof(Src) == 4 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
#pragma unroll
  for (int g = 0; g < I_SPLIT_G; ++g) {
    const int k = k0 + 4 * (g * I_SPLIT_T + threadIdx.x);
    if (vec && k + 3 < K && k + 3 < kend) {
      if constexpr (sizeof(Src) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(row + k);
        v[g][0] = q.x;
        v[g][1] = q.y;
        v[g][2] = q.z;
        v[g][3] = q.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[g][j] = k + j < K && k + j < kend ? row[k + j] : Src(0);
    }
  }
#pragma unroll
  for (int g = 0; g < I_SPLIT_G; ++g)
#pragma unroll
    for (int j = 0; j < 4; ++j) m = fmax(m, nonfinite_abs(v[g][j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < I_SPLIT_T / 32; ++w) m = fmax(m, red[w]);
  const int code = enc_exp(m);
  if (threadIdx.x == 0) ex[(size_t)r * nchunk + c] = code;
  const int e = dec_exp(code);
#pragma unroll
  for (int g = 0; g < I_SPLIT_G; ++g) {
    const int k = k0 + 4 * (g * I_SPLIT_T + threadIdx.x);
    if (k >= kend) continue;
    uint32_t word[I_S] = {};
    if (code != kExpNaN) {   // non-finite chunk: zero slices, the epilogue writes NaN
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // |t| < 1; each step t*128 and t - trunc(t) is exact in the source precision
        Src t = (Src)ldexp((double)v[g][j], -e);
#pragma unroll
        for (int s_ = 0; s_ < I_S; ++s_) {
          t *= Src(128);
          const Src a = trunc(t);
          word[s_] |= ((uint32_t)(int)a & 0xFFu) << (8 * j);
          t -= a;
        }
      }
    }
    const size_t o = (size_t)r * Kp + k;
#pragma unroll
    for (int s_ = 0; s_ < I_S; ++s_) *reinterpret_cast<uint32_t*>(planes + s_ * plane + o) = word[s_];
  }
}

// One pass for the rows-contiguous case with a single K chunk (K <= kRcMaxK: the M-major factor of
// M^- U / M^- (M^-T x)): block = 32 rows, the whole [K][32] tile staged in shared memory with coalesced
// row loads, the per-row maximum -> exponent, then the slices from shared memory.  Same codes and slicing
// arithmetic as i8_exps_rc_kernel + i8_planes_kernel<RC>.
constexpr int kRcMaxK = 1024;
template <typename Src>
constexpr int rc_max_k() { return sizeof(Src) == 4 ? kRcMaxK : kRcMaxK / 2; }
template <typename Src>
__global__ void __launch_bounds__(256) i8_split_rc_kernel(const Src* __restrict__ src, int R, int K, int Kp, size_t ld,
                                                          int* __restrict__ ex, int8_t* __restrict__ planes,
                                                          size_t plane) {
  extern __shared__ __align__(16) unsigned char rc_raw[];
  Src* tile = reinterpret_cast<Src*>(rc_raw);   // [Kp][33]
  __shared__ Src red[8][32];
  __shared__ int codes[32];
  const int r0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  {
    const int r = r0 + tx;
    Src m = Src(0);
#pragma unroll 16
    for (int k = ty; k < Kp; k += 8) {
      const Src v = (k < K && r < R) ? src[r + (size_t)k * ld] : Src(0);
      tile[k * 33 + tx] = v;
      m = fmax(m, nonfinite_abs(v));
    }
    red[ty][tx] = m;
  }
  __syncthreads();
  if (ty == 0) {
    Src m = red[0][tx];
#pragma unroll
    for (int y = 1; y < 8; ++y) m = fmax(m, red[y][tx]);
    const int code = enc_exp(m);
    codes[tx] = code;
    if (r0 + tx < R) ex[r0 + tx] = code;   // one chunk: ex[r * 1 + 0]
  }
  __syncthreads();
  for (int kw = 0; kw < Kp; kw += 128) {
    const int k = kw + 4 * tx;
    if (k >= Kp) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = ty + 8 * i, r = r0 + rl;
      if (r >= R) continue;
      const int code = codes[rl];
      const int e = dec_exp(code);
      uint32_t word[I_S] = {};
      if (code != kExpNaN) {   // non-finite chunk: zero slices, the epilogue writes NaN
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          Src t = (Src)ldexp((double)tile[(k + j) * 33 + rl], -e);
#pragma unroll
          for (int s_ = 0; s_ < I_S; ++s_) {
            t *= Src(128);
            const Src a = trunc(t);
            word[s_] |= ((uint32_t)(int)a & 0xFFu) << (8 * j);
            t -= a;
          }
        }
      }
      const size_t o = (size_t)r * Kp + k;
#pragma unroll
      for (int s_ = 0; s_ < I_S; ++s_) *reinterpret_cast<uint32_t*>(planes + s_ * plane + o) = word[s_];
    }
  }
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

bool make_i8_map(CUtensorMap* tm, const int8_t* planes, int rows, int Kp, int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t gd[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)I_S};
  const cuuint64_t gs[2] = {(cuuint64_t)Kp, (cuuint64_t)Kp * rows};
  const cuuint32_t box[3] = {I_BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)planes, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int gemm_i8_kp(int K) { return (K + 15) / 16 * 16; }
int gemm_i8_nchunk(int K) { return K <= 0 ? 1 : (K + I_KC - 1) / I_KC; }
size_t gemm_i8_plane_bytes(int rows, int K) { return (size_t)I_S * rows * gemm_i8_kp(K); }

template <typename Src>
cudaError_t gemm_i8_split(const Src* src, int R, int K, size_t ld, bool k_contig, int8_t* planes, int* ex,
                          cudaStream_t st) {
  if (R <= 0 || K <= 0) return cudaSuccess;
  const int Kp = gemm_i8_kp(K), nchunk = gemm_i8_nchunk(K);
  if (k_contig && use_i8_split_fused()) {   // one pass: chunk exponents and slices
    i8_split_kc_kernel<Src><<<dim3(nchunk, R), I_SPLIT_T, 0, st>>>(src, K, Kp, ld, nchunk, ex, planes,
                                                                    (size_t)R * Kp);
    return note_launch_err();
  }
  if (!k_contig && Kp <= rc_max_k<Src>() && use_i8_split_fused()) {   // one pass: row exponents and slices
    const size_t smem = (size_t)Kp * 33 * sizeof(Src);
    static PerDeviceOnce once_rc;
    const cudaError_t ce = once_per_device(once_rc, [] {
      return cudaFuncSetAttribute(i8_split_rc_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((size_t)rc_max_k<Src>() * 33 * sizeof(Src)));
    });
    if (ce != cudaSuccess) return ce;
    i8_split_rc_kernel<Src><<<(R + 31) / 32, 256, smem, st>>>(src, R, K, Kp, ld, ex, planes, (size_t)R * Kp);
    return note_launch_err();
  }
  cudaError_t e = cudaMemsetAsync(ex, 0, (size_t)R * nchunk * sizeof(int), st);
  if (e != cudaSuccess) return e;
  if (k_contig) i8_exps_kc_kernel<Src><<<dim3(R, (K + 2047) / 2048), 256, 0, st>>>(src, R, K, ld, nchunk, ex);
  else i8_exps_rc_kernel<Src><<<dim3((R + 255) / 256, (K + 63) / 64), 256, 0, st>>>(src, R, K, ld, nchunk, ex);
  e = note_launch_err();
  if (e != cudaSuccess) return e;
  dim3 grid((Kp + 127) / 128, (R + 31) / 32);
  const size_t plane = (size_t)R * Kp;
  if (k_contig) i8_planes_kernel<Src, true><<<grid, 256, 0, st>>>(src, R, K, Kp, ld, nchunk, ex, planes, plane);
  else i8_planes_kernel<Src, false><<<grid, 256, 0, st>>>(src, R, K, Kp, ld, nchunk, ex, planes, plane);
  return note_launch_err();
}
template cudaError_t gemm_i8_split<float>(const float*, int, int, size_t, bool, int8_t*, int*, cudaStream_t);
template cudaError_t gemm_i8_split<double>(const double*, int, int, size_t, bool, int8_t*, int*, cudaStream_t);

cudaError_t gemm_i8_run(const int8_t* Ap, const int* expA, int M, const int8_t* Bp, const int* expB, int N, int K,
                        double alpha, double beta, float* C, double* Cd, size_t ldc, bool lower, double* work,
                        size_t work_doubles, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  const int Kp = gemm_i8_kp(K), nchunk = gemm_i8_nchunk(K);
  const int nkb = (Kp + I_BK - 1) / I_BK;
  // stacked-B MMAs for one K chunk (the tall M-major products, K <= 8192): ntile <= 48 with double-buffered
  // accumulators, the drain overlapping the next tile (S2 2.16 -> 1.82 ms).  Several chunks (K = D, long MMA
  // runs per drain) stay on one MMA per slice pair with ntile <= 96: stacking there measured slower (ntile 48:
  // more A re-reads; ntile 96 with N split at 256: 1.43 -> 1.60 ms for M^-T x)
  const bool stack = use_i8_stack() && nchunk == 1;
  static const int stack_maxn = [] {   // CAKF_I8_STACK_MAXN=96: one buffer, half the A re-reads (A/B only)
    const char* e = getenv("CAKF_I8_STACK_MAXN");
    const int v = e ? std::atoi(e) : I_STACK_MAXN;
    return v == 96 ? 96 : I_STACK_MAXN;
  }();
  const int maxn = stack ? stack_maxn : I_MAXN;
  // CTA pairs sharing the A planes by multicast (stacked single-chunk products with >= 2 n tiles)
  const int mc = (stack && !lower && use_i8_pair() && N > maxn) ? 2 : 1;
  int ntiles = (N + maxn - 1) / maxn;
  ntiles = (ntiles + mc - 1) / mc * mc;   // whole pairs (a tile past N computes padding only)
  int ntile = (N + ntiles - 1) / ntiles;
  ntile = std::max(16, (ntile + 15) / 16 * 16);
  const int mt = (M + I_BM - 1) / I_BM;
  const uint32_t stage_bytes = ((uint32_t)I_S * I_APLANE + (uint32_t)I_S * ntile * I_BK + 1023u) & ~1023u;
  const int stages = std::max(2, std::min(6, (int)((I_SMEM_BUDGET - 1024 - 256) / stage_bytes)));
  const size_t smem = (size_t)stages * stage_bytes + 1024 + 256;
  static PerDeviceOnce once;
  {
    const cudaError_t e = once_per_device(once, [] {
      return cudaFuncSetAttribute(gemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, I_SMEM_BUDGET);
    });
    if (e != cudaSuccess) return e;
  }
  // one work item per (tile, chunk) when the fp64 partials fit (the persistent CTAs then balance many
  // small items), else whole chunks grouped per split; every chunk count >= 2 goes through work
  int splits = nchunk;
  int cps = 1;
  while (nchunk > 1 && (size_t)splits * M * N > work_doubles && splits > 1) {
    ++cps;
    splits = (nchunk + cps - 1) / cps;
  }
  const bool reduce = nchunk > 1;
  if (reduce && (size_t)splits * M * N > work_doubles) return cudaErrorInvalidValue;
  CUtensorMap tmA, tmB;
  if (!make_i8_map(&tmA, Ap, M, Kp, I_BM) || !make_i8_map(&tmB, Bp, N, Kp, ntile)) return cudaErrorInvalidValue;
  const int nunits = ntiles / mc;   // items: (m tile, n tile or pair of n tiles, K split)
  const int nwork = mt * nunits * splits;
  cudaError_t e;
  if (mc > 1) {
    const int grid = mc * std::min(nwork, sm_count() / mc);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(I_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, gemm_i8_kernel, tmA, tmB, expA, expB, M, N, nkb, nchunk, cps, ntile, nunits, mt,
                           nwork, stages, lower ? 1 : 0, stack ? 1 : 0, mc, alpha, beta, C, Cd, ldc,
                           reduce ? work : nullptr);
    ++launch_counter();
    if (e == cudaSuccess) e = cudaGetLastError();
  } else {
    const int grid = std::min(nwork, sm_count());
    gemm_i8_kernel<<<grid, I_THREADS, smem, st>>>(tmA, tmB, expA, expB, M, N, nkb, nchunk, cps, ntile, nunits, mt,
                                                  nwork, stages, lower ? 1 : 0, stack ? 1 : 0, 1, alpha, beta, C, Cd,
                                                  ldc, reduce ? work : nullptr);
    e = note_launch_err();
  }
  if (e != cudaSuccess || !reduce) return e;
  const size_t tot = (size_t)M * N;
  if (Cd)
    i8_reduce_kernel<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, splits, lower ? 1 : 0, work, alpha,
                                                                             beta, Cd, ldc);
  else
    i8_reduce_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, splits, lower ? 1 : 0, work, alpha,
                                                                            beta, C, ldc);
  return note_launch_err();
}

bool use_i8_pair() {   // off by default: measured no faster on the tall products (S2 1.86 -> 1.99 ms)
  static const bool v = env_is("CAKF_I8_PAIR", '1');
  return v;
}

bool use_i8_stack() {
  static const bool v = !env_is("CAKF_I8_STACK", '0');
  return v;
}

bool use_i8_split_fused() {
  static const bool v = !env_is("CAKF_I8_SPLIT_FUSED", '0');
  return v;
}

bool use_i8_gemm() {
  static const bool v = !env_is("CAKF_GEMM_F64", '1');
  return v;
}

}  // namespace cakf
