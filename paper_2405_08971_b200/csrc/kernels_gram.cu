// kernels_gram.cu — fused kernel-evaluation x vector / x matrix products (sm_100a).
//
// The paper's bottleneck: products with the spatial Gram matrix
// Sigma^x(X, X) that is never materialised.  Two shapes occur on the hot path:
//   K1  single right-hand side (the inner-loop matvec G s):
//       ALU bound (FP32 pipe + MUFU sqrt/ex2 per pair) — register-blocked rows,
//       column chunk staged once in shared memory, broadcast LDS.128 reads.
//   K2  many right-hand sides (post-loop a7, smoother a9): a GEMM whose A operand
//       is generated on the fly; SIMT register-tiled version (8x8 per thread).
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace cakf {

namespace {


template <typename T> constexpr int kRowsPerThread = sizeof(T) == 4 ? 4 : 2;
constexpr int kMvThreads = 256;
template <typename T> constexpr int kMaxChunk = sizeof(T) == 4 ? 2048 : 1024;

// ------------------------------------------------------------------ K1
template <typename T, int NU2, int R>
__global__ void __launch_bounds__(kMvThreads)
matvec_partial_kernel(const V4<T>* __restrict__ xr, int nrows, const V4<T>* __restrict__ xc, int ncols,
                      int chunk, int ch0, T* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V4<T>* sc = reinterpret_cast<V4<T>*>(smem_raw);
  const int ch = ch0 + blockIdx.y;
  const int j0 = ch * chunk;
  const int n = min(chunk, ncols - j0);
  for (int j = threadIdx.x; j < n; j += kMvThreads) sc[j] = xc[j0 + j];

  T px[R], py[R], pz[R], acc[R];
  const int base = blockIdx.x * (kMvThreads * R) + threadIdx.x;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int row = base + k * kMvThreads;
    V4<T> p{};
    if (row < nrows) p = xr[row];
    px[k] = p.x; py[k] = p.y; pz[k] = p.z;
    acc[k] = T(0);
  }
  __syncthreads();
#pragma unroll 2
  for (int j = 0; j < n; ++j) {
    const V4<T> c = sc[j];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const T dx = px[k] - c.x, dy = py[k] - c.y, dz = pz[k] - c.z;
      const T d2 = fma(dz, dz, fma(dy, dy, dx * dx));
      acc[k] = fma(matern_from_d2<NU2>(d2), c.w, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int row = base + k * kMvThreads;
    if (row < nrows) partial[(size_t)ch * nrows + row] = acc[k];
  }
}

// ------------------------------------------------------------------ K1, symmetric (fp32)
// K_TT is symmetric: each unordered pair of 128-point tiles is evaluated once.  Tiles are
// grouped into blocks of SYM_S tiles; a work unit is one block pair (bi <= bj), whose
// 2 * SYM_S tiles are staged once in shared memory.  The 16 x 16 threads own 8 x 8
// micro-tiles of each 128 x 128 tile pair; row sums accumulate in registers across the
// unit's J tiles, column sums in shared memory, and the unit writes
//   partial[bj][rows of its I tiles]  and  partial[bi][rows of its J tiles]
// (for a diagonal unit both go to partial[bi], summed), so every row receives exactly one
// partial per block and stage A's fixed-order sum over the nb blocks reduces them
// (deterministic, no atomics).
constexpr int SYM_T = 128;
constexpr int SYM_S = 4;
__device__ __forceinline__ void sym_unit_decode(long long u, int nb, int& bi, int& bj) {
  const double bb = 2.0 * nb + 1.0;
  bi = (int)floor((bb - sqrt(bb * bb - 8.0 * (double)u)) * 0.5);
  while ((long long)bi * nb - (long long)bi * (bi - 1) / 2 > u) --bi;
  while ((long long)(bi + 1) * nb - (long long)(bi + 1) * bi / 2 <= u) ++bi;
  bj = bi + (int)(u - ((long long)bi * nb - (long long)bi * (bi - 1) / 2));
}

// SUB: the exact-zero test and the work run per 16-row group x 32-column sub-tile (sphJ = 32-point
// spheres; each lane owns one packed column pair of the sub-tile), else per 16-row group x 128-column
// J tile (sphJ = 128-point spheres; each lane owns 8 columns).  Row -> lane mapping is the same.
// 72 registers (no spills) leave 10240 of an SM's 65536 registers beside three resident 256-thread CTAs:
// room for one 128-thread side-stream HM CTA, so the HBM-bound HM passes overlap the MUFU-bound K1
#ifndef CAKF_K1_MAXREG
#define CAKF_K1_MAXREG 72
#endif
template <int NU2, bool SUB>
__global__ void __maxnreg__(CAKF_K1_MAXREG)
matvec_sym_kernel(const float4* __restrict__ x, int n, int nt, int nb, long long u_begin, long long u_end,
                  float* __restrict__ partial,
                  unsigned long long* __restrict__ done_pairs, const int* __restrict__ ulist,
                  const int* __restrict__ ucount, const unsigned short* __restrict__ umask,
                  const float4* __restrict__ sph16, const float4* __restrict__ sphJ, float cut,
                  unsigned* __restrict__ sched, const float4* __restrict__ box16, const float4* __restrict__ boxJ) {
  griddep_wait();   // PDL: the actions (xcs .w) come from the preceding stage kernel
  constexpr int NJS = SUB ? SYM_S * 4 : SYM_S;   // J spheres per unit
  extern __shared__ __align__(16) unsigned char sm_raw[];
  __shared__ float4 s16[SYM_S * 8], s128[NJS];   // this unit's 16-row group / J (sub-)tile spheres
  __shared__ float4 b16[SYM_S * 8 * 2], bJ[NJS * 2];   // and their bounding boxes {lo, hi} (SUB)
  __shared__ unsigned s_done;                        // evaluated 16 x 128 warp blocks of this unit
  __shared__ unsigned s_next;                        // dynamic scheduling: this CTA's next work item
  float4* tI = reinterpret_cast<float4*>(sm_raw);                    // [SYM_S][128]
  float4* tJ = tI + SYM_S * SYM_T;                                    // [SYM_S][128]
  float* rowacc = reinterpret_cast<float*>(tJ + SYM_S * SYM_T);       // [SYM_S][128]
  float* colp = rowacc + SYM_S * SYM_T;                               // [16 ty][SYM_S][128] private slots
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float* mycol = colp + ty * SYM_S * SYM_T + tx * 8;                  // this thread's 8 columns of each J tile
  // ulist: compact ascending list of the units with an active tile pair (exact-zero culling); the
  // skipped units' partial slots were zeroed once per update
  const long long nwork = ulist ? (long long)*ucount : u_end - u_begin;
  // sched != nullptr: the first item is blockIdx.x, later ones are taken from a global counter in list
  // order (longest first => greedy LPT balance); the assignment cannot change any result because every
  // unit owns its partial slots.  The last CTA to finish resets the counters for the next launch.
  for (long long w = blockIdx.x; w < nwork;) {
    const long long u = ulist ? (long long)ulist[w] : u_begin + w;
    // active tile pairs of this unit, bit a*SYM_S+b (exact-zero culling; all ones without)
    const unsigned amask = ulist ? (unsigned)umask[w] : 0xFFFFu;
    if (tid == 0) s_done = 0u;
    // u -> (bi, bj), bi <= bj, row-major over the upper triangle of blocks
    int bi, bj;
    sym_unit_decode(u, nb, bi, bj);
    const bool diag = bi == bj;
    const int na = min(SYM_S, nt - bi * SYM_S), nbj = min(SYM_S, nt - bj * SYM_S);
    __syncthreads();
    // tiles stored as point pairs {x0,x1,y0,y1},{z0,z1,s0,s1} so the packed f32x2 operands load ready-paired
    for (int e = tid; e < SYM_S * SYM_T / 2; e += 256) {
      const int gi = bi * SYM_S * SYM_T + 2 * e, gj = bj * SYM_S * SYM_T + 2 * e;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 p0 = gi < n ? x[gi] : z4, p1 = gi + 1 < n ? x[gi + 1] : z4;
      tI[2 * e] = make_float4(p0.x, p1.x, p0.y, p1.y);
      tI[2 * e + 1] = make_float4(p0.z, p1.z, p0.w, p1.w);
      if (!diag) {
        p0 = gj < n ? x[gj] : z4;
        p1 = gj + 1 < n ? x[gj + 1] : z4;
        tJ[2 * e] = make_float4(p0.x, p1.x, p0.y, p1.y);
        tJ[2 * e + 1] = make_float4(p0.z, p1.z, p0.w, p1.w);
      }
    }
    for (int e = tid; e < SYM_S * SYM_T; e += 256) rowacc[e] = 0.f;
#pragma unroll
    for (int b = 0; b < SYM_S; ++b)
#pragma unroll
      for (int c = 0; c < 8; ++c) mycol[b * SYM_T + c] = 0.f;
    const float4* sJ = diag ? tI : tJ;
    if (ulist) {
      // a missing box is the whole space (no constraint beyond the sphere test)
      const float4 blo = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f), bhi = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
      if (tid < SYM_S * 8) {
        const int g = bi * SYM_S * 8 + tid;
        const bool in = g < (n + 15) / 16;
        s16[tid] = in ? sph16[g] : make_float4(0.f, 0.f, 0.f, 0.f);
        if (SUB) {
          b16[2 * tid] = in && box16 ? box16[2 * g] : blo;
          b16[2 * tid + 1] = in && box16 ? box16[2 * g + 1] : bhi;
        }
      } else if (tid < SYM_S * 8 + NJS) {
        const int t = bj * NJS + tid - SYM_S * 8;
        const bool in = t < (SUB ? (n + 31) / 32 : nt);
        s128[tid - SYM_S * 8] = in ? sphJ[t] : make_float4(0.f, 0.f, 0.f, 0.f);
        if (SUB) {
          bJ[2 * (tid - SYM_S * 8)] = in && boxJ ? boxJ[2 * t] : blo;
          bJ[2 * (tid - SYM_S * 8) + 1] = in && boxJ ? boxJ[2 * t + 1] : bhi;
        }
      }
    }
    __syncthreads();
    for (int a = 0; a < na; ++a) {
      if (!((amask >> (a * SYM_S)) & ((1u << SYM_S) - 1u))) continue;   // no active tile pair in this row tile
      // row groups rotate with the row tile (warp w takes 16-row group (w + a) mod 8 of tile a): a warp whose
      // rows sit far from this unit's columns in one row tile is near them in another, which evens out the
      // culled work per warp before the unit-end barrier
      const int tyr = (ty + 2 * a) & 15, wg = ((tid >> 5) + a) & 7;
      // rows kept negated (d = c - r) as scalars: the packed f32x2 ops broadcast a scalar operand
      float nrx[8], nry[8], nrz[8], rs[8];
      float2 racc2[8];   // per row: even / odd column partial sums
      // SUB: the exact-zero test of this warp's 16 rows against all (<= 16) sub-tiles of the unit's J tiles at
      // once, one sub-tile per lane (lane = 4 b + q4), one ballot: bit 4 b + q4 set = possibly nonzero.
      // Both tests compare squares (no square root): sphere |c_A - c_B|^2 <= (cut + r_A + r_B)^2 and box
      // gap^2 <= cut^2 — each a lower bound on every pair distance, so a skipped sub-tile holds exact zeros
      unsigned act16 = 0u;
      if constexpr (SUB) {
        const int lane = tid & 31, b = lane >> 2, q4 = lane & 3;
        bool on = false;
        if (b < nbj && b >= (diag ? a : 0) && ((amask >> (a * SYM_S + b)) & 1u)) {
          on = bj * SYM_S * SYM_T + b * SYM_T + q4 * 32 < n;   // beyond: only padding
          if (ulist && on) {
            const float4 A = s16[a * 8 + wg], B = s128[lane];
            const float ex = A.x - B.x, ey = A.y - B.y, ez = A.z - B.z, rr = cut + A.w + B.w;
            const float4 Al = b16[2 * (a * 8 + wg)], Ah = b16[2 * (a * 8 + wg) + 1], Bl = bJ[2 * lane], Bh = bJ[2 * lane + 1];
            const float gx = fmaxf(fmaxf(Bl.x - Ah.x, Al.x - Bh.x), 0.f), gy = fmaxf(fmaxf(Bl.y - Ah.y, Al.y - Bh.y), 0.f),
                        gz = fmaxf(fmaxf(Bl.z - Ah.z, Al.z - Bh.z), 0.f);
            on = fmaf(ez, ez, fmaf(ey, ey, ex * ex)) <= rr * rr && fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= cut * cut;
          }
        }
        act16 = __ballot_sync(0xffffffffu, on);
        if (!act16) continue;   // nothing of this row tile for this warp (its row sums gain exact zeros only)
        if (ulist && lane == 0) atomicAdd(&s_done, (unsigned)__popc(act16));
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float4 A = tI[(a * SYM_T / 2 + tyr * 4 + h) * 2], B = tI[(a * SYM_T / 2 + tyr * 4 + h) * 2 + 1];
        nrx[2 * h] = -A.x; nrx[2 * h + 1] = -A.y; nry[2 * h] = -A.z; nry[2 * h + 1] = -A.w;
        nrz[2 * h] = -B.x; nrz[2 * h + 1] = -B.y; rs[2 * h] = B.z; rs[2 * h + 1] = B.w;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) racc2[q] = make_float2(0.f, 0.f);
      for (int b = diag ? a : 0; b < nbj; ++b) {
        if (SUB ? !((act16 >> (4 * b)) & 0xFu) : !((amask >> (a * SYM_S + b)) & 1u)) continue;   // all exact zeros
        const bool offdiag = !(diag && a == b);
        if constexpr (SUB) {
          // 4 sub-tiles of 32 columns; lane tx owns the packed column pairs q4*32 + 2tx, +1 (q4 < 4).
          // act: sub-tiles of this warp's 16 rows with a possibly nonzero value (warp-uniform).  A fully
          // active J tile runs all four pairs at once; otherwise the active sub-tiles run one by one in
          // the same order, so every accumulator sees the same operation sequence (skipped = exact zeros).
          const unsigned act = (act16 >> (4 * b)) & 0xFu;
          if (!act) continue;
          if (act == 0xFu) {
            float2 cx2[4], cy2[4], cz2[4], cs2[4], cacc2[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 P = sJ[(b * SYM_T / 2 + q * 16 + tx) * 2], Q = sJ[(b * SYM_T / 2 + q * 16 + tx) * 2 + 1];
              cx2[q] = make_float2(P.x, P.y); cy2[q] = make_float2(P.z, P.w);
              cz2[q] = make_float2(Q.x, Q.y); cs2[q] = make_float2(Q.z, Q.w);
              cacc2[q] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 dx = __fadd2_rn(cx2[q], make_float2(nrx[r], nrx[r]));
                const float2 dy = __fadd2_rn(cy2[q], make_float2(nry[r], nry[r]));
                const float2 dz = __fadd2_rn(cz2[q], make_float2(nrz[r], nrz[r]));
                const float2 d2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
                const float2 k = matern2_from_d2<NU2>(d2);
                racc2[r] = __ffma2_rn(k, cs2[q], racc2[r]);
                cacc2[q] = __ffma2_rn(k, make_float2(rs[r], rs[r]), cacc2[q]);
              }
            }
            if (offdiag) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float2* m2 = reinterpret_cast<float2*>(colp + ty * SYM_S * SYM_T + b * SYM_T + q * 32 + 2 * tx);
                float2 u = *m2;
                u.x += cacc2[q].x;
                u.y += cacc2[q].y;
                *m2 = u;
              }
            }
            continue;
          }
#pragma unroll 1
          for (int q4 = 0; q4 < 4; ++q4) {
            if (!((act >> q4) & 1u)) continue;
            const float4 P = sJ[(b * SYM_T / 2 + q4 * 16 + tx) * 2], Q = sJ[(b * SYM_T / 2 + q4 * 16 + tx) * 2 + 1];
            const float2 cx2 = make_float2(P.x, P.y), cy2 = make_float2(P.z, P.w);
            const float2 cz2 = make_float2(Q.x, Q.y), cs2 = make_float2(Q.z, Q.w);
            float2 cacc2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const float2 dx = __fadd2_rn(cx2, make_float2(nrx[r], nrx[r]));
              const float2 dy = __fadd2_rn(cy2, make_float2(nry[r], nry[r]));
              const float2 dz = __fadd2_rn(cz2, make_float2(nrz[r], nrz[r]));
              const float2 d2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
              const float2 k = matern2_from_d2<NU2>(d2);
              racc2[r] = __ffma2_rn(k, cs2, racc2[r]);
              cacc2 = __ffma2_rn(k, make_float2(rs[r], rs[r]), cacc2);
            }
            if (offdiag) {   // column sums into this thread's private slots (no barrier)
              float2* m2 = reinterpret_cast<float2*>(colp + ty * SYM_S * SYM_T + b * SYM_T + q4 * 32 + 2 * tx);
              float2 u = *m2;
              u.x += cacc2.x;
              u.y += cacc2.y;
              *m2 = u;
            }
          }
          continue;
        }
        if (ulist) {   // same test for this warp's 16 rows against the J tile (warp-uniform)
          const float4 A = s16[a * 8 + wg], B = s128[b];
          const float ex = A.x - B.x, ey = A.y - B.y, ez = A.z - B.z;
          if (sqrtf(ex * ex + ey * ey + ez * ez) - A.w - B.w > cut) continue;
          if ((tid & 31) == 0) atomicAdd(&s_done, 1u);
        }
        // 8 columns as 4 packed pairs: every elementwise op below is one FADD2 / FMUL2 / FFMA2 for two
        // pairs, leaving the two MUFU ops per pair (sqrt, ex2) as the only scalar work
        float2 cx2[4], cy2[4], cz2[4], cs2[4], cacc2[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 A = sJ[(b * SYM_T / 2 + tx * 4 + q) * 2], B = sJ[(b * SYM_T / 2 + tx * 4 + q) * 2 + 1];
          cx2[q] = make_float2(A.x, A.y); cy2[q] = make_float2(A.z, A.w);
          cz2[q] = make_float2(B.x, B.y); cs2[q] = make_float2(B.z, B.w);
          cacc2[q] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 dx = __fadd2_rn(cx2[q], make_float2(nrx[r], nrx[r]));
            const float2 dy = __fadd2_rn(cy2[q], make_float2(nry[r], nry[r]));
            const float2 dz = __fadd2_rn(cz2[q], make_float2(nrz[r], nrz[r]));
            const float2 d2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
            const float2 k = matern2_from_d2<NU2>(d2);
            racc2[r] = __ffma2_rn(k, cs2[q], racc2[r]);
            cacc2[q] = __ffma2_rn(k, make_float2(rs[r], rs[r]), cacc2[q]);
          }
        }
        float cacc[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) { cacc[2 * q] = cacc2[q].x; cacc[2 * q + 1] = cacc2[q].y; }
        if (offdiag) {   // column sums of this tile pair into this thread's private slots (no barrier)
          float4* m4 = reinterpret_cast<float4*>(mycol + b * SYM_T);
          float4 u0 = m4[0], u1 = m4[1];
          u0.x += cacc[0]; u0.y += cacc[1]; u0.z += cacc[2]; u0.w += cacc[3];
          u1.x += cacc[4]; u1.y += cacc[5]; u1.z += cacc[6]; u1.w += cacc[7];
          m4[0] = u0;
          m4[1] = u1;
        }
      }
      // row sums over the unit's J tiles: reduce the 8 rows over tx (16 lanes of a half-warp) as a
      // reduce-scatter (4 + 2 + 1 + 1 shuffles instead of 8 x 4); lane pair (tx, tx ^ 1) ends with row
      // rsel = 4 (tx>>3 & 1) + 2 (tx>>2 & 1) + (tx>>1 & 1)
      float v8[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) v8[r] = racc2[r].x + racc2[r].y;
      const bool h8 = tx & 8, h4 = tx & 4, h2 = tx & 2;
      float w4[4], w2[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float send = h8 ? v8[i] : v8[i + 4], keep = h8 ? v8[i + 4] : v8[i];
        w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float send = h4 ? w4[i] : w4[i + 2], keep = h4 ? w4[i + 2] : w4[i];
        w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      float w1;
      {
        const float send = h2 ? w2[0] : w2[1], keep = h2 ? w2[1] : w2[0];
        w1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
      if (!(tx & 1)) rowacc[a * SYM_T + tyr * 8 + (h8 ? 4 : 0) + (h4 ? 2 : 0) + (h2 ? 1 : 0)] += w1;
    }
    __syncthreads();
    if (tid == 0 && done_pairs && ulist) atomicAdd(done_pairs, (unsigned long long)s_done);
    for (int e = tid; e < SYM_S * SYM_T; e += 256) {
      float cs_ = 0.f;                       // column sums: fixed-order reduction over the 16 ty slots
#pragma unroll
      for (int t = 0; t < 16; ++t) cs_ += colp[t * SYM_S * SYM_T + e];
      const int gi = bi * SYM_S * SYM_T + e;
      if (gi < n) partial[(size_t)bj * n + gi] = rowacc[e] + (diag ? cs_ : 0.f);
      if (!diag) {
        const int gj = bj * SYM_S * SYM_T + e;
        if (gj < n) partial[(size_t)bi * n + gj] = cs_;
      }
    }
    if (sched) {
      if (tid == 0) s_next = gridDim.x + atomicAdd(sched, 1u);
      __syncthreads();   // the next write of s_next is behind the next unit's barriers
      w = s_next;
    } else {
      w += gridDim.x;
    }
  }
  if (sched && tid == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
      sched[0] = 0u;
      sched[1] = 0u;
    }
  }
}

// Coordinate actions: K_TT e_j is column j of the kernel matrix — N evaluations instead of N^2
// (SURVEY §8a a4).  out[row + c*ldo] = k(x_row, x_{order[i0 - 1 + c]}) for c < nb.
template <typename T, int NU2>
__global__ void kernel_columns_kernel(const V4<T>* __restrict__ x, int N, const int* __restrict__ order, int i0, int nb,
                                      T* __restrict__ out, size_t ldo) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * nb) return;
  const int row = (int)(e % N), c = (int)(e / N);
  out[row + (size_t)c * ldo] = matern_from_d2<NU2>(dist2<T>(x[row], x[order[i0 - 1 + c]]));
}

// Bounding sphere (center, radius inflated for rounding) of each tile of `tile` consecutive points.
// box (nullable): the tile's axis-aligned bounding box {lo, hi} (exact coordinates, .w unused), a second
// lower bound on the distance between two tiles (the K1 sub-tile test takes the larger of the two)
__global__ void tile_spheres_kernel(const float4* __restrict__ x, int n, int tile, float4* __restrict__ out,
                                    float4* __restrict__ box) {
  __shared__ double red[4][32];
  __shared__ float bred[6][32];
  __shared__ double cen[3];
  const int t0 = blockIdx.x * tile, t1 = min(n, t0 + tile);
  double sx = 0, sy = 0, sz = 0;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const float4 p = x[i];
    sx += p.x; sy += p.y; sz += p.z;
    lo[0] = fminf(lo[0], p.x); lo[1] = fminf(lo[1], p.y); lo[2] = fminf(lo[2], p.z);
    hi[0] = fmaxf(hi[0], p.x); hi[1] = fmaxf(hi[1], p.y); hi[2] = fmaxf(hi[2], p.z);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  sx = warp_sum(sx); sy = warp_sum(sy); sz = warp_sum(sz);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if (lane == 0) {
    red[0][w] = sx; red[1][w] = sy; red[2][w] = sz;
#pragma unroll
    for (int c = 0; c < 3; ++c) { bred[c][w] = lo[c]; bred[3 + c][w] = hi[c]; }
  }
  __syncthreads();
  if (box && threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) { bred[c][0] = fminf(bred[c][0], bred[c][q]); bred[3 + c][0] = fmaxf(bred[3 + c][0], bred[3 + c][q]); }
    box[2 * blockIdx.x] = make_float4(bred[0][0], bred[1][0], bred[2][0], 0.f);
    box[2 * blockIdx.x + 1] = make_float4(bred[3][0], bred[4][0], bred[5][0], 0.f);
  }
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { a += red[0][q]; b += red[1][q]; c += red[2][q]; }
    const double cnt = (double)max(1, t1 - t0);
    cen[0] = a / cnt; cen[1] = b / cnt; cen[2] = c / cnt;
  }
  __syncthreads();
  double r = 0;
  for (int i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const float4 p = x[i];
    const double dx = p.x - cen[0], dy = p.y - cen[1], dz = p.z - cen[2];
    r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if (lane == 0) red[3][w] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) m = fmax(m, red[3][q]);
    out[blockIdx.x] = make_float4((float)cen[0], (float)cen[1], (float)cen[2], (float)(m * (1.0 + 1e-5) + 1e-3));
  }
}

template <typename T>
__global__ void sum_partials_kernel(int nrows, int nch, const T* __restrict__ partial, double alpha, T* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double acc = 0.0;
  for (int c = 0; c < nch; ++c) acc += (double)partial[(size_t)c * nrows + i];
  y[i] = (T)(alpha * acc);
}

// ------------------------------------------------------------------ K2 (SIMT)
template <typename T, int NU2, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gram_gemm_kernel(const V4<T>* __restrict__ xr, int M, const V4<T>* __restrict__ xc, int K,
                 const T* __restrict__ B, size_t ldb, int C, T* __restrict__ Y, size_t ldy, T alpha) {
  constexpr int NT = (BM / TM) * (BN / TN);
  static_assert(NT % BM == 0, "thread count must be a multiple of BM");
  constexpr int KSTEP = NT / BM;
  constexpr int AG = BK / KSTEP;
  __shared__ __align__(16) T As[BK][BM];
  __shared__ __align__(16) T Bs[BK][BN];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int tid = threadIdx.x;
  const int arow = tid % BM, akk0 = tid / BM;
  V4<T> xa{};
  if (m0 + arow < M) xa = xr[m0 + arow];
  const int ty = tid / (BN / TN), tx = tid % (BN / TN);
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[i][c] = T(0);

  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int q = 0; q < AG; ++q) {
      const int kk = akk0 + q * KSTEP;
      const int j = k0 + kk;
      T v = T(0);
      if (j < K) {
        const V4<T> c = xc[j];
        v = matern_from_d2<NU2>(dist2<T>(xa, c));
      }
      As[kk][arow] = v;
    }
    for (int e = tid; e < BK * BN; e += NT) {
      const int kk = e % BK, nn = e / BK;
      const int j = k0 + kk, n = n0 + nn;
      Bs[kk][nn] = (j < K && n < C) ? B[j + (size_t)n * ldb] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int c = 0; c < TN; ++c) b[c] = Bs[kk][tx * TN + c];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[i][c] = fma(a[i], b[c], acc[i][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < TN; ++c) {
    const int n = n0 + tx * TN + c;
    if (n >= C) continue;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = m0 + ty * TM + i;
      if (m < M) Y[m + (size_t)n * ldy] = alpha * acc[i][c];
    }
  }
}

template <typename T>
__global__ void prescale_kernel(int n, int dim, const double* __restrict__ xyz, double scale, V4<T>* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c[3] = {0.0, 0.0, 0.0};
  for (int d = 0; d < dim; ++d) c[d] = xyz[(size_t)i * dim + d] * scale;
  V4<T> v;
  v.x = (T)c[0]; v.y = (T)c[1]; v.z = (T)c[2]; v.w = T(0);
  out[i] = v;
}

template <typename T, int NU2>
cudaError_t matvec_partial_nu(const V4<T>* xr, int nrows, const V4<T>* xc, int ncols, int nchunks, int ch0, int ch1,
                              T* partial, cudaStream_t st) {
  constexpr int R = kRowsPerThread<T>;
  const int chunk = (ncols + nchunks - 1) / nchunks;
  if (ch1 <= ch0) return cudaSuccess;
  dim3 grid((nrows + kMvThreads * R - 1) / (kMvThreads * R), ch1 - ch0);
  const size_t smem = (size_t)chunk * sizeof(V4<T>);
  matvec_partial_kernel<T, NU2, R><<<grid, kMvThreads, smem, st>>>(xr, nrows, xc, ncols, chunk, ch0, partial);
  return note_launch_err();
}

template <typename T, int NU2>
cudaError_t gram_gemm_nu(const V4<T>* xr, int M, const V4<T>* xc, int K, const T* B, size_t ldb, int C, T* Y,
                         size_t ldy, double alpha, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (C <= 64) {
      dim3 grid((M + 127) / 128, (C + 63) / 64);
      gram_gemm_kernel<T, NU2, 128, 64, 16, 8, 4><<<grid, 256, 0, st>>>(xr, M, xc, K, B, ldb, C, Y, ldy, (T)alpha);
    } else {
      dim3 grid((M + 127) / 128, (C + 127) / 128);
      gram_gemm_kernel<T, NU2, 128, 128, 16, 8, 8><<<grid, 256, 0, st>>>(xr, M, xc, K, B, ldb, C, Y, ldy, (T)alpha);
    }
  } else {
    dim3 grid((M + 63) / 64, (C + 63) / 64);
    gram_gemm_kernel<T, NU2, 64, 64, 16, 4, 4><<<grid, 256, 0, st>>>(xr, M, xc, K, B, ldb, C, Y, ldy, (T)alpha);
  }
  return note_launch_err();
}

}  // namespace

int matvec_chunks(int nrows, int ncols, int elem_bytes) {
  const int R = elem_bytes == 4 ? kRowsPerThread<float> : kRowsPerThread<double>;
  const int maxchunk = elem_bytes == 4 ? kMaxChunk<float> : kMaxChunk<double>;
  const long tiles = (nrows + kMvThreads * R - 1) / (kMvThreads * R);
  const long slots = (long)num_sms() * (2048 / kMvThreads);  // resident CTAs per wave
  const double pairs = (double)nrows * (double)ncols;
  long waves = std::max(1L, (long)(pairs / ((double)slots * 262144.0)));
  waves = std::min(waves, std::max(1L, 128L * tiles / slots));
  long ch = std::max(1L, waves * slots / tiles);
  const long ch_max = std::max(1L, (long)(ncols + 31) / 32);
  const long ch_min = (ncols + maxchunk - 1) / maxchunk;
  ch = std::min(ch, ch_max);
  ch = std::max(ch, std::max(1L, ch_min));
  return (int)ch;
}

template <typename T>
cudaError_t launch_matvec_partial(int nu2, const V4<T>* xr, int nrows, const V4<T>* xc, int ncols, int nchunks,
                                  T* partial, cudaStream_t st, int ch0, int ch1) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  if (ch1 < 0) ch1 = nchunks;
  switch (nu2) {
    case 1: return matvec_partial_nu<T, 1>(xr, nrows, xc, ncols, nchunks, ch0, ch1, partial, st);
    case 3: return matvec_partial_nu<T, 3>(xr, nrows, xc, ncols, nchunks, ch0, ch1, partial, st);
    case 5: return matvec_partial_nu<T, 5>(xr, nrows, xc, ncols, nchunks, ch0, ch1, partial, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tile_spheres(const float4* x, int n, int tile, float4* out, cudaStream_t st, float4* box) {
  if (n <= 0) return cudaSuccess;
  tile_spheres_kernel<<<(n + tile - 1) / tile, 128, 0, st>>>(x, n, tile, out, box);
  return note_launch_err();
}

template <typename T>
cudaError_t launch_kernel_columns(int nu2, const V4<T>* x, int N, const int* order, int i0, int nb, T* out, size_t ldo,
                                  cudaStream_t st) {
  const size_t n = (size_t)N * nb;
  if (!n) return cudaSuccess;
  const unsigned g = (unsigned)((n + 255) / 256);
  switch (nu2) {
    case 1: kernel_columns_kernel<T, 1><<<g, 256, 0, st>>>(x, N, order, i0, nb, out, ldo); break;
    case 3: kernel_columns_kernel<T, 3><<<g, 256, 0, st>>>(x, N, order, i0, nb, out, ldo); break;
    case 5: kernel_columns_kernel<T, 5><<<g, 256, 0, st>>>(x, N, order, i0, nb, out, ldo); break;
    default: return cudaErrorInvalidValue;
  }
  return note_launch_err();
}
template cudaError_t launch_kernel_columns<float>(int, const V4<float>*, int, const int*, int, int, float*, size_t,
                                                  cudaStream_t);
template cudaError_t launch_kernel_columns<double>(int, const V4<double>*, int, const int*, int, int, double*, size_t,
                                                   cudaStream_t);

int matvec_sym_tiles(int n) { return ((n + SYM_T - 1) / SYM_T + SYM_S - 1) / SYM_S; }   // = partials per row

bool use_sym_k1() {
  static const bool v = !env_is("CAKF_K1_DENSE", '1');
  return v;
}

int matvec_sym_block_points() { return SYM_S * SYM_T; }

long long matvec_sym_units(int n) {
  const long long nt = (n + SYM_T - 1) / SYM_T;
  const long long nb = (nt + SYM_S - 1) / SYM_S;
  return nb * (nb + 1) / 2;
}

// tile-pair activity mask of unit u (bit a*SYM_S+b): pairs whose bounding spheres are within `cut`
__device__ unsigned sym_unit_mask(const float4* __restrict__ sph, int nt, int nb, long long u, float cut) {
  int bi, bj;
  sym_unit_decode(u, nb, bi, bj);
  const int na = min(SYM_S, nt - bi * SYM_S), nbj = min(SYM_S, nt - bj * SYM_S);
  unsigned m = 0;
  for (int a = 0; a < na; ++a)
    for (int b = (bi == bj) ? a : 0; b < nbj; ++b) {
      const float4 A = sph[bi * SYM_S + a], B = sph[bj * SYM_S + b];
      const float ex = A.x - B.x, ey = A.y - B.y, ez = A.z - B.z;
      if (!(sqrtf(ex * ex + ey * ey + ez * ez) - A.w - B.w > cut)) m |= 1u << (a * SYM_S + b);
    }
  return m;
}

// one block: compact list of the units in [u_lo, u_hi) with at least one active tile pair, ordered by
// decreasing number of active pairs (longest first, so the strided assignment of the K1 grid balances);
// the order inside a bucket is arbitrary, which cannot change any result (each unit owns its partial slots)
// Active-unit list of the symmetric K1 (units with at least one tile pair inside the cut), grouped by their
// number of active tile pairs, most first (longest-first dynamic scheduling).  Three grid-wide launches:
// count per group, offsets, scatter (the unit masks are recomputed, no per-unit buffer).  ws = count: [0] the
// list length, [1 + c] group sizes, [1 + kGroups + c] running offsets.  The order inside a group is not
// deterministic and does not need to be: every unit writes its own partial slots.
constexpr int kK1Groups = SYM_S * SYM_S + 1;
__device__ __forceinline__ void k1_unit_range(const long long* urange, long long& u_lo, long long& u_hi) {
  if (urange) {   // this rank's unit range, balanced by active tile pairs (k1_balanced_range_kernel)
    u_lo = urange[0];
    u_hi = urange[1];
  }
}
__global__ void k1_units_count_kernel(const float4* __restrict__ sph, int nt, int nb, long long u_lo, long long u_hi,
                                      float cut, int* __restrict__ ws, const long long* __restrict__ urange) {
  k1_unit_range(urange, u_lo, u_hi);
  __shared__ int bucket[kK1Groups];
  if (threadIdx.x < kK1Groups) bucket[threadIdx.x] = 0;
  __syncthreads();
  for (long long u = u_lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; u < u_hi;
       u += (long long)gridDim.x * blockDim.x) {
    const unsigned m = sym_unit_mask(sph, nt, nb, u, cut);
    if (m) atomicAdd(&bucket[__popc(m)], 1);
  }
  __syncthreads();
  if (threadIdx.x < kK1Groups && bucket[threadIdx.x]) atomicAdd(&ws[1 + threadIdx.x], bucket[threadIdx.x]);
}
__global__ void k1_units_offsets_kernel(int* __restrict__ ws) {   // one thread: 16 active pairs first
  int run = 0;
  for (int c = kK1Groups - 1; c >= 1; --c) {
    ws[1 + kK1Groups + c] = run;
    run += ws[1 + c];
  }
  ws[0] = run;
}
__global__ void k1_units_scatter_kernel(const float4* __restrict__ sph, int nt, int nb, long long u_lo, long long u_hi,
                                        float cut, int* __restrict__ list, unsigned short* __restrict__ mask,
                                        int* __restrict__ ws, const long long* __restrict__ urange) {
  k1_unit_range(urange, u_lo, u_hi);
  for (long long u = u_lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; u < u_hi;
       u += (long long)gridDim.x * blockDim.x) {
    const unsigned m = sym_unit_mask(sph, nt, nb, u, cut);
    if (m) {
      const int pos = atomicAdd(&ws[1 + kK1Groups + __popc(m)], 1);
      list[pos] = (int)u;
      mask[pos] = (unsigned short)m;
    }
  }
}

cudaError_t launch_k1_active_units(const float4* sph, int n, long long u_lo, long long u_hi, float cut, int* list,
                                   unsigned short* mask, int* count, cudaStream_t st, const long long* urange) {
  const int nt = (n + SYM_T - 1) / SYM_T;
  const int nb = (nt + SYM_S - 1) / SYM_S;
  const long long U = (long long)nb * (nb + 1) / 2;   // upper bound of the unit range (urange lies inside)
  const int grid = (int)std::max<long long>(1, std::min<long long>((U + 255) / 256, 8LL * num_sms()));
  cudaError_t e = cudaMemsetAsync(count, 0, (size_t)(1 + 2 * kK1Groups) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  k1_units_count_kernel<<<grid, 256, 0, st>>>(sph, nt, nb, u_lo, u_hi, cut, count, urange);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  k1_units_offsets_kernel<<<1, 1, 0, st>>>(count);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  k1_units_scatter_kernel<<<grid, 256, 0, st>>>(sph, nt, nb, u_lo, u_hi, cut, list, mask, count, urange);
  return note_launch_err();
}

// Per 512-row block B of the symmetric K1: the partner blocks p whose unit (min(B, p), max(B, p)) is active
// (the same predicate as the unit list; every partner without culling, sph == nullptr), ascending, and the
// list positions of the quarter boundaries w * nb / 4 (step.h SlotList).  One block per B.
__global__ void k1_block_partners_kernel(const float4* __restrict__ sph, int nt, int nb, float cut,
                                         int* __restrict__ plist, int* __restrict__ pq) {
  const int B = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ int wsum[32];
  __shared__ int base_s;
  if (tid == 0) base_s = 0;
  __syncthreads();
  int* pl = plist + (size_t)B * nb;
  for (int p0 = 0; p0 < nb; p0 += blockDim.x) {
    const int p = p0 + tid;
    bool act = false;
    if (p < nb) {
      if (!sph) {
        act = true;
      } else {
        const long long bi = min(B, p), bj = max(B, p);
        act = sym_unit_mask(sph, nt, nb, bi * nb - bi * (bi - 1) / 2 + (bj - bi), cut) != 0u;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int off = base_s;
    for (int q = 0; q < w; ++q) off += wsum[q];
    if (act) pl[off + __popc(bal & ((1u << lane) - 1u))] = p;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += wsum[q];
      base_s += t;
    }
    __syncthreads();
  }
  if (tid < 5) {   // first list entry with partner >= tid * nb / 4 (binary search of the ascending list)
    const int P = (int)(((long long)tid * nb) / 4);
    int lo = 0, hi = base_s;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pl[mid] < P) lo = mid + 1;
      else hi = mid;
    }
    pq[B * 5 + tid] = lo;
  }
}

cudaError_t launch_k1_block_partners(const float4* sph, int n, float cut, int* plist, int* pq, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int nt = (n + SYM_T - 1) / SYM_T;
  const int nb = (nt + SYM_S - 1) / SYM_S;
  k1_block_partners_kernel<<<nb, 256, 0, st>>>(sph, nt, nb, cut, plist, pq);
  return note_launch_err();
}
int matvec_sym_blocks(int n) {
  const int nt = (n + SYM_T - 1) / SYM_T;
  return (nt + SYM_S - 1) / SYM_S;
}

// Multi-GPU split of K1 by work (not by unit index): the units in index order carry popc(mask) active tile
// pairs each; rank p takes the contiguous unit range whose prefix work falls in [W p / world, W (p+1) / world).
// One block, each thread a contiguous chunk of units; deterministic (the same range on every rank).
__global__ void k1_balanced_range_kernel(const float4* __restrict__ sph, int nt, int nb, long long U, float cut,
                                         int rank, int world, long long* __restrict__ urange) {
  __shared__ long long csum[1025];
  const int t = threadIdx.x, nthr = blockDim.x;
  const long long per = (U + nthr - 1) / nthr, a = min(U, per * t), b = min(U, a + per);
  long long w = 0;
  for (long long u = a; u < b; ++u) w += __popc(sym_unit_mask(sph, nt, nb, u, cut));
  csum[t + 1] = w;
  if (t == 0) csum[0] = 0;
  __syncthreads();
  if (t == 0)
    for (int x = 1; x <= nthr; ++x) csum[x] += csum[x - 1];
  __syncthreads();
  const long long total = csum[nthr];
  const long long lo_w = total * rank / world, hi_w = total * (rank + 1) / world;
  // boundary unit for a work target: the first unit whose inclusive prefix exceeds the target
  auto boundary = [&](long long target, bool last) -> long long {
    if (last) return U;
    if (target <= 0) return 0;
    // chunk containing the target, then a sequential scan inside it (only one thread calls this)
    int lo = 0, hi = nthr;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (csum[mid + 1] <= target) lo = mid + 1;
      else hi = mid;
    }
    long long acc = csum[lo], u = min(U, per * lo);
    const long long ue = min(U, u + per);
    for (; u < ue; ++u) {
      acc += __popc(sym_unit_mask(sph, nt, nb, u, cut));
      if (acc > target) return u + 1;
    }
    return ue;
  };
  if (t == 0) {
    urange[0] = rank == 0 ? 0 : boundary(lo_w, false);
    urange[1] = boundary(hi_w, rank == world - 1);
  }
}

cudaError_t launch_k1_balanced_range(const float4* sph, int n, float cut, int rank, int world, long long* urange,
                                     cudaStream_t st) {
  const int nt = (n + SYM_T - 1) / SYM_T;
  const int nb = (nt + SYM_S - 1) / SYM_S;
  const long long U = (long long)nb * (nb + 1) / 2;
  k1_balanced_range_kernel<<<1, 1024, 0, st>>>(sph, nt, nb, U, cut, rank, world, urange);
  return note_launch_err();
}

bool use_k1_dyn() {   // CAKF_K1_DYN=0: static strided unit assignment instead of the global work counter
  static const bool v = !env_is("CAKF_K1_DYN", '0');
  return v;
}

bool use_k1_box() {   // CAKF_K1_BOX=0: sphere test only (no bounding boxes) for the sub-tiles
  static const bool v = !env_is("CAKF_K1_BOX", '0');
  return v;
}

bool use_k1_sub() {   // CAKF_K1_SUB=0: exact-zero test per 128-column J tile instead of per 32-column sub-tile
  static const bool v = !env_is("CAKF_K1_SUB", '0');
  return v;
}

template <int NU2, bool SUB>
cudaError_t launch_sym_t(const float4* x, int n, int nt, int nb, float* partial, long long u_begin, long long u_end,
                         cudaStream_t st, unsigned long long* done_pairs, const int* ulist, const int* ucount,
                         const unsigned short* umask, const float4* sph16, const float4* sphJ, float cut,
                         unsigned* sched, const float4* box16, const float4* boxJ) {
  const size_t smem = (size_t)2 * SYM_S * SYM_T * sizeof(float4) + (size_t)SYM_S * SYM_T * sizeof(float) +
                      (size_t)16 * SYM_S * SYM_T * sizeof(float);
  // resident CTAs per SM (one full wave; the units are strided over it), set up once per device (thread-safe)
  static PerDeviceOnce once;
  static int per_sm_dev[PerDeviceOnce::kMaxDev] = {};
  const cudaError_t ce = once_per_device(once, [&] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PerDeviceOnce::kMaxDev) dev = 0;
    cudaError_t r = cudaFuncSetAttribute(matvec_sym_kernel<NU2, SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(matvec_sym_kernel<NU2, SUB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int ps = 0;
    if (r == cudaSuccess &&
        (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, matvec_sym_kernel<NU2, SUB>, 256, smem) != cudaSuccess ||
         ps < 1))
      ps = 1;
    if (const char* e = getenv("CAKF_K1_CTAS")) ps = std::max(1, std::min(ps, atoi(e)));
    per_sm_dev[dev] = ps;
    return r;
  });
  if (ce != cudaSuccess) return ce;
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess || cur < 0 || cur >= PerDeviceOnce::kMaxDev) cur = 0;
  const int per_sm = std::max(1, per_sm_dev[cur]);
  const long long grid = std::min<long long>(u_end - u_begin, (long long)num_sms() * per_sm);
  return launch_pdl(matvec_sym_kernel<NU2, SUB>, dim3((unsigned)grid), dim3(256), smem, st, x, n, nt, nb, u_begin,
                    u_end, partial, done_pairs, ulist, ucount, umask, sph16, sphJ, cut,
                    use_k1_dyn() ? sched : (unsigned*)nullptr, box16, boxJ);
}

cudaError_t launch_matvec_sym(int nu2, const float4* x, int n, float* partial, long long u_begin, long long u_end,
                              cudaStream_t st, unsigned long long* done_pairs, const int* ulist,
                              const int* ucount, const unsigned short* umask, const float4* sph16,
                              const float4* sph128, const float4* sph32, float cut, unsigned* sched,
                              const float4* box16, const float4* box32) {
  if (n <= 0 || u_end <= u_begin) return cudaSuccess;
  if (!use_k1_box()) box16 = box32 = nullptr;
  const int nt = (n + SYM_T - 1) / SYM_T;
  const int nb = (nt + SYM_S - 1) / SYM_S;
  const bool sub = use_k1_sub();
  if (ulist && sub && !sph32) return cudaErrorInvalidValue;
  switch (nu2) {
#define CAKF_SYM_CASE(NU)                                                                                           \
  case NU:                                                                                                         \
    return sub ? launch_sym_t<NU, true>(x, n, nt, nb, partial, u_begin, u_end, st, done_pairs, ulist, ucount,    \
                                        umask, sph16, sph32, cut, sched, box16, box32)                            \
               : launch_sym_t<NU, false>(x, n, nt, nb, partial, u_begin, u_end, st, done_pairs, ulist, ucount,   \
                                         umask, sph16, sph128, cut, sched, nullptr, nullptr);
    CAKF_SYM_CASE(1)
    CAKF_SYM_CASE(3)
    CAKF_SYM_CASE(5)
#undef CAKF_SYM_CASE
    default: return cudaErrorInvalidValue;
  }
}

// dense-equivalent work units counted by done_pairs per 128 x 128 tile pair
int matvec_sym_blocks_per_tile_pair() { return use_k1_sub() ? 32 : 8; }

template <typename T>
cudaError_t launch_sum_partials(int nrows, int nchunks, const T* partial, double alpha, T* y, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  sum_partials_kernel<T><<<(nrows + 255) / 256, 256, 0, st>>>(nrows, nchunks, partial, alpha, y);
  return note_launch_err();
}

template <typename T>
cudaError_t launch_gram_gemm(int nu2, const V4<T>* xr, int M, const V4<T>* xc, int K, const T* B, size_t ldb, int C,
                             T* Y, size_t ldy, double alpha, cudaStream_t st) {
  if (M <= 0 || C <= 0) return cudaSuccess;
  switch (nu2) {
    case 1: return gram_gemm_nu<T, 1>(xr, M, xc, K, B, ldb, C, Y, ldy, alpha, st);
    case 3: return gram_gemm_nu<T, 3>(xr, M, xc, K, B, ldb, C, Y, ldy, alpha, st);
    case 5: return gram_gemm_nu<T, 5>(xr, M, xc, K, B, ldb, C, Y, ldy, alpha, st);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_prescale_coords(int n, int dim, const double* xyz, double scale, V4<T>* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  prescale_kernel<T><<<(n + 255) / 256, 256, 0, st>>>(n, dim, xyz, scale, out);
  return note_launch_err();
}

#define INST(T)                                                                                           \
  template cudaError_t launch_matvec_partial<T>(int, const V4<T>*, int, const V4<T>*, int, int, T*,       \
                                                cudaStream_t, int, int);                                  \
  template cudaError_t launch_sum_partials<T>(int, int, const T*, double, T*, cudaStream_t);              \
  template cudaError_t launch_gram_gemm<T>(int, const V4<T>*, int, const V4<T>*, int, const T*, size_t,   \
                                           int, T*, size_t, double, cudaStream_t);                        \
  template cudaError_t launch_prescale_coords<T>(int, int, const double*, double, V4<T>*, cudaStream_t);
INST(float)
INST(double)
#undef INST

}  // namespace cakf
