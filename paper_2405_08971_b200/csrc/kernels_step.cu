// kernels_step.cu — streaming kernels of one CAKF/CAKS time step (sm_100a).
//
// Inner loop of alg:update_pls per iteration i, with
// G s = Sigma^t_00 K_TT s + Lambda s - (H M^-)((H M^-)^T s):
//   [K1 matvec partials]                       kernels_gram.cu
//   stage A  g' = sig00 * sum(partials) + lam2 .* s ;  u = (HM)^T s ; alpha = s^T r
//   stage B  g  = g' - HM u ;  c = V^T g ;  s^T g
//   stage C  d  = s - V c ;  Gd = g - Z c (Z = G V kept, R18) ; eta = s^T Gd ; accept (R2)
//   stage D  v += (alpha/eta) d ; V_i = d/sqrt(eta) ; Z_i = Gd/sqrt(eta) ;
//            r -= (alpha/eta) Gd ; next action s (policy) packed into the column coords
// Each reduction writes per-block partials (fp64); the last block to arrive sums them
// in block order (deterministic, no float atomics).
#include <algorithm>

#include "internal.h"
#include "step.h"

namespace cakf {

namespace {

// stage kernels: one 128-row tile per block, one row per thread (row-wise ops), 4 warps splitting the
// columns of the column dots; per-block partial rows reduced in two deterministic levels
constexpr int kTile = 128;

// out[j] = sum_{rows of this tile} A[row + j*ld] * v[row]: each lane owns 4 rows; 8 columns per warp pass
// (32 independent loads in flight per lane), lane sums fp32/fp64, cross-lane sums fp64 by a multi-value
// butterfly (9 shuffles for 8 columns)
// the butterfly: 8 -> 4 -> 2 -> 1 values per lane, then a 4-lane sum; lane holds column
// ((l>>4)&1)*4+((l>>3)&1)*2+((l>>2)&1); lanes with (l & 3) == 0 store it
__device__ __forceinline__ void cols8_store(const double (&w8)[8], int j, int ncols, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  double w4[4], w2[2];
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double send = h16 ? w8[c] : w8[c + 4], keep = h16 ? w8[c + 4] : w8[c];
    w4[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double send = h8 ? w4[c] : w4[c + 2], keep = h8 ? w4[c + 2] : w4[c];
    w2[c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double t = (h4 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? w2[0] : w2[1], 4);
  t += __shfl_xor_sync(0xffffffffu, t, 2);
  t += __shfl_xor_sync(0xffffffffu, t, 1);
  const int col = (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
  if ((lane & 3) == 0 && j + col < ncols) out[j + col] = t;
}

// fp32, ld % 4 == 0, 16-byte aligned A and v: each lane owns 4 consecutive rows (one 16-byte load per column),
// 8 columns per warp pass — a quarter of the load instructions of the scalar form (the MIO queue is shared
// with K1's MUFU and shared-memory traffic when this runs beside it on the side stream)
__device__ void tile_cols_dot_v4(const float* __restrict__ A, size_t ld, int ncols, const float* __restrict__ v, int r0,
                                 int r1, double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int row = r0 + 4 * lane;
  const bool in = row < r1;   // r1 - r0 is a multiple of 4
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 x = in ? *reinterpret_cast<const float4*>(v + row) : z4;
  const int rr = in ? row : r0;
  int j = warp * 8;
  for (; j + nw * 8 < ncols; j += 2 * nw * 8) {   // two 8-column groups per pass: 16 loads in flight per lane
    const int j2 = j + nw * 8;
    float4 xv[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      xv[c] = j + c < ncols ? __ldg(reinterpret_cast<const float4*>(A + (size_t)(j + c) * ld + rr)) : z4;
      xv[8 + c] = j2 + c < ncols ? __ldg(reinterpret_cast<const float4*>(A + (size_t)(j2 + c) * ld + rr)) : z4;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double w8[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float acc = fmaf(xv[8 * h + c].x, x.x, 0.f);
        acc = fmaf(xv[8 * h + c].y, x.y, acc);
        acc = fmaf(xv[8 * h + c].z, x.z, acc);
        acc = fmaf(xv[8 * h + c].w, x.w, acc);
        w8[c] = (double)acc;
      }
      cols8_store(w8, h ? j2 : j, ncols, out);
    }
  }
  for (; j < ncols; j += nw * 8) {
    float4 xv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      xv[c] = j + c < ncols ? __ldg(reinterpret_cast<const float4*>(A + (size_t)(j + c) * ld + rr)) : z4;
    double w8[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float acc = fmaf(xv[c].x, x.x, 0.f);
      acc = fmaf(xv[c].y, x.y, acc);
      acc = fmaf(xv[c].z, x.z, acc);
      acc = fmaf(xv[c].w, x.w, acc);
      w8[c] = (double)acc;
    }
    cols8_store(w8, j, ncols, out);
  }
}

template <typename T>
__device__ void tile_cols_dot(const T* __restrict__ A, size_t ld, int ncols, const T* __restrict__ v, int r0, int r1,
                              double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (r1 <= r0) {
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) out[j] = 0.0;
    return;
  }
  if constexpr (sizeof(T) == 4) {
    if ((ld & 3) == 0 && ((((uintptr_t)A) | ((uintptr_t)v)) & 15) == 0 && (r0 & 3) == 0 && blockDim.x <= 128) {
      tile_cols_dot_v4(A, ld, ncols, v, r0, r1, out);
      return;
    }
  }
  T x[4];
  int rr[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = r0 + lane + 32 * q;
    x[q] = row < r1 ? v[row] : T(0);
    rr[q] = row < r1 ? row : r0;
  }
  const int nfull = ncols & ~7;
  for (int j = warp * 8; j < ncols; j += nw * 8) {
    double w8[8];
    if (j < nfull) {   // full group: all 32 loads issued before the first use
      T xv[8][4];
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[c][q] = A[(size_t)(j + c) * ld + rr[q]];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = fma(xv[c][q], x[q], acc);
        w8[c] = (double)acc;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        T acc = T(0);
        if (j + c < ncols) {
          const T* col = A + (size_t)(j + c) * ld;
#pragma unroll
          for (int q = 0; q < 4; ++q) acc = fma(col[rr[q]], x[q], acc);
        }
        w8[c] = (double)acc;
      }
    }
    // 8 -> 4 -> 2 -> 1 values per lane, then a 4-lane sum; lane holds column ((l>>4)&1)*4+((l>>3)&1)*2+((l>>2)&1)
    double w4[4], w2[2];
    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double send = h16 ? w8[c] : w8[c + 4], keep = h16 ? w8[c + 4] : w8[c];
      w4[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double send = h8 ? w4[c] : w4[c + 2], keep = h8 ? w4[c + 2] : w4[c];
      w2[c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double t = (h4 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? w2[0] : w2[1], 4);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    const int col = (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
    if ((lane & 3) == 0 && j + col < ncols) out[j + col] = t;
  }
}

// fp32, ld % 4 == 0, 16-byte aligned V and Z: rows [r0, r1) of V c and Z c in fp64 with 16-byte loads — lane
// owns 4 consecutive rows, warp w the columns j = w (mod 4) in ascending order; the warp partials go to
// sv / sz [4 warps][128 rows] (shared), summed per row in warp order by the caller after a barrier
__device__ void tile_rows_gemv2_v4(const float* __restrict__ V, const float* __restrict__ Z, size_t ld, int ncols,
                                   const double* c, int r0, int r1, double* sv, double* sz) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = r0 + 4 * lane;
  const int rr = row < r1 ? row : r0;
  double av[4] = {0.0, 0.0, 0.0, 0.0}, az[4] = {0.0, 0.0, 0.0, 0.0};
  int j = warp;
  for (; j + 28 < ncols; j += 32) {   // 16 loads in flight per lane
    float4 xv[8], xz[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      xv[q] = __ldg(reinterpret_cast<const float4*>(V + (size_t)(j + 4 * q) * ld + rr));
      xz[q] = __ldg(reinterpret_cast<const float4*>(Z + (size_t)(j + 4 * q) * ld + rr));
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double cj = c[j + 4 * q];
      av[0] = fma((double)xv[q].x, cj, av[0]); av[1] = fma((double)xv[q].y, cj, av[1]);
      av[2] = fma((double)xv[q].z, cj, av[2]); av[3] = fma((double)xv[q].w, cj, av[3]);
      az[0] = fma((double)xz[q].x, cj, az[0]); az[1] = fma((double)xz[q].y, cj, az[1]);
      az[2] = fma((double)xz[q].z, cj, az[2]); az[3] = fma((double)xz[q].w, cj, az[3]);
    }
  }
  for (; j + 12 < ncols; j += 16) {
    float4 xv[4], xz[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      xv[q] = __ldg(reinterpret_cast<const float4*>(V + (size_t)(j + 4 * q) * ld + rr));
      xz[q] = __ldg(reinterpret_cast<const float4*>(Z + (size_t)(j + 4 * q) * ld + rr));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double cj = c[j + 4 * q];
      av[0] = fma((double)xv[q].x, cj, av[0]); av[1] = fma((double)xv[q].y, cj, av[1]);
      av[2] = fma((double)xv[q].z, cj, av[2]); av[3] = fma((double)xv[q].w, cj, av[3]);
      az[0] = fma((double)xz[q].x, cj, az[0]); az[1] = fma((double)xz[q].y, cj, az[1]);
      az[2] = fma((double)xz[q].z, cj, az[2]); az[3] = fma((double)xz[q].w, cj, az[3]);
    }
  }
  for (; j < ncols; j += 4) {
    const float4 xv = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ld + rr));
    const float4 xz = __ldg(reinterpret_cast<const float4*>(Z + (size_t)j * ld + rr));
    const double cj = c[j];
    av[0] = fma((double)xv.x, cj, av[0]); av[1] = fma((double)xv.y, cj, av[1]);
    av[2] = fma((double)xv.z, cj, av[2]); av[3] = fma((double)xv.w, cj, av[3]);
    az[0] = fma((double)xz.x, cj, az[0]); az[1] = fma((double)xz.y, cj, az[1]);
    az[2] = fma((double)xz.z, cj, az[2]); az[3] = fma((double)xz.w, cj, az[3]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    sv[warp * kTile + 4 * lane + e] = av[e];
    sz[warp * kTile + 4 * lane + e] = az[e];
  }
}

// fp32, N % 4 == 0, 16-byte aligned partial: sum over the nch K1 partial slots of rows [r0, r1) with 16-byte
// loads — lane owns 4 consecutive rows, warp w the slots c = w (mod 4) ascending (fp64); the warp partials go
// to sk [4 warps][128 rows] (shared), summed per row in warp order by the caller after a barrier
__device__ void tile_slots_sum_v4(const float* __restrict__ partial, int N, int nch, int r0, int r1, double* sk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = r0 + 4 * lane;
  const int rr = row < r1 ? row : r0;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  int c = warp;
  for (; c + 60 < nch; c += 64) {   // 16 loads in flight per lane
    float4 x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = __ldg(reinterpret_cast<const float4*>(partial + (size_t)(c + 4 * q) * N + rr));
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      a[0] += (double)x[q].x; a[1] += (double)x[q].y; a[2] += (double)x[q].z; a[3] += (double)x[q].w;
    }
  }
  for (; c + 28 < nch; c += 32) {
    float4 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldg(reinterpret_cast<const float4*>(partial + (size_t)(c + 4 * q) * N + rr));
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      a[0] += (double)x[q].x; a[1] += (double)x[q].y; a[2] += (double)x[q].z; a[3] += (double)x[q].w;
    }
  }
  for (; c < nch; c += 4) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(partial + (size_t)c * N + rr));
    a[0] += (double)x.x; a[1] += (double)x.y; a[2] += (double)x.z; a[3] += (double)x.w;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) sk[warp * kTile + 4 * lane + e] = a[e];
}

// the same over the listed slots of the tile's 512-row block: warp w sums the active partners of quarter w
// (slot lists, SlotList) in ascending order — skipped slots hold exact zeros, so the sums equal the full ones
__device__ void tile_slots_list_v4(const float* __restrict__ partial, int N, const SlotList& sl, int r0, int r1,
                                   double* sk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = r0 + 4 * lane;
  const int rr = row < r1 ? row : r0;
  const int B = r0 / 512;
  const int* pl = sl.plist + (size_t)B * sl.nb;
  const int k1 = sl.pq[B * 5 + warp + 1];
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  int k = sl.pq[B * 5 + warp];
  for (; k + 16 <= k1; k += 16) {
    float4 x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = __ldg(reinterpret_cast<const float4*>(partial + (size_t)__ldg(pl + k + q) * N + rr));
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      a[0] += (double)x[q].x; a[1] += (double)x[q].y; a[2] += (double)x[q].z; a[3] += (double)x[q].w;
    }
  }
  for (; k < k1; k += 8) {   // the tail (most lists: ~29 partners over 4 warps) as one predicated batch
    float4 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      x[q] = k + q < k1 ? __ldg(reinterpret_cast<const float4*>(partial + (size_t)__ldg(pl + k + q) * N + rr))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k + q < k1) {
        a[0] += (double)x[q].x; a[1] += (double)x[q].y; a[2] += (double)x[q].z; a[3] += (double)x[q].w;
      }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) sk[warp * kTile + 4 * lane + e] = a[e];
}

// the K1 row sums of this block's rows: the 16-byte-load form when it applies (same in stage A and stage AB,
// so the two stay bit-identical), else per row with 32 loads in flight
template <typename T>
__device__ __forceinline__ double tile_ksum(const T* __restrict__ partial, int N, int nch, int r0, int r1,
                                            const SlotList& sl) {
  const int row = r0 + threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    if ((N & 3) == 0 && ((uintptr_t)partial & 15) == 0 && blockDim.x == kTile) {
      __shared__ double sk[4 * kTile];
      if (sl.plist) tile_slots_list_v4(partial, N, sl, r0, r1, sk);
      else tile_slots_sum_v4(partial, N, nch, r0, r1, sk);
      __syncthreads();
      const int t = threadIdx.x;
      return (sk[t] + sk[kTile + t]) + (sk[2 * kTile + t] + sk[3 * kTile + t]);
    }
  }
  if (row >= r1) return 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int c = 0;
  // 32 loads in flight per thread, then one 16-batch and the scalar tail: each acc[j] sees
  // partial[c + j], partial[c + j + 4], ... in the same order as with 16-batches alone
  for (; c + 32 <= nch; c += 32) {
    T x[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) x[q] = partial[(size_t)(c + q) * N + row];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q & 3] += (double)x[q];
  }
  for (; c + 16 <= nch; c += 16) {
    T x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = partial[(size_t)(c + q) * N + row];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q & 3] += (double)x[q];
  }
  for (; c < nch; ++c) acc[0] += (double)partial[(size_t)c * N + row];
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// sum_j A[row + j*ld] c[j] in fp64 (c in shared memory); 16 independent loads in flight per thread
template <typename T>
__device__ __forceinline__ double row_gemv(const T* __restrict__ A, size_t ld, int ncols, const double* c, int row) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int j = 0;
  for (; j + 32 <= ncols; j += 32) {
    T x[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) x[q] = A[row + (size_t)(j + q) * ld];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q & 3] = fma((double)x[q], c[j + q], acc[q & 3]);
  }
  for (; j + 8 <= ncols; j += 8) {
    T x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = A[row + (size_t)(j + q) * ld];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q & 3] = fma((double)x[q], c[j + q], acc[q & 3]);
  }
  for (; j < ncols; ++j) acc[0] = fma((double)A[row + (size_t)j * ld], c[j], acc[0]);
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// Two-level deterministic reduction of the per-block partial rows part[b*W + j], j < n (no float atomics):
// the last block of each group of gs consecutive blocks sums its group (ascending) into the group row
// part[(nb + g)*W + j]; the last group sums the group rows (ascending) into red.  cnt[0] = top counter,
// cnt[1 + g] = group counters (<= 32 groups), reset by their finalisers.  Returns true in exactly one block,
// with red[0..n) written by that block (visible to it after the return).
__device__ bool reduce_blocks(int n, int W, double* part, unsigned* cnt, double* red) {
  __shared__ unsigned s_flag;
  const int nb = gridDim.x;
  const int gs = max(8, (nb + 31) / 32);
  const int g = blockIdx.x / gs, ng = (nb + gs - 1) / gs;
  const int b0 = g * gs, b1 = min(nb, b0 + gs);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_flag = atomicAdd(cnt + 1 + g, 1u) == (unsigned)(b1 - b0 - 1);
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  double* grow = ng == 1 ? red : part + (size_t)(nb + g) * W;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double sum = 0.0;
    for (int b = b0; b < b1; ++b) sum += __ldcg(part + (size_t)b * W + j);
    grow[j] = sum;
  }
  if (threadIdx.x == 0) cnt[1 + g] = 0u;
  __threadfence();
  __syncthreads();
  if (ng == 1) return true;
  if (threadIdx.x == 0) s_flag = atomicAdd(cnt, 1u) == (unsigned)(ng - 1);
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double sum = 0.0;
    for (int q = 0; q < ng; ++q) sum += __ldcg(part + (size_t)(nb + q) * W + j);
    red[j] = sum;
  }
  if (threadIdx.x == 0) cnt[0] = 0u;
  __syncthreads();
  return true;
}

bool side_slim() {   // CAKF_SIDE_SLIM=0: side-stream HM kernels without the 80-register cap (then they only fit in the K1 tail)
  static const bool v = !env_is("CAKF_SIDE_SLIM", '0');
  return v;
}

// ------------------------------------------------------------------ update prologue
// BLOCKRES region of the observation at user position u: floor(u b / N)  (CAKF_POLICY_BLOCKRES)
__device__ __forceinline__ int block_region(int u, int N, int b) { return (int)(((long long)u * b) / N); }

template <typename T>
__global__ void prep_kernel(int N, const int* __restrict__ idx, const V4<T>* __restrict__ coords, const T* __restrict__ y,
                            const T* __restrict__ mpred, int policy, const int* __restrict__ order, uint64_t seed, int k,
                            const int* __restrict__ sigma, T* __restrict__ r, T* __restrict__ s, T* __restrict__ v,
                            V4<T>* __restrict__ xcs, int nblk_pol, T* __restrict__ rbs) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= N) return;
  const int p = idx[row];
  const T r0 = y[row] - mpred[row];                    // r^(0) = y - H m^-   (P:1515); mpred = H m^- (gathered)
  T s0;
  if (policy == 0) s0 = r0;                            // CG: s_1 = r^(1) = r^(0)  (R1)
  else if (policy == 1) s0 = (order[0] == row) ? T(1) : T(0);
  else if (policy == 3) s0 = block_region(sigma ? sigma[row] : row, N, nblk_pol) == 0 ? r0 : T(0);   // BLOCKRES
  else s0 = (T)philox_normal(seed, (uint32_t)k, 1u, (uint32_t)(sigma ? sigma[row] : row));   // R16: user position
  r[row] = r0;
  s[row] = s0;
  v[row] = T(0);
  if (rbs) rbs[row] = r0;   // BLOCKRES: residual at the block's start
  V4<T> c = coords[p];
  c.w = s0;
  xcs[row] = c;
}

// actions s_{i0} .. s_{i0+nb-1} of a non-adaptive policy at once (block execution): the same
// formulas as prep / stageD — coordinate e_{order[i-1]}, random Philox(seed; j = user position, i, k)
template <typename T>
__global__ void gen_actions_kernel(int N, int i0, int nb, int policy, const int* __restrict__ order, uint64_t seed,
                                   int k, const int* __restrict__ sigma, T* __restrict__ S, size_t ldS,
                                   const T* __restrict__ rbs, int nblk_pol) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * nb) return;
  const int row = (int)(e % N), j = (int)(e / N);
  const int i = i0 + j;
  T v;
  if (policy == 3) v = block_region(sigma ? sigma[row] : row, N, nblk_pol) == (i - 1) % nblk_pol ? rbs[row] : T(0);
  else if (policy == 1) v = (order[i - 1] == row) ? T(1) : T(0);
  else v = (T)philox_normal(seed, (uint32_t)k, (uint32_t)i, (uint32_t)(sigma ? sigma[row] : row));
  S[row + (size_t)j * ldS] = v;
}

// ------------------------------------------------------------------ stage A
template <typename T>
__global__ void __launch_bounds__(kTile)
stageA_kernel(int N, int nch, const T* __restrict__ partial, double sig00, const T* __restrict__ lam2,
              const T* __restrict__ s, const T* __restrict__ r, T* __restrict__ gp, const T* __restrict__ HM, int rin,
              double* __restrict__ part, int W, double* __restrict__ red, unsigned* cnt, SlotList sl) {
  griddep_wait();
  __shared__ double scratch[32 * 3];
  const int r0 = blockIdx.x * kTile, r1 = min(N, r0 + kTile), row = r0 + threadIdx.x;
  double a[3] = {0.0, 0.0, 0.0};  // s.r, s.g', r.r
  const double ksum = tile_ksum(partial, N, nch, r0, r1, sl);
  if (row < r1) {
    const T si = s[row], ri = r[row];
    const T g = (T)(sig00 * ksum) + lam2[row] * si;
    gp[row] = g;
    a[0] = (double)si * (double)ri;
    a[1] = (double)si * (double)g;
    a[2] = (double)ri * (double)ri;
  }
  block_sum<3>(a, scratch);
  double* slot = part + (size_t)blockIdx.x * W;
  if (!HM) {   // u = (HM)^T s runs concurrently on the side stream (hmts_kernel) into red[0, rin)
    if (threadIdx.x == 0) { slot[0] = a[0]; slot[1] = a[1]; slot[2] = a[2]; }
    reduce_blocks(3, W, part, cnt, red + rin);
    return;
  }
  if (threadIdx.x == 0) { slot[rin] = a[0]; slot[rin + 1] = a[1]; slot[rin + 2] = a[2]; }
  tile_cols_dot(HM, (size_t)N, rin, s, r0, r1, slot);            // u = (HM)^T s
  reduce_blocks(rin + 3, W, part, cnt, red);
}

// u = (HM^-)^T s alone (red[0, rin)): the HBM-bound half of stage A, launched on a side stream so it
// overlaps the MUFU-bound K1 of the same iteration (both only need s)
// MINB = 6 caps the kernel at 80 registers so one of its CTAs fits beside three resident K1 CTAs
// (3 x 256 x 72 = 55296 of 65536 registers): the HBM-bound HM passes then run concurrently with the
// MUFU-bound K1 instead of only in its tail
template <typename T, int MINB>
__global__ void __launch_bounds__(kTile, MINB)
hmts_kernel(int N, const T* __restrict__ HM, int rin, const T* __restrict__ s, double* __restrict__ part, int W,
            double* __restrict__ red, unsigned* cnt) {
  const int r0 = blockIdx.x * kTile, r1 = min(N, r0 + kTile);
  tile_cols_dot(HM, (size_t)N, rin, s, r0, r1, part + (size_t)blockIdx.x * W);
  reduce_blocks(rin, W, part, cnt, red);
}

// w = HM u (fp64 rows) on the side stream right after hmts, so stage B's second HM pass also overlaps K1
template <typename T, int MINB>
__global__ void __launch_bounds__(kTile, MINB)
hmu_kernel(int N, const T* __restrict__ HM, int rin, const double* __restrict__ ured, double* __restrict__ w) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* u = reinterpret_cast<double*>(sm_raw);
  for (int j = threadIdx.x; j < rin; j += blockDim.x) u[j] = ured[j];
  __syncthreads();
  const int row = blockIdx.x * kTile + threadIdx.x;
  if (row < N) w[row] = row_gemv(HM, (size_t)N, rin, u, row);
}

// hmu with 4 consecutive rows per thread (one 16-byte load per column; fp32, N % 4 == 0, 16-byte aligned HM):
// 4 rows per thread; every row's fp64 accumulation is row_gemv's (columns ascending, column j into
// acc[j & 3] below the last multiple of 8, the tail into acc[0]), so w is the same bits
template <int MINB>
__global__ void __launch_bounds__(kTile, MINB)
hmu4_kernel(int N, const float* __restrict__ HM, int rin, const double* __restrict__ ured, double* __restrict__ w) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* u = reinterpret_cast<double*>(sm_raw);
  for (int j = threadIdx.x; j < rin; j += blockDim.x) u[j] = ured[j];
  __syncthreads();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (row >= N) return;
  double acc[4][4] = {};
  const int n8 = rin & ~7;
  int j = 0;
  for (; j < n8; j += 8) {
    float4 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldg(reinterpret_cast<const float4*>(HM + row + (size_t)(j + q) * N));
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double c = u[j + q];
      acc[0][q & 3] = fma((double)x[q].x, c, acc[0][q & 3]);
      acc[1][q & 3] = fma((double)x[q].y, c, acc[1][q & 3]);
      acc[2][q & 3] = fma((double)x[q].z, c, acc[2][q & 3]);
      acc[3][q & 3] = fma((double)x[q].w, c, acc[3][q & 3]);
    }
  }
  for (; j < rin; ++j) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(HM + row + (size_t)j * N));
    const double c = u[j];
    acc[0][0] = fma((double)x.x, c, acc[0][0]);
    acc[1][0] = fma((double)x.y, c, acc[1][0]);
    acc[2][0] = fma((double)x.z, c, acc[2][0]);
    acc[3][0] = fma((double)x.w, c, acc[3][0]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) w[row + e] = (acc[e][0] + acc[e][1]) + (acc[e][2] + acc[e][3]);
}

// ------------------------------------------------------------------ stage B
// wpre (nullable): HM u already formed by hmu_kernel (same fp64 row sums), else formed here
template <typename T>
__global__ void __launch_bounds__(kTile)
stageB_kernel(int N, const T* __restrict__ HM, int rin, const double* __restrict__ ured, const T* __restrict__ gp,
              const T* __restrict__ s, T* __restrict__ g, const T* __restrict__ V, int nV, double* __restrict__ part,
              int W, double* __restrict__ red, unsigned* cnt, const double* __restrict__ wpre) {
  griddep_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* u = reinterpret_cast<double*>(sm_raw);
  __shared__ double scratch[32];
  __shared__ T gs_[kTile];
  if (!wpre)
    for (int j = threadIdx.x; j < rin; j += blockDim.x) u[j] = ured[j];
  __syncthreads();
  const int r0 = blockIdx.x * kTile, r1 = min(N, r0 + kTile), row = r0 + threadIdx.x;
  double a[1] = {0.0};
  if (row < r1) {
    const double acc = wpre ? wpre[row] : row_gemv(HM, (size_t)N, rin, u, row);   // fp64: rin ~1e3
    const T gi = (T)((double)gp[row] - acc);                      // G s
    g[row] = gi;
    a[0] = (double)s[row] * (double)gi;
  }
  block_sum<1>(a, scratch);
  double* slot = part + (size_t)blockIdx.x * W;
  if (threadIdx.x == 0) slot[nV] = a[0];
  tile_cols_dot(V, (size_t)N, nV, g, r0, r1, slot);               // c = V^T G s (g rows of this tile: own writes)
  reduce_blocks(nV + 1, W, part, cnt, red);
}

// ------------------------------------------------------------------ stage A + B in one pass
// When u = (HM)^T s and w = HM u come from the side stream (hmw) — or r_in = 0 — stage A's g' feeds only
// stage B, so one kernel forms g' and g = g' - w per row (the same arithmetic as the two kernels, so the
// same bits), c = V^T g, s^T g and stage A's three dots in one block-wide + grid-wide reduction: one launch
// and one reduction fewer per inner iteration, and no g' round trip through HBM.  red: [c | s^T g | s^T r,
// s^T g', r^T r]; the finalising block copies the last three to ared_tail (= redA + r_in, stage C's ared).
template <typename T>
__global__ void __launch_bounds__(kTile)
stageAB_kernel(int N, int nch, const T* __restrict__ partial, double sig00, const T* __restrict__ lam2,
               const T* __restrict__ s, const T* __restrict__ r, const double* __restrict__ wpre, T* __restrict__ g,
               const T* __restrict__ V, int nV, double* __restrict__ part, int W, double* __restrict__ red,
               double* __restrict__ ared_tail, unsigned* cnt, SlotList sl) {
  griddep_wait();
  __shared__ double scratch[32 * 4];
  const int r0 = blockIdx.x * kTile, r1 = min(N, r0 + kTile), row = r0 + threadIdx.x;
  double a[4] = {0.0, 0.0, 0.0, 0.0};   // s.g, s.r, s.g', r.r
  const double ksum = tile_ksum(partial, N, nch, r0, r1, sl);
  if (row < r1) {
    const T si = s[row], ri = r[row];
    const T gpv = (T)(sig00 * ksum) + lam2[row] * si;                // g'  (stage A)
    const T gi = wpre ? (T)((double)gpv - wpre[row]) : gpv;          // G s (stage B)
    g[row] = gi;
    a[0] = (double)si * (double)gi;
    a[1] = (double)si * (double)ri;
    a[2] = (double)si * (double)gpv;
    a[3] = (double)ri * (double)ri;
  }
  block_sum<4>(a, scratch);
  double* slot = part + (size_t)blockIdx.x * W;
  if (threadIdx.x == 0) {
    slot[nV] = a[0];
    slot[nV + 1] = a[1];
    slot[nV + 2] = a[2];
    slot[nV + 3] = a[3];
  }
  tile_cols_dot(V, (size_t)N, nV, g, r0, r1, slot);               // c = V^T G s (g rows of this tile: own writes)
  if (reduce_blocks(nV + 4, W, part, cnt, red) && threadIdx.x < 3) ared_tail[threadIdx.x] = red[nV + 1 + threadIdx.x];
}

// ------------------------------------------------------------------ stage C
// d = sin - V c ; Gd = gin - Z c  (line 11; Z = G V so G d needs no second matvec, R18).
// pass == 1 (first pass of CGS2, R19): also c2 = V^T Gd -> red[0..nV).
// pass == 0 (final pass): eta = s^T Gd (line 12) and the accept / reject decision (R2).
// sin/gin may alias d/Gd (second pass runs in place), hence no __restrict__ on them.
template <typename T>
__global__ void __launch_bounds__(kTile)
stageC_kernel(int N, const T* __restrict__ V, const T* __restrict__ Z, int nV, const double* __restrict__ cred,
              const T* sin, const T* gin, T* d, T* Gd, const T* __restrict__ s_eta, const double* __restrict__ ared,
              int rin, const double* __restrict__ sgs, double* __restrict__ part, int W, double* __restrict__ red,
              unsigned* cnt, IterCtl* ctl, double eps, int iter, int pass) {
  griddep_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* c = reinterpret_cast<double*>(sm_raw);
  __shared__ double scratch[32];
  for (int j = threadIdx.x; j < nV; j += blockDim.x) c[j] = cred[j];
  __syncthreads();
  const int r0 = blockIdx.x * kTile, r1 = min(N, r0 + kTile), row = r0 + threadIdx.x;
  double a[1] = {0.0};
  double vc = 0.0, zc = 0.0;   // (V c)[row], (Z c)[row]
  bool v4 = false;
  if constexpr (sizeof(T) == 4) {
    if ((N & 3) == 0 && ((((uintptr_t)V) | ((uintptr_t)Z)) & 15) == 0 && blockDim.x == kTile) {
      __shared__ double sv[4 * kTile], sz[4 * kTile];
      tile_rows_gemv2_v4(V, Z, (size_t)N, nV, c, r0, r1, sv, sz);
      __syncthreads();
      const int t = threadIdx.x;
      vc = (sv[t] + sv[kTile + t]) + (sv[2 * kTile + t] + sv[3 * kTile + t]);
      zc = (sz[t] + sz[kTile + t]) + (sz[2 * kTile + t] + sz[3 * kTile + t]);
      v4 = true;
    }
  }
  if (row < r1) {
    if (!v4) {
      vc = row_gemv(V, (size_t)N, nV, c, row);
      zc = row_gemv(Z, (size_t)N, nV, c, row);
    }
    const double dv = (double)sin[row] - vc;   // d = (I - V V^T G) s  (line 11)
    const double gd = (double)gin[row] - zc;   // G d = G s - Z c
    d[row] = (T)dv;
    Gd[row] = (T)gd;
    a[0] = (double)s_eta[row] * gd;                               // eta = s^T G d        (line 12)
  }
  if (pass == 1) {
    __syncthreads();                                              // Gd of this tile visible to the block
    tile_cols_dot(V, (size_t)N, nV, Gd, r0, r1, part + (size_t)blockIdx.x * W);   // c2 = V^T G d
    reduce_blocks(nV, W, part, cnt, red);
    return;
  }
  block_sum<1>(a, scratch);
  if (threadIdx.x == 0) part[(size_t)blockIdx.x * W] = a[0];
  if (reduce_blocks(1, W, part, cnt, &ctl->eta)) {
    if (threadIdx.x == 0) {
      const double eta = ctl->eta;
      const double alpha = ared[rin];
      const double sGs = *sgs;
      const double floor_ = 64.0 * eps * fabs(sGs);
      const bool accept = eta > floor_ && isfinite(eta);
      ctl->alpha = alpha;
      ctl->gamma = accept ? alpha / eta : 0.0;
      ctl->inv_sqrt_eta = accept ? 1.0 / sqrt(eta) : 0.0;
      if (iter == 1) ctl->res0_sq = ared[rin + 2];
      if (accept) {
        ctl->n_acc += 1;
        ctl->eta_min = fmin(ctl->eta_min, eta);
      } else {
        ctl->rejected += 1;
      }
      if (!isfinite(eta) || !isfinite(alpha)) ctl->nonfinite = 1;
    }
  }
}

// ------------------------------------------------------------------ stage D
template <typename T>
__global__ void stageD_kernel(int N, int iter, int niter, const IterCtl* __restrict__ ctl, const T* __restrict__ d,
                              const T* __restrict__ Gd, T* __restrict__ XV, T* __restrict__ Z, T* __restrict__ r,
                              T* __restrict__ s, V4<T>* __restrict__ xcs, int policy, const int* __restrict__ order,
                              uint64_t seed, int k, const int* __restrict__ sigma, int nblk_pol, T* __restrict__ rbs) {
  griddep_wait();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= N) return;
  const T gamma = (T)ctl->gamma, isq = (T)ctl->inv_sqrt_eta;
  const T di = d[row], gdi = Gd[row];
  XV[row] = fma(gamma, di, XV[row]);                              // v += alpha/eta d   (line 13)
  XV[row + (size_t)iter * N] = di * isq;                          // V_i = d / sqrt(eta) (line 14)
  Z[row + (size_t)(iter - 1) * N] = gdi * isq;
  const T rn = fma(-gamma, gdi, r[row]);                          // r^(i+1) = r^(i) - alpha/eta G d
  r[row] = rn;
  if (iter < niter) {
    T sn;
    if (policy == 0) sn = rn;
    else if (policy == 1) sn = (order[iter] == row) ? T(1) : T(0);
    else if (policy == 3) {   // BLOCKRES: iteration iter+1 is in-block position iter % b; a new block restarts
      const int jb = iter % nblk_pol;   // from the current residual
      T base;
      if (jb == 0) {
        rbs[row] = rn;
        base = rn;
      } else {
        base = rbs[row];
      }
      sn = block_region(sigma ? sigma[row] : row, N, nblk_pol) == jb ? base : T(0);
    }
    else sn = (T)philox_normal(seed, (uint32_t)k, (uint32_t)(iter + 1), (uint32_t)(sigma ? sigma[row] : row));
    s[row] = sn;
    xcs[row].w = sn;
  }
}

template <typename T>
__global__ void __launch_bounds__(kTile)
dot_final_kernel(int N, const T* __restrict__ a_, const T* __restrict__ b_, double* part, double* out, unsigned* cnt) {
  __shared__ double scratch[32];
  const int row = blockIdx.x * kTile + threadIdx.x;
  double a[1] = {row < N ? (double)a_[row] * (double)b_[row] : 0.0};
  block_sum<1>(a, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = a[0];
  reduce_blocks(1, 1, part, cnt, out);
}

// ------------------------------------------------------------------ gathers / mixing
// HM[row + j*N] = M[idx[row] - lo + j*ldm]   (rows of block 0 picked by H) for the points this rank owns
// (lo <= idx < lo + nl, M holds the local rows), zero for the others (summed across the ranks)
template <typename T>
__global__ void gather_rows_kernel(int N, int C, const int* __restrict__ idx, const T* __restrict__ M, size_t ldm,
                                   T* __restrict__ out, size_t ldo, int lo, int nl) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;   // grid (rows, columns)
  if (row >= N) return;
  const int p = idx[row] - lo;
  out[row + (size_t)j * ldo] = (p >= 0 && p < nl) ? M[p + (size_t)j * ldm] : T(0);
}

// out = (A (x) I) in  or (A^T (x) I) in, column by column (Lemma B.1 structure)
template <typename T>
__global__ void mix_kernel(int NX, int Dp, int C, Mat3 A, int transpose, const T* __restrict__ in, size_t ldi,
                           T* __restrict__ out, size_t ldo) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;   // grid (points, columns)
  if (q >= NX) return;
  double x[3] = {0.0, 0.0, 0.0};
  for (int t = 0; t < Dp; ++t) x[t] = (double)in[q + (size_t)t * NX + (size_t)j * ldi];
  for (int dd = 0; dd < Dp; ++dd) {
    double acc = 0.0;
    for (int t = 0; t < Dp; ++t) acc += (transpose ? A.a[t][dd] : A.a[dd][t]) * x[t];
    out[q + (size_t)dd * NX + (size_t)j * ldo] = (T)acc;
  }
}

// fp32, 16-byte aligned columns: 4 points per thread (float4 loads / stores, Dp loads in flight of 16 B
// instead of 4 B), the same per-element fp64 arithmetic as mix_kernel
// float4 version: each thread owns kMixQ point quads (strided by the block, so every load instruction is
// coalesced) of one column; all DP x kMixQ loads are issued before the first use (HBM-bound: bytes in flight)
constexpr int kMixQ = 4;
template <int DP>
__global__ void __launch_bounds__(256) mix4_kernel(int NX4, int C, Mat3 A, int transpose, const float4* __restrict__ in,
                                                   size_t ldi4, float4* __restrict__ out, size_t ldo4) {
  const int j = blockIdx.y;   // grid (point quads / (256 kMixQ), columns)
  const int q0 = blockIdx.x * blockDim.x * kMixQ + threadIdx.x;
  double c[DP][DP];
#pragma unroll
  for (int dd = 0; dd < DP; ++dd)
#pragma unroll
    for (int t = 0; t < DP; ++t) c[dd][t] = transpose ? A.a[t][dd] : A.a[dd][t];
  float4 x[kMixQ][DP];
#pragma unroll
  for (int u = 0; u < kMixQ; ++u) {
    const int q = q0 + u * blockDim.x;
#pragma unroll
    for (int t = 0; t < DP; ++t)
      x[u][t] = q < NX4 ? in[q + (size_t)t * NX4 + (size_t)j * ldi4] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < kMixQ; ++u) {
    const int q = q0 + u * blockDim.x;
    if (q >= NX4) continue;
#pragma unroll
    for (int dd = 0; dd < DP; ++dd) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int t = 0; t < DP; ++t) {
        a0 += c[dd][t] * (double)x[u][t].x;
        a1 += c[dd][t] * (double)x[u][t].y;
        a2 += c[dd][t] * (double)x[u][t].z;
        a3 += c[dd][t] * (double)x[u][t].w;
      }
      out[q + (size_t)dd * NX4 + (size_t)j * ldo4] = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
    }
  }
}

// post-loop: out[p, j] = Sigma^t_{d,0} Y[q, j] - tmp[p, j]  (p = d*NX + q)
template <typename T>
__global__ void post_combine_kernel(int NX, int Dp, int C, Mat3 S, const T* __restrict__ Y, const T* __restrict__ tmp,
                                    const T* __restrict__ mpred, T* __restrict__ m, T* __restrict__ Mk, int rin) {
  const size_t D = (size_t)NX * Dp;
  const int q = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, dd = blockIdx.z;   // grid (points, cols, D')
  if (q >= NX) return;
  const size_t p = (size_t)dd * NX + q;
  T val = (T)S.a[dd][0] * Y[q + (size_t)j * NX];
  if (tmp) val -= tmp[p + (size_t)j * D];
  if (j == 0) m[p] = mpred[p] + val;                              // m = m^- + P^- w
  else Mk[p + (size_t)(rin + j - 1) * D] = val;                   // B = P^- W
}

// var[p] = base[p] - sum_c M[p + c*ld]^2 ; base = Sigma^t_{dd} when base_vec == nullptr
template <typename T>
__global__ void rowvar_kernel(int NX, int Dp, Mat3 S, const T* __restrict__ base_vec, const T* __restrict__ M,
                              size_t ld, int cols, T* __restrict__ var) {
  const size_t D = (size_t)NX * Dp;
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= D) return;
  double acc = 0.0;
  for (int c = 0; c < cols; ++c) {
    const double x = (double)M[p + (size_t)c * ld];
    acc += x * x;
  }
  const double base = base_vec ? (double)base_vec[p] : S.a[p / NX][p / NX];
  var[p] = (T)(base - acc);
}

// ------------------------------------------------------------------ Gram (fp64 accumulation)
// part[z][a + b*c] = sum_{rows in split z} M[row, a] M[row, b], 32x32 tiles, upper tiles only
template <typename T>
__global__ void __launch_bounds__(256)
gram_partial_kernel(size_t D, int c, const T* __restrict__ M, size_t ld, size_t rows_per_split, double* __restrict__ part) {
  const int ti = blockIdx.x, tj = blockIdx.y;
  if (tj < ti) return;
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const size_t row_lo = (size_t)blockIdx.z * rows_per_split;
  const size_t row_hi = min(D, row_lo + rows_per_split);
  const int a0 = ti * 32, b0 = tj * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // ty in [0, 8)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (size_t r = row_lo; r < row_hi; r += 32) {
    for (int q = ty; q < 32; q += 8) {
      const size_t row = r + tx;
      const int ca = a0 + q, cb = b0 + q;
      As[q][tx] = (row < row_hi && ca < c) ? (double)M[row + (size_t)ca * ld] : 0.0;
      Bs[q][tx] = (row < row_hi && cb < c) ? (double)M[row + (size_t)cb * ld] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double b = Bs[tx][rr];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][rr], b, acc[q]);
    }
    __syncthreads();
  }
  double* out = part + (size_t)blockIdx.z * c * c;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = a0 + ty + 8 * q, b = b0 + tx;
    if (a < c && b < c) out[a + (size_t)b * c] = acc[q];
  }
}

__global__ void gram_reduce_kernel(int c, int nsplit, const double* __restrict__ part, double* __restrict__ G) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)c * c) return;
  const int a = (int)(e % c), b = (int)(e / c);
  const int lo = min(a, b), hi = max(a, b);
  const int tlo = lo / 32, thi = hi / 32;
  // element (lo, hi) lives in tile (tlo, thi) which is an upper tile (tlo <= thi)
  double s = 0.0;
  if (tlo <= thi) {
    for (int z = 0; z < nsplit; ++z) s += part[(size_t)z * c * c + lo + (size_t)hi * c];
  }
  G[e] = s;
}

// Qr[a + j*c] = evec[a + (c-1-j)*c]  (descending eigenvalue order), kept[j] = w[c-1-j]
template <typename T>
__global__ void take_top_kernel(int c, int r, const double* __restrict__ evec, const double* __restrict__ w,
                                T* __restrict__ Qr, double* __restrict__ kept, double* dropped_mass) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (size_t)c * r) {
    const int a = (int)(e % c), j = (int)(e / c);
    Qr[a + (size_t)j * c] = (T)evec[a + (size_t)(c - 1 - j) * c];
  }
  if (e < (size_t)r && kept) kept[e] = w[c - 1 - e];
  if (e == 0 && dropped_mass) {
    double s = 0.0;
    for (int i = 0; i < c - r; ++i) s += w[i];
    *dropped_mass = s;
  }
}

// ------------------------------------------------------------------ smoother helpers
// Sigma_k x: y[d*NX + q, j] = sum_e S[d][e] Y[q, j*Dp + e]
// smoother state: ms = m + y[:,0]; var = var_f - rowsumsq(y[:, 1:C])
template <typename T>
__global__ void smooth_out_kernel(size_t D, int C, const T* __restrict__ m, const T* __restrict__ varf,
                                  const T* __restrict__ y, T* __restrict__ ms, T* __restrict__ vs) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= D) return;
  ms[p] = m[p] + y[p];
  double acc = 0.0;
  for (int j = 1; j < C; ++j) {
    const double x = (double)y[p + (size_t)j * D];
    acc += x * x;
  }
  vs[p] = (T)((double)varf[p] - acc);
}

// fp32, D % 4 == 0, 16-byte aligned: 4 rows per thread (float4), 8 column loads in flight, the same
// per-row fp64 accumulation order (j = 1, 2, ...) as smooth_out_kernel
__global__ void smooth_out4_kernel(size_t D4, int C, const float4* __restrict__ m, const float4* __restrict__ varf,
                                   const float4* __restrict__ y, float4* __restrict__ ms, float4* __restrict__ vs) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= D4) return;
  const float4 m4 = m[p], y0 = y[p];
  ms[p] = make_float4(m4.x + y0.x, m4.y + y0.y, m4.z + y0.z, m4.w + y0.w);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 1;
  for (; j + 8 <= C; j += 8) {
    float4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = y[p + (size_t)(j + u) * D4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 += (double)x[u].x * (double)x[u].x;
      a1 += (double)x[u].y * (double)x[u].y;
      a2 += (double)x[u].z * (double)x[u].z;
      a3 += (double)x[u].w * (double)x[u].w;
    }
  }
  for (; j < C; ++j) {
    const float4 x = y[p + (size_t)j * D4];
    a0 += (double)x.x * (double)x.x;
    a1 += (double)x.y * (double)x.y;
    a2 += (double)x.z * (double)x.z;
    a3 += (double)x.w * (double)x.w;
  }
  const float4 v = varf[p];
  vs[p] = make_float4((float)((double)v.x - a0), (float)((double)v.y - a1), (float)((double)v.z - a2),
                      (float)((double)v.w - a3));
}

// W^s_full = [H^T V, x[:,1:] - H^T R[:,1:]],  w^s = H^T v + x[:,0] - H^T R[:,0]
// step 1: dense part (copy x columns, zero the H^T V block)
template <typename T>
__global__ void ws_dense_kernel(size_t D, int n, int q, const T* __restrict__ X, T* __restrict__ Wf, T* __restrict__ ws) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;   // grid (rows, n + q + 1 columns)
  const int j = blockIdx.y;
  if (p >= D) return;
  if (j == 0) ws[p] = X[p];
  else if (j <= n) Wf[p + (size_t)(j - 1) * D] = T(0);
  else Wf[p + (size_t)(j - 1) * D] = X[p + (size_t)(j - n) * D];
}
// float4 forms of ws_dense / kcar_build (D and N_X multiples of 4, 16-byte aligned buffers): the same values,
// one 16-byte access per thread (these are pure streaming passes over D x (1 + n + q))
__global__ void ws_dense4_kernel(size_t D4, int n, const float4* __restrict__ X, float4* __restrict__ Wf,
                                 float4* __restrict__ ws) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= D4) return;
  if (j == 0) ws[p] = X[p];
  else if (j <= n) Wf[p + (size_t)(j - 1) * D4] = make_float4(0.f, 0.f, 0.f, 0.f);
  else Wf[p + (size_t)(j - 1) * D4] = X[p + (size_t)(j - n) * D4];
}
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) {
  return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__global__ void kcar_build4_kernel(size_t NX4, size_t D4, int n, int q, const float4* __restrict__ KV,
                                   const float4* __restrict__ Z, const float4* __restrict__ Kx,
                                   float4* __restrict__ KWf, float4* __restrict__ Kws) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= D4) return;
  const bool b0 = p < NX4;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j == 0) {
    float4 v = Kx ? Kx[p] : zero;
    if (b0 && n) v = f4add(v, Z ? f4sub(KV[p], Z[p]) : KV[p]);
    Kws[p] = v;
  } else if (j <= n) {
    KWf[p + (size_t)(j - 1) * D4] = b0 ? KV[p + (size_t)j * NX4] : zero;
  } else {
    const int c = j - n;
    float4 v = Kx[p + (size_t)c * D4];
    if (b0 && n && Z) v = f4sub(v, Z[p + (size_t)c * NX4]);
    KWf[p + (size_t)(j - 1) * D4] = v;
  }
}

// kernel-applied carriers: (I (x) K) of ws_dense + ws_scatter, from K(X,T)[v V] and K(X,T) V t (block 0 only,
// H = [E_train, 0]); grid (rows of D, 1 + n + q columns)
template <typename T>
__global__ void kcar_build_kernel(size_t NX, size_t D, int n, int q, const T* __restrict__ KV, const T* __restrict__ Z,
                                  const T* __restrict__ Kx, T* __restrict__ KWf, T* __restrict__ Kws) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= D) return;
  const bool b0 = p < NX;
  if (j == 0) {
    T v = Kx ? Kx[p] : T(0);
    if (b0 && n) v += Z ? KV[p] - Z[p] : KV[p];   // n = 0: no observation-space term (as ws_build)
    Kws[p] = v;
  } else if (j <= n) {
    KWf[p + (size_t)(j - 1) * D] = b0 ? KV[p + (size_t)j * NX] : T(0);
  } else {
    const int c = j - n;
    T v = Kx[p + (size_t)c * D];
    if (b0 && n && Z) v -= Z[p + (size_t)c * NX];
    KWf[p + (size_t)(j - 1) * D] = v;
  }
}

// step 2: scatter the observation-space terms into the train rows of block 0
template <typename T>
__global__ void ws_scatter_kernel(int N, size_t D, int n, int q, const int* __restrict__ idx, const T* __restrict__ XV,
                                  const T* __restrict__ R, T* __restrict__ Wf, T* __restrict__ ws, int lo, int nl) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)N * (n + q + 1);
  if (e >= total) return;
  const int row = (int)(e % N), j = (int)(e / N);
  const int pl = idx[row] - lo;   // local row of the observed point (rows owned by this rank only)
  if (pl < 0 || pl >= nl) return;
  const size_t p = (size_t)pl;
  if (j == 0) ws[p] += XV[row] - R[row];                          // H^T v - H^T V t_0
  else if (j <= n) Wf[p + (size_t)(j - 1) * D] = XV[row + (size_t)j * N];   // H^T V
  else Wf[p + (size_t)(j - 1) * D] -= R[row + (size_t)(j - n) * N];         // - H^T V t_{1:}
}

// Y[row + c*ldy] = G[p][(row - p*slice) + c*slice] with p = row / slice (all-gathered K2 row slices)
template <typename T>
__global__ void assemble_slices_kernel(int M, int C, int slice, const T* __restrict__ G, T* __restrict__ Y, size_t ldy) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)M * C) return;
  const int row = (int)(e % M), c = (int)(e / M);
  const int p = row / slice;
  Y[row + (size_t)c * ldy] = G[(size_t)p * slice * C + (row - (size_t)p * slice) + (size_t)c * slice];
}

// ---- posterior sampler (alg:cakf-caks-sampler), S samples as columns
// out[d*NX + map[i] + s*ldo] = in[d*NX + i + s*ldi]
template <typename T>
__global__ void permute_cols_kernel(int NX, int Dp, int S, const int* __restrict__ map, const T* __restrict__ in,
                                    size_t ldi, T* __restrict__ out, size_t ldo) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t D = (size_t)NX * Dp;
  if (e >= D * S) return;
  const size_t s = e / D, r = e % D;
  const int d = (int)(r / NX), i = (int)(r % NX);
  out[(size_t)d * NX + map[i] + s * ldo] = in[r + s * ldi];
}
// res[j, s] = y[j] - x^-[idx[j], s] - eps_user[sigma[j], s]   (R25: full-space noise draws)
template <typename T>
__global__ void sample_residual_kernel(int N, int S, const T* __restrict__ y, const int* __restrict__ idx,
                                       const int* __restrict__ sigma, const T* __restrict__ xp, size_t D,
                                       const T* __restrict__ eps, T* __restrict__ res) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * S) return;
  const int j = (int)(e % N), s = (int)(e / N);
  res[e] = y[j] - xp[idx[j] + (size_t)s * D] - eps[sigma[j] + (size_t)s * N];
}
// x[p, s] = x^-[p, s] + Sigma^t_{d,0} Y[q, s] - tmp[p, s]   (p = d*NX + q): x^- + P^- w for w in block 0
template <typename T>
__global__ void sample_combine_kernel(int NX, int Dp, int S, Mat3 Sg, const T* __restrict__ Y,
                                      const T* __restrict__ tmp, int has_tmp, const T* __restrict__ xp,
                                      T* __restrict__ x) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t D = (size_t)NX * Dp;
  if (e >= D * S) return;
  const size_t s = e / D, p = e % D;
  const int d = (int)(p / NX), q = (int)(p % NX);
  T v = xp[e] + (T)Sg.a[d][0] * Y[q + s * NX];
  if (has_tmp) v -= tmp[e];
  x[e] = v;
}
// w[idx[j], s] += sign * R[j, s]  (H^T R into the block-0 rows)
template <typename T>
__global__ void scatter_rows_kernel(int N, int S, const int* __restrict__ idx, const T* __restrict__ R, T sign,
                                    T* __restrict__ w, size_t D) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * S) return;
  const int j = (int)(e % N), s = (int)(e / N);
  w[idx[j] + (size_t)s * D] += sign * R[e];
}
template <typename T>
__global__ void gather_coords_kernel(int N, const int* __restrict__ idx, const V4<T>* __restrict__ coords,
                                     V4<T>* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  V4<T> c = coords[idx[j]];
  c.w = T(0);
  out[j] = c;
}

// ---- observation sort: internal index order (spatially compact tiles), fully on device; every kernel
// returns at once when the (nullable) device flag *run is 0 (the observation cache hit, decided on device)
__device__ __forceinline__ bool obs_skip(const int* run) { return run != nullptr && *run == 0; }
__global__ void obs_mark_kernel(int N, const int* __restrict__ run, const int64_t* __restrict__ obs,
                                const int* __restrict__ invperm, int* __restrict__ posof) {
  if (obs_skip(run)) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) posof[invperm[obs[j]]] = j;
}
__global__ void obs_count_kernel(int NX, const int* __restrict__ run, const int* __restrict__ posof,
                                 int* __restrict__ counts) {
  if (obs_skip(run)) return;
  __shared__ int wsum[32];
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const unsigned b = __ballot_sync(0xffffffffu, i < NX && posof[i] >= 0);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 32; ++w) t += wsum[w];
    counts[blockIdx.x] = t;
  }
}
__global__ void obs_scan_kernel(int nb, const int* __restrict__ run, int* __restrict__ counts) {
  // one warp: exclusive scan of the per-block counts, 32 at a time
  if (obs_skip(run) || blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31;
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const int c = b < nb ? counts[b] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (b < nb) counts[b] = carry + inc - c;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}
__global__ void obs_scatter_kernel(int NX, const int* __restrict__ run, const int* __restrict__ posof,
                                   const int* __restrict__ offsets, int* __restrict__ idx_out, int* __restrict__ sigma,
                                   int* __restrict__ sigma_inv) {
  if (obs_skip(run)) return;
  __shared__ int wpre[33];
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int p = i < NX ? posof[i] : -1;
  const unsigned b = __ballot_sync(0xffffffffu, p >= 0);
  if (lane == 0) wpre[w + 1] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    wpre[0] = 0;
    for (int k = 1; k <= 32; ++k) wpre[k] += wpre[k - 1];
  }
  __syncthreads();
  if (p >= 0) {
    const int dst = offsets[blockIdx.x] + wpre[w] + __popc(b & ((1u << lane) - 1u));
    idx_out[dst] = i;
    sigma[dst] = p;
    sigma_inv[p] = dst;
  }
}
template <typename T>
__global__ void gather_vec_kernel(int N, const int* __restrict__ sigma, const T* __restrict__ in, T* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) out[j] = in[sigma[j]];
}
__global__ void map_order_kernel(int n, const int64_t* __restrict__ order_user, const int* __restrict__ sigma_inv,
                                 int* __restrict__ order_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) order_out[i] = sigma_inv[order_user[i]];
}
// out[d*NX + perm[i]] = in[d*NX + i]   (internal -> user point order)
template <typename T>
__global__ void unpermute_kernel(int NX, int Dp, const int* __restrict__ perm, const T* __restrict__ in,
                                 T* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)NX * Dp) return;
  const int i = (int)(e % NX), d = (int)(e / NX);
  out[(size_t)d * NX + perm[i]] = in[e];
}

template <typename S, typename D_>
__global__ void convert_kernel(int rows, int cols, const S* __restrict__ src, size_t lds, D_* __restrict__ dst, size_t ldd) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;   // grid (rows, columns)
  if (i >= rows) return;
  dst[i + (size_t)j * ldd] = (D_)src[i + (size_t)j * lds];
}

// C = (float)(beta * C + Cd): the fp64 GEMM result folded into an fp32 C in one pass (no fp64 copy of C)
__global__ void accum_d2f_kernel(int rows, double beta, const double* __restrict__ Cd, size_t ldcd,
                                 float* __restrict__ C, size_t ldc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;   // grid (rows, columns)
  if (i >= rows) return;
  float* c = C + i + (size_t)j * ldc;
  *c = (float)(beta * (double)*c + Cd[i + (size_t)j * ldcd]);
}

template <typename T>
__global__ void fill_kernel(size_t n, T val, T* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = val;
}

template <typename T>
__global__ void idx64_to32_kernel(int n, const int64_t* __restrict__ in, int* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = (int)in[e];
}

inline unsigned nblk(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int stage_blocks(int N) { return N > 0 ? (N + kTile - 1) / kTile : 1; }

template <typename T>
cudaError_t StepKernels<T>::prep(int N, const int* idx, const V4<T>* coords, const T* y, const T* mpred, int policy,
                                 const int* order, uint64_t seed, int k, const int* sigma, T* r, T* s, T* v, V4<T>* xcs,
                                 cudaStream_t st, int nblk_pol, T* rbs) {
  if (N <= 0) return cudaSuccess;
  prep_kernel<T><<<nblk(N), 256, 0, st>>>(N, idx, coords, y, mpred, policy, order, seed, k, sigma, r, s, v, xcs,
                                          std::max(nblk_pol, 1), policy == 3 ? rbs : nullptr);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::gen_actions(int N, int i0, int nb, int policy, const int* order, uint64_t seed, int k,
                                        const int* sigma, T* S, size_t ldS, cudaStream_t st, const T* rbs,
                                        int nblk_pol) {
  if ((size_t)N * nb == 0) return cudaSuccess;
  gen_actions_kernel<T><<<nblk((size_t)N * nb), 256, 0, st>>>(N, i0, nb, policy, order, seed, k, sigma, S, ldS, rbs,
                                                              std::max(nblk_pol, 1));
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::stageA(int N, int nch, const T* partial, double sig00, const T* lam2, const T* s,
                                   const T* r, T* gp, const T* HM, int rin, double* part, int W, double* red,
                                   unsigned* cnt, cudaStream_t st, SlotList sl) {
  return launch_pdl(stageA_kernel<T>, dim3(stage_blocks(N)), dim3(kTile), 0, st, N, nch, partial, sig00, lam2, s, r,
                    gp, HM, rin, part, W, red, cnt, sl);
}

template <typename T>
cudaError_t StepKernels<T>::hmts(int N, const T* HM, int rin, const T* s, double* part, int W, double* red,
                                 unsigned* cnt, cudaStream_t st) {
  if (rin <= 0 || N <= 0) return cudaSuccess;
  if (side_slim())
    hmts_kernel<T, 6><<<stage_blocks(N), kTile, 0, st>>>(N, HM, rin, s, part, W, red, cnt);
  else
    hmts_kernel<T, 1><<<stage_blocks(N), kTile, 0, st>>>(N, HM, rin, s, part, W, red, cnt);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::hmu(int N, const T* HM, int rin, const double* ured, double* w, cudaStream_t st) {
  if (rin <= 0 || N <= 0) return cudaSuccess;
  if constexpr (sizeof(T) == 4) {
    if ((N & 3) == 0 && ((uintptr_t)HM & 15) == 0) {
      constexpr int kHmu4Threads = 64;   // 256 rows per block: more, smaller blocks (two per slot beside K1)
      const int nb = (N / 4 + kHmu4Threads - 1) / kHmu4Threads;
      if (side_slim())
        hmu4_kernel<6><<<nb, kHmu4Threads, sizeof(double) * rin, st>>>(N, HM, rin, ured, w);
      else
        hmu4_kernel<1><<<nb, kHmu4Threads, sizeof(double) * rin, st>>>(N, HM, rin, ured, w);
      return note_launch_err();
    }
  }
  if (side_slim())
    hmu_kernel<T, 6><<<stage_blocks(N), kTile, sizeof(double) * rin, st>>>(N, HM, rin, ured, w);
  else
    hmu_kernel<T, 1><<<stage_blocks(N), kTile, sizeof(double) * rin, st>>>(N, HM, rin, ured, w);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::stageB(int N, const T* HM, int rin, const double* ured, const T* gp, const T* s, T* g,
                                   const T* V, int nV, double* part, int W, double* red, unsigned* cnt, cudaStream_t st,
                                   const double* wpre) {
  return launch_pdl(stageB_kernel<T>, dim3(stage_blocks(N)), dim3(kTile),
                    wpre ? 8 : sizeof(double) * (rin > 0 ? rin : 1), st, N, HM, rin, ured, gp, s, g, V, nV, part, W,
                    red, cnt, wpre);
}

template <typename T>
cudaError_t StepKernels<T>::stageAB(int N, int nch, const T* partial, double sig00, const T* lam2, const T* s,
                                    const T* r, const double* wpre, T* g, const T* V, int nV, double* part, int W,
                                    double* red, double* ared_tail, unsigned* cnt, cudaStream_t st, SlotList sl) {
  return launch_pdl(stageAB_kernel<T>, dim3(stage_blocks(N)), dim3(kTile), 0, st, N, nch, partial, sig00, lam2, s, r,
                    wpre, g, V, nV, part, W, red, ared_tail, cnt, sl);
}

template <typename T>
cudaError_t StepKernels<T>::stageC(int N, const T* V, const T* Z, int nV, const double* cred, const T* sin,
                                   const T* gin, T* d, T* Gd, const T* s_eta, const double* ared, int rin,
                                   const double* sgs, double* part, int W, double* red, unsigned* cnt, IterCtl* ctl,
                                   double eps, int iter, int pass, cudaStream_t st) {
  return launch_pdl(stageC_kernel<T>, dim3(stage_blocks(N)), dim3(kTile), sizeof(double) * (nV > 0 ? nV : 1), st, N,
                    V, Z, nV, cred, sin, gin, d, Gd, s_eta, ared, rin, sgs, part, W, red, cnt, ctl, eps, iter, pass);
}

template <typename T>
cudaError_t StepKernels<T>::stageD(int N, int iter, int niter, const IterCtl* ctl, const T* d, const T* Gd, T* XV,
                                   T* Z, T* r, T* s, V4<T>* xcs, int policy, const int* order, uint64_t seed, int k,
                                   const int* sigma, cudaStream_t st, int nblk_pol, T* rbs) {
  return launch_pdl(stageD_kernel<T>, dim3(nblk(N)), dim3(256), 0, st, N, iter, niter, ctl, d, Gd, XV, Z, r, s, xcs,
                    policy, order, seed, k, sigma, std::max(nblk_pol, 1), rbs);
}

template <typename T>
cudaError_t StepKernels<T>::dot(int N, const T* a, const T* b, double* part, double* out, unsigned* cnt,
                                cudaStream_t st) {
  dot_final_kernel<T><<<stage_blocks(N), kTile, 0, st>>>(N, a, b, part, out, cnt);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::gather_rows(int N, int C, const int* idx, const T* M, size_t ldm, T* out, size_t ldo,
                                        int lo, int nl,
                                        cudaStream_t st) {
  if ((size_t)N * C == 0) return cudaSuccess;
  if (N <= 0 || C <= 0) return cudaSuccess;
  gather_rows_kernel<T><<<dim3(nblk(N), C), 256, 0, st>>>(N, C, idx, M, ldm, out, ldo, lo, nl);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::mix(int NX, int Dp, int C, const Mat3& A, bool transpose, const T* in, size_t ldi, T* out,
                                size_t ldo, cudaStream_t st) {
  if ((size_t)NX * C == 0) return cudaSuccess;
  if (NX <= 0 || C <= 0) return cudaSuccess;
  if constexpr (sizeof(T) == 4) {
    if (NX % 4 == 0 && ldi % 4 == 0 && ldo % 4 == 0 && reinterpret_cast<uintptr_t>(in) % 16 == 0 &&
        reinterpret_cast<uintptr_t>(out) % 16 == 0) {
      const int nq = NX / 4;
      const dim3 grid((unsigned)((nq + 256 * kMixQ - 1) / (256 * kMixQ)), (unsigned)C);
      const float4* in4 = reinterpret_cast<const float4*>(in);
      float4* out4 = reinterpret_cast<float4*>(out);
      if (Dp == 1) mix4_kernel<1><<<grid, 256, 0, st>>>(nq, C, A, transpose ? 1 : 0, in4, ldi / 4, out4, ldo / 4);
      else if (Dp == 2) mix4_kernel<2><<<grid, 256, 0, st>>>(nq, C, A, transpose ? 1 : 0, in4, ldi / 4, out4, ldo / 4);
      else mix4_kernel<3><<<grid, 256, 0, st>>>(nq, C, A, transpose ? 1 : 0, in4, ldi / 4, out4, ldo / 4);
      return note_launch_err();
    }
  }
  mix_kernel<T><<<dim3(nblk(NX), C), 256, 0, st>>>(NX, Dp, C, A, transpose ? 1 : 0, in, ldi, out, ldo);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::post_combine(int NX, int Dp, int C, const Mat3& S, const T* Y, const T* tmp,
                                         const T* mpred, T* m, T* Mk, int rin, cudaStream_t st) {
  const size_t D = (size_t)NX * Dp;
  if (D == 0 || C <= 0) return cudaSuccess;
  post_combine_kernel<T><<<dim3(nblk(NX), C, Dp), 256, 0, st>>>(NX, Dp, C, S, Y, tmp, mpred, m, Mk, rin);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::rowvar(int NX, int Dp, const Mat3& S, const T* base, const T* M, size_t ld, int cols,
                                   T* var, cudaStream_t st) {
  const size_t D = (size_t)NX * Dp;
  rowvar_kernel<T><<<nblk(D), 256, 0, st>>>(NX, Dp, S, base, M, ld, cols, var);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::gram(size_t D, int c, const T* M, size_t ld, double* part, int nsplit, double* G,
                                 cudaStream_t st) {
  const size_t rps = (D + nsplit - 1) / nsplit;
  const int nt = (c + 31) / 32;
  dim3 grid(nt, nt, nsplit);
  gram_partial_kernel<T><<<grid, 256, 0, st>>>(D, c, M, ld, rps, part);
  cudaError_t e = note_launch_err();
  if (e != cudaSuccess) return e;
  gram_reduce_kernel<<<nblk((size_t)c * c), 256, 0, st>>>(c, nsplit, part, G);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::take_top(int c, int r, const double* evec, const double* w, T* Qr, double* kept,
                                     double* dropped, cudaStream_t st) {
  take_top_kernel<T><<<nblk((size_t)c * r > 0 ? (size_t)c * r : 1), 256, 0, st>>>(c, r, evec, w, Qr, kept, dropped);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::sigma_apply(int NX, int Dp, int C, const Mat3& S, const T* Y, T* y, cudaStream_t st) {
  const size_t D = (size_t)NX * Dp;
  if (NX <= 0 || C <= 0) return cudaSuccess;
  // Y[q + (j*Dp + t)*NX] = Y[q + t*NX + j*D]: the (Sigma^t (x) I) mixing of mix() with column stride D
  return mix(NX, Dp, C, S, false, Y, D, y, D, st);
}

template <typename T>
cudaError_t StepKernels<T>::smooth_out(size_t D, int C, const T* m, const T* varf, const T* y, T* ms, T* vs,
                                       cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
    if (D % 4 == 0 && al(m) && al(varf) && al(y) && al(ms) && al(vs)) {
      smooth_out4_kernel<<<nblk(D / 4), 256, 0, st>>>(D / 4, C, reinterpret_cast<const float4*>(m),
                                                     reinterpret_cast<const float4*>(varf),
                                                     reinterpret_cast<const float4*>(y), reinterpret_cast<float4*>(ms),
                                                     reinterpret_cast<float4*>(vs));
      return note_launch_err();
    }
  }
  smooth_out_kernel<T><<<nblk(D), 256, 0, st>>>(D, C, m, varf, y, ms, vs);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::kcar_build(int64_t NX, int Dp, int n, int q, const T* KV, const T* Z, const T* Kx, T* KWf,
                                       T* Kws, cudaStream_t st) {
  const size_t D = (size_t)NX * Dp;
  if (D == 0) return cudaSuccess;
  if (n && !Z && (Kx || q)) return cudaErrorInvalidValue;
  if constexpr (sizeof(T) == 4) {
    auto al = [](const void* x) { return reinterpret_cast<uintptr_t>(x) % 16 == 0; };
    if (NX % 4 == 0 && al(KV) && al(Z) && al(Kx) && al(KWf) && al(Kws)) {
      kcar_build4_kernel<<<dim3(nblk(D / 4), 1 + n + q), 256, 0, st>>>(
          (size_t)NX / 4, D / 4, n, q, reinterpret_cast<const float4*>(KV), reinterpret_cast<const float4*>(Z),
          reinterpret_cast<const float4*>(Kx), reinterpret_cast<float4*>(KWf), reinterpret_cast<float4*>(Kws));
      return note_launch_err();
    }
  }
  kcar_build_kernel<T><<<dim3(nblk(D), 1 + n + q), 256, 0, st>>>((size_t)NX, D, n, q, KV, Z, Kx, KWf, Kws);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::ws_build(int N, size_t D, int n, int q, const int* idx, const T* X, const T* XV,
                                     const T* R, T* Wf, T* ws, int lo, int nl, cudaStream_t st) {
  bool vec = false;
  if constexpr (sizeof(T) == 4) {
    auto al = [](const void* x) { return reinterpret_cast<uintptr_t>(x) % 16 == 0; };
    vec = D % 4 == 0 && al(X) && al(Wf) && al(ws);
    if (vec)
      ws_dense4_kernel<<<dim3(nblk(D / 4), n + q + 1), 256, 0, st>>>(D / 4, n, reinterpret_cast<const float4*>(X),
                                                                     reinterpret_cast<float4*>(Wf),
                                                                     reinterpret_cast<float4*>(ws));
  }
  if (!vec) ws_dense_kernel<T><<<dim3(nblk(D), n + q + 1), 256, 0, st>>>(D, n, q, X, Wf, ws);
  cudaError_t e = note_launch_err();
  if (e != cudaSuccess || N == 0) return e;
  ws_scatter_kernel<T><<<nblk((size_t)N * (n + q + 1)), 256, 0, st>>>(N, D, n, q, idx, XV, R, Wf, ws, lo, nl);
  return note_launch_err();
}

// row-sharded D vectors: pack a rank's local [d * nl + i] into [d * S + i] (zero padded), and assemble the
// all-gathered packs into the full internal order [d * NX + p * S + i]
template <typename T>
__global__ void pack_dslice_kernel(int Dp, int nl, int S, const T* __restrict__ in, T* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)Dp * S) return;
  const int d = (int)(e / S), i = (int)(e % S);
  out[e] = i < nl ? in[(size_t)d * nl + i] : T(0);
}
template <typename T>
__global__ void unpack_dslices_kernel(int NX, int Dp, int S, const T* __restrict__ G, T* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)Dp * NX) return;
  const int d = (int)(e / NX), g = (int)(e % NX), p = g / S, i = g % S;
  out[e] = G[(size_t)p * Dp * S + (size_t)d * S + i];
}
template <typename T>
cudaError_t StepKernels<T>::pack_dslice(int Dp, int nl, int S, const T* in, T* out, cudaStream_t st) {
  pack_dslice_kernel<T><<<nblk((size_t)Dp * S), 256, 0, st>>>(Dp, nl, S, in, out);
  return note_launch_err();
}
template <typename T>
cudaError_t StepKernels<T>::unpack_dslices(int NX, int Dp, int S, const T* G, T* out, cudaStream_t st) {
  unpack_dslices_kernel<T><<<nblk((size_t)Dp * NX), 256, 0, st>>>(NX, Dp, S, G, out);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::assemble_slices(int M, int C, int slice, const T* G, T* Y, size_t ldy, cudaStream_t st) {
  if ((size_t)M * C == 0) return cudaSuccess;
  assemble_slices_kernel<T><<<nblk((size_t)M * C), 256, 0, st>>>(M, C, slice, G, Y, ldy);
  return note_launch_err();
}

template <typename T>
cudaError_t StepKernels<T>::fill(size_t n, T val, T* out, cudaStream_t st) {
  if (!n) return cudaSuccess;
  fill_kernel<T><<<nblk(n), 256, 0, st>>>(n, val, out);
  return note_launch_err();
}

template <typename S, typename D_>
cudaError_t convert(int rows, int cols, const S* src, size_t lds, D_* dst, size_t ldd, cudaStream_t st) {
  if ((size_t)rows * cols == 0) return cudaSuccess;
  for (int j0 = 0; j0 < cols; j0 += 65535) {   // grid.y <= 65535 columns per launch
    const int nc = std::min(65535, cols - j0);
    convert_kernel<S, D_><<<dim3(nblk(rows), nc), 256, 0, st>>>(rows, nc, src + (size_t)j0 * lds, lds,
                                                                 dst + (size_t)j0 * ldd, ldd);
    if (j0 + nc < cols) {
      const cudaError_t e = note_launch_err();
      if (e != cudaSuccess) return e;
    }
  }
  return note_launch_err();
}
cudaError_t accum_d2f(int rows, int cols, double beta, const double* Cd, size_t ldcd, float* C, size_t ldc,
                      cudaStream_t st) {
  if ((size_t)rows * cols == 0) return cudaSuccess;
  for (int j0 = 0; j0 < cols; j0 += 65535) {
    const int nc = std::min(65535, cols - j0);
    accum_d2f_kernel<<<dim3(nblk(rows), nc), 256, 0, st>>>(rows, beta, Cd + (size_t)j0 * ldcd, ldcd,
                                                          C + (size_t)j0 * ldc, ldc);
    const cudaError_t e = note_launch_err();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t convert<float, double>(int, int, const float*, size_t, double*, size_t, cudaStream_t);
template cudaError_t convert<double, float>(int, int, const double*, size_t, float*, size_t, cudaStream_t);
template cudaError_t convert<double, double>(int, int, const double*, size_t, double*, size_t, cudaStream_t);

template <typename T>
cudaError_t sampler_ops<T>::permute_cols(int NX, int Dp, int S, const int* map, const T* in, size_t ldi, T* out,
                                         size_t ldo, cudaStream_t st) {
  const size_t n = (size_t)NX * Dp * S;
  if (!n) return cudaSuccess;
  permute_cols_kernel<T><<<nblk(n), 256, 0, st>>>(NX, Dp, S, map, in, ldi, out, ldo);
  return note_launch_err();
}
template <typename T>
cudaError_t sampler_ops<T>::residual(int N, int S, const T* y, const int* idx, const int* sigma, const T* xp, size_t D,
                                     const T* eps, T* res, cudaStream_t st) {
  if ((size_t)N * S == 0) return cudaSuccess;
  sample_residual_kernel<T><<<nblk((size_t)N * S), 256, 0, st>>>(N, S, y, idx, sigma, xp, D, eps, res);
  return note_launch_err();
}
template <typename T>
cudaError_t sampler_ops<T>::combine(int NX, int Dp, int S, const Mat3& Sg, const T* Y, const T* tmp, const T* xp, T* x,
                                    cudaStream_t st) {
  const size_t n = (size_t)NX * Dp * S;
  if (!n) return cudaSuccess;
  sample_combine_kernel<T><<<nblk(n), 256, 0, st>>>(NX, Dp, S, Sg, Y, tmp, tmp ? 1 : 0, xp, x);
  return note_launch_err();
}
template <typename T>
cudaError_t sampler_ops<T>::scatter_rows(int N, int S, const int* idx, const T* R, T sign, T* w, size_t D,
                                         cudaStream_t st) {
  if ((size_t)N * S == 0) return cudaSuccess;
  scatter_rows_kernel<T><<<nblk((size_t)N * S), 256, 0, st>>>(N, S, idx, R, sign, w, D);
  return note_launch_err();
}
template <typename T>
cudaError_t sampler_ops<T>::gather_coords(int N, const int* idx, const V4<T>* coords, V4<T>* out, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  gather_coords_kernel<T><<<nblk(N), 256, 0, st>>>(N, idx, coords, out);
  return note_launch_err();
}
template struct sampler_ops<float>;
template struct sampler_ops<double>;

cudaError_t obs_sort(int N, int NX, const int64_t* obs, const int* invperm, int* posof, int* counts, int* idx_out,
                     int* sigma, int* sigma_inv, cudaStream_t st, const int* run) {
  if (N <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(posof, 0xff, (size_t)NX * sizeof(int), st);   // -1 (scratch: harmless on a skip)
  if (e != cudaSuccess) return e;
  obs_mark_kernel<<<nblk(N), 256, 0, st>>>(N, run, obs, invperm, posof);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  const int nb = (NX + 1023) / 1024;
  obs_count_kernel<<<nb, 1024, 0, st>>>(NX, run, posof, counts);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  obs_scan_kernel<<<1, 32, 0, st>>>(nb, run, counts);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  obs_scatter_kernel<<<nb, 1024, 0, st>>>(NX, run, posof, counts, idx_out, sigma, sigma_inv);
  return note_launch_err();
}

// obs_equal: neq_out = 1 if a[0:n] != b[0:n] (the observation-order cache of cakf_update)
__global__ void obs_neq_kernel(int n, const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                               int* __restrict__ neq) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n && a[j] != b[j]) *neq = 1;
}
cudaError_t obs_neq(int n, const int64_t* a, const int64_t* b, int* neq, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(neq, 0, sizeof(int), st);
  if (e != cudaSuccess || n <= 0) return e;
  obs_neq_kernel<<<nblk(n), 256, 0, st>>>(n, a, b, neq);
  return note_launch_err();
}

template <typename T>
cudaError_t gather_vec(int N, const int* sigma, const T* in, T* out, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  gather_vec_kernel<T><<<nblk(N), 256, 0, st>>>(N, sigma, in, out);
  return note_launch_err();
}
template cudaError_t gather_vec<float>(int, const int*, const float*, float*, cudaStream_t);
template cudaError_t gather_vec<double>(int, const int*, const double*, double*, cudaStream_t);

template <typename T>
__global__ void scatter_vec_kernel(int N, const int* __restrict__ sigma, const T* __restrict__ in, T* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) out[sigma[j]] = in[j];
}
template <typename T>
cudaError_t scatter_vec(int N, const int* sigma, const T* in, T* out, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  scatter_vec_kernel<T><<<nblk(N), 256, 0, st>>>(N, sigma, in, out);
  return note_launch_err();
}
template cudaError_t scatter_vec<float>(int, const int*, const float*, float*, cudaStream_t);
template cudaError_t scatter_vec<double>(int, const int*, const double*, double*, cudaStream_t);

template <typename T>
__global__ void set_w_kernel(int N, const T* __restrict__ w, V4<T>* __restrict__ xc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) xc[j].w = w[j];
}
template <typename T>
cudaError_t set_w(int N, const T* w, V4<T>* xc, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  set_w_kernel<T><<<nblk(N), 256, 0, st>>>(N, w, xc);
  return note_launch_err();
}
template cudaError_t set_w<float>(int, const float*, V4<float>*, cudaStream_t);
template cudaError_t set_w<double>(int, const double*, V4<double>*, cudaStream_t);

cudaError_t map_order(int n, const int64_t* order_user, const int* sigma_inv, int* order_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  map_order_kernel<<<nblk(n), 256, 0, st>>>(n, order_user, sigma_inv, order_out);
  return note_launch_err();
}

template <typename T>
cudaError_t unpermute(int NX, int Dp, const int* perm, const T* in, T* out, cudaStream_t st) {
  unpermute_kernel<T><<<nblk((size_t)NX * Dp), 256, 0, st>>>(NX, Dp, perm, in, out);
  return note_launch_err();
}
template cudaError_t unpermute<float>(int, int, const int*, const float*, float*, cudaStream_t);
template cudaError_t unpermute<double>(int, int, const int*, const double*, double*, cudaStream_t);

cudaError_t idx64_to32(int n, const int64_t* in, int* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  idx64_to32_kernel<int><<<nblk(n), 256, 0, st>>>(n, in, out);
  return note_launch_err();
}

template struct StepKernels<float>;
template struct StepKernels<double>;

}  // namespace cakf

namespace cakf {
bool pdl_enabled() {   // CAKF_PDL=0: plain launches for the inner-loop kernels
  static const bool v = !env_is("CAKF_PDL", '0');
  return v;
}
}  // namespace cakf
