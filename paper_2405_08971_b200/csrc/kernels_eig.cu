// kernels_eig.cu — the truncation's symmetric eigensolver (a8 / a9 Truncate, Sec. 3.2 P:334-369,
// "SVD of M M^T" P:367, reading R4: eigh of the c x c Gram M^T M), fp64, entirely on the device.
//
//   1. Householder tridiagonalisation  C = H T H^T  in ONE thread-block cluster (16 CTAs; the matrix
//      resident in their shared memory for c <= ~600, else in L2-resident global memory), one cluster
//      barrier per column: every CTA owns whole columns (cyclically); the rank-2 update of step j is
//      fused into the matvec pass of step j+1; p and the partial dots are pushed into every CTA's shared
//      memory (DSMEM stores before the barrier), the next column goes through L2; every CTA then computes
//      the next reflector itself.
//   2. Cuppen divide and conquer on T (leaves of size 1, six launches per level): rank-one merges with
//      deflation (negligible weight; close poles by Givens rotation), the secular equation per root by a
//      safeguarded two-pole rational iteration in the distance to the nearer pole, Gu-Eisenstat
//      recomputation of z (orthogonal vectors without reorthogonalisation), and the eigenvector update
//      Q_block B as an fp64 GEMM per merge (B = sort permutation x deflation rotations x secular vectors).
//   3. Back-transformation of the r wanted eigenvectors (descending eigenvalues) in compact-WY panels of
//      32 reflectors (T factors by dlarft, then Z <- (I - V T V^T) Z per panel, 4 columns per CTA).
// The outputs replace cusolverDnDsyevd + take_top: Q_r (c x r, column-major), the kept eigenvalues
// (descending), the dropped mass (sum of the c - r smallest) and optionally all eigenvalues ascending.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace cakf {

namespace {

constexpr int kTrdThreads = 1024;
constexpr int kTrdCluster = 16;
constexpr int kTrdSmemBytes = 227 * 1024;
constexpr int kTrdRed = 96;          // doubles of the tridiagonalisation's reduction / exchange scratch
constexpr int kTrdReflWarps = 4;     // warps computing the next reflector while the others apply the rank-2 update (8: no better)

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum (blockDim.x multiple of 32); valid in every thread; red >= 33 doubles of smem
__device__ double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
    t = warp_sum_d(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

struct TrdArgs {
  int c;
  const double* G;   // c x c, lower triangle read (ld c)
  double* V;         // c x c: column j = Householder vector v_j in rows j+1.. (v_j[j+1] = 1)
  double* tau;       // c
  double* d;         // c   diagonal of T
  double* e;         // c   sub-diagonal of T (e[j] = T[j+1][j])
  double* pglob;     // 2 x c  p of the step (double-buffered by step parity)
  double* colglob;   // 2 x c  the next column after all but the latest update
  double* sglob;     // 2 x kTrdCluster partial dots p^T v
  double* Aglob;     // global-memory mode: slabs of L x c per CTA
};


// Householder tridiagonalisation in one cluster of NC CTAs, ONE cluster barrier per step:
//   step j: (a) pass over my columns i > j (one column per warp, two rows per lane as double2): form
//               p_i = tau_j A[:, i] . v_j (update(j-1) was applied in step j-1) and push it to every CTA; the
//               owner of column j+1 also publishes that column in L2;
//           (b) cluster barrier;
//           (c) every CTA finds p and the partial dots in its own shared memory (pushed by their owners over
//               DSMEM during (a)), reads column j+1 (L2), forms w_j and applies update(j) to column j+1; then
//               the first warps compute reflector j+1 (identical arithmetic in every CTA, no second cluster
//               barrier) while the other warps apply update(j) to the CTA's columns i > j+1.
// Layout: local columns with an even stride ldA >= c + 1 (the rows in [c, ldA) and the row entries of v / w
// at and above c are zero), so the double2 pass may start one row early and run one row past the end.
// Reflector convention (LAPACK dlarfg): H = I - tau v v^T, H x = beta e_1, v[j+1] = 1, v[j] = 0.
__host__ __device__ constexpr int trd_ld(int c) { return (c + 2) & ~1; }

template <int NC, bool SMEM>
__global__ void __launch_bounds__(kTrdThreads, 1) sytrd_cluster_kernel(TrdArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int c = a.c, ld = trd_ld(c);
  const int L = (c + NC - 1) / NC;
  extern __shared__ __align__(16) double sm[];
  double* A = SMEM ? sm : a.Aglob + (size_t)q * L * ld;
  double* vb = SMEM ? sm + (size_t)L * ld : sm;   // [2][ld]  v_j by step parity
  double* wb = vb + 2 * (size_t)ld;                // [2][ld]  w_j by step parity
  double* pb = wb + 2 * (size_t)ld;                // [2][ld]  p of every row by step parity (pushed by the column owners)
  double* xb = pb + 3 * (size_t)ld;                // [ld]     column j+1 (one spare ld before it)
  double* red = xb + (size_t)ld;                   // [kTrdRed] red[40 + parity] = tau_j, red[48 + 16 parity + q] = CTA q's partial dot
  const int nloc = q < c ? (c - q + NC - 1) / NC : 0;   // my columns i = q + NC * lc
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5, bd = blockDim.x;
  const bool writer = q == 0;
  for (size_t x = tid; x < (size_t)nloc * ld; x += bd) {
    const int lc = (int)(x / ld), l = (int)(x % ld), i = q + NC * lc;
    A[x] = l >= c ? 0.0 : l >= i ? a.G[l + (size_t)i * c] : a.G[i + (size_t)l * c];
  }
  for (int x = tid; x < 8 * ld; x += bd) vb[x] = 0.0;   // v, w, p, x buffers incl. the padding rows
  if (c <= 2) {
    if (writer && tid == 0) {
      a.d[0] = a.G[0];
      if (c == 2) {
        a.d[1] = a.G[3];
        a.e[0] = a.G[1];
      }
    }
    return;
  }
  // reflector jr from x = xs[jr+1 .. c) (smem), into vout; tau -> red[40 + (jr & 1)]; CTA 0 writes the outputs.
  // s2_own >= 0: this thread's share of sum_{l >= jr+2} x_l^2 was already formed (with the column update)
  auto reflector = [&](int jr, const double* xs, double dj, double* vout, double s2_own) {
    double s2 = 0.0;
    if (s2_own >= 0.0) s2 = s2_own;
    else
      for (int l = jr + 2 + tid; l < c; l += bd) s2 += xs[l] * xs[l];
    s2 = warp_sum_d(s2);
    if (lane == 0) red[warp] = s2;
    __syncthreads();
    double t = lane < nwarps ? red[lane] : 0.0;   // every warp reduces the partials itself (no 2nd barrier)
    t = warp_sum_d(t);
    const double alpha = xs[jr + 1];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (t > 0.0) {
      const double nrm = sqrt(alpha * alpha + t);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int l = jr + 1 + tid; l < c; l += bd) {
      const double v = l == jr + 1 ? 1.0 : xs[l] * scal;
      vout[l] = v;
      if (writer) a.V[l + (size_t)jr * c] = v;
    }
    if (tid == 0) {
      vout[jr] = 0.0;
      red[40 + (jr & 1)] = tau;
      if (writer) {
        a.tau[jr] = tau;
        a.d[jr] = dj;
        a.e[jr] = beta;
      }
    }
  };
  // the same reflector run by the first nthr threads only, with red[0, nwarps) already holding the warps'
  // partial sums of sum_{l >= jr+2} x_l^2 (identical arithmetic: same partials, same reductions)
  auto reflector_part = [&](int jr, const double* xs, double dj, double* vout, int nthr) {
    double t = lane < nwarps ? red[lane] : 0.0;
    t = warp_sum_d(t);
    const double alpha = xs[jr + 1];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (t > 0.0) {
      const double nrm = sqrt(alpha * alpha + t);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int l = jr + 1 + tid; l < c; l += nthr) {
      const double v = l == jr + 1 ? 1.0 : xs[l] * scal;
      vout[l] = v;
      if (writer) a.V[l + (size_t)jr * c] = v;
    }
    if (tid == 0) {
      vout[jr] = 0.0;
      red[40 + (jr & 1)] = tau;
      if (writer) {
        a.tau[jr] = tau;
        a.d[jr] = dj;
        a.e[jr] = beta;
      }
    }
  };
  __syncthreads();
  for (int l = tid; l < c; l += bd) xb[l] = a.G[l];   // column 0 of G: no update yet
  __syncthreads();
  reflector(0, xb, xb[0], vb, -1.0);
  __syncthreads();
#ifdef CAKF_TRD_TIMING
  long long tacc[8] = {};
  long long tprev = clock64();
#define TRD_T(k)                       \
  {                                    \
    const long long tn_ = clock64();   \
    tacc[k] += tn_ - tprev;            \
    tprev = tn_;                       \
  }
#else
#define TRD_T(k)
#endif
  for (int j = 0; j + 3 <= c; ++j) {
    const int par = j & 1;
    const double* vj = vb + (size_t)par * ld;
    double* wj = wb + (size_t)par * ld;
    double* cg_ = a.colglob + (size_t)par * c;
    double* pbp = pb + (size_t)par * ld;
    const double tj = red[40 + par];
    // ---- (a) fused pass: one column per warp (two when more than 32 are live: only while j < 16 (c - 32)),
    // row pairs per lane — with the live columns shrinking to (c - j) / NC, one column per warp keeps twice
    // the warps busy of the earlier column-pair form
    const int lc0 = q > j ? 0 : (j - q) / NC + 1;   // first local column with i > j
    const int r0 = (j + 1) & ~1;                     // first row pair (row j is dead: v_j[j] = 0)
    double sq = 0.0;
    for (int lcA = lc0 + warp; lcA < nloc; lcA += nwarps) {
      const int iA = q + NC * lcA;
      // SMEM: update(j-1) already applied (step j-1, beside its reflector); global-memory columns (large c):
      // update(j-1) fused into this pass, one L2 read and write of the trailing matrix per step
      double* colA = A + (size_t)lcA * ld;
      const bool pubA = iA == j + 1;
      const bool fuse = !SMEM && j > 0;
      const double* vprev = vb + (size_t)(par ^ 1) * ld;
      const double* wprev = wb + (size_t)(par ^ 1) * ld;
      const double vpA = fuse ? vprev[iA] : 0.0, wpA = fuse ? wprev[iA] : 0.0;
      double accA = 0.0;
      for (int r = r0 + 2 * lane; r < c; r += 64) {
        const double2 vv = *reinterpret_cast<const double2*>(vj + r);
        double2 xa = *reinterpret_cast<const double2*>(colA + r);
        if (fuse) {
          const double2 vp = *reinterpret_cast<const double2*>(vprev + r);
          const double2 wp = *reinterpret_cast<const double2*>(wprev + r);
          xa.x -= vp.x * wpA + wp.x * vpA;
          xa.y -= vp.y * wpA + wp.y * vpA;
          *reinterpret_cast<double2*>(colA + r) = xa;
        }
        accA += xa.x * vv.x + xa.y * vv.y;
        if (pubA) {
          if (r >= j + 1) cg_[r] = xa.x;
          if (r + 1 < c) cg_[r + 1] = xa.y;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) accA += __shfl_xor_sync(0xffffffffu, accA, off);
      // p_i into every CTA's p buffer of this parity (DSMEM push, lane q -> CTA q; visible after the barrier;
      // staging p locally and pushing with the whole CTA after the pass measured slower, r4t)
      const double pA = tj * accA;
      if (lane < NC) cl.map_shared_rank(pbp, lane)[iA] = pA;
      if (lane == 0) sq += pA * vj[iA];
    }
    TRD_T(0)
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    TRD_T(1)
    if (warp == 0) {   // my partial dot into every CTA's slot q of this parity
      double t = lane < nwarps ? red[lane] : 0.0;
      t = warp_sum_d(t);
      if (lane < NC) cl.map_shared_rank(red, lane)[48 + 16 * par + q] = t;
    }
    // ---- (b)
    cl.sync();
    TRD_T(2)
    // ---- (c) p and the partial dots are local (pushed before the barrier); column j+1 from L2
    const double* prw = pbp;
    for (int l = j + 1 + tid; l < c; l += bd) xb[l] = __ldcg(cg_ + l);
    if (warp == 0) {
      double t = lane < NC ? red[48 + 16 * par + lane] : 0.0;
      t = warp_sum_d(t);
      if (lane == 0) red[35] = t;
    }
    __syncthreads();
    TRD_T(3)
    const double hk = 0.5 * tj * red[35];
    const double vn = vj[j + 1], wn = prw[j + 1] - hk * vn;
    double s2n = 0.0;   // the next reflector's sum_{l >= j+3} x_l^2, formed with the update (one pass, one sync)
    for (int l = j + 1 + tid; l < c; l += bd) {
      const double w = prw[l] - hk * vj[l];
      wj[l] = w;
      const double x = xb[l] - (vj[l] * wn + w * vn);   // update(j) of column j+1
      xb[l] = x;
      if (l >= j + 3) s2n += x * x;
    }
    if (!SMEM && j + 4 <= c) {   // global-memory columns: the reflector on all warps, update(j) in the next pass
      TRD_T(4)
      reflector(j + 1, xb, tid == 0 ? xb[j + 1] : 0.0, vb + (size_t)(par ^ 1) * ld, s2n);
      TRD_T(5)
    } else if (j + 4 <= c) {
      TRD_T(4)
      s2n = warp_sum_d(s2n);
      if (lane == 0) red[warp] = s2n;
      __syncthreads();   // xb, wj and the partial sums complete
      if (warp < kTrdReflWarps) {
        // the next reflector on the first warps (dj = x_{j+1}: thread 0 wrote that row itself) ...
        reflector_part(j + 1, xb, tid == 0 ? xb[j + 1] : 0.0, vb + (size_t)(par ^ 1) * ld, kTrdReflWarps * 32);
      } else {
        // ... while the other warps apply update(j) (A -= v_j w_j^T + w_j v_j^T) to my columns i > j+1, rows
        // from (j+2) & ~1: the next step's pass then only forms the dots (the same values it formed before)
        const int lc1 = q > j + 1 ? 0 : (j + 1 - q) / NC + 1;
        const int r1 = (j + 2) & ~1;
        // column pairs per warp: v_j, w_j rows loaded once for two columns (the update is bound by
        // shared-memory traffic; 18 pairs at most against 28 warps)
        for (int lcA = lc1 + 2 * (warp - kTrdReflWarps); lcA < nloc; lcA += 2 * (nwarps - kTrdReflWarps)) {
          const bool hasB = lcA + 1 < nloc;
          const int iA = q + NC * lcA, iB = iA + NC;
          double* colA = A + (size_t)lcA * ld;
          double* colB = A + (size_t)(lcA + 1) * ld;
          const double vA = vj[iA], wA = wj[iA];
          const double vB = hasB ? vj[iB] : 0.0, wB = hasB ? wj[iB] : 0.0;
          for (int r = r1 + 2 * lane; r < c; r += 64) {
            const double2 vp = *reinterpret_cast<const double2*>(vj + r);
            const double2 wp = *reinterpret_cast<const double2*>(wj + r);
            double2 xa = *reinterpret_cast<double2*>(colA + r);
            xa.x -= vp.x * wA + wp.x * vA;
            xa.y -= vp.y * wA + wp.y * vA;
            *reinterpret_cast<double2*>(colA + r) = xa;
            if (hasB) {
              double2 xb2 = *reinterpret_cast<double2*>(colB + r);
              xb2.x -= vp.x * wB + wp.x * vB;
              xb2.y -= vp.y * wB + wp.y * vB;
              *reinterpret_cast<double2*>(colB + r) = xb2;
            }
          }
        }
      }
      TRD_T(5)
    } else {   // j + 1 == c - 2: the last 2 x 2 block's column c-2 (rows c-2, c-1: lanes 0, 1 of warp 0)
      __syncwarp();
      if (writer && tid == 0) {
        a.d[c - 2] = xb[c - 2];
        a.e[c - 2] = xb[c - 1];
      }
    }
    __syncthreads();   // xb / wj / vb complete before the next pass; pb, red[36..] are double-buffered
    TRD_T(6)
  }
#ifdef CAKF_TRD_TIMING
  if (tid == 0 && (q == 0 || q == 1 || q == NC - 1))
    printf("trd cta %d c %d: pass %lld sync1 %lld cl.sync %lld loads %lld xupd %lld refl %lld end %lld (cycles/step)\n", q,
           c, tacc[0] / (c - 2), tacc[1] / (c - 2), tacc[2] / (c - 2), tacc[3] / (c - 2), tacc[4] / (c - 2),
           tacc[5] / (c - 2), tacc[6] / (c - 2));
#endif
  // ---- d[c-1]: column c-1 (owner) after update(c-3): row c-1 only
  {
    const int j = c - 3, par = j & 1, i = c - 1;
    const double* vj = vb + (size_t)par * ld;
    const double* wj = wb + (size_t)par * ld;
    if (q == i % NC && tid == 0) {
      const double* col = A + (size_t)(i / NC) * ld;
      a.d[c - 1] = col[c - 1] - 2.0 * vj[c - 1] * wj[c - 1];
    }
  }
}

// ------------------------------------------------------------------ divide and conquer
// Merge m at level s (blocks of size s merged in pairs): rows/cols [o, o + n), L = [o, o + s),
// R = [o + s, o + n), o = 2 s m, n = min(2 s, c - o); valid iff o + s < c.
// Per merge, with P the sort permutation of the poles and G the deflation rotations:
//   T_block = Q P G (Dhat + rho zhat zhat^T) G^T P^T Q^T,   new eigenvectors  Q P G [U | E_defl]
// The new block is computed as Qnew = Q_block B with B = P G [U | E_defl] (n x n, built per column),
// so no permuted copy of Q is materialised; Q and the output alternate between two buffers.
struct DcArgs {
  int c, s;
  const double* e;     // sub-diagonal of T
  double* dl;          // c: eigenvalues of the current blocks (ascending within a block)
  const double* Q;     // c x c: eigenvectors of the current blocks (block-diagonal)
  double* Qn;          // c x c: eigenvectors of the merged blocks (output)
  double* B;           // c x c: per merge, n x n block at (o, o): rows = local columns of Q
  double* dK;          // c: non-deflated poles (sorted)
  double* zK;          // c: non-deflated weights
  double* org_tau;     // c: tau of root t (signed distance to its origin pole)
  double* zhat;        // c
  double* lam;         // c: merged eigenvalues in (K, deflated) order
  double* rotc;        // c: deflation rotation cosines (per merge, in scan order)
  double* rots;        // c: sines
  int* rota;           // c: rotated sorted positions (pj)
  int* rotb;           // c: (nj)
  int* nrot;           // per merge
  int* perm;           // c: sorted position -> local column
  int* org;            // c: origin pole index of root t
  int* kmap;           // c: (K, deflated) order -> sorted position
  int* rank;           // c: (K, deflated) order -> final ascending position
  int* kcnt;           // per merge: number of non-deflated
  double* rho;         // per merge: rho * ||z||^2
};

__device__ __forceinline__ bool dc_merge(int c, int s, int m, int& o, int& n) {
  o = 2 * s * m;
  if (o + s >= c) return false;
  n = min(2 * s, c - o);
  return true;
}

// initial leaves: every point is a split point (leaf size 1): d_i - |e_{i-1}| - |e_i|, Q = I
__global__ void dc_init_kernel(int c, const double* __restrict__ d, const double* __restrict__ e,
                               double* __restrict__ dl, double* __restrict__ Q) {
  const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < (size_t)c * c) {
    const int i = (int)(x % c), j = (int)(x / c);
    Q[x] = i == j ? 1.0 : 0.0;
  }
  if (x < (size_t)c) {
    const int i = (int)x;
    double v = d[i];
    if (i > 0) v -= fabs(e[i - 1]);
    if (i + 1 < c) v -= fabs(e[i]);
    dl[i] = v;
  }
}

constexpr int kDcPrepThreads = 256;

// Per merge: z = Q^T u, sort the poles (merge of two ascending lists), deflate (dlaed2: negligible
// weight; close poles -> Givens rotation).  Dynamic smem: 2 n doubles + n ints.
__global__ void __launch_bounds__(kDcPrepThreads) dc_prep_kernel(DcArgs a) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  int o, n;
  const int m = blockIdx.x;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int c = a.c, s = a.s, n1 = s;
  extern __shared__ __align__(16) double sh[];
  double* ds = sh;              // sorted poles
  double* zs = ds + n;          // sorted weights
  int* km = reinterpret_cast<int*>(zs + n);   // (K, deflated) order -> sorted position
  __shared__ double red[40];
  __shared__ int k_s;
  const double rho0 = fabs(a.e[o + s - 1]);
  const double sgn = a.e[o + s - 1] < 0.0 ? -1.0 : 1.0;
  double z2 = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double z = t < n1 ? a.Q[(o + s - 1) + (size_t)(o + t) * c] : sgn * a.Q[(o + s) + (size_t)(o + t) * c];
    z2 += z * z;
  }
  z2 = block_sum_d(z2, red);
  const double zn = sqrt(z2);
  const double rho = rho0 * z2;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const bool left = t < n1;
    const double dv = a.dl[o + t];
    int lo = left ? n1 : 0, hi = left ? n : n1;   // rank in the other list (ties: L first)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const double dm = a.dl[o + mid];
      if (left ? (dm < dv) : (dm <= dv)) lo = mid + 1;
      else hi = mid;
    }
    const int pos = left ? t + (lo - n1) : (t - n1) + lo;
    const double z = left ? a.Q[(o + s - 1) + (size_t)(o + t) * c] : sgn * a.Q[(o + s) + (size_t)(o + t) * c];
    ds[pos] = dv;
    zs[pos] = zn > 0.0 ? z / zn : 0.0;
    a.perm[o + pos] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // sequential deflation scan (cheap reject of far poles: |gap C S| <= |gap| / 2)
    double dmax = 0.0, zmax = 0.0;
    for (int t = 0; t < n; ++t) {
      dmax = fmax(dmax, fabs(ds[t]));
      zmax = fmax(zmax, fabs(zs[t]));
    }
    const double tol = 8.0 * DBL_EPSILON * fmax(dmax, rho * zmax);
    int k = 0, ndef = 0, nr = 0, pj = -1;
    for (int t = 0; t < n; ++t) {
      if (rho * fabs(zs[t]) <= tol) {
        km[n - 1 - ndef++] = t;
        continue;
      }
      if (pj < 0) {
        pj = t;
        continue;
      }
      const double gap = ds[t] - ds[pj];
      bool defl = false;
      if (fabs(gap) <= 2.0 * tol) {
        double S = zs[pj], C = zs[t];
        const double tz = hypot(C, S);
        C /= tz;
        S = -S / tz;
        if (fabs(gap * C * S) <= tol) {
          defl = true;
          zs[t] = tz;
          zs[pj] = 0.0;
          a.rota[o + nr] = pj;
          a.rotb[o + nr] = t;
          a.rotc[o + nr] = C;
          a.rots[o + nr] = S;
          ++nr;
          const double tt = ds[pj] * C * C + ds[t] * S * S;
          ds[t] = ds[pj] * S * S + ds[t] * C * C;
          ds[pj] = tt;
          km[n - 1 - ndef++] = pj;
        }
      }
      if (!defl) km[k++] = pj;
      pj = t;
    }
    if (pj >= 0) km[k++] = pj;
    for (int x = 0; x < ndef / 2; ++x) {   // deflated part in scan order
      const int tmp = km[k + x];
      km[k + x] = km[n - 1 - x];
      km[n - 1 - x] = tmp;
    }
    k_s = k;
    a.kcnt[m] = k;
    a.nrot[m] = nr;
    a.rho[m] = rho;
  }
  __syncthreads();
  const int k = k_s;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int sp = km[t];
    a.kmap[o + t] = sp;
    if (t < k) {
      a.dK[o + t] = ds[sp];
      a.zK[o + t] = zs[sp];
    } else {
      a.lam[o + t] = ds[sp];   // deflated eigenvalue
    }
  }
}

// secular equation g(tau) = 1/rho + sum_i z_i^2 / ((d_i - d_org) - tau) = 0 for root t of merge m (one warp):
// lambda_t = d_org + tau, origin = the nearer pole.  Safeguarded iteration: the two-pole rational model
// of psi (poles <= t) and phi (poles > t) matched in value and slope (Bunch-Nielsen-Sorensen), falling back to
// bisection (geometric while the bracket spans orders of magnitude) whenever the model step leaves the bracket.
__global__ void dc_secular_kernel(DcArgs a) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= a.c) return;
  const int m = gw / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int t = gw - o, k = a.kcnt[m];
  if (t >= k) return;
  const double* dK = a.dK + o;
  const double* zK = a.zK + o;
  const double rho = a.rho[m], irho = 1.0 / rho;
  const bool last = t == k - 1;
  int orgi;
  double tlo, thi;   // signed bracket of tau, g(tlo) < 0 <= g(thi)
  if (last) {
    orgi = t;
    tlo = DBL_TRUE_MIN;
    thi = rho * 1.0000000001 + 4.0 * DBL_EPSILON * fabs(dK[t]);
  } else {
    const double gap = dK[t + 1] - dK[t];
    double acc = 0.0;
    const double mid = 0.5 * gap;
    for (int i = lane; i < k; i += 32) acc += zK[i] * zK[i] / ((dK[i] - dK[t]) - mid);
    const bool right = warp_sum_d(acc) + irho >= 0.0;
    orgi = right ? t : t + 1;
    tlo = right ? DBL_TRUE_MIN : -0.5 * gap;
    thi = right ? 0.5 * gap : -DBL_TRUE_MIN;
  }
  const double dor = dK[orgi];
  const double dl_ = dK[t] - dor;                          // left pole (origin-relative)
  const double dr_ = last ? 0.0 : dK[t + 1] - dor;         // right pole
  double tau = 0.5 * (tlo + thi);
  for (int it = 0; it < 100; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double inv = 1.0 / ((dK[i] - dor) - tau);
      const double tv = zK[i] * zK[i] * inv;
      if (i <= t) {
        psi += tv;
        dpsi += tv * inv;
      } else {
        phi += tv;
        dphi += tv * inv;
      }
    }
    psi = warp_sum_d(psi);
    dpsi = warp_sum_d(dpsi);
    phi = warp_sum_d(phi);
    dphi = warp_sum_d(dphi);
    const double g = irho + psi + phi;
    if (g < 0.0) tlo = tau;
    else thi = tau;
    const double erretm = 8.0 * (irho + fabs(psi) + fabs(phi)) + fabs(tau) * (dpsi + dphi);
    if (fabs(g) <= DBL_EPSILON * erretm || thi - tlo <= 2.0 * DBL_EPSILON * fmax(fabs(tlo), fabs(thi))) break;
    // rational model step
    double x;
    const double b = dpsi * (dl_ - tau) * (dl_ - tau), av = psi - dpsi * (dl_ - tau);
    if (last) {
      const double A = irho + av;
      x = dl_ + b / A;
    } else {
      const double dd = dphi * (dr_ - tau) * (dr_ - tau), cv = phi - dphi * (dr_ - tau);
      const double A = irho + av + cv;
      // A x^2 - (A (dl + dr) + b + dd) x + (A dl dr + b dr + dd dl) = 0
      const double Bq = -(A * (dl_ + dr_) + b + dd);
      const double Cq = A * dl_ * dr_ + b * dr_ + dd * dl_;
      const double disc = fmax(Bq * Bq - 4.0 * A * Cq, 0.0);
      const double qv = -0.5 * (Bq + copysign(sqrt(disc), Bq));
      const double x1 = qv / A, x2 = Cq / qv;
      x = (x1 > tlo && x1 < thi) ? x1 : x2;
    }
    if (!(x > tlo && x < thi)) {   // bisection (geometric when the bracket spans orders of magnitude)
      if (tlo > 0.0 && thi > 4.0 * tlo) x = sqrt(tlo) * sqrt(thi);
      else if (thi < 0.0 && -tlo > -4.0 * thi) x = -sqrt(-tlo) * sqrt(-thi);
      else x = 0.5 * (tlo + thi);
      if (!(x > tlo && x < thi)) break;
    }
    tau = x;
  }
  if (lane == 0) {
    a.org[o + t] = orgi;
    a.org_tau[o + t] = tau;
  }
}

// lambda_j - d_i from the (origin, tau) representation (accurate for nearby poles)
__device__ __forceinline__ double lam_minus_d(const double* dK, const int* org, const double* tau, int j, int i) {
  return (dK[org[j]] - dK[i]) + tau[j];
}

// Gu-Eisenstat: zhat_i^2 = (lambda_i - d_i)/rho * prod_{j != i} (lambda_j - d_i)/(d_j - d_i); one warp per i
__global__ void dc_zhat_kernel(DcArgs a) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= a.c) return;
  const int m = gw / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int i = gw - o, k = a.kcnt[m];
  if (i >= k) return;
  const double* dK = a.dK + o;
  const int* org = a.org + o;
  const double* tau = a.org_tau + o;
  double mant = 1.0;   // product with explicit exponent tracking (no overflow / underflow for any k)
  int ex = 0;
  for (int j = lane; j < k; j += 32) {
    double f = lam_minus_d(dK, org, tau, j, i);
    if (j != i) f /= (dK[j] - dK[i]);
    else f /= a.rho[m];
    int e2;
    mant = frexp(mant * f, &e2);
    ex += e2;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, mant, off);
    const int oe = __shfl_xor_sync(0xffffffffu, ex, off);
    int e2;
    mant = frexp(mant * om, &e2);
    ex += e2 + oe;
  }
  if (lane == 0) a.zhat[o + i] = copysign(sqrt(ldexp(fabs(mant), ex)), a.zK[o + i]);
}

// column t of B = P G [U | E_defl] (one warp per t < n; n doubles of smem per warp):
//   t < k: U[:, t] = zhat_u / (d_u - lambda_t) normalised, placed at the sorted positions kmap[u];
//   t >= k: the unit vector at sorted position kmap[t];
// then the deflation rotations in reverse order, then the rows scattered to the local columns perm[s].
constexpr int kVecWarps = 4;
__global__ void __launch_bounds__(kVecWarps * 32) dc_vec_kernel(DcArgs a, int nmax) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  extern __shared__ __align__(16) double vbuf[];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= a.c) return;
  const int m = gw / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int t = gw - o, k = a.kcnt[m], c = a.c;
  double* col = vbuf + (size_t)(threadIdx.x >> 5) * nmax;
  for (int x = lane; x < n; x += 32) col[x] = 0.0;
  __syncwarp();
  if (t < k) {
    const double* dK = a.dK + o;
    const int* org = a.org + o;
    const double* tau = a.org_tau + o;
    double ss = 0.0;
    for (int u = lane; u < k; u += 32) {
      const double v = a.zhat[o + u] / -lam_minus_d(dK, org, tau, t, u);
      col[a.kmap[o + u]] = v;
      ss += v * v;
    }
    ss = warp_sum_d(ss);
    __syncwarp();
    const double inv = 1.0 / sqrt(ss);
    for (int u = lane; u < k; u += 32) col[a.kmap[o + u]] *= inv;
    if (lane == 0) a.lam[o + t] = dK[org[t]] + tau[t];
  } else if (lane == 0) {
    col[a.kmap[o + t]] = 1.0;
  }
  __syncwarp();
  if (lane == 0) {
    for (int x = a.nrot[m] - 1; x >= 0; --x) {   // G x = G_1 (G_2 (... G_nrot x))
      const int pa = a.rota[o + x], pb = a.rotb[o + x];
      const double C = a.rotc[o + x], S = a.rots[o + x];
      const double xa = col[pa], xb = col[pb];
      col[pa] = C * xa - S * xb;
      col[pb] = S * xa + C * xb;
    }
  }
  __syncwarp();
  for (int sp = lane; sp < n; sp += 32) a.B[(o + a.perm[o + sp]) + (size_t)(o + t) * c] = col[sp];
}

// final ascending position of each merged eigenvalue (ties by (K, deflated) order index)
__global__ void dc_rank_kernel(DcArgs a) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.c) return;
  const int m = x / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int t = x - o;
  const double v = a.lam[o + t];
  int r = 0;
  for (int u = 0; u < n; ++u) {
    const double w = a.lam[o + u];
    r += (w < v) || (w == v && u < t);
  }
  a.rank[o + t] = r;
  a.dl[o + r] = v;
}

// Qn[o:o+n, o+rank(t)] = Q[o:o+n, o:o+n] B[o:o+n, o+t]; the carried (unmerged) last block is copied.
// 32 x 32 output tiles (many CTAs: the GEMMs are small and latency-bound), 64 threads with 4 x 4 outputs each,
// K chunks of 32 double-buffered through registers.
constexpr int kGT = 32, kGK = 32, kGThreads = 64;
__global__ void __launch_bounds__(kGThreads) dc_gemm_kernel(DcArgs a) {
  griddep_wait();   // PDL: the previous divide-and-conquer launch's outputs
  const int c = a.c, s = a.s;
  const int tpm = (2 * s + kGT - 1) / kGT;   // tiles per merge side
  const int tiles_per_merge = tpm * tpm;
  const int m = blockIdx.x / tiles_per_merge, tt = blockIdx.x % tiles_per_merge;
  int o, n;
  const int r0 = (tt % tpm) * kGT, c0 = (tt / tpm) * kGT;
  if (!dc_merge(c, s, m, o, n)) {
    o = 2 * s * m;
    if (o >= c) return;
    n = c - o;
    for (int x = threadIdx.x; x < kGT * kGT; x += kGThreads) {
      const int rr = r0 + x % kGT, cc = c0 + x / kGT;
      if (rr < n && cc < n) a.Qn[(o + rr) + (size_t)(o + cc) * c] = a.Q[(o + rr) + (size_t)(o + cc) * c];
    }
    return;
  }
  if (r0 >= n || c0 >= n) return;
  __shared__ double As[kGK][kGT + 1];   // [inner][row]
  __shared__ double Bs[kGK][kGT + 1];   // [inner][col]
  const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;   // 8 x 8 threads, outputs (ty + 8p, tx + 8q)
  double acc[4][4] = {};
  double ra[16], rb[16];
  // Q_block is block-diagonal (L = [0, s), R = [s, n)): its off-diagonal blocks are never stored (they hold
  // stale data) and contribute zero; a row tile entirely in L (R) runs over the inner range of L (R) only
  const int ulo = r0 >= s ? s : 0, uhi = r0 + kGT <= s ? s : n;
  auto fetch = [&](int u0) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int x = threadIdx.x + e * kGThreads;     // 0 .. 1023
      const int rr = x % kGT, uu = x / kGT;          // A: rows contiguous
      const int u = u0 + uu, row = r0 + rr;
      ra[e] = (u < uhi && row < n && ((row < s) == (u < s))) ? a.Q[(o + row) + (size_t)(o + u) * c] : 0.0;
      const int ub = x % kGK, cc = x / kGK;          // B: inner contiguous
      rb[e] = (u0 + ub < uhi && c0 + cc < n) ? a.B[(o + u0 + ub) + (size_t)(o + c0 + cc) * c] : 0.0;
    }
  };
  fetch(ulo);
  for (int u0 = ulo; u0 < uhi; u0 += kGK) {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int x = threadIdx.x + e * kGThreads;
      As[x / kGT][x % kGT] = ra[e];
      Bs[x % kGK][x / kGK] = rb[e];
    }
    __syncthreads();
    if (u0 + kGK < uhi) fetch(u0 + kGK);
#pragma unroll
    for (int uu = 0; uu < kGK; ++uu) {
      double av[4], bv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) av[p] = As[uu][ty + 8 * p];
#pragma unroll
      for (int p = 0; p < 4; ++p) bv[p] = Bs[uu][tx + 8 * p];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) acc[p][q2] = fma(av[p], bv[q2], acc[p][q2]);
    }
  }
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    const int t = c0 + tx + 8 * q2;
    if (t >= n) continue;
    const int dst = o + a.rank[o + t];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int row = r0 + ty + 8 * p;
      if (row < n) a.Qn[(o + row) + (size_t)dst * c] = acc[p][q2];
    }
  }
}

// ---- blocked (compact WY) back-transformation: panels of kBtNb reflectors, H_j0 ... H_j0+b-1 = I - V T V^T
constexpr int kBtNb = 32, kBtCols = 4, kBtThreads = 256;

// T of panel p (upper triangular b x b, column-major ld kBtNb): dlarft (forward, columnwise)
__global__ void __launch_bounds__(kBtThreads) bt_larft_kernel(int c, const double* __restrict__ V,
                                                              const double* __restrict__ tau, double* __restrict__ Tall) {
  const int p = blockIdx.x, nref = c - 2, j0 = p * kBtNb, b = min(kBtNb, nref - j0);
  if (b <= 0) return;
  __shared__ double S[kBtNb][kBtNb + 1];
  __shared__ double T[kBtNb][kBtNb + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kBtThreads / 32;
  // S[a][e] = v_{j0+a} . v_{j0+e}, a < e: rows j0+e+1 .. c-1 (the support of v_{j0+e})
  for (int pr = warp; pr < b * b; pr += nw) {
    const int a = pr % b, e = pr / b;
    if (a >= e) continue;
    const double* va = V + (size_t)(j0 + a) * c;
    const double* ve = V + (size_t)(j0 + e) * c;
    double acc = 0.0;
    for (int l = j0 + e + 1 + lane; l < c; l += 32) acc += va[l] * ve[l];
    acc = warp_sum_d(acc);
    if (lane == 0) S[a][e] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    for (int i = 0; i < b; ++i) {
      const double ti = tau[j0 + i];
      // T[0:i, i] = -tau_i T[0:i, 0:i] S[0:i, i]   (lane r computes row r)
      double acc = 0.0;
      if (lane < i)
        for (int x = lane; x < i; ++x) acc += T[lane][x] * S[x][i];
      __syncwarp();
      if (lane < i) T[lane][i] = -ti * acc;
      if (lane == 0) T[i][i] = ti;
      if (lane > i && lane < kBtNb) T[lane][i] = 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < kBtNb * kBtNb; x += kBtThreads) {
    const int r = x % kBtNb, e = x / kBtNb;
    Tall[(size_t)p * kBtNb * kBtNb + x] = (r < b && e < b) ? T[r][e] : 0.0;
  }
}

// kBtCols output columns per CTA: Z = Q_T[:, c-1-j] (descending eigenvalues), then Z <- (I - V_p T_p V_p^T) Z
// for the panels from the last to the first; Z in shared memory (c x kBtCols), the panel's V rows staged
// once per panel into shared memory (in chunks of `rmax` rows only when the panel does not fit).
// Thread t owns the output (a, col) = (t % 32, t / 32) of W = V_p^T Z.
constexpr int kBtPad = kBtNb + 1;
static_assert(kBtNb * kBtCols <= kBtThreads, "one W output per thread");
__global__ void __launch_bounds__(kBtThreads) bt_apply_kernel(int c, int r, int rmax, const double* __restrict__ V,
                                                              const double* __restrict__ Tall,
                                                              const double* __restrict__ Q, double* __restrict__ Qr) {
  extern __shared__ __align__(16) double Zs[];   // [kBtCols][c], then Vs[rmax][kBtPad]
  double* Vs = Zs + (size_t)kBtCols * c;
  __shared__ double W[kBtNb][kBtCols], Ts[kBtNb][kBtNb + 1], Wh[2][kBtNb][kBtCols];
  const int j0c = blockIdx.x * kBtCols, ncol = min(kBtCols, r - j0c);
  for (int x = threadIdx.x; x < kBtCols * c; x += kBtThreads) {
    const int col = x / c, l = x % c;
    Zs[x] = col < ncol ? Q[l + (size_t)(c - 1 - (j0c + col)) * c] : 0.0;
  }
  const int nref = c - 2;
  const int np = nref > 0 ? (nref + kBtNb - 1) / kBtNb : 0;
  const int ta = threadIdx.x % kBtNb, tcol = threadIdx.x / kBtNb;
  const bool wown = threadIdx.x < kBtNb * kBtCols;
  const int half = threadIdx.x / (kBtNb * kBtCols), tcol2 = (threadIdx.x / kBtNb) % kBtCols;
  static_assert(kBtThreads == 2 * kBtNb * kBtCols, "two row halves of the W = V^T Z outputs");
  auto stage = [&](int j0, int b, int r0, int nr) {   // Vs[rr][a] = v_{j0+a}[r0+rr] (zero above its support)
    for (int x = threadIdx.x; x < nr * kBtNb; x += kBtThreads) {
      const int rr = x % nr, a = x / nr, l = r0 + rr;
      Vs[(size_t)rr * kBtPad + a] = (a < b && l > j0 + a) ? __ldg(V + l + (size_t)(j0 + a) * c) : 0.0;
    }
  };
  for (int p = np - 1; p >= 0; --p) {
    const int j0 = p * kBtNb, b = min(kBtNb, nref - j0);
    const int r00 = j0 + 1, nrows = c - r00;
    const bool one = nrows <= rmax;
    for (int x = threadIdx.x; x < kBtNb * kBtNb; x += kBtThreads) Ts[x % kBtNb][x / kBtNb] = Tall[(size_t)p * kBtNb * kBtNb + x];
    // W = V_p^T Z: the even rows of each chunk on threads [0, 128), the odd rows on [128, 256) (the two
    // accumulators of one thread before), summed even + odd
    double acc = 0.0;
    for (int r0 = r00; r0 < c; r0 += rmax) {
      const int nr = min(rmax, c - r0);
      __syncthreads();
      stage(j0, b, r0, nr);
      __syncthreads();
      const double* z = Zs + (size_t)tcol2 * c + r0;
      for (int rr = half; rr < nr; rr += 2) acc += Vs[(size_t)rr * kBtPad + ta] * z[rr];
    }
    Wh[half][ta][tcol2] = acc;
    __syncthreads();
    if (wown) W[ta][tcol] = Wh[0][ta][tcol] + Wh[1][ta][tcol];
    __syncthreads();
    double w2 = 0.0;   // W2 = T W
    if (wown)
      for (int e = ta; e < b; ++e) w2 += Ts[ta][e] * W[e][tcol];
    __syncthreads();
    if (wown) W[ta][tcol] = w2;
    // Z -= V_p W2
    for (int r0 = r00; r0 < c; r0 += rmax) {
      const int nr = min(rmax, c - r0);
      if (!one) {
        __syncthreads();
        stage(j0, b, r0, nr);
      }
      __syncthreads();
      for (int x = threadIdx.x; x < nr * kBtCols; x += kBtThreads) {
        const int rr = x % nr, col = x / nr;
        const double* vr = Vs + (size_t)rr * kBtPad;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int a = 0; a < kBtNb; a += 2) {
          s0 += vr[a] * W[a][col];
          s1 += vr[a + 1] * W[a + 1][col];
        }
        Zs[(size_t)col * c + r0 + rr] -= s0 + s1;
      }
    }
    __syncthreads();
  }
  for (int x = threadIdx.x; x < ncol * c; x += kBtThreads) {
    const int col = x / c, l = x % c;
    Qr[l + (size_t)(j0c + col) * c] = Zs[x];
  }
}

// eigenvalue outputs: kept (descending top r), dropped mass, all (ascending); non-finite -> *fail = 1
__global__ void eig_values_kernel(int c, int r, const double* __restrict__ dl, double* kept, double* dropped,
                                  double* w_all, int* fail) {
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    if (w_all) w_all[i] = dl[i];
    if (kept && i < r) kept[i] = dl[c - 1 - i];
    if (!isfinite(dl[i]) && fail) *fail = 1;
  }
  if (threadIdx.x == 0 && dropped) {
    double s = 0.0;
    for (int i = 0; i < c - r; ++i) s += dl[i];
    *dropped = s;
  }
}

size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

int trd_smem_max_c(int nc) {
  // L x c doubles of columns + 4 c doubles of v / w buffers + 64 doubles, L = ceil(c / nc)
  int best = 0;
  for (int c = 1; c <= 4096; ++c) {
    const size_t L = (c + nc - 1) / nc;
    const size_t ld = trd_ld(c);
    const size_t bytes = (L * ld + 8 * ld + kTrdRed) * sizeof(double);
    if (bytes <= (size_t)kTrdSmemBytes) best = c;
  }
  return best;
}

// 16-CTA clusters need the non-portable size; fall back to 8 if the device cannot co-schedule 16
int trd_cluster_size() {
  static const int nc = [] {
    cudaFuncSetAttribute(sytrd_cluster_kernel<16, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(sytrd_cluster_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrdSmemBytes);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kTrdCluster);
    cfg.blockDim = dim3(kTrdThreads);
    cfg.dynamicSmemBytes = kTrdSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kTrdCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, sytrd_cluster_kernel<16, true>, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      return 8;
    }
    return kTrdCluster;
  }();
  return nc;
}

size_t eig_workspace_bytes(int cmax) {
  const size_t c = (size_t)std::max(cmax, 1);
  size_t b = 0;
  b += align_up(c * c * 8) * 4;                 // V, Q, Qp, U
  b += align_up(c * 8) * 13;                    // tau, d, e, dl, dK, zK, org_tau, zhat, lam, colglob(2), pglob(2)
  b += align_up(c * 4) * 8;                     // org, kmap, rank, kcnt, perm, rota, rotb, nrot
  b += align_up(c * 8) * 2;                     // rotc, rots
  b += align_up(c * 8) + align_up(64 * 8);      // rho, sglob
  b += align_up((c + kTrdCluster) * (c + 2) * 8);   // global-memory tridiagonalisation slabs (nc x ceil(c/nc) x ld)
  b += align_up((c / 32 + 2) * 32 * 32 * 8);    // compact-WY T factors of the back-transformation
  return b + 4096;
}

cudaError_t eig_top(int c, int r, const double* G, void* ws, size_t ws_bytes, double* Qr, double* kept,
                    double* dropped, double* w_all, int* fail, cudaStream_t st, cudaStream_t side, cudaEvent_t ev_a,
                    cudaEvent_t ev_b) {
  if (c <= 0 || r < 0 || r > c) return cudaErrorInvalidValue;
  if (eig_workspace_bytes(c) > ws_bytes) return cudaErrorInvalidValue;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += align_up(bytes);
    return q;
  };
  const size_t cc = (size_t)c * c;
  double* V = reinterpret_cast<double*>(take(cc * 8));
  double* Q = reinterpret_cast<double*>(take(cc * 8));
  double* Qp = reinterpret_cast<double*>(take(cc * 8));
  double* U = reinterpret_cast<double*>(take(cc * 8));
  double* tau = reinterpret_cast<double*>(take(c * 8));
  double* d = reinterpret_cast<double*>(take(c * 8));
  double* e = reinterpret_cast<double*>(take(c * 8));
  double* dl = reinterpret_cast<double*>(take(c * 8));
  double* dK = reinterpret_cast<double*>(take(c * 8));
  double* zK = reinterpret_cast<double*>(take(c * 8));
  double* otau = reinterpret_cast<double*>(take(c * 8));
  double* zhat = reinterpret_cast<double*>(take(c * 8));
  double* lam = reinterpret_cast<double*>(take(c * 8));
  double* colglob = reinterpret_cast<double*>(take(2 * (size_t)c * 8));
  double* pglob = reinterpret_cast<double*>(take(2 * (size_t)c * 8));
  int* org = reinterpret_cast<int*>(take(c * 4));
  int* kmap = reinterpret_cast<int*>(take(c * 4));
  int* rank = reinterpret_cast<int*>(take(c * 4));
  int* kcnt = reinterpret_cast<int*>(take(c * 4));
  int* perm = reinterpret_cast<int*>(take(c * 4));
  int* rota = reinterpret_cast<int*>(take(c * 4));
  int* rotb = reinterpret_cast<int*>(take(c * 4));
  int* nrot = reinterpret_cast<int*>(take(c * 4));
  double* rotc = reinterpret_cast<double*>(take(c * 8));
  double* rots = reinterpret_cast<double*>(take(c * 8));
  double* rho = reinterpret_cast<double*>(take(c * 8));
  double* sglob = reinterpret_cast<double*>(take(64 * 8));
  double* Aglob = reinterpret_cast<double*>(take(((size_t)c + kTrdCluster) * ((size_t)c + 2) * 8));
  double* Tp = reinterpret_cast<double*>(take(((size_t)c / 32 + 2) * 32 * 32 * 8));
  (void)p;
  // ---- 1. tridiagonalisation (one cluster of nc CTAs: 16 where the device can co-schedule it, else 8)
  {
    static const int smem_max_c16 = trd_smem_max_c(16), smem_max_c8 = trd_smem_max_c(8);
    static const int nc_env = [] { const char* e = getenv("CAKF_TRD_NC"); return e ? std::atoi(e) : 0; }();
    const int nc = nc_env == 8 ? 8 : trd_cluster_size();   // CAKF_TRD_NC=8: the 8-CTA cluster (A/B only)
    auto kern = nc == 16 ? (c <= smem_max_c16 ? sytrd_cluster_kernel<16, true> : sytrd_cluster_kernel<16, false>)
                         : (c <= smem_max_c8 ? sytrd_cluster_kernel<8, true> : sytrd_cluster_kernel<8, false>);
    const size_t L = (c + nc - 1) / nc;
    const bool in_smem = c <= (nc == 16 ? smem_max_c16 : smem_max_c8);
    const size_t ldt = trd_ld(c);
    const size_t smem = in_smem ? (L * ldt + 8 * ldt + kTrdRed) * sizeof(double) : (8 * ldt + kTrdRed) * sizeof(double);
    if (smem > (size_t)kTrdSmemBytes) return cudaErrorInvalidValue;
    static PerDeviceOnce once;
    const cudaError_t ce = once_per_device(once, [] {
      cudaError_t r1 = cudaSuccess;
      for (auto k : {sytrd_cluster_kernel<16, true>, sytrd_cluster_kernel<16, false>, sytrd_cluster_kernel<8, true>,
                     sytrd_cluster_kernel<8, false>}) {
        if (r1 == cudaSuccess) r1 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrdSmemBytes);
        if (r1 == cudaSuccess) r1 = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }
      return r1;
    });
    if (ce != cudaSuccess) return ce;
    TrdArgs ta{c, G, V, tau, d, e, pglob, colglob, sglob, Aglob};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc);
    cfg.blockDim = dim3(kTrdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, kern, ta);
    ++launch_counter();
    if (le != cudaSuccess) return le;
    le = cudaGetLastError();
    if (le != cudaSuccess) return le;
  }
  // the back-transformation's T factors need only the reflectors: on the side stream (when given), beside the
  // divide and conquer, joined before bt_apply
  const int np = c > 2 ? (c - 2 + kBtNb - 1) / kBtNb : 0;
  const bool larft_side = side && ev_a && ev_b && r > 0 && np > 0;
  if (larft_side) {
    cudaError_t e1 = cudaEventRecord(ev_a, st);
    if (e1 == cudaSuccess) e1 = cudaStreamWaitEvent(side, ev_a, 0);
    if (e1 != cudaSuccess) return e1;
    bt_larft_kernel<<<np, kBtThreads, 0, side>>>(c, V, tau, Tp);
    if ((e1 = note_launch_err()) != cudaSuccess) return e1;
    if ((e1 = cudaEventRecord(ev_b, side)) != cudaSuccess) return e1;
  }
  // ---- 2. divide and conquer on T
  dc_init_kernel<<<(unsigned)((cc + 255) / 256), 256, 0, st>>>(c, d, e, dl, Q);
  cudaError_t err = note_launch_err();
  if (err != cudaSuccess) return err;
  DcArgs da{c, 1, e, dl, Q, Qp, U, dK, zK, otau, zhat, lam, rotc, rots, rota, rotb, nrot, perm, org, kmap, rank,
            kcnt, rho};
  static PerDeviceOnce once_dc;
  err = once_per_device(once_dc, [] {
    cudaError_t r1 = cudaFuncSetAttribute(dc_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (r1 == cudaSuccess) r1 = cudaFuncSetAttribute(dc_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return r1;
  });
  if (err != cudaSuccess) return err;
  double* Qcur = Q;
  double* Qnext = Qp;
  for (int s = 1; s < c; s *= 2) {
    da.s = s;
    da.Q = Qcur;
    da.Qn = Qnext;
    const int nmerge = (c + 2 * s - 1) / (2 * s);
    const size_t nmax = (size_t)std::min(2 * s, c);
    const size_t psmem = nmax * (2 * sizeof(double) + sizeof(int));
    const size_t vsmem = (size_t)kVecWarps * nmax * sizeof(double);
    if (psmem > 200 * 1024 || vsmem > 200 * 1024) return cudaErrorInvalidValue;
    // programmatic dependent launches: each kernel's launch and prologue overlap its predecessor's tail
    // (every kernel waits with griddepcontrol.wait before touching memory)
    if ((err = launch_pdl(dc_prep_kernel, dim3(nmerge), dim3(kDcPrepThreads), psmem, st, da)) != cudaSuccess) return err;
    const unsigned wblocks = (unsigned)((c * 32 + 255) / 256);
    if ((err = launch_pdl(dc_secular_kernel, dim3(wblocks), dim3(256), 0, st, da)) != cudaSuccess) return err;
    if ((err = launch_pdl(dc_zhat_kernel, dim3(wblocks), dim3(256), 0, st, da)) != cudaSuccess) return err;
    if ((err = launch_pdl(dc_vec_kernel, dim3((unsigned)((c + kVecWarps - 1) / kVecWarps)), dim3(kVecWarps * 32), vsmem,
                          st, da, (int)nmax)) != cudaSuccess)
      return err;
    if ((err = launch_pdl(dc_rank_kernel, dim3((c + 255) / 256), dim3(256), 0, st, da)) != cudaSuccess) return err;
    const int tpm = (2 * s + kGT - 1) / kGT;
    if ((err = launch_pdl(dc_gemm_kernel, dim3(nmerge * tpm * tpm), dim3(kGThreads), 0, st, da)) != cudaSuccess) return err;
    std::swap(Qcur, Qnext);
  }
  // ---- 3. back-transformation of the r wanted eigenvectors (compact WY panels), eigenvalue outputs
  eig_values_kernel<<<1, 256, 0, st>>>(c, r, dl, kept, dropped, w_all, fail);
  if ((err = note_launch_err()) != cudaSuccess) return err;
  if (r == 0) return cudaSuccess;
  if (larft_side) {
    if ((err = cudaStreamWaitEvent(st, ev_b, 0)) != cudaSuccess) return err;
  } else if (np) {
    bt_larft_kernel<<<np, kBtThreads, 0, st>>>(c, V, tau, Tp);
    if ((err = note_launch_err()) != cudaSuccess) return err;
  }
  constexpr size_t kBtSmem = 200 * 1024;   // + ~9 KB static (W, T)
  const size_t zbytes = (size_t)kBtCols * c * sizeof(double);
  if (zbytes + 64 * kBtPad * sizeof(double) > kBtSmem) return cudaErrorInvalidValue;
  const int rmax = (int)std::min<size_t>((size_t)std::max(c - 1, 1), (kBtSmem - zbytes) / (kBtPad * sizeof(double)));
  const size_t bsmem = zbytes + (size_t)rmax * kBtPad * sizeof(double);
  static PerDeviceOnce once_bt;
  err = once_per_device(once_bt, [] {
    return cudaFuncSetAttribute(bt_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBtSmem);
  });
  if (err != cudaSuccess) return err;
  bt_apply_kernel<<<(r + kBtCols - 1) / kBtCols, kBtThreads, bsmem, st>>>(c, r, rmax, V, Tp, Qcur, Qr);
  return note_launch_err();
}

}  // namespace cakf
