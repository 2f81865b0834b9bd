// kernels_eig.cu — the truncation's symmetric eigensolver (a8 / a9 Truncate, Sec. 3.2 P:334-369,
// "SVD of M M^T" P:367, reading R4: eigh of the c x c Gram M^T M), fp64, entirely on the device.
//
//   1. Householder tridiagonalisation  C = H T H^T  in ONE thread-block cluster (16 CTAs, the
//      matrix resident in their shared memory for c <= kTrdSmemMaxC, else in L2-resident global
//      memory): reflector j is computed by the CTA owning column j; the symmetric matvec p = tau A v
//      is column-parallel (every CTA owns whole columns, cyclically), the rank-2 update of step j is
//      fused into the matvec pass of step j+1 (one pass over the trailing matrix per step), v and p
//      are exchanged through L2 between two cluster barriers per step.
//   2. Cuppen divide and conquer on T (leaves of size 1, one level per launch group): rank-one
//      merges with deflation (small z, close poles by Givens rotation), the secular equation solved
//      per root by bisection in the distance to the nearest pole (full relative accuracy, one warp
//      per root), Gu-Eisenstat recomputation of z so the merged eigenvectors are orthogonal, and
//      the eigenvector update as an fp64 GEMM per merge.
//   3. Back-transformation of the r wanted eigenvectors (descending eigenvalues): q <- H_0 ... H_{c-3} q,
//      one warp per column.
// The outputs replace cusolverDnDsyevd + take_top: Q_r (c x r, column-major), the kept eigenvalues
// (descending), the dropped mass (sum of the c - r smallest) and optionally all eigenvalues ascending.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace cakf {

namespace {

constexpr int kTrdThreads = 1024;
constexpr int kTrdCluster = 16;
constexpr int kTrdSmemBytes = 227 * 1024;

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
  double* vglob;     // 2 x c  broadcast of v (double-buffered by step parity)
  double* pglob;     // c      broadcast of p
  double* sglob;     // kTrdCluster partial dots
  double* Aglob;     // global-memory mode: kTrdCluster slabs of L x c
};

// Householder reflector of column j (owned by this CTA, local column lc): x = A[j+1:, j].
// LAPACK dlarfg convention: H = I - tau v v^T, H x = beta e_1, v[j+1] = 1.
__device__ void trd_householder(const TrdArgs& a, const double* Acol, int j, double* red) {
  const int c = a.c;
  double s2 = 0.0;
  for (int l = j + 2 + threadIdx.x; l < c; l += blockDim.x) s2 += Acol[l] * Acol[l];
  s2 = block_sum_d(s2, red);
  const double alpha = Acol[j + 1];
  double tau = 0.0, beta = alpha, scal = 0.0;
  if (s2 > 0.0) {
    const double nrm = sqrt(alpha * alpha + s2);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  double* vg = a.vglob + (size_t)(j & 1) * c;
  for (int l = j + 1 + threadIdx.x; l < c; l += blockDim.x) {
    const double v = l == j + 1 ? 1.0 : Acol[l] * scal;
    vg[l] = v;
    a.V[l + (size_t)j * c] = v;
  }
  if (threadIdx.x == 0) {
    a.tau[j] = tau;
    a.d[j] = Acol[j];
    a.e[j] = beta;
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(kTrdThreads, 1) sytrd_cluster_kernel(TrdArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int NC = (int)cl.num_blocks();
  const int c = a.c;
  const int L = (c + NC - 1) / NC;
  extern __shared__ __align__(16) double sm[];
  double* A = SMEM ? sm : a.Aglob + (size_t)q * L * c;
  double* vb = SMEM ? sm + (size_t)L * c : sm;   // [2][c]
  double* wb = vb + 2 * (size_t)c;                // [2][c]
  double* red = wb + 2 * (size_t)c;               // [64]
  const int nloc = q < c ? (c - q + NC - 1) / NC : 0;   // my columns i = q + NC * lc
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // load my columns of the symmetric matrix (lower triangle mirrored)
  for (size_t x = threadIdx.x; x < (size_t)nloc * c; x += blockDim.x) {
    const int lc = (int)(x / c), l = (int)(x % c), i = q + NC * lc;
    A[x] = l >= i ? a.G[l + (size_t)i * c] : a.G[i + (size_t)l * c];
  }
  __syncthreads();
  if (c >= 3 && q == 0) trd_householder(a, A, 0, red);   // column 0 lives in CTA 0 (lc 0)
  cl.sync();
  for (int j = 0; j + 3 <= c; ++j) {
    const int par = j & 1;
    double* vj = vb + (size_t)par * c;
    double* vprev = vb + (size_t)(par ^ 1) * c;
    double* wprev = wb + (size_t)(par ^ 1) * c;
    double* wj = wb + (size_t)par * c;
    // ---- v_j from L2 (written by the owner before the barrier)
    const double* vg = a.vglob + (size_t)par * c;
    for (int l = j + 1 + threadIdx.x; l < c; l += blockDim.x) vj[l] = __ldcg(vg + l);
    const double tj = __ldcg(a.tau + j);
    __syncthreads();
    // ---- fused pass over my columns i > j: apply update(j-1) to rows >= j+1, then p_i = tau_j A[:, i] . v_j
    const int lc0 = q > j ? 0 : (j - q) / NC + 1;   // first local column with i > j
    double sq = 0.0;
    for (int lc = lc0 + warp; lc < nloc; lc += nwarps) {
      const int i = q + NC * lc;
      double* col = A + (size_t)lc * c;
      double acc = 0.0;
      if (j > 0) {
        const double vpi = vprev[i], wpi = wprev[i];
        for (int l = j + 1 + lane; l < c; l += 32) {
          const double x = col[l] - vprev[l] * wpi - wprev[l] * vpi;
          col[l] = x;
          acc += x * vj[l];
        }
      } else {
        for (int l = j + 1 + lane; l < c; l += 32) acc += col[l] * vj[l];
      }
      acc = warp_sum_d(acc);
      if (lane == 0) {
        const double p = tj * acc;
        a.pglob[i] = p;
        sq += p * vj[i];
      }
    }
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += red[w];
      a.sglob[q] = t;
    }
    cl.sync();
    // ---- w_j = p - (tau/2)(p^T v) v, every CTA, full vector
    double K = 0.0;
    for (int r = 0; r < NC; ++r) K += __ldcg(a.sglob + r);
    const double hk = 0.5 * tj * K;
    for (int l = j + 1 + threadIdx.x; l < c; l += blockDim.x) wj[l] = __ldcg(a.pglob + l) - hk * vj[l];
    __syncthreads();
    // ---- owner of column j+1: apply update(j) to it now (look-ahead), then its reflector
    const int jn = j + 1;
    if (q == jn % NC) {
      double* col = A + (size_t)(jn / NC) * c;
      const double vi = vj[jn], wi = wj[jn];
      for (int l = jn + threadIdx.x; l < c; l += blockDim.x) col[l] -= vj[l] * wi + wj[l] * vi;
      __syncthreads();
      if (jn + 3 <= c) trd_householder(a, col, jn, red);
    }
    cl.sync();
  }
  // ---- epilogue: the last 2 x 2 block (column c-2 got update(c-3) in the loop; column c-1 gets it here)
  if (c >= 3) {
    const int j = c - 3, par = j & 1;
    const double* vj = vb + (size_t)par * c;
    const double* wj = wb + (size_t)par * c;
    const int i = c - 1;
    if (q == i % NC && threadIdx.x < 2) {
      double* col = A + (size_t)(i / NC) * c;
      const int l = c - 2 + threadIdx.x;
      col[l] -= vj[l] * wj[i] + wj[l] * vj[i];
    }
    __syncthreads();
  }
  if (c >= 2) {
    if (q == (c - 2) % NC && threadIdx.x == 0) {
      const double* col = A + (size_t)((c - 2) / NC) * c;
      a.d[c - 2] = col[c - 2];
      a.e[c - 2] = col[c - 1];
    }
  }
  if (q == (c - 1) % NC && threadIdx.x == 0) a.d[c - 1] = A[(size_t)((c - 1) / NC) * c + (c - 1)];
}

// ------------------------------------------------------------------ divide and conquer
// Merge m at level s (blocks of size s merged in pairs): rows/cols [o, o + n), L = [o, o + s),
// R = [o + s, o + n), o = 2 s m, n = min(2 s, c - o); valid iff o + s < c.
struct DcArgs {
  int c, s;
  const double* e;     // sub-diagonal of T
  double* dl;          // c: eigenvalues of the current blocks (ascending within a block)
  double* Q;           // c x c: eigenvectors of the current blocks (block-diagonal)
  double* Qp;          // c x c: gathered (sorted, rotated) columns of the merge
  double* U;           // c x c: secular eigenvectors, block (o, o)
  double* dK;          // c: non-deflated poles (sorted), then deflated values
  double* zK;          // c: non-deflated weights
  double* org_tau;     // c: tau of root t (distance to its origin pole)
  double* zhat;        // c
  double* lam;         // c: merged eigenvalues in (K, deflated) order
  int* org;            // c: origin pole index of root t
  int* kmap;           // c: (K, deflated) order -> sorted position (column of Qp)
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

// Per merge: z = Q^T u, sort the poles, deflate (dlaed2), gather the sorted columns and apply the
// deflation rotations.  Dynamic smem: n doubles (d sorted) + n doubles (z sorted) + n ints (perm)
// + n ints (kmap) + n x (2 ints + 2 doubles) rotations.
__global__ void __launch_bounds__(kDcPrepThreads) dc_prep_kernel(DcArgs a) {
  int o, n;
  const int m = blockIdx.x;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int c = a.c, s = a.s, n1 = s, n2 = n - s;
  extern __shared__ __align__(16) double sh[];
  double* ds = sh;              // sorted poles
  double* zs = ds + n;          // sorted weights
  double* rc = zs + n;          // rotation cosines
  double* rs = rc + n;          // rotation sines
  int* perm = reinterpret_cast<int*>(rs + n);   // sorted position -> local column
  int* ra = perm + n;           // rotation column a (sorted positions)
  int* rb = ra + n;
  int* km = rb + n;             // (K, deflated) order -> sorted position
  __shared__ double red[40];
  __shared__ int nrot_s, k_s;
  const double rho0 = fabs(a.e[o + s - 1]);
  const double sgn = a.e[o + s - 1] < 0.0 ? -1.0 : 1.0;
  // z and its norm
  double z2 = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double z = t < n1 ? a.Q[(o + s - 1) + (size_t)(o + t) * c] : sgn * a.Q[(o + s) + (size_t)(o + t) * c];
    z2 += z * z;
  }
  z2 = block_sum_d(z2, red);
  const double zn = sqrt(z2);
  const double rho = rho0 * z2;
  // merge the two ascending lists (ties: L first)
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const bool left = t < n1;
    const double dv = a.dl[o + t];
    int lo = left ? n1 : 0, hi = left ? n : n1;   // search the other list
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const double dm = a.dl[o + mid];
      if (left ? (dm < dv) : (dm <= dv)) lo = mid + 1;
      else hi = mid;
    }
    const int pos = left ? t + (lo - n1) : (t - n1) + lo;
    const double z = t < n1 ? a.Q[(o + s - 1) + (size_t)(o + t) * c] : sgn * a.Q[(o + s) + (size_t)(o + t) * c];
    ds[pos] = dv;
    zs[pos] = zn > 0.0 ? z / zn : 0.0;
    perm[pos] = t;
  }
  __syncthreads();
  // deflation scan (sequential, dlaed2)
  if (threadIdx.x == 0) {
    double dmax = 0.0, zmax = 0.0;
    for (int t = 0; t < n; ++t) {
      dmax = fmax(dmax, fabs(ds[t]));
      zmax = fmax(zmax, fabs(zs[t]));
    }
    const double tol = 8.0 * DBL_EPSILON * fmax(dmax, rho * zmax);
    int k = 0, ndef = 0, nrot = 0, pj = -1;
    // deflated entries are written from the back of km (reverse order, fixed below)
    for (int t = 0; t < n; ++t) {
      if (rho * fabs(zs[t]) <= tol) {   // negligible weight
        km[n - 1 - ndef++] = t;
        continue;
      }
      if (pj < 0) {
        pj = t;
        continue;
      }
      double S = zs[pj], C = zs[t];
      const double tz = hypot(C, S);
      C /= tz;
      S = -S / tz;
      const double gap = ds[t] - ds[pj];
      if (fabs(gap * C * S) <= tol) {   // close poles: rotate the weight of pj into t
        zs[t] = tz;
        zs[pj] = 0.0;
        ra[nrot] = pj;
        rb[nrot] = t;
        rc[nrot] = C;
        rs[nrot] = S;
        ++nrot;
        const double tt = ds[pj] * C * C + ds[t] * S * S;
        ds[t] = ds[pj] * S * S + ds[t] * C * C;
        ds[pj] = tt;
        km[n - 1 - ndef++] = pj;
        pj = t;
      } else {
        km[k++] = pj;
        pj = t;
      }
    }
    if (pj >= 0) km[k++] = pj;
    // deflated part in ascending scan order
    for (int x = 0; x < ndef / 2; ++x) {
      const int tmp = km[k + x];
      km[k + x] = km[n - 1 - x];
      km[n - 1 - x] = tmp;
    }
    nrot_s = nrot;
    k_s = k;
    a.kcnt[m] = k;
    a.rho[m] = rho;
  }
  __syncthreads();
  const int k = k_s, nrot = nrot_s;
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
  // gather the columns in sorted order (rows of the merge only), then the rotations row by row
  for (size_t x = threadIdx.x; x < (size_t)n * n; x += blockDim.x) {
    const int r = (int)(x % n), sp = (int)(x / n);
    a.Qp[(o + r) + (size_t)(o + sp) * c] = a.Q[(o + r) + (size_t)(o + perm[sp]) * c];
  }
  __syncthreads();
  if (nrot) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double* row = a.Qp + (o + r);
      for (int x = 0; x < nrot; ++x) {
        double* pa = row + (size_t)(o + ra[x]) * c;
        double* pb = row + (size_t)(o + rb[x]) * c;
        const double qa = *pa, qb = *pb, C = rc[x], S = rs[x];
        *pa = C * qa + S * qb;
        *pb = C * qb - S * qa;
      }
    }
  }
}

// secular equation 1/rho + sum_i z_i^2 / (d_i - lambda) = 0, root t of merge m (one warp):
// lambda_t = d[org] + tau with org the nearer pole, tau solved by bisection to full relative precision
__global__ void dc_secular_kernel(DcArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= a.c) return;
  const int m = gw / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int t = gw - o, k = a.kcnt[m];
  if (t >= k) return;
  const double* dK = a.dK + o;
  const double* zK = a.zK + o;
  const double rho = a.rho[m];
  auto g_at = [&](int orgi, double tau) {   // 1/rho + sum z^2 / ((d_i - d_org) - tau)
    const double dor = dK[orgi];
    double acc = 0.0;
    for (int i = lane; i < k; i += 32) acc += zK[i] * zK[i] / ((dK[i] - dor) - tau);
    return warp_sum_d(acc) + 1.0 / rho;
  };
  int orgi;
  double lo, hi;   // |tau| bracket (lo > 0 tiny, hi), direction by orgi
  bool right;      // tau > 0 (origin on the left)
  if (t == k - 1) {
    orgi = t;
    right = true;
    hi = rho * 1.0000000001 + 4.0 * DBL_EPSILON * fabs(dK[t]);   // ||z|| = 1
  } else {
    const double gap = dK[t + 1] - dK[t];
    const double gm = g_at(t, 0.5 * gap);
    right = gm >= 0.0;
    orgi = right ? t : t + 1;
    hi = 0.5 * gap;
  }
  lo = DBL_TRUE_MIN;
  for (int it = 0; it < 200; ++it) {
    const double mid = hi > 4.0 * lo ? sqrt(lo) * sqrt(hi) : 0.5 * (lo + hi);
    if (!(mid > lo && mid < hi)) break;
    const double g = g_at(orgi, right ? mid : -mid);
    // g increasing in lambda: right (tau = +mid): g < 0 -> larger; left (tau = -mid): g < 0 -> smaller |tau|
    if ((g < 0.0) == right) lo = mid;
    else hi = mid;
    if (hi - lo <= 2.0 * DBL_EPSILON * hi) break;
  }
  if (lane == 0) {
    const double tau = 0.5 * (lo + hi);
    a.org[o + t] = orgi;
    a.org_tau[o + t] = right ? tau : -tau;
  }
}

// lambda_j - d_i from the (origin, tau) representation (accurate for nearby poles)
__device__ __forceinline__ double lam_minus_d(const double* dK, const int* org, const double* tau, int j, int i) {
  return (dK[org[j]] - dK[i]) + tau[j];
}

// Gu-Eisenstat: zhat_i^2 = (lambda_i - d_i)/rho * prod_{j != i} (lambda_j - d_i)/(d_j - d_i); one warp per i
__global__ void dc_zhat_kernel(DcArgs a) {
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
  // product with explicit exponent tracking (no overflow / underflow for any k)
  double mant = 1.0;
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
  if (lane == 0) {
    const double z2 = ldexp(fabs(mant), ex);
    const double zs = a.zK[o + i];
    a.zhat[o + i] = copysign(sqrt(z2), zs);
  }
}

// secular eigenvectors U[:, j] = zhat_i / (d_i - lambda_j), normalised (one warp per j), the merged
// eigenvalues, and (one thread per element) the final ascending rank of all n eigenvalues
__global__ void dc_vec_kernel(DcArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= a.c) return;
  const int m = gw / (2 * a.s);
  int o, n;
  if (!dc_merge(a.c, a.s, m, o, n)) return;
  const int j = gw - o, k = a.kcnt[m];
  const int c = a.c;
  if (j < k) {
    const double* dK = a.dK + o;
    const int* org = a.org + o;
    const double* tau = a.org_tau + o;
    double ss = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double u = a.zhat[o + i] / -lam_minus_d(dK, org, tau, j, i);
      ss += u * u;
    }
    ss = warp_sum_d(ss);
    const double inv = 1.0 / sqrt(ss);
    for (int i = lane; i < k; i += 32)
      a.U[(o + i) + (size_t)(o + j) * c] = a.zhat[o + i] / -lam_minus_d(dK, org, tau, j, i) * inv;
    if (lane == 0) a.lam[o + j] = dK[org[j]] + tau[j];
  }
}

// final ascending position of each merged eigenvalue (ties by (K, deflated) order index)
__global__ void dc_rank_kernel(DcArgs a) {
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

// Q[o:o+n, o+rank(t)] = Qp[o:o+n, o+kmap[u]] U[o+u, o+t] (u < k) for t < k; = Qp[:, o+kmap[t]] for t >= k.
// Tiles of 64 x 64 outputs (rows x (K, deflated)-order columns) within one merge; 256 threads, 4 x 4 each.
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256) dc_gemm_kernel(DcArgs a) {
  const int c = a.c, s = a.s;
  // tile -> (merge, row tile, col tile); merges have n <= 2s, tiles per merge = ceil(n/64)^2
  const int tpm = (2 * s + kGT - 1) / kGT;   // tiles per merge side
  const int tiles_per_merge = tpm * tpm;
  const int m = blockIdx.x / tiles_per_merge, tt = blockIdx.x % tiles_per_merge;
  int o, n;
  if (!dc_merge(c, s, m, o, n)) return;
  const int r0 = (tt % tpm) * kGT, c0 = (tt / tpm) * kGT;
  if (r0 >= n || c0 >= n) return;
  const int k = a.kcnt[m];
  __shared__ double As[kGK][kGT + 1];   // Qp rows x u
  __shared__ double Bs[kGK][kGT + 1];   // u x cols
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  const int kend = min(k, n);
  if (c0 < k) {
    for (int u0 = 0; u0 < kend; u0 += kGK) {
      for (int x = threadIdx.x; x < kGK * kGT; x += 256) {
        const int uu = x / kGT, rr = x % kGT;
        const int u = u0 + uu, row = r0 + rr;
        As[uu][rr] = (u < kend && row < n) ? a.Qp[(o + row) + (size_t)(o + a.kmap[o + u]) * c] : 0.0;
        const int col = c0 + rr;
        Bs[uu][rr] = (u < kend && col < k) ? a.U[(o + u) + (size_t)(o + col) * c] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int uu = 0; uu < kGK; ++uu) {
        double av[4], bv[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) av[p] = As[uu][ty + 16 * p];
#pragma unroll
        for (int p = 0; p < 4; ++p) bv[p] = Bs[uu][tx + 16 * p];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) acc[p][q2] = fma(av[p], bv[q2], acc[p][q2]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    const int t = c0 + tx + 16 * q2;
    if (t >= n) continue;
    const int dst = o + a.rank[o + t];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int row = r0 + ty + 16 * p;
      if (row >= n) continue;
      a.Q[(o + row) + (size_t)dst * c] = t < k ? acc[p][q2] : a.Qp[(o + row) + (size_t)(o + a.kmap[o + t]) * c];
    }
  }
}

// back-transformation of the r wanted eigenvectors (descending eigenvalues): out[:, j] = H_0 ... H_{c-3} Q[:, c-1-j],
// one warp per column, the column in shared memory; kept / dropped / all eigenvalues; non-finite -> *fail = 1
constexpr int kBtWarps = 8;
__global__ void __launch_bounds__(kBtWarps * 32) eig_backtransform_kernel(int c, int r, const double* __restrict__ V,
                                                                         const double* __restrict__ tau,
                                                                         const double* __restrict__ Q,
                                                                         const double* __restrict__ dl, double* Qr,
                                                                         double* kept, double* dropped, double* w_all,
                                                                         int* fail) {
  extern __shared__ __align__(16) double colbuf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * kBtWarps + warp;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < c; i += blockDim.x) {
      if (w_all) w_all[i] = dl[i];
      if (!isfinite(dl[i]) && fail) *fail = 1;
    }
    if (threadIdx.x == 0 && dropped) {
      double s = 0.0;
      for (int i = 0; i < c - r; ++i) s += dl[i];
      *dropped = s;
    }
  }
  if (j >= r) return;
  double* q = colbuf + (size_t)warp * c;
  const int src = c - 1 - j;
  for (int l = lane; l < c; l += 32) q[l] = Q[l + (size_t)src * c];
  __syncwarp();
  for (int h = c - 3; h >= 0; --h) {
    const double th = tau[h];
    if (th == 0.0) continue;
    const double* v = V + (size_t)h * c;
    double acc = 0.0;
    for (int l = h + 1 + lane; l < c; l += 32) acc += __ldg(v + l) * q[l];
    acc = warp_sum_d(acc) * th;
    for (int l = h + 1 + lane; l < c; l += 32) q[l] -= acc * __ldg(v + l);
    __syncwarp();
  }
  for (int l = lane; l < c; l += 32) Qr[l + (size_t)j * c] = q[l];
  if (lane == 0 && kept) kept[j] = dl[src];
}

size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

int trd_smem_max_c(int nc) {
  // L x c doubles of columns + 4 c doubles of v / w buffers + 64 doubles, L = ceil(c / nc)
  int best = 0;
  for (int c = 1; c <= 4096; ++c) {
    const size_t L = (c + nc - 1) / nc;
    const size_t bytes = (L * c + 4 * (size_t)c + 64) * sizeof(double);
    if (bytes <= (size_t)kTrdSmemBytes) best = c;
  }
  return best;
}

// 16-CTA clusters need the non-portable size; fall back to 8 if the device cannot co-schedule 16
int trd_cluster_size() {
  static const int nc = [] {
    cudaFuncSetAttribute(sytrd_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(sytrd_cluster_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrdSmemBytes);
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
    if (cudaOccupancyMaxActiveClusters(&n, sytrd_cluster_kernel<true>, &cfg) != cudaSuccess || n < 1) {
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
  b += align_up(c * 8) * 12;                    // tau, d, e, dl, dK, zK, org_tau, zhat, lam, vglob(2), pglob
  b += align_up(c * 4) * 4;                     // org, kmap, rank, kcnt
  b += align_up(c * 8) + align_up(64 * 8);      // rho, sglob
  b += align_up((c + kTrdCluster) * c * 8);     // global-memory tridiagonalisation slabs (nc x ceil(c/nc) x c)
  return b + 4096;
}

cudaError_t eig_top(int c, int r, const double* G, void* ws, size_t ws_bytes, double* Qr, double* kept,
                    double* dropped, double* w_all, int* fail, cudaStream_t st) {
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
  double* vglob = reinterpret_cast<double*>(take(2 * (size_t)c * 8));
  double* pglob = reinterpret_cast<double*>(take(c * 8));
  int* org = reinterpret_cast<int*>(take(c * 4));
  int* kmap = reinterpret_cast<int*>(take(c * 4));
  int* rank = reinterpret_cast<int*>(take(c * 4));
  int* kcnt = reinterpret_cast<int*>(take(c * 4));
  double* rho = reinterpret_cast<double*>(take(c * 8));
  double* sglob = reinterpret_cast<double*>(take(64 * 8));
  double* Aglob = reinterpret_cast<double*>(take(((size_t)c + kTrdCluster) * c * 8));
  (void)p;
  // ---- 1. tridiagonalisation (one cluster of nc CTAs: 16 where the device can co-schedule it, else 8)
  {
    static const int smem_max_c16 = trd_smem_max_c(16), smem_max_c8 = trd_smem_max_c(8);
    const int nc = trd_cluster_size();
    const size_t L = (c + nc - 1) / nc;
    const bool in_smem = c <= (nc == 16 ? smem_max_c16 : smem_max_c8);
    const size_t smem = in_smem ? (L * c + 4 * (size_t)c + 64) * sizeof(double)
                                : (4 * (size_t)c + 64) * sizeof(double);
    if (smem > (size_t)kTrdSmemBytes) return cudaErrorInvalidValue;
    static PerDeviceOnce once;
    const cudaError_t ce = once_per_device(once, [] {
      cudaError_t r1 = cudaFuncSetAttribute(sytrd_cluster_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kTrdSmemBytes);
      if (r1 == cudaSuccess)
        r1 = cudaFuncSetAttribute(sytrd_cluster_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kTrdSmemBytes);
      if (r1 == cudaSuccess)
        r1 = cudaFuncSetAttribute(sytrd_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (r1 == cudaSuccess)
        r1 = cudaFuncSetAttribute(sytrd_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      return r1;
    });
    if (ce != cudaSuccess) return ce;
    TrdArgs ta{c, G, V, tau, d, e, vglob, pglob, sglob, Aglob};
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
    cudaError_t le = in_smem ? cudaLaunchKernelEx(&cfg, sytrd_cluster_kernel<true>, ta)
                             : cudaLaunchKernelEx(&cfg, sytrd_cluster_kernel<false>, ta);
    ++launch_counter();
    if (le != cudaSuccess) return le;
    le = cudaGetLastError();
    if (le != cudaSuccess) return le;
  }
  // ---- 2. divide and conquer on T
  dc_init_kernel<<<(unsigned)((cc + 255) / 256), 256, 0, st>>>(c, d, e, dl, Q);
  cudaError_t err = note_launch_err();
  if (err != cudaSuccess) return err;
  DcArgs da{c, 1, e, dl, Q, Qp, U, dK, zK, otau, zhat, lam, org, kmap, rank, kcnt, rho};
  static PerDeviceOnce once_prep;
  err = once_per_device(once_prep, [] {
    return cudaFuncSetAttribute(dc_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  if (err != cudaSuccess) return err;
  for (int s = 1; s < c; s *= 2) {
    da.s = s;
    const int nmerge = (c + 2 * s - 1) / (2 * s);
    const size_t nmax = (size_t)std::min(2 * s, c);
    const size_t psmem = nmax * (4 * sizeof(double) + 4 * sizeof(int));
    if (psmem > 200 * 1024) return cudaErrorInvalidValue;
    dc_prep_kernel<<<nmerge, kDcPrepThreads, psmem, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
    const unsigned wblocks = (unsigned)((c * 32 + 255) / 256);
    dc_secular_kernel<<<wblocks, 256, 0, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
    dc_zhat_kernel<<<wblocks, 256, 0, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
    dc_vec_kernel<<<wblocks, 256, 0, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
    dc_rank_kernel<<<(c + 255) / 256, 256, 0, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
    const int tpm = (2 * s + kGT - 1) / kGT;
    dc_gemm_kernel<<<nmerge * tpm * tpm, 256, 0, st>>>(da);
    if ((err = note_launch_err()) != cudaSuccess) return err;
  }
  // ---- 3. back-transformation of the r wanted eigenvectors
  const size_t bsmem = (size_t)kBtWarps * c * sizeof(double);
  static PerDeviceOnce once_bt;
  err = once_per_device(once_bt, [] {
    return cudaFuncSetAttribute(eig_backtransform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  });
  if (err != cudaSuccess) return err;
  if (bsmem > 220 * 1024) return cudaErrorInvalidValue;
  const unsigned bgrid = (unsigned)std::max(1, (r + kBtWarps - 1) / kBtWarps);
  eig_backtransform_kernel<<<bgrid, kBtWarps * 32, bsmem, st>>>(c, r, V, tau, Q, dl, Qr, kept, dropped, w_all, fail);
  return note_launch_err();
}

}  // namespace cakf
