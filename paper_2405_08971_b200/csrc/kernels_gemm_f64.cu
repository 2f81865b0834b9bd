// kernels_gemm_f64.cu — the low-rank contractions with fp64 accumulation on the FP64 pipe, for the
// products the INT8-slice tensor-core GEMM does not take (short K, and every product of the fp64
// parity mode): a7's M^- U and (HM^-)^T [v V] at small rank, a9's B_k t, V t and (K(X,T) V) t
// (alg:mfks P:388-409, K = N^ = 64), and all of them (plus the truncation Gram) in fp64 mode.
//
//   C = alpha op(A) op(B) + beta C,  column-major, op(X) = X or X^T,
//   A, B fp32 or fp64 (converted to fp64 on load), C fp32 or fp64, products and sums in fp64.
//
// 64 x 64 output tiles per CTA (4 warps of 32 x 32 on the FP64 tensor cores, mma.sync m8n8k4 DMMA), K chunks
// of 16 staged through shared memory (converted to fp64 on load) with a register prefetch of the next chunk.  Long reductions (K >> m, n: M^T x, the Gram) are
// split over K into fixed slices whose fp64 partials are summed in slice order by a second kernel, so
// results are bit-reproducible.  The fp32 epilogue rounds once: C = (float)(alpha acc + beta C).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace cakf {

namespace {

constexpr int kFT = 64, kFK = 16, kFThreads = 128;   // 64 x 64 tile, 4 warps of 32 x 32, K chunks of 16

// D (8x8, fp64) += A (8x4) B (4x8) on the tensor cores (DMMA): a = A[g][t], b = B[t][g], d = D[g][2t .. 2t+1]
// with g = lane / 4, t = lane % 4
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename TA, typename TB, typename TC, bool TRA, bool TRB>
__global__ void __launch_bounds__(kFThreads) gemm_f64acc_kernel(int m, int n, int k, int kslice, double alpha,
                                                                 const TA* __restrict__ A, size_t lda,
                                                                 const TB* __restrict__ B, size_t ldb, double beta,
                                                                 TC* __restrict__ C, size_t ldc,
                                                                 double* __restrict__ part) {
  __shared__ double As[kFK][kFT + 1];   // [k][row]
  __shared__ double Bs[kFK][kFT + 1];   // [k][col]
  const int i0 = blockIdx.x * kFT, j0 = blockIdx.y * kFT, z = blockIdx.z;
  const int k0 = z * kslice, k1 = min(k, k0 + kslice);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2] = {};
  constexpr int kPer = kFT * kFK / kFThreads;   // 8 elements of each operand per thread and chunk
  double ra[kPer], rb[kPer];
  // element x of a chunk: the contiguous dimension of the operand fastest across threads
  auto fetch = [&](int kk) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int x = threadIdx.x + e * kFThreads;   // 0 .. 1023 = 64 x 16
      int r, l;
      if (TRA) { l = x % kFK; r = x / kFK; }       // op(A)(r, l) = A[l + r lda]: k contiguous
      else { r = x % kFT; l = x / kFT; }           // op(A)(r, l) = A[r + l lda]: rows contiguous
      const int gi = i0 + r, gl = kk + l;
      ra[e] = (gi < m && gl < k1) ? (double)(TRA ? A[gl + (size_t)gi * lda] : A[gi + (size_t)gl * lda]) : 0.0;
      int cc, lb;
      if (TRB) { cc = x % kFT; lb = x / kFT; }     // op(B)(l, c) = B[c + l ldb]: cols contiguous
      else { lb = x % kFK; cc = x / kFK; }         // op(B)(l, c) = B[l + c ldb]: k contiguous
      const int gj = j0 + cc, glb = kk + lb;
      rb[e] = (gj < n && glb < k1) ? (double)(TRB ? B[gj + (size_t)glb * ldb] : B[glb + (size_t)gj * ldb]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int x = threadIdx.x + e * kFThreads;
      if (TRA) As[x % kFK][x / kFK] = ra[e];
      else As[x / kFT][x % kFT] = ra[e];
      if (TRB) Bs[x / kFT][x % kFT] = rb[e];
      else Bs[x % kFK][x / kFK] = rb[e];
    }
  };
  if (k0 < k1) fetch(k0);
  for (int kk = k0; kk < k1; kk += kFK) {
    __syncthreads();
    store();
    __syncthreads();
    if (kk + kFK < k1) fetch(kk + kFK);
#pragma unroll
    for (int ks = 0; ks < kFK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[ks + t][wm + 8 * mi + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[ks + t][wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = i0 + wm + 8 * mi + g;
    if (i >= m) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + wn + 8 * ni + 2 * t + h;
        if (j >= n) continue;
        const double v = acc[mi][ni][h];
        if (part) {
          part[((size_t)z * n + j) * m + i] = v;
        } else {
          TC* c = C + i + (size_t)j * ldc;
          *c = (TC)(beta != 0.0 ? alpha * v + beta * (double)*c : alpha * v);
        }
      }
    }
  }
}

// Short-K row-strip variant (op(A) = A, op(B) = B, K <= kStripK): a CTA keeps its 64-row strip of A in shared
// memory (fp64) for the whole product and walks the 64-column tiles of C; the next B tile and the current
// C tile (beta != 0) are fetched into registers while the tensor cores work on the current tile.  Used for
// the alg:mfks K = N^ products (B_k t, V t, (K(X,T)V) t) whose tall, thin shape leaves the tiled kernel
// latency-bound.
constexpr int kStripK = 64;
template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(kFThreads) gemm_f64acc_strip_kernel(int m, int n, int k, double alpha,
                                                                       const TA* __restrict__ A, size_t lda,
                                                                       const TB* __restrict__ B, size_t ldb,
                                                                       double beta, TC* __restrict__ C, size_t ldc) {
  extern __shared__ __align__(16) double strip_smem[];
  double(*As)[kFT + 1] = reinterpret_cast<double(*)[kFT + 1]>(strip_smem);                     // [k][row]
  double(*Bs)[kFT + 1] = reinterpret_cast<double(*)[kFT + 1]>(strip_smem + kStripK * (kFT + 1));  // [k][col]
  const int i0 = blockIdx.x * kFT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int kp = (k + 3) & ~3;   // k rounded to the MMA depth (zero padded)
  for (int x = threadIdx.x; x < kStripK * kFT; x += kFThreads) {
    const int r = x % kFT, l = x / kFT;
    As[l][r] = (l < k && i0 + r < m) ? (double)A[(i0 + r) + (size_t)l * lda] : 0.0;
  }
  constexpr int kPerB = kStripK * kFT / kFThreads;   // 32
  double rb[kPerB];
  auto fetchB = [&](int j0) {
#pragma unroll
    for (int e = 0; e < kPerB; ++e) {
      const int x = threadIdx.x + e * kFThreads;
      const int l = x % kStripK, cc = x / kStripK;
      rb[e] = (l < k && j0 + cc < n) ? (double)B[l + (size_t)(j0 + cc) * ldb] : 0.0;
    }
  };
  fetchB(0);
  for (int j0 = 0; j0 < n; j0 += kFT) {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kPerB; ++e) {
      const int x = threadIdx.x + e * kFThreads;
      Bs[x % kStripK][x / kStripK] = rb[e];
    }
    __syncthreads();
    // C of this tile in flight during the MMAs
    float cpre[4][4][2];
    if (beta != 0.0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = i0 + wm + 8 * mi + g, j = j0 + wn + 8 * ni + 2 * t + h;
            cpre[mi][ni][h] = (i < m && j < n) ? (float)C[i + (size_t)j * ldc] : 0.f;
          }
    }
    if (j0 + kFT < n) fetchB(j0 + kFT);
    double acc[4][4][2] = {};
    for (int ks = 0; ks < kp; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[ks + t][wm + 8 * mi + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[ks + t][wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = i0 + wm + 8 * mi + g;
      if (i >= m) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = j0 + wn + 8 * ni + 2 * t + h;
          if (j >= n) continue;
          const double v = acc[mi][ni][h];
          C[i + (size_t)j * ldc] = (TC)(beta != 0.0 ? alpha * v + beta * (double)cpre[mi][ni][h] : alpha * v);
        }
    }
  }
}

// Row-strip variant for fp32 B and C (the fp32 path's K = N^ products): 8 warps (2 x 4 of 32 x 16) per
// 64 x 64 C tile, the A strip converted to fp64 once per CTA, the B tile and the old C tile of the NEXT
// column tile streamed into shared memory with cp.async (fp32, double-buffered) while the DMMAs of the
// current one run — no register prefetch, ~100 registers, two CTAs (16 warps) per SM.
constexpr int kS2Threads = 256, kS2Pad = 68;   // fp32 row stride of the staged B / C tiles (16-byte rows)
constexpr size_t kS2Smem = (size_t)kStripK * (kFT + 1) * sizeof(double) + 4 * (size_t)kFT * kS2Pad * sizeof(float);
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
template <typename TA>
__global__ void __launch_bounds__(kS2Threads, 2) gemm_f64acc_strip2_kernel(int m, int n, int k, double alpha,
                                                                             const TA* __restrict__ A, size_t lda,
                                                                             const float* __restrict__ B, size_t ldb,
                                                                             double beta, float* __restrict__ C,
                                                                             size_t ldc) {
  extern __shared__ __align__(16) double s2_smem[];
  double(*As)[kFT + 1] = reinterpret_cast<double(*)[kFT + 1]>(s2_smem);   // [k][row]
  float* Bsf = reinterpret_cast<float*>(s2_smem + kStripK * (kFT + 1));   // [2][col][k]
  float* Csf = Bsf + 2 * kFT * kS2Pad;                                     // [2][col][row]
  const int i0 = blockIdx.x * kFT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int kp = (k + 3) & ~3;
  const bool readc = beta != 0.0;
  // stage column tile j0 (B: 64 columns x k, C: 64 columns x 64 rows) into buffer b; 16-byte chunks, zero fill
  auto stage = [&](int j0, int b) {
    for (int x = threadIdx.x; x < kFT * 16; x += kS2Threads) {
      const int cc = x >> 4, l0 = (x & 15) * 4, col = j0 + cc;
      const int nb = (col < n && l0 < k) ? 4 * min(4, k - l0) : 0;
      const float* src = B + (nb ? (size_t)col * ldb + l0 : 0);
      cp_async16_zfill((uint32_t)__cvta_generic_to_shared(Bsf + (size_t)b * kFT * kS2Pad + cc * kS2Pad + l0), src, nb);
      if (readc) {
        const int nc = (col < n && i0 + l0 < m) ? 4 * min(4, m - i0 - l0) : 0;
        const float* srcc = C + (nc ? (size_t)col * ldc + i0 + l0 : 0);
        cp_async16_zfill((uint32_t)__cvta_generic_to_shared(Csf + (size_t)b * kFT * kS2Pad + cc * kS2Pad + l0), srcc,
                         nc);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0, 0);
  for (int x = threadIdx.x; x < kStripK * kFT; x += kS2Threads) {
    const int r = x % kFT, l = x / kFT;
    As[l][r] = (l < k && i0 + r < m) ? (double)A[(i0 + r) + (size_t)l * lda] : 0.0;
  }
  const int ntl = (n + kFT - 1) / kFT;
  for (int jt = 0; jt < ntl; ++jt) {
    const int j0 = jt * kFT, b = jt & 1;
    if (jt + 1 < ntl) {
      stage(j0 + kFT, b ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* Bt = Bsf + (size_t)b * kFT * kS2Pad;
    double acc[4][2][2] = {};
    for (int ks = 0; ks < kp; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[ks + t][wm + 8 * mi + g];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = (double)Bt[(wn + 8 * ni + g) * kS2Pad + ks + t];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    const float* Ct = Csf + (size_t)b * kFT * kS2Pad;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int rl = wm + 8 * mi + g, i = i0 + rl;
      if (i >= m) continue;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cl = wn + 8 * ni + 2 * t + h, j = j0 + cl;
          if (j >= n) continue;
          const double v = acc[mi][ni][h];
          C[i + (size_t)j * ldc] = (float)(readc ? alpha * v + beta * (double)Ct[cl * kS2Pad + rl] : alpha * v);
        }
    }
    __syncthreads();   // buffer b is restaged at tile jt + 2
  }
}

template <typename TC>
__global__ void gemm_f64acc_reduce_kernel(int m, int n, int S, const double* __restrict__ part, double alpha,
                                          double beta, TC* __restrict__ C, size_t ldc) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)m * n) return;
  const int i = (int)(e % m), j = (int)(e / m);
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += part[((size_t)z * n + j) * m + i];
  TC* c = C + i + (size_t)j * ldc;
  *c = (TC)(beta != 0.0 ? alpha * s + beta * (double)*c : alpha * s);
}

template <typename TA, typename TB, typename TC, bool TRA, bool TRB>
cudaError_t launch_t(int m, int n, int k, double alpha, const TA* A, size_t lda, const TB* B, size_t ldb, double beta,
                     TC* C, size_t ldc, double* work, size_t work_doubles, cudaStream_t st) {
  const int mt = (m + kFT - 1) / kFT, nt = (n + kFT - 1) / kFT;
  // split K while the tiles do not fill two waves and each slice keeps >= 8 chunks
  int S = 1;
  if (k > 0) {
    const int tiles = mt * nt;
    const int want = (2 * num_sms() + tiles - 1) / tiles;
    S = std::max(1, std::min(want, k / (8 * kFK)));
    while (S > 1 && (size_t)S * m * n > work_doubles) --S;
  }
  const int kslice = S > 1 ? ((k + S - 1) / S + kFK - 1) / kFK * kFK : std::max(k, 1);
  S = k > 0 ? (k + kslice - 1) / kslice : 1;
  const bool split = S > 1;
  dim3 grid(mt, nt, S);
  gemm_f64acc_kernel<TA, TB, TC, TRA, TRB><<<grid, kFThreads, 0, st>>>(m, n, k, kslice, alpha, A, lda, B, ldb, beta,
                                                                      C, ldc, split ? work : nullptr);
  cudaError_t e = note_launch_err();
  if (e != cudaSuccess || !split) return e;
  const size_t tot = (size_t)m * n;
  gemm_f64acc_reduce_kernel<TC><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(m, n, S, work, alpha, beta, C, ldc);
  return note_launch_err();
}

}  // namespace

bool use_strip2() {
  static const bool v = !env_is("CAKF_STRIP2", '0');
  return v;
}

template <typename TA, typename TB, typename TC>
cudaError_t gemm_f64acc(bool transa, bool transb, int m, int n, int k, double alpha, const TA* A, size_t lda,
                        const TB* B, size_t ldb, double beta, TC* C, size_t ldc, double* work, size_t work_doubles,
                        cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if constexpr (sizeof(TB) == 4 && sizeof(TC) == 4) {
    auto al16 = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    if (!transa && !transb && k > 0 && k <= kStripK && m >= 8 * kFT && ldb % 4 == 0 && ldc % 4 == 0 && al16(B) &&
        al16(C) && use_strip2()) {
      static PerDeviceOnce once2;
      const cudaError_t ce = once_per_device(once2, [] {
        return cudaFuncSetAttribute(gemm_f64acc_strip2_kernel<TA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kS2Smem);
      });
      if (ce != cudaSuccess) return ce;
      gemm_f64acc_strip2_kernel<TA><<<(m + kFT - 1) / kFT, kS2Threads, kS2Smem, st>>>(
          m, n, k, alpha, A, lda, reinterpret_cast<const float*>(B), ldb, beta, reinterpret_cast<float*>(C), ldc);
      return note_launch_err();
    }
  }
  if (!transa && !transb && k > 0 && k <= kStripK && sizeof(TC) == 4 && m >= 8 * kFT) {
    constexpr size_t smem = 2 * kStripK * (kFT + 1) * sizeof(double);
    static PerDeviceOnce once;
    const cudaError_t ce = once_per_device(once, [] {
      return cudaFuncSetAttribute(gemm_f64acc_strip_kernel<TA, TB, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem);
    });
    if (ce != cudaSuccess) return ce;
    gemm_f64acc_strip_kernel<TA, TB, TC><<<(m + kFT - 1) / kFT, kFThreads, smem, st>>>(m, n, k, alpha, A, lda, B, ldb,
                                                                                     beta, C, ldc);
    return note_launch_err();
  }
  if (transa) {
    if (transb) return launch_t<TA, TB, TC, true, true>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, work_doubles, st);
    return launch_t<TA, TB, TC, true, false>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, work_doubles, st);
  }
  if (transb) return launch_t<TA, TB, TC, false, true>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, work_doubles, st);
  return launch_t<TA, TB, TC, false, false>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, work_doubles, st);
}

template cudaError_t gemm_f64acc<float, float, float>(bool, bool, int, int, int, double, const float*, size_t,
                                                      const float*, size_t, double, float*, size_t, double*, size_t,
                                                      cudaStream_t);
template cudaError_t gemm_f64acc<float, double, float>(bool, bool, int, int, int, double, const float*, size_t,
                                                       const double*, size_t, double, float*, size_t, double*, size_t,
                                                       cudaStream_t);
template cudaError_t gemm_f64acc<float, float, double>(bool, bool, int, int, int, double, const float*, size_t,
                                                       const float*, size_t, double, double*, size_t, double*, size_t,
                                                       cudaStream_t);
template cudaError_t gemm_f64acc<double, double, double>(bool, bool, int, int, int, double, const double*, size_t,
                                                         const double*, size_t, double, double*, size_t, double*,
                                                         size_t, cudaStream_t);

// ---- small vector helpers replacing the BLAS level-1 calls: y += a x
template <typename T>
__global__ void axpy_kernel(size_t n, double a, const T* __restrict__ x, T* __restrict__ y) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = (T)((double)y[i] + a * (double)x[i]);
}
template <typename T>
cudaError_t axpy(size_t n, double a, const T* x, T* y, cudaStream_t st) {
  if (!n) return cudaSuccess;
  axpy_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, a, x, y);
  return note_launch_err();
}
template cudaError_t axpy<float>(size_t, double, const float*, float*, cudaStream_t);
template cudaError_t axpy<double>(size_t, double, const double*, double*, cudaStream_t);

}  // namespace cakf
