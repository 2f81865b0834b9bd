// internal.h — host launchers of libcakf's device kernels (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace cakf {

// ---- K1: kernel matvec partials  partial[ch][i] = sum_{j in chunk ch} k(xr_i, xc_j) * xc_j.w
// (ch0, ch1): compute only column chunks [ch0, ch1) (multi-GPU shard); ch1 < 0 = all
template <typename T>
cudaError_t launch_matvec_partial(int nu2, const V4<T>* xr, int nrows, const V4<T>* xc, int ncols,
                                  int nchunks, T* partial, cudaStream_t st, int ch0 = 0, int ch1 = -1);
// choose the number of column chunks for a matvec of this shape (fills the GPU in whole waves)
int matvec_chunks(int nrows, int ncols, int elem_bytes);
// symmetric K1 (fp32, one RHS with rows == cols): partial[c][i] for c < matvec_sym_tiles(n)
int matvec_sym_tiles(int n);
long long matvec_sym_units(int n);   // number of symmetric tile-block work units
int matvec_sym_block_points();       // points per tile block of the symmetric K1
// ulist != nullptr (exact-zero culling): evaluate only the *ucount units ulist[w] (ascending), and in each
// only the tile pairs set in umask[w] (bit a*4+b), and in those only the warps whose 16-row group sphere
// (sph16) is within cut of the J tile sphere (sph128); the skipped units' partial slots must hold zeros.
// done_pairs (nullable) accumulates the evaluated 128 x 128 tile pairs.
// With the 32-column sub-tile test (default; CAKF_K1_SUB=0 for the 128-column one) the warp test uses
// sph32 (32-point spheres of the observations) and done_pairs counts 16 x 32 blocks; box16 / box32
// (nullable, launch_tile_spheres' boxes of the same tiles) add the bounding-box distance test.
cudaError_t launch_matvec_sym(int nu2, const float4* x, int n, float* partial, long long u_begin, long long u_end,
                              cudaStream_t st, unsigned long long* done_pairs = nullptr, const int* ulist = nullptr,
                              const int* ucount = nullptr, const unsigned short* umask = nullptr,
                              const float4* sph16 = nullptr, const float4* sph128 = nullptr,
                              const float4* sph32 = nullptr, float cut = 0.f, unsigned* sched = nullptr,
                              const float4* box16 = nullptr, const float4* box32 = nullptr);
// sched (nullable, 2 zero-initialised counters, one per handle): dynamic unit scheduling (CAKF_K1_DYN=0: off)
int matvec_sym_blocks_per_tile_pair();   // warp blocks per 128 x 128 tile pair counted by done_pairs
// list (+ tile-pair masks) of the sym units in [u_lo, u_hi) with a tile pair within `cut`, grouped by their
// active-pair count (most first); count: a device workspace of >= 64 ints, count[0] = the list length.
// urange (nullable, device): read [u_lo, u_hi) from it instead (the balanced multi-GPU split below)
// per 512-row block of the symmetric K1: the active partner blocks (step.h SlotList; sph == nullptr: all)
cudaError_t launch_k1_block_partners(const float4* sph, int n, float cut, int* plist, int* pq, cudaStream_t st);
int matvec_sym_blocks(int n);   // 512-point blocks of the symmetric K1
cudaError_t launch_k1_active_units(const float4* sph, int n, long long u_lo, long long u_hi, float cut, int* list,
                                   unsigned short* mask, int* count, cudaStream_t st, const long long* urange = nullptr);
// multi-GPU: the unit range of `rank` with an equal share of the active tile pairs (deterministic) -> urange[2]
cudaError_t launch_k1_balanced_range(const float4* sph, int n, float cut, int rank, int world, long long* urange,
                                     cudaStream_t st);
// bounding spheres (x, y, z, radius) of consecutive tiles of `tile` points
// box (nullable): per tile {lo, hi} axis-aligned bounding box, 2 float4 per tile
cudaError_t launch_tile_spheres(const float4* x, int n, int tile, float4* out, cudaStream_t st, float4* box = nullptr);
// fp32 exact-zero cut: a prescaled distance above which ex2.approx.ftz(-a log2 e) flushes to 0
constexpr float kCullCut = 88.0f;
bool use_sym_k1();  // false if CAKF_K1_DENSE=1
// reduce partials: y[i] = alpha * sum_ch partial[ch][i]
template <typename T>
cudaError_t launch_sum_partials(int nrows, int nchunks, const T* partial, double alpha, T* y, cudaStream_t st);

// ---- K2: kernel x matrix  Y[i, c] = alpha * sum_j k(xr_i, xc_j) B[j, c]  (column-major)
template <typename T>
cudaError_t launch_gram_gemm(int nu2, const V4<T>* xr, int M, const V4<T>* xc, int K, const T* B, size_t ldb,
                             int C, T* Y, size_t ldy, double alpha, cudaStream_t st);

// ---- K2 on tcgen05 tensor cores (fp32 via 3xTF32): workspace = gram_gemm_tc_workspace(K, C) bytes
size_t gram_gemm_tc_workspace(int K, int C);
// act_cnt / act_list (nullable): per 128-row output tile, the ascending list of 32-column K-blocks that
// are not entirely exactly-zero (exact-zero culling); act_stride = list stride per tile
cudaError_t launch_gram_gemm_tc(int nu2, const float4* xr, int M, const float4* xc, int K, const float* B, size_t ldb,
                                int C, float* Y, size_t ldy, double alpha, float* work, cudaStream_t st,
                                const int* act_cnt = nullptr, const int* act_list = nullptr, int act_stride = 0);
// build the active K-block lists from M-tile (128) and K-block (32) spheres
// (*total += number of active K-blocks, for the cull statistics)
cudaError_t launch_k2_active(const float4* sphM, int nmt, const float4* sphK, int nkb, float cut, int* act_cnt,
                             int* act_list, int act_stride, unsigned long long* total, cudaStream_t st);
// true unless CAKF_K2_SIMT=1 is set in the environment
bool use_tc_k2();

// ---- coordinates
template <typename T>
cudaError_t launch_prescale_coords(int n, int dim, const double* xyz, double scale, V4<T>* out, cudaStream_t st);

// ---- low-rank contractions on tcgen05 (kernels_gemm_tc.cu): fp32 operands as exact bf16x3 planes
int gemm_tc_kp(int K);                              // padded K of the planes (multiple of 8)
size_t gemm_tc_plane_bytes(int rows, int K);        // bytes of the three planes of a rows x K operand
// planes[3][R][Kp] of the R x K operand whose (r, k) element is src[k + r ld] (k_contig) or src[r + k ld]
cudaError_t gemm_tc_split(const float* src, int R, int K, size_t ld, bool k_contig, uint16_t* planes,
                          cudaStream_t st);
// C (M x N, column-major ldc) = alpha A B^T-of-planes + beta C, i.e. sum_k Ap[m][k] Bp[n][k];
// output fp32 C or fp64 Cd (exactly one non-null); K splits reduced in fp64 through work (floats)
cudaError_t gemm_tc_run(const uint16_t* Ap, int M, const uint16_t* Bp, int N, int K, double alpha, double beta,
                        float* C, double* Cd, size_t ldc, float* work, size_t work_floats, cudaStream_t st);
bool use_tc_gemm();   // CAKF_GEMM_F64=1: fp32 contractions through fp64 DGEMM instead
bool use_k2_stack();   // CAKF_K2_STACK=0: six 3xBF16 MMAs per k-step in K2 instead of three stacked ones
bool use_i8_pair();   // CAKF_I8_PAIR=1: CTA-pair A multicast in the stacked INT8 GEMM (A/B only; off)
bool use_i8_stack();   // CAKF_I8_STACK=0: one MMA per slice pair, single accumulator buffer (A/B only)
bool use_i8_split_fused();   // CAKF_I8_SPLIT_FUSED=0: the two-pass exponent + slice kernels (A/B only)
bool use_split_rc8();   // CAKF_SPLIT_RC8=0: the 2-byte-store bf16x3 transpose-split (A/B only)
bool use_tc_persist();   // CAKF_TC_PERSIST=0: un-split 3xBF16 GEMMs on the one-tile-per-CTA kernel (A/B only)
constexpr size_t kGemmWorkFloats = (size_t)32 << 20;

// ---- fp64-accurate contractions of fp32 factors on the INT8 tensor cores (kernels_gemm_i8.cu, Ozaki
// splitting into 7-bit slices with per-(row, K chunk) power-of-two scales; exact int32 accumulation)
int gemm_i8_kp(int K);                              // padded K of the planes (multiple of 16)
int gemm_i8_nchunk(int K);                          // K chunks (one exponent per row and chunk)
size_t gemm_i8_plane_bytes(int rows, int K);        // bytes of the slice planes of a rows x K operand
// planes[S][R][Kp] + exponents ex[R][nchunk] of the R x K operand (r, k) = src[k + r ld] (k_contig) or src[r + k ld]
template <typename Src>
cudaError_t gemm_i8_split(const Src* src, int R, int K, size_t ld, bool k_contig, int8_t* planes, int* ex,
                          cudaStream_t st);
// C (M x N, column-major ldc) = alpha sum_k A(m, k) B(n, k) + beta C from the planes of both operands;
// output fp32 C or fp64 Cd (exactly one non-null); lower: only n <= m is required (symmetric Gram);
// K splits accumulate in fp64 through work (doubles), reduced in a fixed order
cudaError_t gemm_i8_run(const int8_t* Ap, const int* expA, int M, const int8_t* Bp, const int* expB, int N, int K,
                        double alpha, double beta, float* C, double* Cd, size_t ldc, bool lower, double* work,
                        size_t work_doubles, cudaStream_t st);
bool use_i8_gemm();   // CAKF_GEMM_F64=1: fp32 contractions through fp64 DGEMM instead

// ---- low-rank contractions with fp64 accumulation on the FP64 pipe (kernels_gemm_f64.cu):
// C = alpha op(A) op(B) + beta C, column-major, op = transpose when trans*; fp32/fp64 operands converted on
// load, fp64 products and sums, one rounding into C; long K split into fixed slices reduced in order through
// work (doubles; the split shrinks to fit work_doubles)
template <typename TA, typename TB, typename TC>
cudaError_t gemm_f64acc(bool transa, bool transb, int m, int n, int k, double alpha, const TA* A, size_t lda,
                        const TB* B, size_t ldb, double beta, TC* C, size_t ldc, double* work, size_t work_doubles,
                        cudaStream_t st);
// y += a x
template <typename T>
cudaError_t axpy(size_t n, double a, const T* x, T* y, cudaStream_t st);

// ---- the truncation's symmetric eigensolver (kernels_eig.cu): cluster Householder tridiagonalisation,
// divide and conquer, back-transformation of the r wanted eigenvectors.  G: c x c fp64, lower triangle
// (ld c).  Qr: c x r eigenvectors of the r largest eigenvalues, descending; kept (r, nullable) those
// eigenvalues; dropped (nullable) the sum of the c - r smallest; w_all (c, nullable) all eigenvalues
// ascending; fail (nullable device int) set to 1 on a non-finite eigenvalue.
size_t eig_workspace_bytes(int cmax);
// side / ev_a / ev_b (nullable): a stream and two events for the T factors beside the divide and conquer
cudaError_t eig_top(int c, int r, const double* G, void* ws, size_t ws_bytes, double* Qr, double* kept,
                    double* dropped, double* w_all, int* fail, cudaStream_t st, cudaStream_t side = nullptr,
                    cudaEvent_t ev_a = nullptr, cudaEvent_t ev_b = nullptr);

// ---- per-update kd-tree order of the observed points (kd_order.cu)
size_t kd_obs_workspace(int Nmax);
// idx/sig_in_sorted: the observations in internal point order (obs_sort); writes idx_out, sig_out
// (user position of each row) and sig_inv in the kd order.  run (nullable device flag): every kernel
// returns at once when *run == 0.  Sync-free, no library sort.
template <typename T>
cudaError_t kd_obs_order(int N, const int* idx, const V4<T>* coords, int* sig_out, int* sig_inv, int* idx_out,
                         const int* sig_in_sorted, void* ws, size_t ws_bytes, cudaStream_t st,
                         const int* run = nullptr);

// columns k(X, x_{order[i0-1+c]}), c < nb, of the kernel matrix (coordinate actions)
template <typename T>
cudaError_t launch_kernel_columns(int nu2, const V4<T>* x, int N, const int* order, int i0, int nb, T* out, size_t ldo,
                                  cudaStream_t st);

}  // namespace cakf
