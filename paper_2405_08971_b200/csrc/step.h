// step.h — launchers of the per-step streaming kernels (kernels_step.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace cakf {

struct Mat3 {
  double a[3][3];
};

// Device-resident control block of one update's inner loop.
struct IterCtl {
  double alpha, eta, gamma, inv_sqrt_eta;
  double eta_min, res0_sq, res_sq, dropped;
  int n_acc, rejected, nonfinite, pad;
};

int stage_blocks(int N);   // blocks (128-row tiles) of the stage kernels
cudaError_t idx64_to32(int n, const int64_t* in, int* out, cudaStream_t st);
// observations -> internal point order: idx_out ascending, sigma[j] = user position, sigma_inv inverse.
// run (nullable device flag): the kernels return at once when *run == 0
cudaError_t obs_sort(int N, int NX, const int64_t* obs, const int* invperm, int* posof, int* counts, int* idx_out,
                     int* sigma, int* sigma_inv, cudaStream_t st, const int* run = nullptr);
// *neq = (a[0:n] != b[0:n]) (device buffers)
cudaError_t obs_neq(int n, const int64_t* a, const int64_t* b, int* neq, cudaStream_t st);
template <typename T>
cudaError_t gather_vec(int N, const int* sigma, const T* in, T* out, cudaStream_t st);
// out[sigma[j]] = in[j]  (internal observation order -> user order)
template <typename T>
cudaError_t scatter_vec(int N, const int* sigma, const T* in, T* out, cudaStream_t st);
// xc[j].w = w[j]
template <typename T>
cudaError_t set_w(int N, const T* w, V4<T>* xc, cudaStream_t st);
cudaError_t map_order(int n, const int64_t* order_user, const int* sigma_inv, int* order_out, cudaStream_t st);
template <typename T>
cudaError_t unpermute(int NX, int Dp, const int* perm, const T* in, T* out, cudaStream_t st);
template <typename S, typename D_>
cudaError_t convert(int rows, int cols, const S* src, size_t lds, D_* dst, size_t ldd, cudaStream_t st);
// C = (float)(beta C + Cd) (fp64 GEMM result accumulated into fp32 C)
cudaError_t accum_d2f(int rows, int cols, double beta, const double* Cd, size_t ldcd, float* C, size_t ldc,
                      cudaStream_t st);

// The symmetric K1's partial slots that can hold nonzeros for each 512-row block B: plist[B * nb + k], k <
// pq[B * 5 + 4], the active partner blocks of B in ascending order; pq[B * 5 + w] = the first entry with partner
// >= w * nb / 4 (the stage kernels' warp w sums the partners of quarter w in ascending order, so the sums do not
// depend on which slots were skipped).  plist == nullptr: sum all nch slots.
struct SlotList {
  const int* plist = nullptr;
  const int* pq = nullptr;
  int nb = 0;
};

template <typename T>
struct StepKernels {
  static cudaError_t prep(int N, const int* idx, const V4<T>* coords, const T* y, const T* mpred, int policy,
                          const int* order, uint64_t seed, int k, const int* sigma, T* r, T* s, T* v, V4<T>* xcs,
                          cudaStream_t st, int nblk_pol = 1, T* rbs = nullptr);   // BLOCKRES: block size, r^(i0)
  static cudaError_t stageA(int N, int nch, const T* partial, double sig00, const T* lam2, const T* s, const T* r,
                            T* gp, const T* HM, int rin, double* part, int W, double* red, unsigned* cnt,
                            cudaStream_t st, SlotList sl = {});
  static cudaError_t gen_actions(int N, int i0, int nb, int policy, const int* order, uint64_t seed, int k,
                                 const int* sigma, T* S, size_t ldS, cudaStream_t st, const T* rbs = nullptr,
                                 int nblk_pol = 1);
  // HM == nullptr in stageA: u = HM^T s is computed by hmts (side stream) into red[0, rin)
  static cudaError_t hmts(int N, const T* HM, int rin, const T* s, double* part, int W, double* red, unsigned* cnt,
                          cudaStream_t st);
  // w = HM u (fp64) from the reduced u = red[0, rin) (side stream, after hmts)
  static cudaError_t hmu(int N, const T* HM, int rin, const double* ured, double* w, cudaStream_t st);
  // stage A + B in one pass (u, HM u from the side stream in wpre, or r_in = 0 with wpre = nullptr):
  // g = G s; red = [V^T g | s^T g | s^T r, s^T g', r^T r], the last three also to ared_tail
  static cudaError_t stageAB(int N, int nch, const T* partial, double sig00, const T* lam2, const T* s, const T* r,
                             const double* wpre, T* g, const T* V, int nV, double* part, int W, double* red,
                             double* ared_tail, unsigned* cnt, cudaStream_t st, SlotList sl = {});
  static cudaError_t stageB(int N, const T* HM, int rin, const double* ured, const T* gp, const T* s, T* g, const T* V,
                            int nV, double* part, int W, double* red, unsigned* cnt, cudaStream_t st,
                            const double* wpre = nullptr);
  static cudaError_t stageC(int N, const T* V, const T* Z, int nV, const double* cred, const T* sin, const T* gin,
                            T* d, T* Gd, const T* s_eta, const double* ared, int rin, const double* sgs, double* part,
                            int W, double* red, unsigned* cnt, IterCtl* ctl, double eps, int iter, int pass,
                            cudaStream_t st);
  static cudaError_t stageD(int N, int iter, int niter, const IterCtl* ctl, const T* d, const T* Gd, T* XV, T* Z, T* r,
                            T* s, V4<T>* xcs, int policy, const int* order, uint64_t seed, int k, const int* sigma,
                            cudaStream_t st, int nblk_pol = 1, T* rbs = nullptr);
  static cudaError_t dot(int N, const T* a, const T* b, double* part, double* out, unsigned* cnt, cudaStream_t st);
  // rows of the points a rank owns (lo <= idx < lo + nl; M = local rows), zeros for the others
  static cudaError_t gather_rows(int N, int C, const int* idx, const T* M, size_t ldm, T* out, size_t ldo, int lo, int nl,
                                 cudaStream_t st);
  static cudaError_t mix(int NX, int Dp, int C, const Mat3& A, bool transpose, const T* in, size_t ldi, T* out,
                         size_t ldo, cudaStream_t st);
  static cudaError_t post_combine(int NX, int Dp, int C, const Mat3& S, const T* Y, const T* tmp, const T* mpred, T* m,
                                  T* Mk, int rin, cudaStream_t st);
  static cudaError_t rowvar(int NX, int Dp, const Mat3& S, const T* base, const T* M, size_t ld, int cols, T* var,
                            cudaStream_t st);
  static cudaError_t gram(size_t D, int c, const T* M, size_t ld, double* part, int nsplit, double* G, cudaStream_t st);
  static cudaError_t take_top(int c, int r, const double* evec, const double* w, T* Qr, double* kept, double* dropped,
                              cudaStream_t st);
  static cudaError_t sigma_apply(int NX, int Dp, int C, const Mat3& S, const T* Y, T* y, cudaStream_t st);
  static cudaError_t smooth_out(size_t D, int C, const T* m, const T* varf, const T* y, T* ms, T* vs, cudaStream_t st);
  // kernel-applied smoother carriers: with KV = K(X,T)[v V] (NX x (1+n)), Z = K(X,T) V t (NX x C,
  // nullable when n = 0), Kx = (I (x) K) x (D x (1+q), nullable at the first step):
  //   Kws = [KV_0 - Z_0; 0] + Kx_0,  KWf = [[KV_1..n; 0], Kx_1..q - [Z_1..q; 0]]
  static cudaError_t kcar_build(int64_t NX, int Dp, int n, int q, const T* KV, const T* Z, const T* Kx, T* KWf,
                                T* Kws, cudaStream_t st);
  // D = local rows; observations of points outside [lo, lo + nl) are skipped
  static cudaError_t ws_build(int N, size_t D, int n, int q, const int* idx, const T* X, const T* XV, const T* R,
                              T* Wf, T* ws, int lo, int nl, cudaStream_t st);
  static cudaError_t fill(size_t n, T val, T* out, cudaStream_t st);
  static cudaError_t assemble_slices(int M, int C, int slice, const T* G, T* Y, size_t ldy, cudaStream_t st);
  static cudaError_t pack_dslice(int Dp, int nl, int S, const T* in, T* out, cudaStream_t st);
  static cudaError_t unpack_dslices(int NX, int Dp, int S, const T* G, T* out, cudaStream_t st);
};

// posterior sampler helpers (alg:cakf-caks-sampler); S samples as columns
template <typename T>
struct sampler_ops {
  static cudaError_t permute_cols(int NX, int Dp, int S, const int* map, const T* in, size_t ldi, T* out, size_t ldo,
                                  cudaStream_t st);
  static cudaError_t residual(int N, int S, const T* y, const int* idx, const int* sigma, const T* xp, size_t D,
                              const T* eps, T* res, cudaStream_t st);
  static cudaError_t combine(int NX, int Dp, int S, const Mat3& Sg, const T* Y, const T* tmp, const T* xp, T* x,
                             cudaStream_t st);
  static cudaError_t scatter_rows(int N, int S, const int* idx, const T* R, T sign, T* w, size_t D, cudaStream_t st);
  static cudaError_t gather_coords(int N, const int* idx, const V4<T>* coords, V4<T>* out, cudaStream_t st);
};

}  // namespace cakf
