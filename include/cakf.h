/*
 * cakf.h — C-ABI of the B200-native computation-aware Kalman filter / RTS smoother
 * (CAKF / CAKS, Pförtner et al., arXiv 2405.08971).
 *
 * Citations "P:<line>" refer to the paper's LaTeX source; "R<n>" to the
 * readings listed in DESIGN.md §3.
 *
 * Problem statement (Def. A.1; Lemma B.1):
 *   u_k = A_{k-1} u_{k-1} + q_{k-1},  q ~ N(0, Q_{k-1}),  u_0 ~ N(mu_0, Sigma_0)
 *   y_k = H_k u_k + eps_k,            eps ~ N(0, Lambda_k)
 * for a space-time separable Gauss-Markov prior:
 *   A = A^t (x) I_{N_X},  Q = Q^t (x) Sigma^x(X, X),  Sigma_k = Sigma^t_k (x) Sigma^x(X, X)
 * with D' x D' temporal factors (D' = d_time) and an N_X-point spatial Matérn kernel
 * Sigma^x evaluated on the fly (never stored).  The state is derivative-major:
 * u = (f_0(t, X); f_1(t, X); ...), D = D' * N_X.  H_k picks the rows obs_idx of
 * block 0; Lambda_k is diagonal (R22).
 *
 * Call sequence (alg:mfkf P:276-299, alg:mfks P:386-410):
 *   cakf_create
 *   repeat T times: cakf_predict -> cakf_update -> cakf_truncate
 *   caks_smooth
 *   cakf_get / cakf_get_stats (any time after the step exists)
 *   cakf_reset (start a new run on the same handle) ... cakf_destroy
 * Out-of-order calls return CAKF_E_STATE and leave the handle unchanged.
 *
 * Memory and ownership: every pointer argument is borrowed for the duration of
 * the call.  Array arguments may be host or device (CUDA UVA) pointers; they are
 * copied (stream-ordered) before the call returns to the caller's control of the
 * stream.  The handle owns all device state (trace, workspaces); outputs are
 * written to caller buffers.  All device work is enqueued on cfg.stream (or on a
 * stream the handle creates when cfg.stream is NULL); cakf_get, cakf_get_stats
 * and cakf_sync synchronise that stream.
 *
 * Errors: every function returns 0 (CAKF_OK) or a negative code; the message of
 * the last failure on the calling thread is available from cakf_last_error().
 * CAKF_E_ARG / CAKF_E_STATE leave the handle unchanged.  CAKF_E_CUDA and
 * CAKF_E_NUMERIC mark the handle failed: only get_stats, reset and destroy stay
 * valid.  Rejected (G-degenerate) actions are NOT errors (R2): they are counted
 * in cakf_step_stats.rejected.
 *
 * Concurrency: one handle is used by one host thread at a time.
 */
#ifndef CAKF_H
#define CAKF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAKF_VERSION 1

enum cakf_status {
  CAKF_OK = 0,
  CAKF_E_ARG = -1,         /* NULL / out-of-range / inconsistent argument        */
  CAKF_E_STATE = -2,       /* call out of order (see call sequence)              */
  CAKF_E_UNSUPPORTED = -3, /* kernel family, d_time or policy outside the build  */
  CAKF_E_NUMERIC = -4,     /* non-finite values or failed eigendecomposition     */
  CAKF_E_CUDA = -5,        /* CUDA / cuBLAS / cuSOLVER failure                   */
  CAKF_E_NCCL = -6,        /* multi-GPU communication failure                    */
  CAKF_E_NOMEM = -7        /* device allocation failed                           */
};

enum cakf_dtype { CAKF_F32 = 0, CAKF_F64 = 1 };

/* Spatial Matérn family: Sigma^x(x, x') = Matern_nu(|x - x'| / ell_x), unit output
 * scale (the output scale lives in Sigma^t).  Value = 2 nu. */
enum cakf_kernel { CAKF_MATERN12 = 1, CAKF_MATERN32 = 3, CAKF_MATERN52 = 5 };

/* Policy (Sec. 3.3, App. C.3):
 *   CAKF_POLICY_CG     s_i = current residual r^(i)           (R1; the paper's choice)
 *   CAKF_POLICY_COORD  s_i = e_{order[i-1]}                    (coordinate actions)
 *   CAKF_POLICY_RANDOM s_i ~ N(0, I) by Philox4x32-10 (R16)    (randomized actions)
 *   CAKF_POLICY_BLOCKRES  the adaptive block policy of alg:projected_update:
 *                      a block of b = block_actions actions is chosen at once from the residual at the
 *                      block's start, r^(i0) restricted to b regions of the observations:
 *                      s_{i0+j} = r^(i0) * 1[floor(u b / N) == j], u = the observation's position in the
 *                      caller's order (contiguous index ranges: latitude bands on ERA5-shaped grids);
 *                      b = 1 is CG.  Executed as one multi-RHS K2 per block (tensor cores). */
enum cakf_policy { CAKF_POLICY_CG = 0, CAKF_POLICY_COORD = 1, CAKF_POLICY_RANDOM = 2, CAKF_POLICY_BLOCKRES = 3 };

/* which-selector of cakf_get */
enum cakf_which { CAKF_PRED = 0, CAKF_FILTER = 1, CAKF_SMOOTH = 2 };

typedef struct cakf_s* cakf_t;

typedef struct {
  int32_t dtype;            /* CAKF_F32 or CAKF_F64: arithmetic type of all device math      */
  int32_t d_time;           /* D' (1..3); 2 = Matérn-3/2 temporal prior                      */
  int64_t n_space;          /* N_X >= 1                                                       */
  int32_t space_dim;        /* 1..3 (sphere grids are passed already embedded in R^3)        */
  const double* coords;     /* n_space * space_dim, row-major; host or device; copied         */
  int32_t spatial_kernel;   /* enum cakf_kernel                                              */
  double ell_x;             /* spatial lengthscale (coordinate units), > 0                    */
  const double* sigma_t0;   /* D' x D' row-major Sigma^t(t_0, t_0); Sigma_0 = sigma_t0 (x) K  */
  const double* mu0;        /* D (derivative-major) or NULL for a zero prior mean             */
  int32_t policy;           /* enum cakf_policy                                              */
  int32_t max_iter;         /* N^max: iterations (actions) per update, >= 0                   */
  int32_t max_rank;         /* truncation cap r for M (filter) and W^s (smoother); < 0 = never */
  double rtol;              /* stop once ||r|| <= rtol ||r0||; 0 = count-only (R2, default)   */
  int32_t reorth;           /* 1 = second Gram-Schmidt pass d -= V V^T G d (CGS2, R19); 0 = the
                               single classical pass of alg:update_pls line 11 as printed      */
  int32_t cull_zero;        /* 1 = exact-zero culling (fp32 only): skip kernel tiles whose every
                               value underflows to exactly 0 in fp32 (bounding-sphere distance in
                               prescaled units > 88); results are bit-identical to 0 */
  int32_t block_actions;    /* b >= 1: the non-adaptive policies (random, coordinate) evaluate the
                               kernel part of G s for b consecutive actions with one multi-RHS
                               product (K2, tensor cores); same arithmetic as b sequential
                               iterations.  1 = one K1 matvec per iteration.  Ignored
                               for CG (each action depends on the previous residual); the block
                               size of CAKF_POLICY_BLOCKRES                                       */
  int32_t keep_carriers;    /* 1 = keep the smoother carriers w^s_k, W^s_k of every step (an extra
                               (T+1) x D x (1 + r) values) so cakf_interpolate can return smoother
                               states between steps (Cor. A.10); 0 = filter interpolation only */
  uint64_t seed;            /* Philox key of CAKF_POLICY_RANDOM                               */
  int32_t max_steps;        /* T: number of time steps the trace is sized for                */
  int64_t max_obs;          /* max N_k over the run (0 = n_space)                            */
  int32_t rank;             /* multi-GPU rank (0 for a single GPU)                           */
  int32_t world;            /* number of ranks (1 = single GPU); > 1 shards the Gram products */
  const void* nccl_id;      /* 128-byte ncclUniqueId when world > 1, else NULL               */
  void* stream;             /* cudaStream_t to enqueue on, or NULL                           */
} cakf_config;

typedef struct {
  int32_t k;                /* step index                                                     */
  int32_t iters;            /* iterations executed (including rejected actions)              */
  int32_t rejected;         /* actions rejected by the eta floor (R2)                         */
  int32_t rank_in;          /* columns of M^-_k                                               */
  int32_t cols;             /* columns of M_k = rank_in + iters                               */
  int32_t rank_out;         /* columns of M~_k after Truncate                                 */
  int32_t smoother_rank;    /* columns of W^s_k after the smoother's Truncate                 */
  int32_t missing;          /* 1 if the step had no observations (IsMissing)                  */
  double res0;              /* ||r^(0)||_2                                                    */
  double res_final;         /* ||r^(iters)||_2 (recurrence)                                   */
  double eta_min;           /* smallest accepted eta                                          */
  double dropped_mass;      /* sum of dropped Gram eigenvalues = tr(N N^T) (Sec. 3.2)         */
} cakf_step_stats;

/* Create a handle: copies coords (prescaled), allocates the trace for max_steps
 * steps and all workspaces.  Returns CAKF_E_NOMEM if the trace does not fit. */
int cakf_create(const cakf_config* cfg, cakf_t* out);

/* Discard all steps and start again at k = 0 with the same configuration and buffers. */
int cakf_reset(cakf_t h);

/* Predict step k-1 -> k (alg:mfkf lines 4-5; Prop A.3):
 *   Sigma^t_k = A^t Sigma^t_{k-1} A^tT + Q^t         (host, fp64)
 *   m^-_k = (A^t (x) I) m_{k-1} + b,  M^-_k = (A^t (x) I) M~_{k-1}
 * A_t, Q_t: D' x D' row-major (host or device).  b: D or NULL (zero, R9). */
int cakf_predict(cakf_t h, const double* A_t, const double* Q_t, const void* b);

/* Update step k (alg:update_pls), or IsMissing when n_obs == 0
 * (P:283-294).  obs_idx: n_obs int64 spatial indices (f_0 rows of H_k), unique;
 * y, noise_var: n_obs values of the handle's dtype (noise_var = diag Lambda_k);
 * coord_order: for CAKF_POLICY_COORD, >= min(max_iter, n_obs) int64 positions into
 * obs_idx (j(i) of App. C.3), else NULL.  Iterations = min(max_iter, n_obs). */
int cakf_update(cakf_t h, int64_t n_obs, const int64_t* obs_idx, const void* y,
                const void* noise_var, const int64_t* coord_order);

/* Truncate step k (Sec. 3.2; R3/R4): keep the top min(max_rank, cols)
 * eigen-directions of M_k^T M_k, M~_k = M_k Q_r (eigendecomposition on device).
 * Ordering: on a one-GPU fp32 handle the eigensolver and M Q_r may still run on an internal
 * stream when this returns (they overlap the next update's prologue and first K1).  Every later
 * call except cakf_predict / cakf_update (which order themselves after it) first joins that work
 * into the handle's stream, so library calls stay stream-ordered; before synchronising the
 * handle's stream yourself right after cakf_truncate, call cakf_sync (CAKF_TRUNC_OVERLAP=0: off). */
int cakf_truncate(cakf_t h);

/* Backward CAKS sweep k = T-1 .. 0 (alg:mfks; R6, R7) over the steps
 * filtered so far.  Produces smoother means and marginal variances for k = 0..T. */
int caks_smooth(cakf_t h);

/* Copy the mean and/or marginal variance (D values each, dtype of the handle,
 * derivative-major) of state k in {0..T} to mean_D / var_D (host or device; either
 * may be NULL).  which: CAKF_PRED (m^-_k, diag P^-_k), CAKF_FILTER (m_k, diag P_k),
 * CAKF_SMOOTH (m^s_k, diag P^s_k; requires caks_smooth).  Synchronises. */
int cakf_get(cakf_t h, int32_t k, int32_t which, void* mean_D, void* var_D);

/* Per-step statistics (synchronises). */
int cakf_get_stats(cakf_t h, int32_t k, cakf_step_stats* out);

/* Kept Gram eigenvalues of the filter truncation at step k, descending
 * (min(max_rank, cols) values) into vals (host, double); n_out receives the count. */
int cakf_get_kept_eigs(cakf_t h, int32_t k, double* vals, int32_t cap, int32_t* n_out);

/* Wait for all work enqueued by the handle. */
int cakf_sync(cakf_t h);

/* Kernel timing by category with CUDA events recorded on the handle's stream around
 * every launch of that category (for bench.py's live roofline).  enable = 0 stops
 * recording.  cakf_profile_read synchronises, adds the elapsed times recorded since
 * the last reset into ms[CAKF_PROF_NCAT] and launches[CAKF_PROF_NCAT], and clears the
 * record when reset != 0. */
enum cakf_prof_category {
  CAKF_PROF_K1 = 0,         /* fused kernel-eval matvec of the inner loop (a4)         */
  CAKF_PROF_K2_POST = 1,    /* fused kernel-eval x [v V] of the post-loop update (a7)  */
  CAKF_PROF_K2_SMOOTH = 2,  /* fused kernel-eval x [x_0 x_1] of the smoother (a9)      */
  CAKF_PROF_STAGES = 3,     /* inner-loop reduction / update stages (a5, a6)           */
  CAKF_PROF_TRUNCATE = 4,   /* Gram + eigendecomposition + M Q_r (a8, smoother too)    */
  CAKF_PROF_LOWRANK = 5,    /* low-rank fp64-accumulated contractions (a7, a9)         */
  CAKF_PROF_TRUNC_GRAM = 6, /* ... of which: the Gram matrix F^T F                      */
  CAKF_PROF_TRUNC_EIG = 7,  /* ... of which: the symmetric eigendecomposition            */
  CAKF_PROF_TRUNC_GEMM = 8, /* ... of which: F Q_r                                       */
  CAKF_PROF_NCAT = 9
};
int cakf_profile(cakf_t h, int32_t enable);
int cakf_profile_read(cakf_t h, double* ms, int64_t* launches, int32_t reset);

/* Number of libcakf kernels launched by this process so far (all handles). */
int64_t cakf_kernel_launches(void);

/* Temporal interpolation (Cor. A.10 P:1386-1437; alg:cakf-interpolation P:1445-1469,
 * alg:caks-interpolation P:1470-1499): the filter (which = CAKF_FILTER) or smoother
 * (CAKF_SMOOTH) marginal mean and variance at an off-grid time t with t_k <= t < t_{k+1}
 * (k = T: t >= t_T), from the stored step-k state — no data is revisited:
 *   m(t) = (A1 (x) I) m_k, M(t) = (A1 (x) I) M~_k, P(t) = Sigma(t) - M(t) M(t)^T,
 *   Sigma(t) = (A1 Sigma^t_k A1^T + Q1) (x) K_X;  smoother (k < T): m^s(t) = m(t) +
 *   P(t) (A2 (x) I)^T w^s_{k+1}, var^s(t) = var(t) - rowsumsq(P(t) (A2 (x) I)^T W^s_{k+1}).
 * A1 = A^t(t, t_k), Q1 = Q^t(t, t_k), A2 = A^t(t_{k+1}, t): D' x D' row-major doubles, host or
 * device (e.g. cakf_matern_transition with dt = t - t_k and t_{k+1} - t); A2 is ignored for the
 * filter and for k = T.  mean_D / var_D: D values (dtype), user point order, host or device,
 * either may be NULL.  Synchronises the handle's stream.
 * Errors: CAKF_E_ARG (k outside [1, steps done], bad which, NULL matrices), CAKF_E_STATE (step k
 * not truncated yet; smoother query before caks_smooth or without keep_carriers), CAKF_E_NUMERIC
 * (singular A_{k+1}), CAKF_E_CUDA. */
int cakf_interpolate(cakf_t h, int32_t k, const double* A1, const double* Q1, const double* A2, int32_t which,
                     void* mean_D, void* var_D);

/* Posterior sampler (alg:cakf-caks-sampler P:1336-1358; Matheron's rule P:1150-1216, Prop A.9
 * P:1290-1313): S samples of the CAKF (which = CAKF_FILTER) or CAKS (CAKF_SMOOTH) posterior
 * at every step k = 0..T from the stored filter trace, given the caller's prior draws (the
 * random numbers the method consumes are inputs; the smoother does not have to have run):
 *   forward  x^-_k = A_{k-1} x_{k-1} + q_{k-1};  w_k = H_k^T V_k V_k^T (y_k - H_k x^-_k - eps_k);
 *            x_k = x^-_k + P^-_k w_k
 *   backward x^s_k = x_k + P_k A_k^T w^s_{k+1};  w^s_k = w_k + (I - W_k W_k^T P^-_k) A_k^T w^s_{k+1}
 * (R25: eps_k is a full-space draw of N(0, Lambda_k), equivalent to the paper's projected noise).
 *   x0  : D x S column-major draws of N(mu_0, Sigma_0), user point order, dtype
 *   q   : T blocks of D x S, block k-1 = draws of N(0, Q^t_{k-1} (x) K_X) into step k
 *   eps : for k = 1..T, an N_k x S block of N(0, Lambda_k) draws in the observation order passed
 *         to cakf_update at step k (missing steps contribute no block)
 *   out : (T+1) blocks of D x S, user point order.  All host or device.  1 <= S <= 1 + max_iter.
 * Valid after the last cakf_truncate.  Synchronises the handle's stream.
 * Errors: CAKF_E_ARG, CAKF_E_STATE, CAKF_E_CUDA, CAKF_E_NOMEM (workspace). */
int cakf_sample(cakf_t h, int32_t n_samples, const void* x0, const void* q, const void* eps, int32_t which,
                void* out);

/* Test entry point: the inner loop's kernel matvec (a4's K_TT s) launched
 * exactly as cakf_update launches it — the per-update kd order of the observed points, the
 * exact-zero culling lists, the symmetric tile-pair kernel with its dynamic unit scheduler and
 * partial slots — for one vector:  out[j] = sum_l Matern(|x_{obs[j]} - x_{obs[l]}| / ell) s[l].
 * obs_idx (n_obs spatial indices, int64), s and out (n_obs, handle dtype) in the caller's
 * observation order, host or device.  Call between steps (not between predict and update); it
 * overwrites the inner-loop workspaces only.  shares > 1 runs K1 as the multi-GPU split into `shares`
 * contiguous unit ranges with equal active tile pairs (what rank p of `shares` ranks evaluates), one after
 * the other into the same partial slots: the result must equal shares = 1 bit for bit.  Synchronises.
 * Errors: CAKF_E_ARG (NULL, n_obs outside [1, max_obs], index out of range), CAKF_E_STATE, CAKF_E_CUDA. */
int cakf_debug_matvec(cakf_t h, int64_t n_obs, const int64_t* obs_idx, const void* s, void* out, int32_t shares);

/* Exact-zero culling statistics of the handle so far: frac3[0] = fraction of the symmetric K1's
 * pairs evaluated (counted in 16 x 128 warp blocks of its 128 x 128 tile pairs), frac3[1] = fraction of the post-loop K2's 128x32 tiles evaluated,
 * frac3[2] = same for the smoother's K2 (all 1.0 when culling is off).  Synchronises the handle's
 * stream.  Errors: CAKF_E_HANDLE, CAKF_E_ARG (NULL frac3), CAKF_E_CUDA. */
int cakf_cull_stats(cakf_t h, double* frac3);

/* ---- multi-GPU (the spatial rows of the covariance operator and of M are sharded) ----
 * With cfg.world > 1 every rank calls the same sequence with the same full inputs.  Rank p owns the
 * internal (kd-ordered) points [row_lo, row_hi) (128-aligned equal slices) and holds only their rows of
 * every D-length state: m, variances, M_k = [M^-_k | B_k], the truncated factors, the smoother carriers
 * and the post-loop kernel products K(X_p, X_T)[v V].  Exchanges, all NCCL on cfg.stream:
 *   update   all-reduce of [H m^-, H M^-] (N x (1 + r): each rank contributes the observed rows it owns);
 *   loop     K1 (K_TT s): rank p evaluates its share of the symmetric tile-block units (with exact-zero
 *            culling: a contiguous unit range holding 1/world of the active tile pairs, else [u_lo, u_hi)),
 *            then all-reduce of the N-vector; the N-length loop state is replicated;
 *   post     none: K2 and the low-rank algebra produce this rank's rows;
 *   truncate all-reduce of the partial Grams M_p^T M_p (c x c fp64); the eigensolver runs on every rank
 *            on identical bits; M~_p = M_p Q_r;
 *   smoother all-reduce of M^-T x (r x (1+q)) and V^T H y (n x (1+q));
 *   get      all-gather of the row slices.
 * cakf_interpolate / cakf_sample / CAKF_SMOOTH_K2 are single-GPU only (CAKF_E_UNSUPPORTED).
 * cakf_nccl_unique_id writes the 128-byte ncclUniqueId rank 0 creates (broadcast it to all ranks
 * and pass it as cfg.nccl_id). */
int cakf_nccl_unique_id(void* out128);

/* Host-only: the shard of rank `rank` of `world`: out[0..6] = {row_lo, row_hi, u_lo, u_hi,
 * n_units, slice_rows, block_points} for n_space points and n_obs observations (a K1 unit is a
 * pair of blocks of block_points consecutive observations). */
int cakf_shard_plan(int64_t n_space, int64_t n_obs, int32_t world, int32_t rank, int64_t* out);

/* Host-only mirror of the symmetric K1's unit -> (tile block i, tile block j) map, i <= j. */
int cakf_sym_unit_blocks(int64_t n_obs, int64_t unit, int32_t* bi, int32_t* bj);

/* Free everything the handle owns. */
int cakf_destroy(cakf_t h);

/* Thread-local message for the last non-zero status. */
const char* cakf_last_error(void);

int cakf_version(void);

/* Stationary Matérn(nu2/2) temporal SDE, closed forms (Remark B.2; R10):
 * A = expm(F dt) (D' x D', row-major), Q = Sinf - A Sinf A^T, Sinf the stationary
 * covariance, D' = (nu2 + 1) / 2.  Any output pointer may be NULL (host pointers). */
int cakf_matern_transition(int32_t nu2, double ell_t, double sigma, double dt,
                           double* A, double* Q, double* Sinf);

/* Standalone fused kernel-evaluation x matrix product (the "Gramian x matrix" op of
 * P:644-647; a4/a7/a9 of SURVEY §8a):
 *   Y[i, c] = alpha * sum_j Matern_nu(|xr_i - xc_j| / ell) * X[j, c]
 * xr: n_rows x space_dim, xc: n_cols x space_dim (row-major, device, dtype);
 * X: n_cols x n_rhs column-major (ld = n_cols), Y: n_rows x n_rhs column-major
 * (ld = n_rows), both device.  stream may be NULL. */
int cakf_gram_matmul(int32_t dtype, int32_t spatial_kernel, double ell, int32_t space_dim,
                     int64_t n_rows, const void* xr, int64_t n_cols, const void* xc,
                     int32_t n_rhs, const void* X, double alpha, void* Y, void* stream);

/* Standalone low-rank contraction of the fp32 path (a7 post-loop P:1532-1541, a8 truncation Gram
 * and M Q_r Sec. 3.2, a9 smoother products alg:mfks P:388-409):
 *   C = alpha * op(A) op(B) + beta * C,   op(X) = X (trans = 0) or X^T (trans = 1),
 * A, B, C fp32, column-major (BLAS convention: op(A) m x k, op(B) k x n, C m x n, leading
 * dimensions lda / ldb / ldc), device pointers.  Computed on the INT8 tensor cores with exact
 * slice products and fp64 sums (kernels_gemm_i8.cu): the result equals the fp64 product of
 * the fp32 inputs to ~2^-33 relative to sum_k |a||b| per chunk maximum.  k >= 1.
 * Workspaces are allocated on `stream` (may be NULL) and freed before return; synchronises. */
int cakf_lowrank_gemm(int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k, double alpha,
                      const float* A, int64_t lda, const float* B, int64_t ldb, double beta, float* C,
                      int64_t ldc, void* stream);

/* Live ALU peaks for the roofline denominators (bench.py): out3[0] = MUFU ops/s of the sqrt.approx /
 * ex2.approx mix K1 is bound by (2 MUFU ops per kernel pair), out3[1] = fp64 tensor-core
 * (DMMA) flop/s, out3[2] = clock64 cycles of one CTA of the MUFU test (diagnostic).  Microbenchmarks launched on
 * `stream` (may be NULL); synchronises.  Errors: CAKF_E_ARG, CAKF_E_CUDA. */
int cakf_alu_peaks(double* out3, void* stream);

/* Standalone symmetric eigensolver of the truncation (a8 / a9 Truncate, Sec. 3.2; "SVD of
 * M M^T" P:367, reading R4: eigh of the Gram M^T M), fp64, all on the device (kernels_eig.cu:
 * cluster Householder tridiagonalisation, divide and conquer, back-transformation):
 *   G : c x c symmetric, column-major, only the lower triangle is read (host or device)
 *   w : c eigenvalues, ascending (nullable)
 *   Qr: c x r column-major eigenvectors of the r LARGEST eigenvalues, in descending order (nullable)
 * 1 <= c <= 8192, 0 <= r <= c.  Workspaces are allocated on `stream` (may be NULL); synchronises.
 * Errors: CAKF_E_ARG, CAKF_E_NUMERIC (non-finite eigenvalue), CAKF_E_CUDA. */
int cakf_sym_eig(int64_t c, int64_t r, const double* G, double* w, double* Qr, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CAKF_H */
