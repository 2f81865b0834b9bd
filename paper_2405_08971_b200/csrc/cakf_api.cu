// cakf_api.cu — runtime (handle, trace arena, step scheduler) and the C-ABI of libcakf.
//
// One CAKF/CAKS run on one B200 (cfg.world == 1).  Device layout:
//   coords      N_X x {x,y,z,w} (dtype), prescaled by sqrt(2 nu)/ell_x
//   per step k  m^-_k, m_k, var_k, m^s_k, var^s_k (D each)
//               M_k = [M^-_k | B_k]  D x (rin_k + iters_k), column-major, ld = D
//               obs idx (N_k int32), XV = [v | V]  N_k x (1 + N^max), column-major
//               IterCtl (stats), kept Gram eigenvalues
//   workspaces  inner loop (r, s, g, g', d, Gd, Z, HM, K1 partials, fp64 block partials),
//               post-loop (Y, U, tmp), truncation (Gram, eig, Q_r, M~), smoother (X, Y, y, W^s)
// Everything is enqueued on one stream without host synchronisation between the
// calls (iteration counts and ranks are host-known integers, R2/R3).
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <cfloat>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cakf.h"
#include "internal.h"
#include "step.h"

using namespace cakf;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK_CUDA(expr)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      failed_ = true;                                                                           \
      return fail(e_ == cudaErrorMemoryAllocation ? CAKF_E_NOMEM : CAKF_E_CUDA,                 \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                          \
    }                                                                                           \
  } while (0)
#define CK_SOLVER(expr)                                                                         \
  do {                                                                                          \
    cusolverStatus_t s_ = (expr);                                                               \
    if (s_ != CUSOLVER_STATUS_SUCCESS) {                                                        \
      failed_ = true;                                                                           \
      return fail(CAKF_E_CUDA, std::string(#expr) + ": cusolver status " + std::to_string(s_)); \
    }                                                                                           \
  } while (0)
#define CK_NCCL(expr)                                                                           \
  do {                                                                                          \
    ncclResult_t r_ = (expr);                                                                   \
    if (r_ != ncclSuccess) {                                                                    \
      failed_ = true;                                                                           \
      return fail(CAKF_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));             \
    }                                                                                           \
  } while (0)
#define CK(expr)              \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != 0) return rc_; \
  } while (0)

Mat3 mat_from(const double* a, int n) {
  Mat3 m{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) m.a[i][j] = a[i * n + j];
  return m;
}
Mat3 mat_abat_plus_q(const Mat3& A, const Mat3& S, const Mat3& Q, int n) {
  Mat3 AS{}, R{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int t = 0; t < n; ++t) AS.a[i][j] += A.a[i][t] * S.a[t][j];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = Q.a[i][j];
      for (int t = 0; t < n; ++t) acc += AS.a[i][t] * A.a[j][t];
      R.a[i][j] = acc;
    }
  return R;
}

Mat3 mat_mul(const Mat3& A, const Mat3& B, int n) {
  Mat3 R{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int t = 0; t < n; ++t) R.a[i][j] += A.a[i][t] * B.a[t][j];
  return R;
}
// Gauss-Jordan with partial pivoting (n <= 3); false if singular
bool mat_inv(const Mat3& A, int n, Mat3& out) {
  double M[3][6] = {};
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) M[i][j] = A.a[i][j];
    M[i][n + i] = 1.0;
  }
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(M[r][c]) > std::fabs(M[p][c])) p = r;
    if (M[p][c] == 0.0) return false;
    for (int j = 0; j < 2 * n; ++j) std::swap(M[c][j], M[p][j]);
    const double d = M[c][c];
    for (int j = 0; j < 2 * n; ++j) M[c][j] /= d;
    for (int r = 0; r < n; ++r)
      if (r != c) {
        const double f = M[r][c];
        for (int j = 0; j < 2 * n; ++j) M[r][j] -= f * M[c][j];
      }
  }
  out = Mat3{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out.a[i][j] = M[i][n + j];
  return true;
}

// host copy of a small host-or-device array of doubles
bool fetch_doubles(const double* src, size_t n, std::vector<double>& out) {
  out.resize(n);
  if (!n) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, src) == cudaSuccess &&
      (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged)) {
    return cudaMemcpy(out.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaGetLastError();
  std::memcpy(out.data(), src, n * sizeof(double));
  return true;
}
// CAKF_TRUNC_OVERLAP=0: the filter truncation's eigensolver and M Q_r in line (A/B only)
bool trunc_overlap() {
  static const bool v = !env_is("CAKF_TRUNC_OVERLAP", '0');
  return v;
}

// CAKF_SLOT_LISTS=0: the stage kernels sum all K1 partial slots (interleaved over the warps) instead of the
// per-block lists of the slots that can be nonzero (A/B only; a different summation grouping, so not the
// same bits — culling on / off stays bit-identical within either mode)
bool slot_lists_on() {
  static const bool v = !env_is("CAKF_SLOT_LISTS", '0');
  return v;
}

// CAKF_STAGE_AB=0: the inner loop's stages A and B as two kernels (A/B only)
bool stage_ab() {
  static const bool v = !env_is("CAKF_STAGE_AB", '0');
  return v;
}

// CAKF_SMOOTH_OVERLAP=0: the smoother's carrier products run in line with the truncation (A/B only)
bool smooth_overlap() {
  static const bool v = !env_is("CAKF_SMOOTH_OVERLAP", '0');
  return v;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

constexpr bool OP_N = false, OP_T = true;   // op(X) = X / X^T of the low-rank contractions

struct ImplBase {
  virtual ~ImplBase() = default;
  // the filter truncation's eigensolver / M Q_r may still run on the truncation stream (overlapping the next
  // update's prologue and first K1); every entry point except predict / update joins it first
  virtual int join_pending() { return CAKF_OK; }
  virtual int init(const cakf_config& cfg) = 0;
  virtual int reset() = 0;
  virtual int predict(const double* A, const double* Q, const void* b) = 0;
  virtual int update(int64_t n, const int64_t* idx, const void* y, const void* nv, const int64_t* order) = 0;
  virtual int truncate() = 0;
  virtual int smooth() = 0;
  virtual int get(int k, int which, void* mean, void* var) = 0;
  virtual int stats(int k, cakf_step_stats* out) = 0;
  virtual int kept_eigs(int k, double* vals, int cap, int* n_out) = 0;
  virtual int sync() = 0;
  virtual int profile(bool on) = 0;
  virtual int prof_read(double* ms, int64_t* n, bool reset) = 0;
  virtual int cull_stats(double* out) = 0;
  virtual int interpolate(int k, const double* A1, const double* Q1, const double* A2, int which, void* mean,
                          void* var) = 0;
  virtual int sample(int S, const void* x0, const void* q, const void* eps, int which, void* out) = 0;
  virtual int debug_matvec(int64_t n, const int64_t* idx, const void* s, void* out, int shares) = 0;
};

template <typename T>
struct Impl final : ImplBase {
  // ---------------- configuration
  int Dp = 2, dim = 3, nu2 = 3, policy = 0, nhat = 0, rcap = -1, Tmax = 0;
  // Row sharding: this rank owns the internal points [plo, plo + NX) — NX and D = Dp NX are the
  // LOCAL sizes of every D-row array (m, var, M_k, B, carriers, ...); NXf / Df are the full grid.  world = 1:
  // plo = 0, NX = NXf.
  int64_t NX = 0, D = 0, Nmax = 0;
  int64_t NXf = 0, Df = 0, plo = 0, pslice = 0;
  double rtol = 0.0, ell = 1.0;
  uint64_t seed = 0;
  Mat3 sig_t0{};
  bool own_stream = false, failed_ = false;
  cudaStream_t st = nullptr;
  // side stream: u = (HM^-)^T s (HBM-bound) overlaps K1 (MUFU-bound) in every inner iteration
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // smoother: the kernel-applied carriers (Zk GEMM + kcar_build) on the side stream beside the truncation's
  // Gram / eig / first GEMM of the same step (they only feed its second GEMM); ev_kcar joins them
  cudaEvent_t ev_ws = nullptr, ev_kcar = nullptr;
  cudaEvent_t f2_wait = nullptr;   // consumed by truncate_factor*: wait before the second factor's GEMM
  std::function<int()> after_gram;  // consumed by truncate_factor*: enqueued right after the Gram (side work)
  // filter truncation: eigensolver + M Q_r (and the next predict's M^- = A M~) on st_t, beside the next
  // update's prologue and first K1 (they need only m^-); the update joins before gathering H M^-
  cudaStream_t st_t = nullptr;
  cudaEvent_t ev_tf = nullptr, ev_td = nullptr;
  cudaStream_t st_e = nullptr;   // eigensolver side stream (T factors beside the divide and conquer)
  cudaEvent_t ev_ea = nullptr, ev_eb = nullptr;
  bool fork_trunc = false;     // set by truncate() around its truncate_factor call
  bool trunc_pending = false;  // work on st_t not yet joined into st
  int join_pending() override {
    if (!trunc_pending) return CAKF_OK;
    trunc_pending = false;
    CK_CUDA(cudaStreamWaitEvent(st, ev_td, 0));
    return CAKF_OK;
  }
  double* part2 = nullptr;
  double* hmw = nullptr;   // HM u (fp64 rows), formed on the side stream
  bool side = [] { const char* e = getenv("CAKF_NO_SIDE_STREAM"); return !(e && e[0] == '1'); }();
  cusolverDnHandle_t sol = nullptr;

  // ---------------- device memory
  char* arena = nullptr;
  size_t arena_bytes = 0, arena_off = 0;
  V4<T>* coords = nullptr;
  T* mu0 = nullptr;
  struct Step {
    T *m_pred, *m, *var, *ms, *vs, *Mk, *XV;
    T* KV;   // post-loop kernel products K(X, T_k) [v V] (NX x (1 + n)), reused by the smoother
    int* idx;
    double* kept;
    int cap_cols = 0;
    int rin = 0, cols = 0, n = 0, N = 0, rank_out = 0, smoother_rank = 0;
    bool missing = true, truncated = false;
    Mat3 sig_t{}, A_next{};
  };
  std::vector<Step> steps;
  IterCtl* ctl = nullptr;  // [Tmax + 1]
  IterCtl* ctl_init_host = nullptr;

  // inner loop
  V4<T>* xcs = nullptr;
  T *r = nullptr, *s = nullptr, *g = nullptr, *gp = nullptr, *d = nullptr, *Gd = nullptr, *Z = nullptr, *HM = nullptr;
  T* hmx = nullptr;   // [H m^- | H M^-] (N x (1 + rin)): gathered from the owners of the observed rows
  T* rbs = nullptr;   // CAKF_POLICY_BLOCKRES: the residual at the current block's start
  void* samp_ws = nullptr;   // cakf_sample workspace (grow-only, freed at destroy)
  size_t samp_bytes = 0;
  long long* k1_range = nullptr;   // multi-GPU: this rank's K1 unit range, balanced by active tile pairs
  T *ybuf = nullptr, *lam2 = nullptr, *partial = nullptr;
  size_t partial_cap = 0;
  int64_t* stage64 = nullptr;
  int* order32 = nullptr;
  double *part = nullptr, *redA = nullptr, *redB = nullptr, *redC = nullptr;
  bool reorth = true;
  unsigned* cnt = nullptr;
  int W = 0, rin_max = 0, qmax = 0, cmax = 0;
  // post-loop
  T *Yb = nullptr, *Ub = nullptr, *tmp = nullptr;
  // truncation
  double *gpart = nullptr, *Gm = nullptr, *eigw = nullptr, *work = nullptr;
  int* info = nullptr;
  void* eigws = nullptr;   // own eigensolver workspace (kernels_eig.cu)
  size_t eigws_bytes = 0;
  // CAKF_EIG_CUSOLVER=1: cusolverDnDsyevd instead of the repo's eigensolver (A/B only)
  bool eig_cusolver = env_is("CAKF_EIG_CUSOLVER", '1');
  int lwork = 0, nsplit_max = 16;
  T* Mtil = nullptr;
  double* QrD = nullptr;
  // fp64 scratch of the low-rank contractions (fp32 storage, fp64 accumulation)
  size_t dscr = 0;          // largest low-rank operand (elements): sizes the tensor-core operand planes
  double* fwork = nullptr;  // split-K partials of the FP64-pipe GEMM
  static constexpr size_t kF64WorkDoubles = (size_t)4 << 20;
  // smoother
  T *X = nullptr, *Yk = nullptr, *yb = nullptr, *Tm = nullptr, *Hy = nullptr, *tt = nullptr, *R = nullptr;
  T *Wf = nullptr, *Ws = nullptr, *ws = nullptr, *pvar = nullptr;
  // kernel-applied smoother carriers (I (x) K)[w^s, W^s] (and of W^s_full), K(X, T) V t
  T *KWf = nullptr, *KWs = nullptr, *Kws = nullptr, *Zk = nullptr;
  bool smooth_k2 = [] { const char* e = getenv("CAKF_SMOOTH_K2"); return e && e[0] == '1'; }();
  float* tcw = nullptr;  // bf16 planes of the K2 right-hand sides
  // low-rank contractions on tcgen05 (kernels_gemm_tc.cu): operand planes, split-K work, fp32 Q_r
  // (truncation always; the post-loop / smoother contractions only with CAKF_LOWRANK_TC=1 — fp32
  // accumulation there misses the cfg1 1e-4 bound under the variance cancellation)
  bool lowrank_tc = [] { const char* e = getenv("CAKF_LOWRANK_TC"); return e && e[0] == '1'; }();
  bool gram_tc = [] { const char* e = getenv("CAKF_GRAM_TC"); return e && e[0] == '1'; }();
  uint16_t *gpA = nullptr, *gpB = nullptr;
  size_t gp_elems = 0;
  float *gwork = nullptr, *Qf = nullptr;
  int *gexA = nullptr, *gexB = nullptr;   // INT8-slice GEMM: per-(row, K chunk) exponents
  // contractions with K >= i8_min_k (the D- and N-long reductions: truncation Gram, M^T x, (HM)^T [v V],
  // and the K = r_in products M (M^T x), M U, from r_in = 128 on) run on the INT8-slice GEMM; K = N^ = 64
  // (B_k t, V t, (K(X,T)V) t) on the DMMA strip kernel.  (At 512 the early steps' M^- (M^-T x) with
  // r_in = 128 .. 448 fell to the tiled DMMA kernel: 7 - 10 ms per call, ≈ 40 ms per cfg3 pass.)
  // CAKF_I8_MIN_K overrides
  int i8_min_k = [] { const char* e = getenv("CAKF_I8_MIN_K"); return e ? std::atoi(e) : 128; }();
  bool i8_mqr = [] { const char* e = getenv("CAKF_I8_MQR"); return e && e[0] == '1'; }();
  size_t gex_elems = 0;

  // ---------------- exact-zero culling (fp32 only): tile bounding spheres and, per 128-row
  // output tile of K2, the ascending list of 32-column K-blocks not entirely below the fp32 underflow
  bool cull = false;
  float4 *sph_x128 = nullptr, *sph_x32 = nullptr, *sph_o128 = nullptr, *sph_o32 = nullptr, *sph_o16 = nullptr;
  float4 *box_o32 = nullptr, *box_o16 = nullptr;   // bounding boxes {lo, hi} of the 32- / 16-point tiles (K1)
  int *act_cnt_sm = nullptr, *act_list_sm = nullptr, *act_cnt_po = nullptr, *act_list_po = nullptr;
  int act_stride_sm = 0, act_stride_po = 0;
  int *k1_list = nullptr, *k1_count = nullptr;
  int *k1_plist = nullptr, *k1_pq = nullptr;   // per 512-row block: the K1 partial slots that can be nonzero (SlotList)
  unsigned short* k1_mask = nullptr;  // active symmetric K1 units of this update
  unsigned* k1_sched = nullptr;                           // K1 dynamic unit scheduling counters
  unsigned long long* cull_ctr = nullptr;  // [0] K1 tile pairs done, [1] K2-post blocks, [2] K2-smooth blocks
  double k1_pairs_dense = 0, k2_post_dense = 0, k2_sm_dense = 0;
  int64_t k2_sm_launches = 0;

  // ---------------- internal point order (spatially compact tiles for the fused kernels)
  int *perm_d = nullptr, *invperm_d = nullptr;   // internal -> user, user -> internal
  int *posof = nullptr, *obs_cnt = nullptr, *sigma = nullptr, *sigma_inv = nullptr;
  T *ybuf_user = nullptr, *lam2_user = nullptr, *outm = nullptr, *outv = nullptr;
  std::vector<int> perm_h;
  // temporal interpolation (Cor. A.10): smoother carriers w^s_k, W^s_k kept per step
  bool keep = false;
  // block execution of the non-adaptive policies: b actions' G s per K2 launch
  int blk = 1;
  int *act_cnt_tt = nullptr, *act_list_tt = nullptr;
  // per-step observations (internal row order) and their user positions, for the sampler
  T* y_st = nullptr;
  int* sig_st = nullptr;
  T *ws_st = nullptr, *Ws_st = nullptr, *ip_m = nullptr, *ip_v = nullptr, *ip_ms = nullptr, *ip_vs = nullptr;
  // per-update kd order of the observations (kd_order.cu); CAKF_NO_REORDER=1 keeps the sorted order
  bool kd_obs = [] { const char* e = getenv("CAKF_NO_REORDER"); return !(e && e[0] == '1'); }();
  int *idx_tmp = nullptr, *sig_tmp = nullptr;
  // observation-order cache: an update whose obs_idx equals the previous one's reuses that order
  // (idx, sigma, sigma_inv are a pure function of obs_idx; bit-identical to recomputing it)
  int64_t obs_cache_n = -1;
  std::vector<int64_t> obs_cache_h;    // host copy (host-pointer callers)
  int64_t* obs_cache_d = nullptr;      // device copy (device-pointer callers)
  int *idx_cache = nullptr, *sig_cache = nullptr, *siginv_cache = nullptr, *neq_d = nullptr;
  void* kd_ws = nullptr;
  size_t kd_ws_bytes = 0;

  // Internal point order: a balanced kd-tree (recursive bisection at the median of the widest
  // axis), depth-first.  Splits fall on multiples of 128 above 256 points and of 32 below, so every
  // 128-row tile of the K2 output and every 32-column K-block is one compact subtree (bounding
  // spheres ~2x tighter than a Morton order).  CAKF_NO_REORDER=1 keeps the user order.
  void make_perm(const std::vector<double>& xyz) {
    perm_h.resize(NXf);
    for (int64_t i = 0; i < NXf; ++i) perm_h[i] = (int)i;
    const char* e = getenv("CAKF_NO_REORDER");
    if (e && e[0] == '1') return;
    std::vector<std::pair<int64_t, int64_t>> stack{{0, NXf}};
    while (!stack.empty()) {
      const auto [b0, b1] = stack.back();
      stack.pop_back();
      const int64_t n = b1 - b0;
      if (n <= 32) continue;
      double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int d = 0; d < dim; ++d) {
        lo[d] = hi[d] = xyz[(size_t)perm_h[b0] * dim + d];
        for (int64_t i = b0; i < b1; ++i) {
          const double v = xyz[(size_t)perm_h[i] * dim + d];
          lo[d] = std::min(lo[d], v);
          hi[d] = std::max(hi[d], v);
        }
      }
      int ax = 0;
      for (int d = 1; d < dim; ++d)
        if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
      std::sort(perm_h.begin() + b0, perm_h.begin() + b1, [&](int a, int b) {
        const double va = xyz[(size_t)a * dim + ax], vb = xyz[(size_t)b * dim + ax];
        return va < vb || (va == vb && a < b);
      });
      const int64_t al = n > 256 ? 128 : 32;
      int64_t h = ((n / 2 + al / 2) / al) * al;
      h = std::min(std::max(h, al), n - 1);
      stack.push_back({b0 + h, b1});   // right half after the left one (depth-first, left first)
      stack.push_back({b0, b0 + h});
    }
  }

  // ---------------- multi-GPU: the Gram products are sharded, the rest replicated
  int world = 1, rank = 0;
  bool coll = false;   // sharded data path with collectives (world > 1, or CAKF_FORCE_COLLECTIVES=1 at world 1)
  ncclComm_t comm = nullptr;
  T *yloc = nullptr, *yred = nullptr;      // K1: this rank's reduced partial, all-reduced vector
  T *yslice = nullptr, *ygath = nullptr;   // K2: this rank's output row slice, all-gathered slices
  size_t k2_cmax = 0;

  static int k2_slice_rows(int M, int world_) {
    const int per = (M + world_ - 1) / world_;
    return ((per + 127) / 128) * 128;
  }

  cudaError_t k2_local(const V4<T>* xr, int M, const V4<T>* xc, int K, const T* B, size_t ldb, int C, T* Y,
                       size_t ldy, const int* acnt, const int* alist, int astride) {
    if constexpr (sizeof(T) == 4) {
      if (use_tc_k2())
        return launch_gram_gemm_tc(nu2, reinterpret_cast<const float4*>(xr), M, reinterpret_cast<const float4*>(xc), K,
                                   reinterpret_cast<const float*>(B), ldb, C, reinterpret_cast<float*>(Y), ldy, 1.0,
                                   tcw, st, acnt, alist, astride);
    }
    return launch_gram_gemm<T>(nu2, xr, M, xc, K, B, ldb, C, Y, ldy, 1.0, st);
  }

  // K2: Y = K(xr, xc) B — tcgen05 3xBF16 for fp32, SIMT for fp64 (or CAKF_K2_SIMT=1).  With row sharding
  // the callers pass their local rows (coords + plo, NX) and the matching slice of the culling lists.
  // acnt/alist: exact-zero culling lists of the 128-row tiles of xr (nullable)
  int k2(const V4<T>* xr, int M, const V4<T>* xc, int K, const T* B, size_t ldb, int C, T* Y, size_t ldy,
         const int* acnt = nullptr, const int* alist = nullptr, int astride = 0) {
    CK_CUDA(k2_local(xr, M, xc, K, B, ldb, C, Y, ldy, acnt, alist, astride));
    return CAKF_OK;
  }
  // sum of a small replicated-shape partial over the ranks (no-op without collectives)
  template <typename U>
  int allreduce(U* buf, size_t n) {
    if (!coll || !n) return CAKF_OK;
    CK_NCCL(ncclAllReduce(buf, buf, n, sizeof(U) == 4 ? ncclFloat32 : ncclFloat64, ncclSum, comm, st));
    return CAKF_OK;
  }

  // ---------------- profiling: CUDA events around launches of one category (cakf_profile)
  bool prof_on = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_done;  // (category, index of the start event)
  double prof_ms[CAKF_PROF_NCAT] = {0};
  int64_t prof_n[CAKF_PROF_NCAT] = {0};
  size_t prof_begin() {
    if (!prof_on) return SIZE_MAX;
    while (ev_pool.size() < ev_used + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return SIZE_MAX;
      ev_pool.push_back(e);
    }
    const size_t i = ev_used;
    ev_used += 2;
    cudaEventRecord(ev_pool[i], st);
    return i;
  }
  void prof_end(int cat, size_t i) {
    if (i == SIZE_MAX) return;
    cudaEventRecord(ev_pool[i + 1], st);
    ev_done.emplace_back(cat, i);
  }
  // fractions of the dense work performed: [K1 tile pairs, K2-post K-blocks, K2-smooth K-blocks] (1 = no culling)
  int cull_stats(double* out) override {
    out[0] = out[1] = out[2] = 1.0;
    if (!cull) return CAKF_OK;
    unsigned long long h[4];
    CK_CUDA(cudaMemcpyAsync(h, cull_ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    const double nx128 = (double)((NX + 127) / 128), nx32 = (double)((NX + 31) / 32);
    if (k1_pairs_dense > 0) out[0] = (double)h[0] / k1_pairs_dense;
    if (k2_post_dense > 0) out[1] = (double)h[1] / k2_post_dense;
    out[2] = (double)h[2] / (nx128 * nx32);
    return CAKF_OK;
  }

  int prof_read(double* ms, int64_t* n, bool reset_) override {
    CK_CUDA(cudaStreamSynchronize(st));
    for (auto& pr : ev_done) {
      float t = 0.f;
      CK_CUDA(cudaEventElapsedTime(&t, ev_pool[pr.second], ev_pool[pr.second + 1]));
      prof_ms[pr.first] += t;
      prof_n[pr.first] += 1;
    }
    ev_done.clear();
    ev_used = 0;
    for (int c = 0; c < CAKF_PROF_NCAT; ++c) {
      if (ms) ms[c] = prof_ms[c];
      if (n) n[c] = prof_n[c];
      if (reset_) { prof_ms[c] = 0.0; prof_n[c] = 0; }
    }
    return CAKF_OK;
  }

  int kcur = 0, phase = 0;  // phase: 0 ready (expect predict), 1 predicted, 2 updated
  bool smoothed = false;

  ~Impl() override {
    if (st) cudaStreamSynchronize(st);
    if (samp_ws) cudaFree(samp_ws);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (arena) cudaFree(arena);
    if (ctl_init_host) cudaFreeHost(ctl_init_host);
    if (comm) ncclCommDestroy(comm);
    if (sol) cusolverDnDestroy(sol);
    if (own_stream && st) cudaStreamDestroy(st);
    if (st2) cudaStreamDestroy(st2);
    if (st_t) {
      cudaStreamSynchronize(st_t);
      cudaStreamDestroy(st_t);
    }
    if (ev_tf) cudaEventDestroy(ev_tf);
    if (ev_td) cudaEventDestroy(ev_td);
    if (st_e) {
      cudaStreamSynchronize(st_e);
      cudaStreamDestroy(st_e);
    }
    if (ev_ea) cudaEventDestroy(ev_ea);
    if (ev_eb) cudaEventDestroy(ev_eb);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_ws) cudaEventDestroy(ev_ws);
    if (ev_kcar) cudaEventDestroy(ev_kcar);
  }

  template <typename U>
  U* carve(size_t count) {
    const size_t bytes = ((count * sizeof(U) + 255) / 256) * 256;
    if (arena) {
      U* p = reinterpret_cast<U*>(arena + arena_off);
      arena_off += bytes;
      return p;
    }
    arena_off += bytes;
    return nullptr;
  }

  int step_cap_cols(int k) const {
    if (k == 0) return 0;
    const long grow = (long)(k - 1) * nhat;
    const long rin = rcap >= 0 ? std::min<long>(rcap, grow) : grow;
    return (int)(rin + nhat);
  }

  void layout() {
    arena_off = 0;
    coords = carve<V4<T>>(NXf);
    mu0 = carve<T>(D);
    steps.resize(Tmax + 1);
    for (int k = 0; k <= Tmax; ++k) {
      Step& S = steps[k];
      S.cap_cols = step_cap_cols(k);
      S.m_pred = carve<T>(D);
      S.m = carve<T>(D);
      S.var = carve<T>(D);
      S.ms = carve<T>(D);
      S.vs = carve<T>(D);
      S.Mk = carve<T>((size_t)D * S.cap_cols);
      S.XV = k ? carve<T>((size_t)Nmax * (1 + nhat)) : nullptr;
      S.KV = k ? carve<T>((size_t)NX * (1 + nhat)) : nullptr;
      S.idx = k ? carve<int>(Nmax) : nullptr;
      S.kept = rcap > 0 ? carve<double>(rcap) : nullptr;
    }
    ctl = carve<IterCtl>(Tmax + 1);
    rin_max = rcap >= 0 ? rcap : std::max(0, (Tmax - 1) * nhat);
    qmax = rcap >= 0 ? std::max(rcap, nhat) : Tmax * nhat;   // W^s_T = W_T keeps n <= nhat columns (R6)
    cmax = std::max(rin_max + nhat, nhat + qmax);
    W = std::max(rin_max, nhat) + 8;
    xcs = carve<V4<T>>(Nmax);
    r = carve<T>(Nmax); s = carve<T>(Nmax); g = carve<T>(Nmax); gp = carve<T>(Nmax);
    d = carve<T>(Nmax); Gd = carve<T>(Nmax);
    ybuf = carve<T>(Nmax); lam2 = carve<T>(Nmax);
    Z = carve<T>((size_t)Nmax * std::max(nhat, 1));
    hmx = carve<T>((size_t)Nmax * (1 + std::max(rin_max, 1)));
    rbs = carve<T>(Nmax);
    HM = hmx + Nmax;
    const int nch = matvec_chunks((int)Nmax, (int)Nmax, sizeof(T));
    partial_cap = (size_t)std::max<int64_t>({(int64_t)nch, (int64_t)64, (int64_t)matvec_sym_tiles((int)Nmax)}) * Nmax;
    partial = carve<T>(partial_cap);
    stage64 = carve<int64_t>(std::max<int64_t>(Nmax, 3 * NXf));   // also the 3 x NX staged coordinates
    order32 = carve<int>(std::max(nhat, 1));
    part = carve<double>((size_t)(stage_blocks((int)Nmax) + 33) * W);   // block rows + group rows
    redA = carve<double>(W);
    redB = carve<double>(W);
    redC = carve<double>(W);
    cnt = carve<unsigned>(5 * 64);   // per reduction: [0] top, [1..32] group counters
    part2 = carve<double>((size_t)(stage_blocks((int)Nmax) + 33) * W);
    hmw = carve<double>((size_t)Nmax);
    Yb = carve<T>((size_t)std::max<int64_t>(NX, Nmax) * (1 + nhat));   // K2 post output or N x b action block
    Ub = carve<T>((size_t)std::max(rin_max, 1) * (1 + nhat));
    tmp = carve<T>(std::max<size_t>((size_t)D * (1 + nhat), (size_t)Nmax * blk));
    if (rcap >= 0) {
      gpart = carve<double>((size_t)nsplit_max * cmax * cmax);
      Gm = carve<double>((size_t)cmax * cmax);
      eigw = carve<double>(cmax);
      work = carve<double>(std::max(lwork, 1));
      info = carve<int>(4);
      QrD = carve<double>((size_t)cmax * std::max(rcap, 1));
      eigws_bytes = eig_workspace_bytes(cmax);
      eigws = carve<unsigned char>(eigws_bytes);
      Mtil = carve<T>((size_t)D * std::max(rcap, 1));
    }
    if (sizeof(T) == 4) {
      const size_t C1 = (size_t)(1 + qmax);
      dscr = std::max<size_t>({(size_t)D * (size_t)(std::max(cmax, 1 + qmax) + 1), (size_t)Nmax * C1,
                               (size_t)std::max(rin_max, 1) * C1, (size_t)std::max(nhat, 1) * C1,
                               (size_t)cmax * (size_t)std::max(rcap, 1), (size_t)Nmax * (size_t)(1 + nhat),
                               (size_t)std::max(rin_max, 1) * (size_t)(1 + nhat)});
    }
    fwork = carve<double>(kF64WorkDoubles);
    const size_t C = 1 + qmax;
    X = carve<T>((size_t)D * C);
    Yk = carve<T>((size_t)D * C);
    yb = carve<T>((size_t)D * C);
    Tm = carve<T>((size_t)std::max(rin_max, 1) * C);
    Hy = carve<T>((size_t)Nmax * C);
    tt = carve<T>((size_t)std::max(nhat, 1) * C);
    R = carve<T>((size_t)Nmax * C);
    Wf = carve<T>((size_t)D * (nhat + qmax));
    Ws = carve<T>((size_t)D * (nhat + qmax));
    ws = carve<T>(D);
    if (!smooth_k2) {
      KWf = carve<T>((size_t)D * (nhat + qmax));
      KWs = carve<T>((size_t)D * (nhat + qmax));
      Kws = carve<T>(D);
      Zk = carve<T>((size_t)NX * C);
    }
    pvar = carve<T>(D);
    perm_d = carve<int>(NXf);
    invperm_d = carve<int>(NXf);
    posof = carve<int>(NXf);
    obs_cnt = carve<int>((NXf + 1023) / 1024 + 1);
    sigma = carve<int>(Nmax);
    sigma_inv = carve<int>(Nmax);
    ip_m = carve<T>(D); ip_v = carve<T>(D); ip_ms = carve<T>(D); ip_vs = carve<T>(D);
    if (keep) {
      ws_st = carve<T>((size_t)(Tmax + 1) * D);
      Ws_st = carve<T>((size_t)(Tmax + 1) * D * std::max(qmax, 1));
    }
    y_st = carve<T>((size_t)(Tmax + 1) * Nmax);
    sig_st = carve<int>((size_t)(Tmax + 1) * Nmax);
    idx_tmp = carve<int>(Nmax);
    sig_tmp = carve<int>(Nmax);
    obs_cache_d = carve<int64_t>(Nmax);
    idx_cache = carve<int>(Nmax);
    sig_cache = carve<int>(Nmax);
    siginv_cache = carve<int>(Nmax);
    neq_d = carve<int>(1);
    kd_ws_bytes = kd_obs_workspace((int)Nmax);
    kd_ws = carve<unsigned char>(kd_ws_bytes);
    ybuf_user = carve<T>(Nmax);
    lam2_user = carve<T>(Nmax);
    outm = carve<T>(Df);
    outv = carve<T>(Df);
    if (coll) {
      yloc = carve<T>(Nmax);
      yred = carve<T>(Nmax);
      const size_t slice = (size_t)pslice;   // cakf_get: pack + all-gather of the local D rows
      yslice = carve<T>(slice * Dp);
      ygath = carve<T>(slice * Dp * world);
    }
    if (sizeof(T) == 4) {
      const size_t wb = std::max(gram_gemm_tc_workspace((int)Nmax, 1 + nhat),
                                 gram_gemm_tc_workspace((int)NX, Dp * (1 + qmax)));
      tcw = carve<float>(wb / sizeof(float) + 64);
      gp_elems = 3 * (dscr + 8 * (size_t)std::max<int64_t>({D, Nmax, (int64_t)cmax}) + 64);
      gpA = carve<uint16_t>(gp_elems);
      gpB = carve<uint16_t>(gp_elems);
      gwork = carve<float>(kGemmWorkFloats);
      gex_elems = (size_t)std::max<int64_t>({D, Nmax, (int64_t)cmax}) + gp_elems / 4096 + 1024;
      gexA = carve<int>(gex_elems);
      gexB = carve<int>(gex_elems);
      if (rcap >= 0) Qf = carve<float>((size_t)cmax * std::max(rcap, 1));
    }
    if (cull) {
      const int nx128 = (int)((NXf + 127) / 128), nx32 = (int)((NXf + 31) / 32);
      const int no128 = (int)((Nmax + 127) / 128), no32 = (int)((Nmax + 31) / 32);
      sph_x128 = carve<float4>(nx128); sph_x32 = carve<float4>(nx32);
      sph_o128 = carve<float4>(no128); sph_o32 = carve<float4>(no32);
      sph_o16 = carve<float4>((Nmax + 15) / 16 + 1);
      box_o32 = carve<float4>(2 * (size_t)no32); box_o16 = carve<float4>(2 * (size_t)((Nmax + 15) / 16 + 1));
      act_stride_sm = nx32; act_stride_po = no32;
      act_cnt_sm = carve<int>(nx128); act_list_sm = carve<int>((size_t)nx128 * nx32);
      act_cnt_po = carve<int>(nx128); act_list_po = carve<int>((size_t)nx128 * no32);
      cull_ctr = carve<unsigned long long>(4);
      k1_list = carve<int>((size_t)matvec_sym_units((int)Nmax) + 1);
      k1_mask = carve<unsigned short>((size_t)matvec_sym_units((int)Nmax) + 1);
      act_cnt_tt = carve<int>(no128);
      act_list_tt = carve<int>((size_t)no128 * no32);
      k1_count = carve<int>(64);   // [0] active-unit count, then launch_k1_active_units' group counters
    }
    k1_sched = carve<unsigned>(4);
    if (sizeof(T) == 4) {
      const size_t nbk = (size_t)matvec_sym_blocks((int)Nmax);
      k1_plist = carve<int>(nbk * nbk);
      k1_pq = carve<int>(nbk * 5);
    }
    k1_range = carve<long long>(2);
  }

  int init(const cakf_config& c) override {
    Dp = c.d_time; dim = c.space_dim; nu2 = c.spatial_kernel; policy = c.policy;
    nhat = c.max_iter; rcap = c.max_rank; Tmax = c.max_steps; NXf = c.n_space; Df = NXf * Dp;
    Nmax = c.max_obs > 0 ? std::min<int64_t>(c.max_obs, NXf) : NXf;
    rtol = c.rtol; ell = c.ell_x; seed = c.seed; reorth = c.reorth != 0;
    keep = c.keep_carriers != 0;
    blk = std::max(1, std::min<int>(c.block_actions, std::max(1, 1 + nhat)));
    cull = c.cull_zero != 0 && sizeof(T) == 4;
    world = std::max(1, c.world); rank = c.rank;
    {
      const char* fc = std::getenv("CAKF_FORCE_COLLECTIVES");
      coll = world > 1 || (fc && fc[0] == '1');
    }
    if (coll) {
      ncclUniqueId id;
      if (world == 1) {
        // single-rank communicator: the sharded path (slices, all-reduce, all-gather) runs on one GPU
        rank = 0;
        CK_NCCL(ncclGetUniqueId(&id));
      } else {
        if (!c.nccl_id || rank < 0 || rank >= world)
          return fail(CAKF_E_ARG, "multi-GPU: nccl_id and 0 <= rank < world needed");
        std::memcpy(&id, c.nccl_id, sizeof(id));
      }
      const ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
      if (r != ncclSuccess) return fail(CAKF_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    // this rank's rows: 128-aligned equal slices of the internal (kd-ordered, spatially compact) point order
    pslice = coll ? k2_slice_rows((int)NXf, world) : NXf;
    plo = std::min<int64_t>(NXf, (int64_t)rank * pslice);
    NX = std::max<int64_t>(0, std::min<int64_t>(NXf, plo + pslice) - plo);
    D = NX * Dp;
    if (NX < 1) return fail(CAKF_E_ARG, "multi-GPU: every rank needs at least one 128-point slice of the grid");
    if (world > 1 && smooth_k2) return fail(CAKF_E_UNSUPPORTED, "CAKF_SMOOTH_K2=1 is single-GPU only");
    if (rtol != 0.0) return fail(CAKF_E_UNSUPPORTED, "rtol != 0 is not supported by the device path (R2)");
    std::vector<double> st0;
    if (!fetch_doubles(c.sigma_t0, (size_t)Dp * Dp, st0)) return fail(CAKF_E_ARG, "cannot read sigma_t0");
    sig_t0 = mat_from(st0.data(), Dp);
    if (c.stream) st = (cudaStream_t)c.stream;
    else {
      CK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      own_stream = true;
    }
    if (c.max_rank >= 0 && eig_cusolver) {
      if (cusolverDnCreate(&sol) != CUSOLVER_STATUS_SUCCESS) return fail(CAKF_E_CUDA, "cusolverDnCreate failed");
      CK_SOLVER(cusolverDnSetStream(sol, st));
    }
    // size pass, then workspace query, then the real allocation
    layout();
    // the stage kernels keep one fp64 per kept column / previous action in (default, <= 48 KB) dynamic smem
    if (std::max(rin_max, nhat) > 6144)
      return fail(CAKF_E_UNSUPPORTED, "max_rank (or (T-1) max_iter without a cap) and max_iter must be <= 6144");
    if (rcap >= 0 && cmax > 0 && eig_cusolver) {
      CK_SOLVER(cusolverDnDsyevd_bufferSize(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, cmax, nullptr, cmax,
                                            nullptr, &lwork));
    }
    layout();
    arena_bytes = arena_off;
    cudaError_t e = cudaMalloc(&arena, arena_bytes);
    if (e != cudaSuccess) {
      arena = nullptr;
      return fail(CAKF_E_NOMEM, "trace arena of " + std::to_string(arena_bytes) + " bytes: " + cudaGetErrorString(e));
    }
    layout();
    CK_CUDA(cudaMemsetAsync(cnt, 0, 5 * 64 * sizeof(unsigned), st));
    CK_CUDA(cudaMemsetAsync(k1_sched, 0, 4 * sizeof(unsigned), st));
    if (side) {
      {  // highest priority: the side HM passes take SM slots ahead of queued K1 CTAs
        int lo = 0, hi = 0;
        CK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const char* e = getenv("CAKF_SIDE_PRIO");
        CK_CUDA(cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, (e && e[0] == '0') ? lo : hi));
      }
      CK_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      CK_CUDA(cudaStreamCreateWithFlags(&st_e, cudaStreamNonBlocking));
      CK_CUDA(cudaEventCreateWithFlags(&ev_ea, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&ev_eb, cudaEventDisableTiming));
      if (sizeof(T) == 4 && world == 1 && trunc_overlap()) {
        CK_CUDA(cudaStreamCreateWithFlags(&st_t, cudaStreamNonBlocking));
        CK_CUDA(cudaEventCreateWithFlags(&ev_tf, cudaEventDisableTiming));
        CK_CUDA(cudaEventCreateWithFlags(&ev_td, cudaEventDisableTiming));
      }
      CK_CUDA(cudaEventCreateWithFlags(&ev_ws, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&ev_kcar, cudaEventDisableTiming));
    }
    CK_CUDA(cudaMallocHost(&ctl_init_host, sizeof(IterCtl)));
    std::memset(ctl_init_host, 0, sizeof(IterCtl));
    ctl_init_host->eta_min = INFINITY;
    // coordinates: copy (host or device doubles) and prescale by sqrt(2 nu)/ell
    std::vector<double> xyz;
    if (!fetch_doubles(c.coords, (size_t)NXf * dim, xyz)) return fail(CAKF_E_ARG, "cannot read coords");
    make_perm(xyz);
    std::vector<int> inv(NXf);
    std::vector<double> xyz_int((size_t)NXf * dim);
    for (int64_t i = 0; i < NXf; ++i) {
      inv[perm_h[i]] = (int)i;
      for (int d = 0; d < dim; ++d) xyz_int[i * dim + d] = xyz[(size_t)perm_h[i] * dim + d];
    }
    CK_CUDA(cudaMemcpyAsync(perm_d, perm_h.data(), NXf * sizeof(int), cudaMemcpyHostToDevice, st));
    CK_CUDA(cudaMemcpyAsync(invperm_d, inv.data(), NXf * sizeof(int), cudaMemcpyHostToDevice, st));
    double* dxyz = reinterpret_cast<double*>(stage64);
    CK_CUDA(cudaMemcpyAsync(dxyz, xyz_int.data(), (size_t)NXf * dim * sizeof(double), cudaMemcpyHostToDevice, st));
    CK_CUDA(launch_prescale_coords<T>((int)NXf, dim, dxyz, std::sqrt((double)nu2) / ell, coords, st));
    if (cull) {  // the smoother's K2 lists depend on the (fixed) grid only
      const float4* xf = reinterpret_cast<const float4*>(coords);
      const int nx128 = (int)((NXf + 127) / 128), nx32 = (int)((NXf + 31) / 32);
      CK_CUDA(cudaMemsetAsync(cull_ctr, 0, 4 * sizeof(unsigned long long), st));
      CK_CUDA(launch_tile_spheres(xf, (int)NXf, 128, sph_x128, st));
      CK_CUDA(launch_tile_spheres(xf, (int)NXf, 32, sph_x32, st));
      CK_CUDA(launch_k2_active(sph_x128, nx128, sph_x32, nx32, kCullCut, act_cnt_sm, act_list_sm, act_stride_sm,
                               cull_ctr + 2, st));
    }
    std::vector<T> mu(D, T(0));   // this rank's rows of the prior mean, internal order
    if (c.mu0) {
      std::vector<double> m0;
      if (!fetch_doubles(c.mu0, Df, m0)) return fail(CAKF_E_ARG, "cannot read mu0");
      for (int d = 0; d < Dp; ++d)
        for (int64_t i = 0; i < NX; ++i) mu[d * NX + i] = (T)m0[d * NXf + perm_h[plo + i]];
    }
    CK_CUDA(cudaMemcpyAsync(mu0, mu.data(), D * sizeof(T), cudaMemcpyHostToDevice, st));
    CK_CUDA(cudaStreamSynchronize(st));
    return reset();
  }

  int reset() override {
    Step& S0 = steps[0];
    S0.sig_t = sig_t0;
    S0.rin = S0.cols = S0.n = S0.N = S0.rank_out = 0;
    S0.missing = true;
    S0.truncated = false;
    CK_CUDA(cudaMemcpyAsync(S0.m_pred, mu0, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(cudaMemcpyAsync(S0.m, mu0, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(StepKernels<T>::rowvar((int)NX, Dp, S0.sig_t, nullptr, S0.Mk, D, 0, S0.var, st));
    CK_CUDA(cudaMemcpyAsync(&ctl[0], ctl_init_host, sizeof(IterCtl), cudaMemcpyHostToDevice, st));
    kcur = 0;
    phase = 0;
    smoothed = false;
    failed_ = false;
    return CAKF_OK;
  }

  int predict(const double* A_t, const double* Q_t, const void* b) override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (phase != 0) return fail(CAKF_E_STATE, "predict: expected after create/reset/truncate");
    if (kcur >= Tmax) return fail(CAKF_E_ARG, "predict: max_steps exhausted");
    if (!A_t || !Q_t) return fail(CAKF_E_ARG, "predict: A_t and Q_t are required");
    std::vector<double> a, q;
    if (!fetch_doubles(A_t, (size_t)Dp * Dp, a) || !fetch_doubles(Q_t, (size_t)Dp * Dp, q))
      return fail(CAKF_E_ARG, "predict: cannot read A_t/Q_t");
    Step& P = steps[kcur];
    Step& S = steps[kcur + 1];
    const Mat3 A = mat_from(a.data(), Dp), Q = mat_from(q.data(), Dp);
    P.A_next = A;
    S.sig_t = mat_abat_plus_q(A, P.sig_t, Q, Dp);                     // Sigma^t_k
    CK_CUDA(StepKernels<T>::mix((int)NX, Dp, 1, A, false, P.m, D, S.m_pred, D, st));   // m^- = A m
    if (b) {   // user point order -> internal order (unpermute with the inverse permutation), this rank's rows
      CK_CUDA(cudaMemcpyAsync(outm, b, Df * sizeof(T), cudaMemcpyDefault, st));
      CK_CUDA(unpermute<T>((int)NXf, Dp, invperm_d, outm, outv, st));
      for (int d = 0; d < Dp; ++d)
        CK_CUDA(axpy<T>((size_t)NX, 1.0, outv + (size_t)d * NXf + plo, S.m_pred + (size_t)d * NX, st));
    }
    const T* src = P.truncated ? Mtil : P.Mk;
    const int rin = P.truncated ? P.rank_out : P.cols;
    S.rin = rin;                                                      // M^- = A M~   (Prop A.3)
    if (rin) {
      // M~ may still be in flight on the truncation stream: the mix follows it there (the update joins)
      cudaStream_t ms = trunc_pending ? st_t : st;
      CK_CUDA(StepKernels<T>::mix((int)NX, Dp, rin, A, false, src, D, S.Mk, D, ms));
      if (trunc_pending) CK_CUDA(cudaEventRecord(ev_td, st_t));
    }
    S.cols = rin;
    S.n = S.N = 0;
    S.missing = true;
    S.truncated = false;
    S.rank_out = rin;
    CK_CUDA(cudaMemcpyAsync(&ctl[kcur + 1], ctl_init_host, sizeof(IterCtl), cudaMemcpyHostToDevice, st));
    kcur += 1;
    phase = 1;
    smoothed = false;
    return CAKF_OK;
  }

  // Observations in the internal point order of this update: idx_out (kd order over the observed points),
  // sigma[j] = the user's position of row j, sigma_inv its inverse.  The order is a pure function of obs_idx
  // and is kept in a cache (idx_cache, sig_cache, siginv_cache): host-pointer callers compare on the host and
  // skip the recompute; device-pointer callers compare ON THE DEVICE (neq_d) and every kernel of the
  // recompute returns at once on a hit — no host round trip, the update stays stream-ordered.
  int stage_obs(int N, const int64_t* obs_idx, int* idx_out) {
    CK_CUDA(cudaMemcpyAsync(stage64, obs_idx, (size_t)N * sizeof(int64_t), cudaMemcpyDefault, st));
    const bool obs_host = !is_device_ptr(obs_idx);
    const int* run = nullptr;   // nullptr: recompute unconditionally
    bool recompute = true;
    if (obs_host) {
      recompute = !(obs_cache_n == N && obs_cache_h.size() == (size_t)N &&
                    std::memcmp(obs_idx, obs_cache_h.data(), (size_t)N * sizeof(int64_t)) == 0);
    } else if (obs_cache_n == N) {
      CK_CUDA(obs_neq(N, stage64, obs_cache_d, neq_d, st));   // *neq_d = 1 iff the set changed
      run = neq_d;
    }
    if (recompute) {
      if (kd_obs) {   // internal order, then the per-update kd order over the observed points
        CK_CUDA(obs_sort(N, (int)NXf, stage64, invperm_d, posof, obs_cnt, idx_tmp, sig_tmp, siginv_cache, st, run));
        CK_CUDA(kd_obs_order<T>(N, idx_tmp, coords, sig_cache, siginv_cache, idx_cache, sig_tmp, kd_ws, kd_ws_bytes,
                                st, run));
      } else {
        CK_CUDA(obs_sort(N, (int)NXf, stage64, invperm_d, posof, obs_cnt, idx_cache, sig_cache, siginv_cache, st,
                         run));
      }
      CK_CUDA(cudaMemcpyAsync(obs_cache_d, stage64, (size_t)N * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      if (obs_host) obs_cache_h.assign(obs_idx, obs_idx + N);
      else obs_cache_h.clear();
      obs_cache_n = N;
    }
    CK_CUDA(cudaMemcpyAsync(idx_out, idx_cache, (size_t)N * sizeof(int), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(cudaMemcpyAsync(sigma, sig_cache, (size_t)N * sizeof(int), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(cudaMemcpyAsync(sigma_inv, siginv_cache, (size_t)N * sizeof(int), cudaMemcpyDeviceToDevice, st));
    return CAKF_OK;
  }

  // K1 exactly as the inner loop launches it (observation order, exact-zero culling lists, dynamic unit
  // scheduler, symmetric partial slots), for one user vector s: out = K(X_obs, X_obs) s in the user's
  // observation order.  Test entry point (cakf_debug_matvec); clobbers the inner-loop workspaces.
  int debug_matvec(int64_t n_obs, const int64_t* obs_idx, const void* s_user, void* out_user, int shares) override {
    if (phase == 1) return fail(CAKF_E_STATE, "debug_matvec: not between predict and update");
    if (n_obs < 1 || n_obs > Nmax || !obs_idx || !s_user || !out_user) return fail(CAKF_E_ARG, "debug_matvec: bad argument");
    const int N = (int)n_obs;
    if (!is_device_ptr(obs_idx))
      for (int i = 0; i < N; ++i)
        if (obs_idx[i] < 0 || obs_idx[i] >= NXf) return fail(CAKF_E_ARG, "debug_matvec: obs_idx out of range");
    int* idx = sig_st;   // scratch index list: the sampler's per-step slot 0 (step 0 is never observed)
    CK(stage_obs(N, obs_idx, idx));
    CK_CUDA(cudaMemcpyAsync(ybuf_user, s_user, (size_t)N * sizeof(T), cudaMemcpyDefault, st));
    CK_CUDA(gather_vec<T>(N, sigma, ybuf_user, ybuf, st));
    CK_CUDA(sampler_ops<T>::gather_coords(N, idx, coords, xcs, st));
    CK_CUDA(set_w<T>(N, ybuf, xcs, st));
    const bool sym = sizeof(T) == 4 && use_sym_k1();
    const int nch = sym ? matvec_sym_tiles(N)
                        : std::max(1, std::min<int>(matvec_chunks(N, N, sizeof(T)), (int)(partial_cap / N)));
    if constexpr (sizeof(T) == 4) {
      if (sym) {
        if (cull) {
          const float4* xf = reinterpret_cast<const float4*>(xcs);
          CK_CUDA(launch_tile_spheres(xf, N, 128, sph_o128, st));
          CK_CUDA(launch_tile_spheres(xf, N, 32, sph_o32, st, box_o32));
          CK_CUDA(launch_tile_spheres(xf, N, 16, sph_o16, st, box_o16));
          CK_CUDA(cudaMemsetAsync(partial, 0, (size_t)matvec_sym_tiles(N) * N * sizeof(T), st));
        }
        // shares > 1: the multi-GPU split (units balanced by active tile pairs), every share in turn into the
        // same partial slots (disjoint units: the sum is the one-launch result bit for bit)
        const long long U = matvec_sym_units(N);
        for (int p = 0; p < std::max(1, shares); ++p) {
          if (cull) {
            if (shares > 1) {
              CK_CUDA(launch_k1_balanced_range(sph_o128, N, kCullCut, p, shares, k1_range, st));
              CK_CUDA(launch_k1_active_units(sph_o128, N, 0, U, kCullCut, k1_list, k1_mask, k1_count, st, k1_range));
            } else {
              CK_CUDA(launch_k1_active_units(sph_o128, N, 0, U, kCullCut, k1_list, k1_mask, k1_count, st));
            }
          }
          CK_CUDA(launch_matvec_sym(nu2, reinterpret_cast<const float4*>(xcs), N, reinterpret_cast<float*>(partial),
                                    cull ? 0 : U * p / std::max(1, shares), cull ? U : U * (p + 1) / std::max(1, shares),
                                    st, nullptr, cull ? k1_list : nullptr, k1_count, k1_mask, sph_o16, sph_o128,
                                    sph_o32, kCullCut, k1_sched, box_o16, box_o32));
        }
      } else {
        CK_CUDA(launch_matvec_partial<T>(nu2, xcs, N, xcs, N, nch, partial, st));
      }
    } else {
      CK_CUDA(launch_matvec_partial<T>(nu2, xcs, N, xcs, N, nch, partial, st));
    }
    CK_CUDA(launch_sum_partials<T>(N, nch, partial, 1.0, r, st));
    CK_CUDA(scatter_vec<T>(N, sigma, r, ybuf_user, st));
    CK_CUDA(cudaMemcpyAsync(out_user, ybuf_user, (size_t)N * sizeof(T), cudaMemcpyDefault, st));
    CK_CUDA(cudaStreamSynchronize(st));
    return CAKF_OK;
  }

  int update(int64_t n_obs, const int64_t* obs_idx, const void* y, const void* noise_var,
             const int64_t* coord_order) override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (phase != 1) return fail(CAKF_E_STATE, "update: expected after predict");
    if (n_obs < 0 || n_obs > Nmax) return fail(CAKF_E_ARG, "update: n_obs outside [0, max_obs]");
    Step& S = steps[kcur];
    const int k = kcur;
    const int N = (int)n_obs;
    if (N == 0) {                                                     // IsMissing
      CK(join_pending());   // rowvar reads M^-
      CK_CUDA(cudaMemcpyAsync(S.m, S.m_pred, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
      S.cols = S.rin;
      S.n = 0;
      S.N = 0;
      S.missing = true;
      CK_CUDA(StepKernels<T>::rowvar((int)NX, Dp, S.sig_t, nullptr, S.Mk, D, S.cols, S.var, st));
      phase = 2;
      return CAKF_OK;
    }
    if (!obs_idx || !y || !noise_var) return fail(CAKF_E_ARG, "update: obs_idx, y and noise_var are required");
    const int niter = std::min<int>(nhat, N);
    if (policy == CAKF_POLICY_COORD && niter > 0 && !coord_order)
      return fail(CAKF_E_ARG, "update: coordinate policy needs coord_order");
    if (!is_device_ptr(obs_idx)) {
      for (int i = 0; i < N; ++i)
        if (obs_idx[i] < 0 || obs_idx[i] >= NXf) return fail(CAKF_E_ARG, "update: obs_idx out of range");
    }
    if (policy == CAKF_POLICY_COORD && niter > 0 && !is_device_ptr(coord_order)) {
      for (int i = 0; i < niter; ++i)
        if (coord_order[i] < 0 || coord_order[i] >= N) return fail(CAKF_E_ARG, "update: coord_order out of range");
    }
    S.N = N;
    S.n = niter;
    S.missing = false;
    // ---- stage inputs (host or device pointers)
    CK(stage_obs(N, obs_idx, S.idx));
    CK_CUDA(cudaMemcpyAsync(ybuf_user, y, (size_t)N * sizeof(T), cudaMemcpyDefault, st));
    CK_CUDA(cudaMemcpyAsync(lam2_user, noise_var, (size_t)N * sizeof(T), cudaMemcpyDefault, st));
    CK_CUDA(gather_vec<T>(N, sigma, ybuf_user, ybuf, st));
    CK_CUDA(gather_vec<T>(N, sigma, lam2_user, lam2, st));
    CK_CUDA(cudaMemcpyAsync(y_st + (size_t)k * Nmax, ybuf, (size_t)N * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(cudaMemcpyAsync(sig_st + (size_t)k * Nmax, sigma, (size_t)N * sizeof(int), cudaMemcpyDeviceToDevice, st));
    if (policy == CAKF_POLICY_COORD && niter > 0) {
      CK_CUDA(cudaMemcpyAsync(stage64, coord_order, (size_t)niter * sizeof(int64_t), cudaMemcpyDefault, st));
      CK_CUDA(map_order(niter, stage64, sigma_inv, order32, st));
    }
    const int rin = S.rin;
    IterCtl* C = &ctl[k];
    // ---- [H m^-, H M^-] (N x (1 + rin)) from the ranks owning the observed rows (zeros elsewhere, summed),
    // then r^(0) and the first action
    HM = hmx + N;
    CK_CUDA(StepKernels<T>::gather_rows(N, 1, S.idx, S.m_pred, D, hmx, N, (int)plo, (int)NX, st));
    // H M^- needs M^- = A M~ (possibly still on the truncation stream): gathered after the first K1 then
    if (niter == 0) CK(join_pending());   // no first K1 to hide the truncation behind
    bool hm_ready = !trunc_pending;
    if (hm_ready) {
      if (rin) CK_CUDA(StepKernels<T>::gather_rows(N, rin, S.idx, S.Mk, D, HM, N, (int)plo, (int)NX, st));
      CK(allreduce(hmx, (size_t)N * (1 + rin)));
    } else {
      CK(allreduce(hmx, (size_t)N));   // H m^- now, H M^- after the first K1
    }
    CK_CUDA(StepKernels<T>::prep(N, S.idx, coords, ybuf, hmx, policy, order32, seed, k, sigma, r, s, S.XV, xcs, st, blk,
                                 rbs));
    const double sig00 = S.sig_t.a[0][0];
    const double eps = sizeof(T) == 4 ? (double)FLT_EPSILON : DBL_EPSILON;
    const bool sym = sizeof(T) == 4 && use_sym_k1();
    if (cull && N > 0) {  // spheres of the sorted observation tiles; K2-post lists against them
      const float4* xf = reinterpret_cast<const float4*>(xcs);
      CK_CUDA(launch_tile_spheres(xf, N, 128, sph_o128, st));
      CK_CUDA(launch_tile_spheres(xf, N, 32, sph_o32, st, box_o32));
      CK_CUDA(launch_tile_spheres(xf, N, 16, sph_o16, st, box_o16));
      CK_CUDA(launch_k2_active(sph_x128 + plo / 128, (int)((NX + 127) / 128), sph_o32, (N + 31) / 32, kCullCut,
                               act_cnt_po, act_list_po, act_stride_po, cull_ctr + 1, st));
      k2_post_dense += (double)((NX + 127) / 128) * ((N + 31) / 32);
      if (sym) {  // active K1 units of this rank; the skipped units' partial slots stay zero
        const long long U = matvec_sym_units(N);
        if (world > 1) {   // contiguous unit range holding 1/world of the active tile pairs (same on every rank)
          CK_CUDA(launch_k1_balanced_range(sph_o128, N, kCullCut, rank, world, k1_range, st));
          CK_CUDA(launch_k1_active_units(sph_o128, N, 0, U, kCullCut, k1_list, k1_mask, k1_count, st, k1_range));
        } else {
          CK_CUDA(launch_k1_active_units(sph_o128, N, 0, U, kCullCut, k1_list, k1_mask, k1_count, st));
        }
        CK_CUDA(cudaMemsetAsync(partial, 0, (size_t)matvec_sym_tiles(N) * N * sizeof(T), st));
      }
    }
    // the stage kernels sum only the K1 partial slots that can be nonzero, per 512-row block (all of them
    // without culling: the same sums in the same order, so culling stays bit-identical); single rank only
    // (the sharded K1 is summed by sum_partials before its all-reduce)
    const bool slot_lists = sym && !coll && k1_plist && N > 0 && slot_lists_on();
    if (slot_lists)
      CK_CUDA(launch_k1_block_partners(cull ? sph_o128 : nullptr, N, kCullCut, k1_plist, k1_pq, st));
    auto slots_for = [&](const T* kp) {
      SlotList sl;
      if (slot_lists && kp == partial) {
        sl.plist = k1_plist;
        sl.pq = k1_pq;
        sl.nb = matvec_sym_blocks(N);
      }
      return sl;
    };
    const int nch = sym ? matvec_sym_tiles(N)
                        : std::max(1, std::min<int>(matvec_chunks(N, N, sizeof(T)), (int)(partial_cap / N)));
    T* V = S.XV + N;
    // Non-adaptive policies (random, coordinate) with block_actions = b > 1: the actions of b
    // consecutive iterations are known in advance, so K_TT [s_i .. s_{i+b-1}] is one multi-RHS K2
    // product (tensor cores, each kernel value evaluated once for b columns) and the b iterations
    // then run the unchanged stage kernels on its columns — the same arithmetic as b sequential
    // iterations up to summation order (iterative = projected update for the same S).
    const bool blocked = blk > 1 && policy != CAKF_POLICY_CG && niter > 0;
    if (blocked && cull) {
      CK_CUDA(launch_k2_active(sph_o128, (N + 127) / 128, sph_o32, (N + 31) / 32, kCullCut, act_cnt_tt, act_list_tt,
                               act_stride_po, nullptr, st));
    }
    T* Sblk = tmp;   // N x b actions   (post-loop scratch, free during the loop)
    T* Yblk = Yb;    // N x b   K_TT S
    auto fork_hm = [&]() -> int {   // u = HM^T s and HM u on the side stream (joined before stage B)
      CK_CUDA(cudaEventRecord(ev_fork, st));
      CK_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
      CK_CUDA(StepKernels<T>::hmts(N, HM, rin, s, part2, W, redA, cnt + 256, st2));
      CK_CUDA(StepKernels<T>::hmu(N, HM, rin, redA, hmw, st2));
      CK_CUDA(cudaEventRecord(ev_join, st2));
      return CAKF_OK;
    };
    for (int i = 1; i <= niter; ++i) {
      // G s  (matrix-free: kernel rows on the fly + low-rank downdate + noise)
      bool fork = side && rin > 0;
      if (fork && hm_ready) CK(fork_hm());   // concurrently with K1
      size_t pk = prof_begin();
      const T* kpart = partial;
      int kch = nch;
      if (policy == CAKF_POLICY_COORD) {
        // K_TT e_j: the kernel columns of the chosen points (N evaluations each), b at a time
        const int j = (i - 1) % blk;
        if (j == 0) CK_CUDA(launch_kernel_columns<T>(nu2, xcs, N, order32, i, std::min(blk, niter - i + 1), Yblk, N, st));
        kpart = Yblk + (size_t)j * N;
        kch = 1;
      } else if (blocked) {
        const int j = (i - 1) % blk;
        if (j == 0) {
          const int nb = std::min(blk, niter - i + 1);
          CK_CUDA(StepKernels<T>::gen_actions(N, i, nb, policy, order32, seed, k, sigma, Sblk, N, st, rbs, blk));
          CK(k2(xcs, N, xcs, N, Sblk, N, nb, Yblk, N, cull ? act_cnt_tt : nullptr, act_list_tt, act_stride_po));
        }
        kpart = Yblk + (size_t)j * N;
        kch = 1;
      } else {
      // multi-GPU: this rank evaluates its share of the kernel work (sym units / column chunks),
      // the rest of the partial buffer is zero, and the reduced vector is all-reduced
      if (coll) CK_CUDA(cudaMemsetAsync(partial, 0, (size_t)nch * N * sizeof(T), st));
      if constexpr (sizeof(T) == 4) {
        if (sym) {
          const long long U = matvec_sym_units(N);
          // culling: the unit list (this rank's balanced share) defines the work; else the unit-index range
          CK_CUDA(launch_matvec_sym(nu2, reinterpret_cast<const float4*>(xcs), N, reinterpret_cast<float*>(partial),
                                    cull ? 0 : U * rank / world, cull ? U : U * (rank + 1) / world, st,
                                    cull ? cull_ctr : nullptr,
                                    cull ? k1_list : nullptr, k1_count, k1_mask, sph_o16, sph_o128, sph_o32, kCullCut,
                                    k1_sched, box_o16, box_o32));
          if (cull) {
            const double nt = (double)((N + 127) / 128);
            k1_pairs_dense += (double)matvec_sym_blocks_per_tile_pair() * nt * (nt + 1) / 2 / world;   // warp blocks
          }
        } else {
          CK_CUDA(launch_matvec_partial<T>(nu2, xcs, N, xcs, N, nch, partial, st, nch * rank / world,
                                           nch * (rank + 1) / world));
        }
      } else {
        CK_CUDA(launch_matvec_partial<T>(nu2, xcs, N, xcs, N, nch, partial, st, nch * rank / world,
                                         nch * (rank + 1) / world));
      }
      if (coll) {
        CK_CUDA(launch_sum_partials<T>(N, nch, partial, 1.0, yloc, st));
        CK_NCCL(ncclAllReduce(yloc, yred, (size_t)N, sizeof(T) == 4 ? ncclFloat32 : ncclFloat64, ncclSum, comm, st));
        kpart = yred;
        kch = 1;
      }
      }
      prof_end(CAKF_PROF_K1, pk);
      if (!hm_ready) {   // first iteration beside the previous truncation: join it, gather H M^-, fork now
        CK(join_pending());
        if (rin) CK_CUDA(StepKernels<T>::gather_rows(N, rin, S.idx, S.Mk, D, HM, N, (int)plo, (int)NX, st));
        CK(allreduce(HM, (size_t)N * rin));
        hm_ready = true;
        if (fork) CK(fork_hm());
      }
      pk = prof_begin();
      if ((fork || rin == 0) && stage_ab()) {   // stage A + B in one pass (HM u from the side stream)
        if (fork) CK_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
        CK_CUDA(StepKernels<T>::stageAB(N, kch, kpart, sig00, lam2, s, r, fork ? hmw : nullptr, g, V, i - 1, part, W,
                                        redB, redA + rin, cnt + 64, st, slots_for(kpart)));
      } else {
        CK_CUDA(StepKernels<T>::stageA(N, kch, kpart, sig00, lam2, s, r, gp, fork ? nullptr : HM, rin, part, W, redA,
                                       cnt, st, slots_for(kpart)));
        if (fork) CK_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
        CK_CUDA(StepKernels<T>::stageB(N, HM, rin, redA, gp, s, g, V, i - 1, part, W, redB, cnt + 64, st,
                                       fork ? hmw : nullptr));
      }
      if (reorth && i > 1) {  // CGS2 (R19): d = s - V c, then d -= V (V^T G d)
        CK_CUDA(StepKernels<T>::stageC(N, V, Z, i - 1, redB, s, g, d, Gd, s, redA, rin, redB + (i - 1), part, W, redC,
                                       cnt + 128, C, eps, i, 1, st));
        CK_CUDA(StepKernels<T>::stageC(N, V, Z, i - 1, redC, d, Gd, d, Gd, s, redA, rin, redB + (i - 1), part, W,
                                       nullptr, cnt + 128, C, eps, i, 0, st));
      } else {
        CK_CUDA(StepKernels<T>::stageC(N, V, Z, i - 1, redB, s, g, d, Gd, s, redA, rin, redB + (i - 1), part, W,
                                       nullptr, cnt + 128, C, eps, i, 0, st));
      }
      CK_CUDA(StepKernels<T>::stageD(N, i, niter, C, d, Gd, S.XV, Z, r, s, xcs, policy, order32, seed, k, sigma, st, blk,
                                     rbs));
      prof_end(CAKF_PROF_STAGES, pk);
    }
    CK_CUDA(StepKernels<T>::dot(N, r, r, part, &C->res_sq, cnt + 192, st));
    // ---- post-loop: [P^- w, P^- W] = Sigma H^T [v V] - M^- (H M^-)^T [v V]
    const int Cc = 1 + niter;
    size_t pk = prof_begin();
    CK(k2(coords + plo, (int)NX, xcs, N, S.XV, N, Cc, S.KV, NX, cull ? act_cnt_po : nullptr, act_list_po,
          act_stride_po));
    prof_end(CAKF_PROF_K2_POST, pk);
    if (rin) {
      pk = prof_begin();
      CK(gemm(OP_T, OP_N, rin, Cc, N, 1.0, HM, N, S.XV, N, 0.0, Ub, rin));
      CK(gemm(OP_N, OP_N, (int)D, Cc, rin, 1.0, S.Mk, (int)D, Ub, rin, 0.0, tmp, (int)D));
      prof_end(CAKF_PROF_LOWRANK, pk);
    }
    CK_CUDA(StepKernels<T>::post_combine((int)NX, Dp, Cc, S.sig_t, S.KV, rin ? tmp : nullptr, S.m_pred, S.m, S.Mk, rin,
                                         st));
    S.cols = rin + niter;
    CK_CUDA(StepKernels<T>::rowvar((int)NX, Dp, S.sig_t, nullptr, S.Mk, D, S.cols, S.var, st));
    phase = 2;
    return CAKF_OK;
  }

  // C = alpha op(A) op(B) + beta C with fp64 accumulation for both dtypes (B optionally already fp64):
  // fp32 with K >= i8_min_k on the INT8-slice tensor-core GEMM, everything else (short K, fp64 mode) on the
  // FP64-pipe GEMM of kernels_gemm_f64.cu (fp32 operands converted on load, one rounding of the result)
  int gemm_impl(bool ta, bool tb, int m, int n, int k, double alpha, const T* A, int lda, const T* B, const double* Bd,
                int ldb, double beta, T* C, int ldc) {
    if (m <= 0 || n <= 0) return CAKF_OK;
    if constexpr (sizeof(T) == 8) {
      const double* Bp = Bd ? Bd : reinterpret_cast<const double*>(B);
      CK_CUDA((gemm_f64acc<double, double, double>)(ta, tb, m, n, k, alpha, reinterpret_cast<const double*>(A),
                                                    (size_t)lda, Bp, (size_t)ldb, beta, reinterpret_cast<double*>(C),
                                                    (size_t)ldc, fwork, kF64WorkDoubles, st));
    } else if (!lowrank_tc && !Bd && k >= i8_min_k && use_i8_gemm()) {
      CK(gemm_i8_f32(ta, tb, m, n, k, alpha, reinterpret_cast<const float*>(A), lda,
                     reinterpret_cast<const float*>(B), ldb, beta, reinterpret_cast<float*>(C), nullptr, ldc));
    } else if (lowrank_tc) {
      // tcgen05 3xBF16 (kernels_gemm_tc.cu): op(A) rows m and op(B)^T rows n as K-major planes
      if (Bd) return fail(CAKF_E_ARG, "gemm: fp64 right operand on the tensor-core path");
      if (gemm_tc_plane_bytes(m, k) > gp_elems * 2 || gemm_tc_plane_bytes(n, k) > gp_elems * 2)
        return fail(CAKF_E_ARG, "gemm: operand planes too small");
      CK_CUDA(gemm_tc_split(reinterpret_cast<const float*>(A), m, k, (size_t)lda, ta, gpA, st));
      CK_CUDA(gemm_tc_split(reinterpret_cast<const float*>(B), n, k, (size_t)ldb, !tb, gpB, st));
      CK_CUDA(gemm_tc_run(gpA, m, gpB, n, k, alpha, beta, reinterpret_cast<float*>(C), nullptr, (size_t)ldc, gwork,
                          kGemmWorkFloats, st));
    } else if (Bd) {
      CK_CUDA((gemm_f64acc<float, double, float>)(ta, tb, m, n, k, alpha, reinterpret_cast<const float*>(A),
                                                  (size_t)lda, Bd, (size_t)ldb, beta, reinterpret_cast<float*>(C),
                                                  (size_t)ldc, fwork, kF64WorkDoubles, st));
    } else {
      CK_CUDA((gemm_f64acc<float, float, float>)(ta, tb, m, n, k, alpha, reinterpret_cast<const float*>(A),
                                                 (size_t)lda, reinterpret_cast<const float*>(B), (size_t)ldb, beta,
                                                 reinterpret_cast<float*>(C), (size_t)ldc, fwork, kF64WorkDoubles, st));
    }
    return CAKF_OK;
  }
  // fp32 operands, fp64-accurate product on the INT8 tensor cores (kernels_gemm_i8.cu): op(A) rows m and
  // op(B)^T rows n sliced into K-major planes; fp32 C or fp64 Cd; lower: only n <= m needed (Gram);
  // Bq (nullable) replaces B by an fp64 operand with the same layout
  int gemm_i8_f32(bool ta, bool tb, int m, int n, int k, double alpha, const float* A,
                  int lda, const float* B, int ldb, double beta, float* C, double* Cd, int ldc, bool lower = false,
                  const double* Bq = nullptr) {
    const size_t cap = gp_elems * 2;
    const size_t nch = (size_t)gemm_i8_nchunk(k);
    if (gemm_i8_plane_bytes(m, k) > cap || gemm_i8_plane_bytes(n, k) > cap || (size_t)m * nch > gex_elems ||
        (size_t)n * nch > gex_elems)
      return fail(CAKF_E_ARG, "gemm: INT8 slice planes too small");
    int8_t* pa = reinterpret_cast<int8_t*>(gpA);
    int8_t* pb = reinterpret_cast<int8_t*>(gpB);
    CK_CUDA(gemm_i8_split<float>(A, m, k, (size_t)lda, ta, pa, gexA, st));
    const bool same = B == A && tb != ta && ldb == lda && m == n && !Bq;   // A^T A: one set of planes
    if (Bq) CK_CUDA(gemm_i8_split<double>(Bq, n, k, (size_t)ldb, !tb, pb, gexB, st));
    else if (!same) CK_CUDA(gemm_i8_split<float>(B, n, k, (size_t)ldb, !tb, pb, gexB, st));
    CK_CUDA(gemm_i8_run(pa, gexA, m, same ? pa : pb, same ? gexA : gexB, n, k, alpha, beta, C, Cd, (size_t)ldc,
                        lower, reinterpret_cast<double*>(gwork), kGemmWorkFloats / 2, st));
    return CAKF_OK;
  }

  int gemm(bool ta, bool tb, int m, int n, int k, double alpha, const T* A, int lda,
           const T* B, int ldb, double beta, T* C, int ldc) {
    return gemm_impl(ta, tb, m, n, k, alpha, A, lda, B, nullptr, ldb, beta, C, ldc);
  }

  // Gram Gm = F^T F in fp64 (F fp32 or fp64, D x c, ld D; Gm ld c; the eigensolver reads the lower triangle)
  int gram_fp64(const T* F, int c) {
    if constexpr (sizeof(T) == 8)
      CK_CUDA((gemm_f64acc<double, double, double>)(true, false, c, c, (int)D, 1.0, reinterpret_cast<const double*>(F),
                                                    (size_t)D, reinterpret_cast<const double*>(F), (size_t)D, 0.0, Gm,
                                                    (size_t)c, fwork, kF64WorkDoubles, st));
    else
      CK_CUDA((gemm_f64acc<float, float, double>)(true, false, c, c, (int)D, 1.0, reinterpret_cast<const float*>(F),
                                                  (size_t)D, reinterpret_cast<const float*>(F), (size_t)D, 0.0, Gm,
                                                  (size_t)c, fwork, kF64WorkDoubles, st));
    return CAKF_OK;
  }

  // fp32 truncation on tcgen05: Gram F^T F (3xBF16, K split, fp64 reduction) -> fp64 eig -> F Q_r
  // top-rkeep eigenpairs of the Gram Gm (lower, ld c) -> QrD (c x rkeep, descending), kept, dropped mass;
  // fail: the step's IterCtl::nonfinite (reported by cakf_get_stats)
  int eig(int c, int rkeep, double* kept, double* dropped, int* failflag) {
    if (eig_cusolver) {
      CK_SOLVER(cusolverDnDsyevd(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, c, Gm, c, eigw, work, lwork,
                                 info));
      CK_CUDA(StepKernels<double>::take_top(c, rkeep, Gm, eigw, QrD, kept, dropped, st));
      return CAKF_OK;
    }
    // the eigensolver's own side stream (the T factors beside the divide and conquer)
    CK_CUDA(eig_top(c, rkeep, Gm, eigws, eigws_bytes, QrD, kept, dropped, nullptr, failflag, st, st_e, ev_ea, ev_eb));
    static const bool check = env_is("CAKF_EIG_CHECK", '1');
    if (check) {   // debug: residual of the returned eigenpairs against the (lower) Gram, on the host
      std::vector<double> G((size_t)c * c), Q((size_t)c * rkeep), w(c);
      CK_CUDA(cudaStreamSynchronize(st));
      CK_CUDA(cudaMemcpy(G.data(), Gm, G.size() * 8, cudaMemcpyDeviceToHost));
      CK_CUDA(cudaMemcpy(Q.data(), QrD, Q.size() * 8, cudaMemcpyDeviceToHost));
      double gmax = 0, res = 0, orth = 0;
      for (int i = 0; i < c; ++i)
        for (int j = 0; j <= i; ++j) gmax = std::max(gmax, std::fabs(G[i + (size_t)j * c]));
      for (int t = 0; t < rkeep; ++t) {
        const double* q = &Q[(size_t)t * c];
        std::vector<double> gq(c, 0.0);
        for (int i = 0; i < c; ++i)
          for (int j = 0; j < c; ++j) gq[i] += (i >= j ? G[i + (size_t)j * c] : G[j + (size_t)i * c]) * q[j];
        double lam = 0;
        for (int i = 0; i < c; ++i) lam += q[i] * gq[i];
        double rr = 0;
        for (int i = 0; i < c; ++i) rr += (gq[i] - lam * q[i]) * (gq[i] - lam * q[i]);
        res = std::max(res, std::sqrt(rr) / gmax);
        for (int u = 0; u < t; ++u) {
          double dd = 0;
          for (int i = 0; i < c; ++i) dd += q[i] * Q[(size_t)u * c + i];
          orth = std::max(orth, std::fabs(dd));
        }
      }
      fprintf(stderr, "eig check c=%d r=%d: residual %.3e orthogonality %.3e\n", c, rkeep, res, orth);
    }
    return CAKF_OK;
  }

  int truncate_factor_tc(const float* F, int c, int rkeep, float* out, double* kept, double* dropped, size_t pk,
                         const float* F2, float* out2, int* failflag) {
    size_t ps = prof_begin();
    if (gemm_tc_plane_bytes((int)D, c) > gp_elems * 2) return fail(CAKF_E_ARG, "truncate: operand planes too small");
    const bool i8 = use_i8_gemm();
    if (gram_tc) {
      CK_CUDA(gemm_tc_split(F, c, (int)D, (size_t)D, true, gpA, st));          // F^T rows (K = D contiguous)
      CK_CUDA(gemm_tc_run(gpA, c, gpA, c, (int)D, 1.0, 0.0, nullptr, Gm, (size_t)c, gwork, kGemmWorkFloats, st));
    } else if (i8) {   // exact products, fp64 sums: lower triangle of F^T F on the INT8 tensor cores
      CK(gemm_i8_f32(OP_T, OP_N, c, c, (int)D, 1.0, F, (int)D, F, (int)D, 0.0, nullptr, Gm, c, true));
    } else {   // the Gram decides the kept subspace: fp32 products, fp64 accumulation
      CK_CUDA((gemm_f64acc<float, float, double>)(true, false, c, c, (int)D, 1.0, F, (size_t)D, F, (size_t)D, 0.0, Gm,
                                                  (size_t)c, fwork, kF64WorkDoubles, st));
    }
    CK(allreduce(Gm, (size_t)c * c));   // row-sharded factor: the Gram is the sum of the ranks' partial Grams
    prof_end(CAKF_PROF_TRUNC_GRAM, ps);
    if (after_gram) {   // side-stream work that only the second GEMM needs: it runs beside the eigensolver
      std::function<int()> job;
      job.swap(after_gram);
      CK(job());
    }
    // filter truncation: the eigensolver and M Q_r on st_t (joined by the next update / any other call)
    const bool forked = fork_trunc && !F2;
    cudaStream_t main_st = st;
    if (forked) {
      CK_CUDA(cudaEventRecord(ev_tf, st));
      CK_CUDA(cudaStreamWaitEvent(st_t, ev_tf, 0));
      st = st_t;
    }
    const int rc_t = truncate_eig_gemm(F, c, rkeep, out, kept, dropped, failflag, F2, out2, i8);
    if (forked) {
      st = main_st;
      if (rc_t == CAKF_OK) {
        CK_CUDA(cudaEventRecord(ev_td, st_t));
        trunc_pending = true;
      }
    }
    CK(rc_t);
    prof_end(CAKF_PROF_TRUNCATE, pk);
    return CAKF_OK;
  }

  int truncate_eig_gemm(const float* F, int c, int rkeep, float* out, double* kept, double* dropped, int* failflag,
                        const float* F2, float* out2, bool i8) {
    size_t ps = prof_begin();
    CK(eig(c, rkeep, kept, dropped, failflag));
    prof_end(CAKF_PROF_TRUNC_EIG, ps);
    ps = prof_begin();
    if (i8 && i8_mqr) {   // M~ = F Q_r with the fp64 eigenvectors sliced directly
      CK(gemm_i8_f32(OP_N, OP_N, (int)D, rkeep, c, 1.0, F, (int)D, nullptr, c, 0.0, out, nullptr,
                     (int)D, false, QrD));
      if (F2 && f2_wait) CK_CUDA(cudaStreamWaitEvent(st, f2_wait, 0));
      f2_wait = nullptr;
      if (F2)
        CK(gemm_i8_f32(OP_N, OP_N, (int)D, rkeep, c, 1.0, F2, (int)D, nullptr, c, 0.0, out2, nullptr,
                       (int)D, false, QrD));
    } else {
      CK_CUDA((convert<double, float>)(c, rkeep, QrD, c, Qf, c, st));
      CK_CUDA(gemm_tc_split(F, (int)D, c, (size_t)D, false, gpA, st));           // F rows (K = c, transposed)
      CK_CUDA(gemm_tc_split(Qf, rkeep, c, (size_t)c, true, gpB, st));           // Q_r columns
      CK_CUDA(gemm_tc_run(gpA, (int)D, gpB, rkeep, c, 1.0, 0.0, out, nullptr, (size_t)D, gwork, kGemmWorkFloats,
                          st));
      if (F2 && f2_wait) CK_CUDA(cudaStreamWaitEvent(st, f2_wait, 0));
      f2_wait = nullptr;
      if (F2) {   // same Q_r planes
        CK_CUDA(gemm_tc_split(F2, (int)D, c, (size_t)D, false, gpA, st));
        CK_CUDA(gemm_tc_run(gpA, (int)D, gpB, rkeep, c, 1.0, 0.0, out2, nullptr, (size_t)D, gwork, kGemmWorkFloats,
                            st));
      }
    }
    prof_end(CAKF_PROF_TRUNC_GEMM, ps);
    return CAKF_OK;
  }

  // Truncate a D x c factor F (ld D) to its top-r Gram eigen-directions: out = F Q_r; F2 (nullable, D x c)
  // gets the same Q_r: out2 = F2 Q_r (the smoother's kernel-applied carriers).
  int truncate_factor(const T* F, int c, int rkeep, T* out, double* kept, double* dropped, int* failflag,
                      const T* F2 = nullptr, T* out2 = nullptr) {
    const size_t pk = prof_begin();
    if constexpr (sizeof(T) == 4) {
      if (use_tc_gemm()) return truncate_factor_tc(reinterpret_cast<const float*>(F), c, rkeep,
                                                   reinterpret_cast<float*>(out), kept, dropped, pk,
                                                   reinterpret_cast<const float*>(F2), reinterpret_cast<float*>(out2),
                                                   failflag);
    }
    // fp64 accumulation for the Gram and M Q_r on the FP64 pipe (CAKF_GEMM_F64=1 for fp32, and fp64 mode)
    size_t ps = prof_begin();
    CK(gram_fp64(F, c));
    CK(allreduce(Gm, (size_t)c * c));   // row-sharded factor: the Gram is the sum of the ranks' partial Grams
    prof_end(CAKF_PROF_TRUNC_GRAM, ps);
    if (after_gram) {   // side-stream work that only the second GEMM needs: it runs beside the eigensolver
      std::function<int()> job;
      job.swap(after_gram);
      CK(job());
    }
    ps = prof_begin();
    CK(eig(c, rkeep, kept, dropped, failflag));
    prof_end(CAKF_PROF_TRUNC_EIG, ps);
    ps = prof_begin();
    CK(gemm_impl(false, false, (int)D, rkeep, c, 1.0, F, (int)D, nullptr, QrD, c, 0.0, out, (int)D));
    if (F2 && f2_wait) CK_CUDA(cudaStreamWaitEvent(st, f2_wait, 0));
    f2_wait = nullptr;
    if (F2) CK(gemm_impl(false, false, (int)D, rkeep, c, 1.0, F2, (int)D, nullptr, QrD, c, 0.0, out2, (int)D));
    prof_end(CAKF_PROF_TRUNC_GEMM, ps);
    prof_end(CAKF_PROF_TRUNCATE, pk);
    return CAKF_OK;
  }

  int truncate() override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (phase == 1) CK(update(0, nullptr, nullptr, nullptr, nullptr));
    if (phase != 2) return fail(CAKF_E_STATE, "truncate: expected after update");
    Step& S = steps[kcur];
    if (rcap < 0 || S.cols <= rcap) {
      S.truncated = false;
      S.rank_out = S.cols;
    } else {
      fork_trunc = st_t != nullptr;
      const int trc = truncate_factor(S.Mk, S.cols, rcap, Mtil, S.kept, &ctl[kcur].dropped, &ctl[kcur].nonfinite);
      fork_trunc = false;
      CK(trc);   // Sec. 3.2
      S.truncated = true;
      S.rank_out = rcap;
    }
    phase = 0;
    return CAKF_OK;
  }

  int smooth() override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (phase != 0 || kcur < 1) return fail(CAKF_E_STATE, "caks_smooth: expected after >= 1 truncated step");
    const int T_ = kcur;
    Step& ST = steps[T_];
    CK_CUDA(cudaMemcpyAsync(ST.ms, ST.m, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK_CUDA(cudaMemcpyAsync(ST.vs, ST.var, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
    // w^s_T = H^T v_T, W^s_T = H^T V_T  (alg:mfks lines 2-3)
    int q = ST.n;
    CK_CUDA(StepKernels<T>::fill(D, T(0), X, st));
    CK_CUDA(StepKernels<T>::fill((size_t)std::max(ST.N, 1), T(0), R, st));
    CK_CUDA(StepKernels<T>::ws_build(ST.N, D, ST.n, 0, ST.idx, X, ST.XV, R, Ws, ws, (int)plo, (int)NX, st));
    // (I (x) K) of the carriers: [K(X,T) v_T; 0], [K(X,T) V_T; 0] from the stored post-loop products
    if (!smooth_k2) CK_CUDA(StepKernels<T>::kcar_build(NX, Dp, ST.n, 0, ST.KV, nullptr, nullptr, KWs, Kws, st));
    ST.smoother_rank = q;
    CK(keep_carriers(T_, q));
    for (int k = T_ - 1; k >= 0; --k) {
      Step& S = steps[k];
      const int C = 1 + q;
      // x = A_k^T [w^s_{k+1}, W^s_{k+1}]
      CK_CUDA(StepKernels<T>::mix((int)NX, Dp, 1, S.A_next, true, ws, D, X, D, st));
      if (q) CK_CUDA(StepKernels<T>::mix((int)NX, Dp, q, S.A_next, true, Ws, D, X + D, D, st));
      // Sigma_k x = (Sigma^t_k (x) K) x : K applied to all D' blocks of all C columns at once
      size_t pk = prof_begin();
      if (smooth_k2) {
        CK(k2(coords, (int)NX, coords, (int)NX, X, NX, Dp * C, Yk, NX, cull ? act_cnt_sm : nullptr, act_list_sm,
              act_stride_sm));
        ++k2_sm_launches;
      } else {
        // (I (x) K) x = (A^T (x) I) (I (x) K)[w^s, W^s]: the carriers' kernel products, kept exactly by
        // linearity (K (F Q) = (K F) Q, K H^T V t = (K(X,T) V) t), so no kernel is evaluated here
        CK_CUDA(StepKernels<T>::mix((int)NX, Dp, 1, S.A_next, true, Kws, D, Yk, D, st));
        if (q) CK_CUDA(StepKernels<T>::mix((int)NX, Dp, q, S.A_next, true, KWs, D, Yk + D, D, st));
      }
      prof_end(CAKF_PROF_K2_SMOOTH, pk);
      CK_CUDA(StepKernels<T>::sigma_apply((int)NX, Dp, C, S.sig_t, Yk, yb, st));
      const int rin = S.rin, n = S.n, N = S.N;
      // y = P^-_k x = Sigma x - M^- (M^-^T x)
      pk = prof_begin();
      if (rin) {
        CK(gemm(OP_T, OP_N, rin, C, (int)D, 1.0, S.Mk, (int)D, X, (int)D, 0.0, Tm, rin));
        CK(allreduce(Tm, (size_t)rin * C));   // M^-T x over all rows: sum of the ranks' partial products
        CK(gemm(OP_N, OP_N, (int)D, C, rin, -1.0, S.Mk, (int)D, Tm, rin, 1.0, yb, (int)D));
      }
      // P_k x = y - B_k (V^T H y);  R = V (V^T H y)
      if (n) {
        T* Vk = S.XV + N;
        CK_CUDA(StepKernels<T>::gather_rows(N, C, S.idx, yb, D, Hy, N, (int)plo, (int)NX, st));
        CK(gemm(OP_T, OP_N, n, C, N, 1.0, Vk, N, Hy, N, 0.0, tt, n));
        CK(allreduce(tt, (size_t)n * C));     // V^T H y: each rank holds the observed rows it owns (zeros elsewhere)
        CK(gemm(OP_N, OP_N, (int)D, C, n, -1.0, S.Mk + (size_t)rin * D, (int)D, tt, n, 1.0, yb, (int)D));
        CK(gemm(OP_N, OP_N, N, C, n, 1.0, Vk, N, tt, n, 0.0, R, N));
      }
      prof_end(CAKF_PROF_LOWRANK, pk);
      // m^s_k = m_k + P_k A^T w^s ;  var^s_k = var_k - rowsumsq(P_k A^T W^s)   (lines 5-6)
      // (with the carriers below: nothing else in the step reads m^s_k / var^s_k)
      if (smooth_k2) CK_CUDA(StepKernels<T>::smooth_out(D, C, S.m, S.var, yb, S.ms, S.vs, st));
      // w^s_k, W^s_k = [W_k, (I - W W^T P^-) A^T W^s]   (lines 7-8)
      CK_CUDA(StepKernels<T>::ws_build(n ? N : 0, D, n, q, S.idx, X, S.XV, R, Wf, ws, (int)plo, (int)NX, st));
      bool kcar_side = false;
      if (!smooth_k2) {
        // (I (x) K) W^s_full = [[K(X,T) V; 0], Kx[:,1:] - [K(X,T) V t[:,1:]; 0]], same for w^s with column 0.
        // fp32 with K = n <= 64 (the workspace-free strip GEMM): on the side stream, beside the truncation's
        // Gram and eig (16 SMs) — they only feed its second GEMM and the next step (joined below)
        const int qn_ = n + q;
        kcar_side = sizeof(T) == 4 && side && st2 && n <= 64 && NX >= 512 && smooth_overlap() && rcap >= 0 &&
                    qn_ > rcap;   // a truncation follows: fork after its Gram, beside the eigensolver
        const T* KVk = S.KV;
        T *mk = S.m, *vk = S.var, *msk = S.ms, *vsk = S.vs;
        auto carriers = [this, n, q, C, KVk, mk, vk, msk, vsk](cudaStream_t on) -> int {
          CK_CUDA(StepKernels<T>::smooth_out(D, C, mk, vk, yb, msk, vsk, on));   // m^s_k, var^s_k (lines 5-6)
          cudaStream_t main_st = st;
          st = on;   // gemm() and prof_* use the member stream
          size_t pk2 = prof_begin();
          int rc = CAKF_OK;
          if (n) rc = gemm(OP_N, OP_N, (int)NX, C, n, 1.0, KVk + NX, (int)NX, tt, n, 0.0, Zk, (int)NX);
          prof_end(CAKF_PROF_LOWRANK, pk2);
          st = main_st;
          CK(rc);
          CK_CUDA(StepKernels<T>::kcar_build(NX, Dp, n, q, KVk, n ? Zk : nullptr, Yk, KWf, Kws, on));
          return CAKF_OK;
        };
        if (kcar_side) {
          after_gram = [this, carriers]() -> int {
            CK_CUDA(cudaEventRecord(ev_ws, st));
            CK_CUDA(cudaStreamWaitEvent(st2, ev_ws, 0));
            CK(carriers(st2));
            CK_CUDA(cudaEventRecord(ev_kcar, st2));
            f2_wait = ev_kcar;
            return CAKF_OK;
          };
        } else {
          CK(carriers(st));
        }
      }
      const int qn = n + q;
      if (rcap >= 0 && qn > rcap) {                                   // line 9 (R6)
        const int trc = truncate_factor(Wf, qn, rcap, Ws, nullptr, nullptr, &ctl[k].nonfinite,
                                        smooth_k2 ? nullptr : KWf, KWs);
        after_gram = nullptr;   // (consumed inside unless the truncation failed early)
        CK(trc);
        q = rcap;
      } else {
        if (f2_wait) CK_CUDA(cudaStreamWaitEvent(st, f2_wait, 0));
        f2_wait = nullptr;
        std::swap(Wf, Ws);
        if (!smooth_k2) std::swap(KWf, KWs);
        q = qn;
      }
      if (kcar_side) CK_CUDA(cudaStreamWaitEvent(st, ev_kcar, 0));   // carriers complete before the next step
      f2_wait = nullptr;
      S.smoother_rank = q;
      CK(keep_carriers(k, q));
    }
    smoothed = true;
    return CAKF_OK;
  }

  int keep_carriers(int k, int q) {
    if (!keep) return CAKF_OK;
    if (q > std::max(qmax, 1)) return fail(CAKF_E_ARG, "smoother carrier rank exceeds the kept capacity");
    CK_CUDA(cudaMemcpyAsync(ws_st + (size_t)k * D, ws, D * sizeof(T), cudaMemcpyDeviceToDevice, st));
    if (q)
      CK_CUDA(cudaMemcpyAsync(Ws_st + (size_t)k * D * std::max(qmax, 1), Ws, (size_t)D * q * sizeof(T),
                              cudaMemcpyDeviceToDevice, st));
    return CAKF_OK;
  }

  // Cor. A.10 / alg:cakf-interpolation / alg:caks-interpolation: the filter (and
  // smoother) state at t in [t_k, t_{k+1}) from the stored step-k filter state, the filter factor
  // M~_k and the step-(k+1) smoother carriers; A1 = A(t, t_k), Q1 = Q(t, t_k), A2 = A(t_{k+1}, t).
  // M~_k = (A_{k+1}^-1 (x) I) M^-_{k+1} for k < T (already stored), else the last truncation output.
  int interpolate(int k, const double* A1p, const double* Q1p, const double* A2p, int which, void* mean,
                  void* var) override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (world > 1) return fail(CAKF_E_UNSUPPORTED, "cakf_interpolate: single-GPU handles only");
    if (k < 1 || k > kcur) return fail(CAKF_E_ARG, "interpolate: k outside [1, steps done]");
    if (k == kcur && phase != 0) return fail(CAKF_E_STATE, "interpolate: step k not truncated yet");
    if (which != CAKF_FILTER && which != CAKF_SMOOTH) return fail(CAKF_E_ARG, "interpolate: bad which");
    const bool smooth_q = which == CAKF_SMOOTH;
    if (smooth_q && !smoothed) return fail(CAKF_E_STATE, "interpolate: caks_smooth has not run");
    if (smooth_q && k < kcur && !keep) return fail(CAKF_E_STATE, "interpolate: create with keep_carriers = 1");
    if (!A1p || !Q1p || (smooth_q && k < kcur && !A2p))
      return fail(CAKF_E_ARG, "interpolate: A1, Q1 (and A2) are required");
    std::vector<double> a1, q1, a2;
    if (!fetch_doubles(A1p, (size_t)Dp * Dp, a1) || !fetch_doubles(Q1p, (size_t)Dp * Dp, q1))
      return fail(CAKF_E_ARG, "interpolate: cannot read A1/Q1");
    const Mat3 A1 = mat_from(a1.data(), Dp), Q1 = mat_from(q1.data(), Dp);
    Step& S = steps[k];
    const Mat3 sig_t = mat_abat_plus_q(A1, S.sig_t, Q1, Dp);          // Sigma^t(t)
    CK_CUDA(StepKernels<T>::mix((int)NX, Dp, 1, A1, false, S.m, D, ip_m, D, st));   // m(t) = A1 m_k
    // M(t) = A1 M~_k, into the smoother scratch Wf
    int rt = 0;
    if (k < kcur) {
      const Step& S1 = steps[k + 1];
      Mat3 Ainv{};
      if (!mat_inv(S.A_next, Dp, Ainv)) return fail(CAKF_E_NUMERIC, "interpolate: singular A_{k+1}");
      rt = S1.rin;
      if (rt) CK_CUDA(StepKernels<T>::mix((int)NX, Dp, rt, mat_mul(A1, Ainv, Dp), false, S1.Mk, D, Wf, D, st));
    } else {
      rt = S.truncated ? S.rank_out : S.cols;
      if (rt) CK_CUDA(StepKernels<T>::mix((int)NX, Dp, rt, A1, false, S.truncated ? Mtil : S.Mk, D, Wf, D, st));
    }
    CK_CUDA(StepKernels<T>::rowvar((int)NX, Dp, sig_t, nullptr, Wf, D, rt, ip_v, st));
    const T *pm = ip_m, *pv = ip_v;
    if (smooth_q && k < kcur) {
      if (!fetch_doubles(A2p, (size_t)Dp * Dp, a2)) return fail(CAKF_E_ARG, "interpolate: cannot read A2");
      const Mat3 A2 = mat_from(a2.data(), Dp);
      const int q = steps[k + 1].smoother_rank, C = 1 + q;
      const T* wsk = ws_st + (size_t)(k + 1) * D;
      const T* Wsk = Ws_st + (size_t)(k + 1) * D * std::max(qmax, 1);
      // x = A2^T [w^s_{k+1}, W^s_{k+1}];  y = P(t) x = Sigma(t) x - M(t) (M(t)^T x)
      CK_CUDA(StepKernels<T>::mix((int)NX, Dp, 1, A2, true, wsk, D, X, D, st));
      if (q) CK_CUDA(StepKernels<T>::mix((int)NX, Dp, q, A2, true, Wsk, D, X + D, D, st));
      CK(k2(coords, (int)NX, coords, (int)NX, X, NX, Dp * C, Yk, NX, cull ? act_cnt_sm : nullptr, act_list_sm,
            act_stride_sm));
      CK_CUDA(StepKernels<T>::sigma_apply((int)NX, Dp, C, sig_t, Yk, yb, st));
      if (rt) {
        CK(gemm(OP_T, OP_N, rt, C, (int)D, 1.0, Wf, (int)D, X, (int)D, 0.0, Tm, rt));
        CK(gemm(OP_N, OP_N, (int)D, C, rt, -1.0, Wf, (int)D, Tm, rt, 1.0, yb, (int)D));
      }
      // m^s(t) = m(t) + y_0 ; var^s(t) = var(t) - rowsumsq(y_{1:})
      CK_CUDA(StepKernels<T>::smooth_out(D, C, ip_m, ip_v, yb, ip_ms, ip_vs, st));
      pm = ip_ms;
      pv = ip_vs;
    }
    if (mean) {
      CK_CUDA(unpermute<T>((int)NX, Dp, perm_d, pm, outm, st));
      CK_CUDA(cudaMemcpyAsync(mean, outm, D * sizeof(T), cudaMemcpyDefault, st));
    }
    if (var) {
      CK_CUDA(unpermute<T>((int)NX, Dp, perm_d, pv, outv, st));
      CK_CUDA(cudaMemcpyAsync(var, outv, D * sizeof(T), cudaMemcpyDefault, st));
    }
    CK_CUDA(cudaStreamSynchronize(st));
    return CAKF_OK;
  }

  // alg:cakf-caks-sampler: S posterior samples from the stored filter trace and the
  // caller's prior draws (x0 ~ N(mu_0, Sigma_0), q_{k-1} ~ N(0, Q_{k-1}), eps_k ~ N(0, Lambda_k)).
  // Forward: x^-_k = A x_{k-1} + q_{k-1}; w_k = H^T V_k V_k^T (y_k - H x^-_k - eps_k) (R25);
  // x_k = x^-_k + P^-_k w_k.  Backward: x^s_k = x_k + P_k A_k^T w^s_{k+1};
  // w^s_k = w_k + (I - W_k W_k^T P^-_k) A_k^T w^s_{k+1}.  Same kernels as the update / smoother.
  int sample(int S, const void* x0, const void* q, const void* eps, int which, void* out) override {
    if (failed_) return fail(CAKF_E_STATE, "handle failed earlier");
    if (world > 1) return fail(CAKF_E_UNSUPPORTED, "cakf_sample: single-GPU handles only");
    if (phase != 0 || kcur < 1) return fail(CAKF_E_STATE, "sample: expected after the last truncate");
    if (S < 1 || S > 1 + std::min(nhat, qmax)) return fail(CAKF_E_ARG, "sample: n_samples outside [1, 1 + max_iter]");
    if (which != CAKF_FILTER && which != CAKF_SMOOTH) return fail(CAKF_E_ARG, "sample: bad which");
    if (!x0 || !q || !out || !eps) return fail(CAKF_E_ARG, "sample: x0, q, eps and out are required");
    const int T_ = kcur;
    const size_t DS = (size_t)D * S;
    // device workspace: forward samples x_0..x_T, their w_k (as u_k = V V^T res, N_k x S), staging
    size_t n_obs_total = 0;
    for (int k = 1; k <= T_; ++k) n_obs_total += (size_t)steps[k].N;
    T* xs = nullptr;
    const size_t bytes = ((size_t)(T_ + 1) * DS + 3 * DS + n_obs_total * S * 2 + 1024) * sizeof(T);
    // grow-only workspace kept by the handle (no allocation inside repeated sampler calls)
    if (samp_bytes < bytes) {
      if (samp_ws) CK_CUDA(cudaFreeAsync(samp_ws, st));
      samp_ws = nullptr;
      samp_bytes = 0;
      CK_CUDA(cudaMallocAsync(&samp_ws, bytes, st));
      samp_bytes = bytes;
    }
    xs = static_cast<T*>(samp_ws);
    T* xtmp = xs + (size_t)(T_ + 1) * DS;   // D x S scratch (user order staging)
    T* wsv = xtmp + DS;                     // w^s (D x S)
    T* xsm = wsv + DS;                      // one smoother sample (D x S)
    T* ust = xsm + DS;                      // u_k per step (N_k x S)
    T* epsd = ust + n_obs_total * S;        // eps of all steps (device copy)
    std::vector<size_t> uoff(T_ + 2, 0);
    for (int k = 1; k <= T_; ++k) uoff[k + 1] = uoff[k] + (size_t)steps[k].N * S;
    auto cleanup = [&]() {};
    auto run = [&]() -> int {
      CK_CUDA(cudaMemcpyAsync(epsd, eps, n_obs_total * S * sizeof(T), cudaMemcpyDefault, st));
      // x_0 (user order) -> internal
      CK_CUDA(cudaMemcpyAsync(xtmp, x0, DS * sizeof(T), cudaMemcpyDefault, st));
      CK_CUDA(sampler_ops<T>::permute_cols((int)NX, Dp, S, invperm_d, xtmp, D, xs, D, st));
      for (int k = 1; k <= T_; ++k) {
        Step& P = steps[k - 1];
        Step& K = steps[k];
        T* xk = xs + (size_t)k * DS;
        // x^-_k = A x_{k-1} + q_{k-1}
        CK_CUDA(StepKernels<T>::mix((int)NX, Dp, S, P.A_next, false, xs + (size_t)(k - 1) * DS, D, xk, D, st));
        CK_CUDA(cudaMemcpyAsync(xtmp, static_cast<const T*>(q) + (size_t)(k - 1) * DS, DS * sizeof(T),
                                cudaMemcpyDefault, st));
        CK_CUDA(sampler_ops<T>::permute_cols((int)NX, Dp, S, invperm_d, xtmp, D, xsm, D, st));
        CK_CUDA(axpy<T>(DS, 1.0, xsm, xk, st));
        const int N = K.N, n = K.n, rin = K.rin;
        if (K.missing || N == 0) continue;
        // u = V V^T (y - H x^- - eps)
        T* res = R;                                         // N x S
        CK_CUDA(sampler_ops<T>::residual(N, S, y_st + (size_t)k * Nmax, K.idx, sig_st + (size_t)k * Nmax, xk, D,
                                         epsd + uoff[k], res, st));
        T* u = ust + uoff[k];
        if (n) {
          const T* Vk = K.XV + N;
          CK(gemm(OP_T, OP_N, n, S, N, 1.0, Vk, N, res, N, 0.0, tt, n));
          CK(gemm(OP_N, OP_N, N, S, n, 1.0, Vk, N, tt, n, 0.0, u, N));
        } else {
          CK_CUDA(cudaMemsetAsync(u, 0, (size_t)N * S * sizeof(T), st));
        }
        // x_k = x^-_k + Sigma_k H^T u - M^- (H M^-)^T u
        CK_CUDA(sampler_ops<T>::gather_coords(N, K.idx, coords, xcs, st));
        if (cull) {   // this step's active K-block lists (as in its update)
          CK_CUDA(launch_tile_spheres(reinterpret_cast<const float4*>(xcs), N, 32, sph_o32, st));
          CK_CUDA(launch_k2_active(sph_x128, (int)((NX + 127) / 128), sph_o32, (N + 31) / 32, kCullCut, act_cnt_po,
                                   act_list_po, act_stride_po, nullptr, st));
        }
        CK(k2(coords, (int)NX, xcs, N, u, N, S, Yb, NX, cull ? act_cnt_po : nullptr, act_list_po, act_stride_po));
        const T* tmpp = nullptr;
        if (rin) {
          HM = hmx + N;
          CK_CUDA(StepKernels<T>::gather_rows(N, rin, K.idx, K.Mk, D, HM, N, 0, (int)NX, st));
          CK(gemm(OP_T, OP_N, rin, S, N, 1.0, HM, N, u, N, 0.0, Ub, rin));
          CK(gemm(OP_N, OP_N, (int)D, S, rin, 1.0, K.Mk, (int)D, Ub, rin, 0.0, tmp, (int)D));
          tmpp = tmp;
        }
        CK_CUDA(sampler_ops<T>::combine((int)NX, Dp, S, K.sig_t, Yb, tmpp, xk, xk, st));
      }
      const T* res_out = xs;   // filter samples
      if (which == CAKF_SMOOTH) {
        // w^s_T = w_T = H^T u_T
        CK_CUDA(cudaMemsetAsync(wsv, 0, DS * sizeof(T), st));
        if (!steps[T_].missing && steps[T_].N)
          CK_CUDA(sampler_ops<T>::scatter_rows(steps[T_].N, S, steps[T_].idx, ust + uoff[T_], T(1), wsv, D, st));
        for (int k = T_ - 1; k >= 0; --k) {
          Step& K = steps[k];
          const int N = K.N, n = K.n, rin = K.rin;
          // z = A_k^T w^s_{k+1};  y = P^-_k z = Sigma_k z - M^- (M^-^T z)
          CK_CUDA(StepKernels<T>::mix((int)NX, Dp, S, K.A_next, true, wsv, D, X, D, st));
          CK(k2(coords, (int)NX, coords, (int)NX, X, NX, Dp * S, Yk, NX, cull ? act_cnt_sm : nullptr, act_list_sm,
                act_stride_sm));
          CK_CUDA(StepKernels<T>::sigma_apply((int)NX, Dp, S, K.sig_t, Yk, yb, st));
          if (rin) {
            CK(gemm(OP_T, OP_N, rin, S, (int)D, 1.0, K.Mk, (int)D, X, (int)D, 0.0, Tm, rin));
            CK(gemm(OP_N, OP_N, (int)D, S, rin, -1.0, K.Mk, (int)D, Tm, rin, 1.0, yb, (int)D));
          }
          // w^s_k = w_k + z - H^T V (V^T H y);  P_k z = y - B_k (V^T H y)
          CK_CUDA(cudaMemcpyAsync(wsv, X, DS * sizeof(T), cudaMemcpyDeviceToDevice, st));
          if (!K.missing && N) {
            CK_CUDA(sampler_ops<T>::scatter_rows(N, S, K.idx, ust + uoff[k], T(1), wsv, D, st));
            if (n) {
              const T* Vk = K.XV + N;
              CK_CUDA(StepKernels<T>::gather_rows(N, S, K.idx, yb, D, Hy, N, 0, (int)NX, st));
              CK(gemm(OP_T, OP_N, n, S, N, 1.0, Vk, N, Hy, N, 0.0, tt, n));
              CK(gemm(OP_N, OP_N, N, S, n, 1.0, Vk, N, tt, n, 0.0, R, N));
              CK_CUDA(sampler_ops<T>::scatter_rows(N, S, K.idx, R, T(-1), wsv, D, st));
              CK(gemm(OP_N, OP_N, (int)D, S, n, -1.0, K.Mk + (size_t)rin * D, (int)D, tt, n, 1.0, yb,
                      (int)D));
            }
          }
          // x^s_k = x_k + P_k z  (in place over the forward sample: the forward x_k is not needed again)
          CK_CUDA(axpy<T>(DS, 1.0, yb, xs + (size_t)k * DS, st));
        }
      }
      // internal -> user order, to the caller's buffer: (T+1) x D x S
      for (int k = 0; k <= T_; ++k) {
        CK_CUDA(sampler_ops<T>::permute_cols((int)NX, Dp, S, perm_d, res_out + (size_t)k * DS, D, xtmp, D, st));
        CK_CUDA(cudaMemcpyAsync(static_cast<T*>(out) + (size_t)k * DS, xtmp, DS * sizeof(T), cudaMemcpyDefault, st));
      }
      CK_CUDA(cudaStreamSynchronize(st));
      return CAKF_OK;
    };
    const int rc = run();
    cleanup();
    if (rc == CAKF_OK) CK_CUDA(cudaStreamSynchronize(st));
    return rc;
  }

  int get(int k, int which, void* mean, void* var) override {
    if (k < 0 || k > kcur) return fail(CAKF_E_ARG, "get: step index out of range");
    Step& S = steps[k];
    const T *pm = nullptr, *pv = nullptr;
    if (which == CAKF_PRED) {
      pm = S.m_pred;
      if (var) {
        CK_CUDA(StepKernels<T>::rowvar((int)NX, Dp, S.sig_t, nullptr, S.Mk, D, S.rin, pvar, st));
        pv = pvar;
      }
    } else if (which == CAKF_FILTER) {
      if (k == kcur && phase == 1) return fail(CAKF_E_STATE, "get: step not updated yet");
      pm = S.m;
      pv = S.var;
    } else if (which == CAKF_SMOOTH) {
      if (!smoothed) return fail(CAKF_E_STATE, "get: caks_smooth has not run");
      pm = S.ms;
      pv = S.vs;
    } else {
      return fail(CAKF_E_ARG, "get: bad which");
    }
    // this rank's rows -> all rows (all-gather of the row slices) -> user point order
    if (mean) {
      const T* full = nullptr;
      CK(gather_rows_all(pm, outv, &full));
      CK_CUDA(unpermute<T>((int)NXf, Dp, perm_d, full, outm, st));
      CK_CUDA(cudaMemcpyAsync(mean, outm, Df * sizeof(T), cudaMemcpyDefault, st));
    }
    if (var) {
      const T* full = nullptr;
      CK(gather_rows_all(pv, outm, &full));
      CK_CUDA(unpermute<T>((int)NXf, Dp, perm_d, full, outv, st));
      CK_CUDA(cudaMemcpyAsync(var, outv, Df * sizeof(T), cudaMemcpyDefault, st));
    }
    CK_CUDA(cudaStreamSynchronize(st));
    return CAKF_OK;
  }

  // the full D vector (internal order) from the ranks' local rows: *out = local when one rank holds all rows,
  // else the packed slices all-gathered (ncclAllGather) and unpacked into scratch (Df elements)
  int gather_rows_all(const T* local, T* scratch, const T** out) {
    if (NX == NXf) {
      *out = local;
      return CAKF_OK;
    }
    CK_CUDA(StepKernels<T>::pack_dslice(Dp, (int)NX, (int)pslice, local, yslice, st));
    CK_NCCL(ncclAllGather(yslice, ygath, (size_t)Dp * pslice, sizeof(T) == 4 ? ncclFloat32 : ncclFloat64, comm, st));
    CK_CUDA(StepKernels<T>::unpack_dslices((int)NXf, Dp, (int)pslice, ygath, scratch, st));
    *out = scratch;
    return CAKF_OK;
  }

  int stats(int k, cakf_step_stats* out) override {
    if (k < 0 || k > kcur) return fail(CAKF_E_ARG, "get_stats: step index out of range");
    IterCtl c{};
    CK_CUDA(cudaMemcpyAsync(&c, &ctl[k], sizeof(IterCtl), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    const Step& S = steps[k];
    out->k = k;
    out->iters = S.n;
    out->rejected = c.rejected;
    out->rank_in = S.rin;
    out->cols = S.cols;
    out->rank_out = S.rank_out;
    out->smoother_rank = smoothed ? S.smoother_rank : -1;
    out->missing = S.missing ? 1 : 0;
    out->res0 = std::sqrt(c.res0_sq);
    out->res_final = std::sqrt(c.res_sq);
    out->eta_min = c.eta_min;
    out->dropped_mass = c.dropped;
    if (c.nonfinite) return fail(CAKF_E_NUMERIC, "non-finite eta/alpha in step " + std::to_string(k));
    return CAKF_OK;
  }

  int kept_eigs(int k, double* vals, int cap, int* n_out) override {
    if (k < 0 || k > kcur) return fail(CAKF_E_ARG, "get_kept_eigs: step index out of range");
    const Step& S = steps[k];
    const int n = S.truncated ? S.rank_out : 0;
    if (n_out) *n_out = n;
    if (n && vals) {
      CK_CUDA(cudaMemcpyAsync(vals, S.kept, (size_t)std::min(n, cap) * sizeof(double), cudaMemcpyDefault, st));
      CK_CUDA(cudaStreamSynchronize(st));
    }
    return CAKF_OK;
  }

  int profile(bool on) override {
    prof_on = on;
    return CAKF_OK;
  }

  int sync() override {
    CK_CUDA(cudaStreamSynchronize(st));
    return CAKF_OK;
  }
};

}  // namespace

struct cakf_s {
  ImplBase* impl = nullptr;
  int device = -1;   // CUDA device current at cakf_create; every entry point runs on it
};

namespace {
// Scoped current-device switch: a handle may be driven from a host thread whose current device differs
// from the one it was created on (serving mode); restores the caller's device on exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = -1;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

const char* cakf_last_error(void) { return g_last_error.c_str(); }
int cakf_version(void) { return CAKF_VERSION; }

int cakf_create(const cakf_config* cfg, cakf_t* out) {
  if (!cfg || !out) return fail(CAKF_E_ARG, "cakf_create: NULL argument");
  *out = nullptr;
  if (cfg->world < 0 || cfg->world > 64) return fail(CAKF_E_ARG, "cakf_create: bad world");
  if (cfg->dtype != CAKF_F32 && cfg->dtype != CAKF_F64) return fail(CAKF_E_ARG, "cakf_create: bad dtype");
  if (cfg->d_time < 1 || cfg->d_time > 3) return fail(CAKF_E_UNSUPPORTED, "cakf_create: d_time must be 1..3");
  if (cfg->n_space < 1 || cfg->n_space > (int64_t)1 << 30) return fail(CAKF_E_ARG, "cakf_create: bad n_space");
  if (cfg->space_dim < 1 || cfg->space_dim > 3) return fail(CAKF_E_ARG, "cakf_create: space_dim must be 1..3");
  if (!cfg->coords || !cfg->sigma_t0) return fail(CAKF_E_ARG, "cakf_create: coords and sigma_t0 are required");
  if (cfg->spatial_kernel != 1 && cfg->spatial_kernel != 3 && cfg->spatial_kernel != 5)
    return fail(CAKF_E_UNSUPPORTED, "cakf_create: spatial_kernel must be MATERN12/32/52");
  if (!(cfg->ell_x > 0)) return fail(CAKF_E_ARG, "cakf_create: ell_x must be > 0");
  if (cfg->policy < 0 || cfg->policy > 3) return fail(CAKF_E_UNSUPPORTED, "cakf_create: unknown policy");
  if (cfg->max_iter < 0 || cfg->max_steps < 1) return fail(CAKF_E_ARG, "cakf_create: bad max_iter / max_steps");
  ImplBase* impl = nullptr;
  if (cfg->dtype == CAKF_F32) impl = new Impl<float>();
  else impl = new Impl<double>();
  const int rc = impl->init(*cfg);
  if (rc != CAKF_OK) {
    const std::string msg = g_last_error;
    delete impl;
    g_last_error = msg;
    return rc;
  }
  cakf_s* h = new cakf_s;
  h->impl = impl;
  cudaGetDevice(&h->device);
  *out = h;
  return CAKF_OK;
}

#define HANDLE_CHECK_NOJOIN(h)                                   \
  if (!(h) || !(h)->impl) return fail(CAKF_E_ARG, "NULL handle"); \
  DeviceGuard device_guard_((h)->device)
// every entry point but predict / update first joins the filter truncation still running on its own stream
#define HANDLE_CHECK(h)                                              \
  HANDLE_CHECK_NOJOIN(h);                                            \
  {                                                                  \
    const int join_rc_ = (h)->impl->join_pending();                  \
    if (join_rc_ != CAKF_OK) return join_rc_;                        \
  }

int cakf_reset(cakf_t h) { HANDLE_CHECK(h); return h->impl->reset(); }
int cakf_predict(cakf_t h, const double* A_t, const double* Q_t, const void* b) {
  HANDLE_CHECK_NOJOIN(h);
  return h->impl->predict(A_t, Q_t, b);
}
int cakf_update(cakf_t h, int64_t n_obs, const int64_t* obs_idx, const void* y, const void* noise_var,
                const int64_t* coord_order) {
  HANDLE_CHECK_NOJOIN(h);
  return h->impl->update(n_obs, obs_idx, y, noise_var, coord_order);
}
int cakf_truncate(cakf_t h) { HANDLE_CHECK(h); return h->impl->truncate(); }
int caks_smooth(cakf_t h) { HANDLE_CHECK(h); return h->impl->smooth(); }
int cakf_get(cakf_t h, int32_t k, int32_t which, void* mean_D, void* var_D) {
  HANDLE_CHECK(h);
  return h->impl->get(k, which, mean_D, var_D);
}
int cakf_get_stats(cakf_t h, int32_t k, cakf_step_stats* out) {
  HANDLE_CHECK(h);
  if (!out) return fail(CAKF_E_ARG, "NULL stats");
  return h->impl->stats(k, out);
}
int cakf_get_kept_eigs(cakf_t h, int32_t k, double* vals, int32_t cap, int32_t* n_out) {
  HANDLE_CHECK(h);
  return h->impl->kept_eigs(k, vals, cap, n_out);
}
int cakf_sync(cakf_t h) { HANDLE_CHECK(h); return h->impl->sync(); }
int cakf_profile(cakf_t h, int32_t enable) { HANDLE_CHECK(h); return h->impl->profile(enable != 0); }
int cakf_profile_read(cakf_t h, double* ms, int64_t* launches, int32_t reset) {
  HANDLE_CHECK(h);
  return h->impl->prof_read(ms, launches, reset != 0);
}
int64_t cakf_kernel_launches(void) { return (int64_t)launch_counter().load(); }
int cakf_interpolate(cakf_t h, int32_t k, const double* A1, const double* Q1, const double* A2, int32_t which,
                     void* mean_D, void* var_D) {
  HANDLE_CHECK(h);
  return h->impl->interpolate(k, A1, Q1, A2, which, mean_D, var_D);
}
int cakf_sample(cakf_t h, int32_t n_samples, const void* x0, const void* q, const void* eps, int32_t which,
                void* out) {
  HANDLE_CHECK(h);
  return h->impl->sample(n_samples, x0, q, eps, which, out);
}
int cakf_debug_matvec(cakf_t h, int64_t n_obs, const int64_t* obs_idx, const void* s, void* out, int32_t shares) {
  HANDLE_CHECK(h);
  return h->impl->debug_matvec(n_obs, obs_idx, s, out, shares);
}
int cakf_cull_stats(cakf_t h, double* frac3) {
  HANDLE_CHECK(h);
  if (!frac3) return fail(CAKF_E_ARG, "NULL output");
  return h->impl->cull_stats(frac3);
}

int cakf_nccl_unique_id(void* out) {
  if (!out) return fail(CAKF_E_ARG, "cakf_nccl_unique_id: NULL");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(CAKF_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return CAKF_OK;
}

int cakf_shard_plan(int64_t n_space, int64_t n_obs, int32_t world, int32_t rank, int64_t* out) {
  if (!out || world < 1 || rank < 0 || rank >= world || n_space < 0 || n_obs < 0)
    return fail(CAKF_E_ARG, "cakf_shard_plan: bad argument");
  const int64_t per = (n_space + world - 1) / world;
  const int64_t slice = ((per + 127) / 128) * 128;
  out[0] = std::min<int64_t>(n_space, slice * rank);
  out[1] = std::min<int64_t>(n_space, slice * (rank + 1));
  const long long U = n_obs > 0 ? matvec_sym_units((int)n_obs) : 0;
  out[2] = U * rank / world;
  out[3] = U * (rank + 1) / world;
  out[4] = U;
  out[5] = slice;
  out[6] = matvec_sym_block_points();
  return CAKF_OK;
}

int cakf_sym_unit_blocks(int64_t n_obs, int64_t u, int32_t* bi_out, int32_t* bj_out) {
  // host mirror of the device unit -> (bi, bj) map of the symmetric K1 (tests of the shard plan)
  const long long bp = matvec_sym_block_points(), nb = (n_obs + bp - 1) / bp;
  if (u < 0 || u >= nb * (nb + 1) / 2 || !bi_out || !bj_out) return fail(CAKF_E_ARG, "cakf_sym_unit_blocks: bad unit");
  const double bb = 2.0 * nb + 1.0;
  long long bi = (long long)std::floor((bb - std::sqrt(bb * bb - 8.0 * (double)u)) * 0.5);
  while (bi * nb - bi * (bi - 1) / 2 > u) --bi;
  while ((bi + 1) * nb - (bi + 1) * bi / 2 <= u) ++bi;
  *bi_out = (int32_t)bi;
  *bj_out = (int32_t)(bi + (u - (bi * nb - bi * (bi - 1) / 2)));
  return CAKF_OK;
}
int cakf_destroy(cakf_t h) {
  if (!h) return CAKF_OK;
  DeviceGuard device_guard_(h->device);
  delete h->impl;
  delete h;
  return CAKF_OK;
}

int cakf_matern_transition(int32_t nu2, double ell_t, double sigma, double dt, double* A, double* Q, double* Sinf) {
  // Closed forms of the companion-form SDE (R10); lam = sqrt(2 nu)/ell, e = exp(-lam dt).
  if (!(ell_t > 0) || dt < 0) return fail(CAKF_E_ARG, "cakf_matern_transition: bad ell/dt");
  const double lam = std::sqrt((double)nu2) / ell_t, s2 = sigma * sigma, e = std::exp(-lam * dt);
  double a[9] = {0}, si[9] = {0};
  int n = 0;
  if (nu2 == 1) {
    n = 1;
    a[0] = e;
    si[0] = s2;
  } else if (nu2 == 3) {
    n = 2;
    const double x = lam * dt;
    a[0] = e * (1 + x); a[1] = e * dt;
    a[2] = -e * lam * lam * dt; a[3] = e * (1 - x);
    si[0] = s2; si[3] = s2 * lam * lam;
  } else if (nu2 == 5) {
    n = 3;
    const double t = dt, l = lam, l2 = l * l, l3 = l2 * l, t2 = t * t;
    // expm of F = [[0,1,0],[0,0,1],[-l^3,-3l^2,-3l]]  (triple eigenvalue -l)
    a[0] = e * (1 + l * t + 0.5 * l2 * t2); a[1] = e * (t + l * t2); a[2] = e * 0.5 * t2;
    a[3] = -e * 0.5 * l3 * t2; a[4] = e * (1 + l * t - l2 * t2); a[5] = e * (t - 0.5 * l * t2);
    a[6] = -e * l3 * (t - 0.5 * l * t2); a[7] = -e * l2 * (3 * t - l * t2); a[8] = e * (1 - 2 * l * t + 0.5 * l2 * t2);
    si[0] = s2; si[2] = -s2 * l2 / 3.0; si[4] = s2 * l2 / 3.0; si[6] = -s2 * l2 / 3.0; si[8] = s2 * l2 * l2;
  } else {
    return fail(CAKF_E_UNSUPPORTED, "cakf_matern_transition: nu2 must be 1, 3 or 5");
  }
  if (A) std::memcpy(A, a, sizeof(double) * n * n);
  if (Sinf) std::memcpy(Sinf, si, sizeof(double) * n * n);
  if (Q) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double acc = si[i * n + j];
        for (int p = 0; p < n; ++p)
          for (int q = 0; q < n; ++q) acc -= a[i * n + p] * si[p * n + q] * a[j * n + q];
        Q[i * n + j] = acc;
      }
  }
  return CAKF_OK;
}

int cakf_gram_matmul(int32_t dtype, int32_t spatial_kernel, double ell, int32_t space_dim, int64_t n_rows,
                     const void* xr, int64_t n_cols, const void* xc, int32_t n_rhs, const void* X, double alpha,
                     void* Y, void* stream) {
  if (!xr || !xc || !X || !Y || n_rows < 0 || n_cols < 0 || n_rhs < 0 || space_dim < 1 || space_dim > 3 || !(ell > 0))
    return fail(CAKF_E_ARG, "cakf_gram_matmul: bad argument");
  if (spatial_kernel != 1 && spatial_kernel != 3 && spatial_kernel != 5)
    return fail(CAKF_E_UNSUPPORTED, "cakf_gram_matmul: spatial_kernel");
  cudaStream_t st = (cudaStream_t)stream;
  const double scale = std::sqrt((double)spatial_kernel) / ell;
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    V4<T>*cr = nullptr, *cc = nullptr;
    double* dxyz = nullptr;
    T* part = nullptr;
    bool failed_ = false;
    (void)failed_;
    const size_t nmax = (size_t)std::max(n_rows, n_cols);
    std::vector<double> hx;
    cudaError_t e = cudaMallocAsync(&dxyz, nmax * space_dim * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cr, (size_t)std::max<int64_t>(n_rows, 1) * sizeof(V4<T>), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cc, (size_t)std::max<int64_t>(n_cols, 1) * sizeof(V4<T>), st);
    // device coordinates of the handle dtype -> double staging
    auto stage = [&](const void* src, int64_t n, V4<T>* dst) -> cudaError_t {
      if (n == 0) return cudaSuccess;
      std::vector<T> h((size_t)n * space_dim);
      cudaError_t ee = cudaMemcpyAsync(h.data(), src, h.size() * sizeof(T), cudaMemcpyDefault, st);
      if (ee != cudaSuccess) return ee;
      ee = cudaStreamSynchronize(st);
      if (ee != cudaSuccess) return ee;
      std::vector<double> hd(h.begin(), h.end());
      ee = cudaMemcpyAsync(dxyz, hd.data(), hd.size() * sizeof(double), cudaMemcpyHostToDevice, st);
      if (ee != cudaSuccess) return ee;
      ee = launch_prescale_coords<T>((int)n, space_dim, dxyz, scale, dst, st);
      if (ee != cudaSuccess) return ee;
      return cudaStreamSynchronize(st);
    };
    if (e == cudaSuccess) e = stage(xr, n_rows, cr);
    if (e == cudaSuccess) e = stage(xc, n_cols, cc);
    if (e == cudaSuccess && n_rhs == 1 && n_rows > 0 && n_cols > 0) {
      // K1 path: X is the column vector; pack it into .w of the column coordinates
      std::vector<V4<T>> hc((size_t)n_cols);
      std::vector<T> hxv((size_t)n_cols);
      e = cudaMemcpyAsync(hc.data(), cc, hc.size() * sizeof(V4<T>), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(hxv.data(), X, hxv.size() * sizeof(T), cudaMemcpyDefault, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      for (size_t j = 0; j < hc.size(); ++j) hc[j].w = hxv[j];
      if (e == cudaSuccess) e = cudaMemcpyAsync(cc, hc.data(), hc.size() * sizeof(V4<T>), cudaMemcpyHostToDevice, st);
      // symmetric path when the row and column point sets are the same array (K_TT s of the inner loop)
      const bool sym = sizeof(T) == 4 && xr == xc && n_rows == n_cols && use_sym_k1();
      const int nch = sym ? matvec_sym_tiles((int)n_rows) : matvec_chunks((int)n_rows, (int)n_cols, sizeof(T));
      if (e == cudaSuccess) e = cudaMallocAsync(&part, (size_t)nch * n_rows * sizeof(T), st);
      if (e == cudaSuccess) {
        if constexpr (sizeof(T) == 4) {
          if (sym) e = launch_matvec_sym(spatial_kernel, cc, (int)n_rows, (float*)part, 0, matvec_sym_units((int)n_rows), st);
          else e = launch_matvec_partial<T>(spatial_kernel, cr, (int)n_rows, cc, (int)n_cols, nch, part, st);
        } else {
          e = launch_matvec_partial<T>(spatial_kernel, cr, (int)n_rows, cc, (int)n_cols, nch, part, st);
        }
      }
      if (e == cudaSuccess) e = launch_sum_partials<T>((int)n_rows, nch, part, alpha, (T*)Y, st);
    } else if (e == cudaSuccess) {
      if constexpr (sizeof(T) == 4) {
        if (use_tc_k2()) {
          float* w = nullptr;
          e = cudaMallocAsync(&w, gram_gemm_tc_workspace((int)n_cols, n_rhs), st);
          if (e == cudaSuccess)
            e = launch_gram_gemm_tc(spatial_kernel, cr, (int)n_rows, cc, (int)n_cols, (const float*)X, (size_t)n_cols,
                                    n_rhs, (float*)Y, (size_t)n_rows, alpha, w, st);
          if (w) cudaFreeAsync(w, st);
        } else {
          e = launch_gram_gemm<T>(spatial_kernel, cr, (int)n_rows, cc, (int)n_cols, (const T*)X, (size_t)n_cols, n_rhs,
                                  (T*)Y, (size_t)n_rows, alpha, st);
        }
      } else {
        e = launch_gram_gemm<T>(spatial_kernel, cr, (int)n_rows, cc, (int)n_cols, (const T*)X, (size_t)n_cols, n_rhs,
                                (T*)Y, (size_t)n_rows, alpha, st);
      }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(dxyz, st);
    cudaFreeAsync(cr, st);
    cudaFreeAsync(cc, st);
    if (part) cudaFreeAsync(part, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(CAKF_E_CUDA, std::string("cakf_gram_matmul: ") + cudaGetErrorString(e));
    return CAKF_OK;
  };
  if (dtype == CAKF_F32) return run(float{});
  if (dtype == CAKF_F64) return run(double{});
  return fail(CAKF_E_ARG, "cakf_gram_matmul: bad dtype");
}

int cakf_sym_eig(int64_t c, int64_t r, const double* G, double* w, double* Qr, void* stream) {
  if (c < 1 || c > 8192 || r < 0 || r > c || !G || (!w && !Qr)) return fail(CAKF_E_ARG, "cakf_sym_eig: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t cc = (size_t)c * c, wsb = eig_workspace_bytes((int)c);
  double *Gd = nullptr, *wd = nullptr, *Qd = nullptr;
  int* fl = nullptr;
  // one process-wide workspace, reused by successive calls like a handle's (grown when c grows)
  static std::mutex ws_mu;
  static void* ws_keep = nullptr;
  static size_t ws_keep_bytes = 0;
  std::lock_guard<std::mutex> lock(ws_mu);
  cudaError_t e = cudaSuccess;
  if (ws_keep_bytes < wsb) {
    if (ws_keep) cudaFree(ws_keep);
    ws_keep = nullptr;
    ws_keep_bytes = 0;
    e = cudaMalloc(&ws_keep, wsb);
    if (e == cudaSuccess) ws_keep_bytes = wsb;
  }
  void* ws = ws_keep;
  if (e == cudaSuccess) e = cudaMallocAsync(&Gd, cc * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&wd, (size_t)c * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&Qd, (size_t)c * std::max<int64_t>(r, 1) * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&fl, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(Gd, G, cc * sizeof(double), cudaMemcpyDefault, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(fl, 0, sizeof(int), st);
  if (e == cudaSuccess) e = eig_top((int)c, (int)r, Gd, ws, wsb, Qd, nullptr, nullptr, wd, fl, st);
  int hf = 0;
  if (e == cudaSuccess && w) e = cudaMemcpyAsync(w, wd, (size_t)c * sizeof(double), cudaMemcpyDefault, st);
  if (e == cudaSuccess && Qr && r) e = cudaMemcpyAsync(Qr, Qd, (size_t)c * r * sizeof(double), cudaMemcpyDefault, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hf, fl, sizeof(int), cudaMemcpyDeviceToHost, st);
  for (void* p : {(void*)Gd, (void*)wd, (void*)Qd, (void*)fl})
    if (p) cudaFreeAsync(p, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return fail(CAKF_E_CUDA, std::string("cakf_sym_eig: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
  if (hf) return fail(CAKF_E_NUMERIC, "cakf_sym_eig: non-finite eigenvalue");
  return CAKF_OK;
}

int cakf_lowrank_gemm(int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                      int64_t lda, const float* B, int64_t ldb, double beta, float* C, int64_t ldc, void* stream) {
  if (!A || !B || !C || m < 0 || n < 0 || k < 1 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX ||
      (transa != 0 && transa != 1) || (transb != 0 && transb != 1) || ldc < std::max<int64_t>(m, 1) ||
      lda < std::max<int64_t>(transa ? k : m, 1) || ldb < std::max<int64_t>(transb ? n : k, 1))
    return fail(CAKF_E_ARG, "cakf_lowrank_gemm: bad argument");
  if (m == 0 || n == 0) return CAKF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  static bool pool_kept = [] {   // keep the stream-ordered pool's memory between calls (repeated calls)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return true;
  }();
  (void)pool_kept;
  int8_t *pa = nullptr, *pb = nullptr;
  int *ea = nullptr, *eb = nullptr;
  double* work = nullptr;
  const size_t nch = (size_t)gemm_i8_nchunk((int)k);
  const size_t work_doubles = (size_t)m * n * nch;
  cudaError_t e = cudaMallocAsync(&pa, gemm_i8_plane_bytes((int)m, (int)k), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&pb, gemm_i8_plane_bytes((int)n, (int)k), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&ea, (size_t)m * nch * sizeof(int), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&eb, (size_t)n * nch * sizeof(int), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&work, work_doubles * sizeof(double), st);
  if (e == cudaSuccess) e = gemm_i8_split<float>(A, (int)m, (int)k, (size_t)lda, transa == 1, pa, ea, st);
  if (e == cudaSuccess) e = gemm_i8_split<float>(B, (int)n, (int)k, (size_t)ldb, transb == 0, pb, eb, st);
  if (e == cudaSuccess)
    e = gemm_i8_run(pa, ea, (int)m, pb, eb, (int)n, (int)k, alpha, beta, C, nullptr, (size_t)ldc, false, work,
                    work_doubles, st);
  for (void* p : {(void*)pa, (void*)pb, (void*)ea, (void*)eb, (void*)work})
    if (p) cudaFreeAsync(p, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return fail(CAKF_E_CUDA, std::string("cakf_lowrank_gemm: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
  return CAKF_OK;
}

}  // extern "C"
