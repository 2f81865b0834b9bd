// kd_order.cu — per-update spatial order of the observed points (device-side balanced kd-tree).
//
// The symmetric K1 and the post-loop K2 work on tiles of 128 / blocks of 32 *consecutive observed
// points*.  Restricting the grid's own order (kd-tree over all N_X points) to the observed subset
// breaks the subtrees apart, so each update re-orders its N_k observations with a kd-tree built
// over them alone: recursive bisection at the median of the widest axis, splits on multiples of
// 128 above 256 points and of 32 below, leaves of <= 32 — every 128-tile is one compact subtree
// (cfg3: evaluated K1 tile-pair fraction 32 % -> ~22 %).  The segment boundaries of every
// level depend on N only; the data decide the split axis.
//
// Each level is ONE launch, one block per segment, over a contiguous payload (coordinates + input
// position, float4) that moves with the partition — no gathers after the first: bounding box -> widest axis -> 32-bit orderable keys
// -> radix select of the split key (4 passes of 8-bit histograms) -> stable partition (ties broken by
// position).  A final warp-per-leaf pass orders every leaf (<= 32 points) along its own widest axis.
// No library sort, no host round trip: the whole order is stream-ordered and sync-free (CUB's segmented
// sort copies partition sizes to the host and synchronises), and every kernel can be skipped by a device
// flag (`run`, nullable) — the device-pointer observation cache of cakf_update decides on the device.
// The permutation only changes which observation sits in which row of the inner loop — never a result
// beyond summation order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace cakf {

namespace {

constexpr int kKdThreads = 1024;
constexpr int kKdUnroll = 4;   // elements per thread per pass: independent loads in flight

__host__ __device__ inline int kd_split(int n) {
  const int al = n > 256 ? 128 : 32;
  int h = ((n / 2 + al / 2) / al) * al;
  h = h < al ? al : h;
  return h > n - 1 ? n - 1 : h;
}

int kd_levels(int n) {
  if (n <= 32) return 0;
  const int h = kd_split(n);
  return 1 + std::max(kd_levels(h), kd_levels(n - h));
}

// segment s of level L: walk from the root; segments that stopped splitting keep their range in the
// left child and leave the right child empty
__device__ inline void kd_segment(int N, int level, int s, int& b0, int& b1) {
  b0 = 0;
  b1 = N;
  for (int l = 0; l < level; ++l) {
    const int bit = (s >> (level - 1 - l)) & 1;
    const int n = b1 - b0;
    if (n <= 32) {
      if (bit) b0 = b1;
      continue;
    }
    const int h = kd_split(n);
    if (bit) b0 += h;
    else b1 = b0 + h;
  }
}

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ bool skip(const int* run) { return run != nullptr && *run == 0; }

__device__ __forceinline__ float axis_of(const float4& p, int ax) { return ax == 0 ? p.x : ax == 1 ? p.y : p.z; }

// exclusive prefix count of `f` over the block in thread order, and the block total
__device__ __forceinline__ void block_scan_flag(bool f, int* wc, int& pre, int& tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if (lane == 0) wc[warp] = __popc(b);
  __syncthreads();
  int p = 0, t = 0;
  for (int w = 0; w < nw; ++w) {
    const int c = wc[w];
    p += w < warp ? c : 0;
    t += c;
  }
  pre = p + __popc(b & ((1u << lane) - 1u));
  tot = t;
  __syncthreads();
}

// payload of an observation: its (prescaled) coordinates and, in .w, its position in the input list
template <typename T>
__global__ void kd_gather_kernel(int N, const int* __restrict__ run, const int* __restrict__ idx,
                                 const V4<T>* __restrict__ coords, float4* __restrict__ P) {
  if (skip(run)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const V4<T> c = coords[idx[i]];
  P[i] = make_float4((float)c.x, (float)c.y, (float)c.z, __int_as_float(i));
}

// one level of the tree: block = segment [b0, b1) of the payload array, Pin -> Pout
__global__ void __launch_bounds__(kKdThreads) kd_level_kernel(int N, int level, const int* __restrict__ run,
                                                              const float4* __restrict__ Pin,
                                                              float4* __restrict__ Pout, uint32_t* __restrict__ keys) {
  __shared__ float red[6][32];
  __shared__ unsigned hist[256];
  __shared__ int wc[32];
  __shared__ int sel[2];
  if (skip(run)) return;
  int b0, b1;
  kd_segment(N, level, blockIdx.x, b0, b1);
  const int n = b1 - b0;
  const int bd = blockDim.x, step = kKdUnroll * bd;
  if (n <= 32) {   // leaf already: carried through (ordered by kd_leaf_kernel)
    for (int i = b0 + threadIdx.x; i < b1; i += bd) Pout[i] = Pin[i];
    return;
  }
  const int h = kd_split(n);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = bd >> 5;
  // bounding box -> widest axis
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int base = b0 + threadIdx.x; base < b1; base += step) {
    float4 p[kKdUnroll];
#pragma unroll
    for (int q = 0; q < kKdUnroll; ++q) {
      const int i = base + q * bd;
      p[q] = i < b1 ? Pin[i] : Pin[b0];
    }
#pragma unroll
    for (int q = 0; q < kKdUnroll; ++q) {
      lo[0] = fminf(lo[0], p[q].x);
      lo[1] = fminf(lo[1], p[q].y);
      lo[2] = fminf(lo[2], p[q].z);
      hi[0] = fmaxf(hi[0], p[q].x);
      hi[1] = fmaxf(hi[1], p[q].y);
      hi[2] = fmaxf(hi[2], p[q].z);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  if (lane == 0)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      red[d][w] = lo[d];
      red[3 + d][w] = hi[d];
    }
  __syncthreads();
  int ax = 0;
  {
    float L[3] = {INFINITY, INFINITY, INFINITY}, H[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = 0; q < nw; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        L[d] = fminf(L[d], red[d][q]);
        H[d] = fmaxf(H[d], red[3 + d][q]);
      }
    for (int d = 1; d < 3; ++d)
      if (H[d] - L[d] > H[ax] - L[ax]) ax = d;
  }
  // radix select (MSB first) of kth = the h-th smallest key: after the 4 digits, `need` = how many of the
  // keys equal to kth go left (the first ones in position order).  Digit 3 also writes the keys.
  uint32_t prefix = 0u, pmask = 0u;
  int need = h;
  for (int d = 3; d >= 0; --d) {
    for (int t = threadIdx.x; t < 256; t += bd) hist[t] = 0u;
    __syncthreads();
    const int sh = 8 * d;
    for (int base = b0 + threadIdx.x; base < b1; base += step) {
      uint32_t k[kKdUnroll];
      if (d == 3) {
        float4 p[kKdUnroll];
#pragma unroll
        for (int q = 0; q < kKdUnroll; ++q) {
          const int i = base + q * bd;
          p[q] = i < b1 ? Pin[i] : Pin[b0];
        }
#pragma unroll
        for (int q = 0; q < kKdUnroll; ++q) {
          const int i = base + q * bd;
          k[q] = orderable(axis_of(p[q], ax));
          if (i < b1) keys[i] = k[q];
        }
      } else {
#pragma unroll
        for (int q = 0; q < kKdUnroll; ++q) {
          const int i = base + q * bd;
          k[q] = i < b1 ? keys[i] : 0u;
        }
      }
#pragma unroll
      for (int q = 0; q < kKdUnroll; ++q)
        if (base + q * bd < b1 && (k[q] & pmask) == prefix) atomicAdd(&hist[(k[q] >> sh) & 255u], 1u);
    }
    __syncthreads();
    if (w == 0) {
      int s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += (int)hist[8 * lane + q];
      int inc = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      const int exc = inc - s;
      if (exc < need && need <= inc) {
        int cum = exc;
        for (int q = 0; q < 8; ++q) {
          const int hq = (int)hist[8 * lane + q];
          if (cum + hq >= need) {
            sel[0] = 8 * lane + q;
            sel[1] = need - cum;
            break;
          }
          cum += hq;
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)sel[0] << sh;
    pmask |= 255u << sh;
    need = sel[1];
    __syncthreads();   // sel / hist reused by the next digit
  }
  const uint32_t kth = prefix;
  // stable partition: keys < kth, then the first `need` keys == kth -> left [b0, b0 + h); the rest right
  int run_eq = 0, run_left = 0;
  for (int base = b0; base < b1; base += step) {
    float4 p[kKdUnroll];
    uint32_t k[kKdUnroll];
#pragma unroll
    for (int q = 0; q < kKdUnroll; ++q) {
      const int i = base + q * bd + threadIdx.x;
      k[q] = i < b1 ? keys[i] : 0u;
      p[q] = i < b1 ? Pin[i] : Pin[b0];
    }
#pragma unroll
    for (int q = 0; q < kKdUnroll; ++q) {
      const int i = base + q * bd + threadIdx.x;
      const bool valid = i < b1;
      const bool eq = valid && k[q] == kth;
      int eqpre, eqtot, lpre, ltot;
      block_scan_flag(eq, wc, eqpre, eqtot);
      const bool left = valid && (k[q] < kth || (eq && run_eq + eqpre < need));
      block_scan_flag(left, wc, lpre, ltot);
      if (valid) {
        const int nl = run_left + lpre;
        Pout[left ? b0 + nl : b0 + h + (i - b0) - nl] = p[q];
      }
      run_eq += eqtot;
      run_left += ltot;
    }
  }
}

// leaves (<= 32 points): one warp each, ordered along the leaf's own widest axis (ties by position);
// writes the final permutation (positions into the input list)
__global__ void kd_leaf_kernel(int N, int level, int nseg, const int* __restrict__ run, const float4* __restrict__ P,
                               int* __restrict__ perm) {
  if (skip(run)) return;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  int b0, b1;
  kd_segment(N, level, s, b0, b1);
  const int n = b1 - b0;
  if (n <= 0) return;
  const bool act = lane < n;
  const float4 p = act ? P[b0 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  float lo[3] = {act ? p.x : INFINITY, act ? p.y : INFINITY, act ? p.z : INFINITY};
  float hi[3] = {act ? p.x : -INFINITY, act ? p.y : -INFINITY, act ? p.z : -INFINITY};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  int ax = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
  const uint32_t key = act ? orderable(axis_of(p, ax)) : 0xffffffffu;
  int rank = 0;
  for (int m = 0; m < 32; ++m) {
    const uint32_t km = __shfl_sync(0xffffffffu, key, m);
    rank += (m < n) && (km < key || (km == key && m < lane));
  }
  if (act) perm[b0 + rank] = __float_as_int(p.w);
}

__global__ void apply_perm_kernel(int N, const int* __restrict__ run, const int* __restrict__ perm,
                                  const int* __restrict__ idx_in, const int* __restrict__ sig_in,
                                  int* __restrict__ idx_out, int* __restrict__ sig_out, int* __restrict__ sig_inv) {
  if (skip(run)) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int p = perm[j];
  const int s = sig_in[p];
  idx_out[j] = idx_in[p];
  sig_out[j] = s;
  sig_inv[s] = j;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

size_t kd_obs_workspace(int Nmax) {
  const size_t n = (size_t)std::max(Nmax, 1);
  return 2 * align256(n * 16) + 2 * align256(n * 4) + 1024;
}

template <typename T>
cudaError_t kd_obs_order(int N, const int* idx, const V4<T>* coords, int* sig_io, int* sig_inv, int* idx_out,
                         const int* sig_in_sorted, void* ws, size_t ws_bytes, cudaStream_t st, const int* run) {
  if (N <= 0) return cudaSuccess;
  if (kd_obs_workspace(N) > ws_bytes) return cudaErrorInvalidValue;
  const int L = kd_levels(N);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  auto take = [&](size_t b) { unsigned char* q = p; p += align256(b); return q; };
  float4* PA = reinterpret_cast<float4*>(take((size_t)N * 16));
  float4* PB = reinterpret_cast<float4*>(take((size_t)N * 16));
  uint32_t* keys = reinterpret_cast<uint32_t*>(take((size_t)N * 4));
  int* perm = reinterpret_cast<int*>(take((size_t)N * 4));
  kd_gather_kernel<T><<<(N + 255) / 256, 256, 0, st>>>(N, run, idx, coords, PA);
  cudaError_t e = note_launch_err();
  for (int l = 0; l < L && e == cudaSuccess; ++l) {
    kd_level_kernel<<<1 << l, kKdThreads, 0, st>>>(N, l, run, PA, PB, keys);
    e = note_launch_err();
    std::swap(PA, PB);
  }
  if (e != cudaSuccess) return e;
  const int nseg = 1 << L;
  kd_leaf_kernel<<<(nseg + 7) / 8, 256, 0, st>>>(N, L, nseg, run, PA, perm);
  if ((e = note_launch_err()) != cudaSuccess) return e;
  apply_perm_kernel<<<(N + 255) / 256, 256, 0, st>>>(N, run, perm, idx, sig_in_sorted, idx_out, sig_io, sig_inv);
  return note_launch_err();
}

template cudaError_t kd_obs_order<float>(int, const int*, const V4<float>*, int*, int*, int*, const int*, void*, size_t,
                                         cudaStream_t, const int*);
template cudaError_t kd_obs_order<double>(int, const int*, const V4<double>*, int*, int*, int*, const int*, void*,
                                          size_t, cudaStream_t, const int*);

}  // namespace cakf
