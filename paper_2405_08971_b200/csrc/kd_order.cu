// kd_order.cu — per-update spatial order of the observed points (device-side balanced kd-tree).
//
// The symmetric K1 and the post-loop K2 work on tiles of 128 / blocks of 32 *consecutive observed
// points*.  Restricting the grid's own order (kd-tree over all N_X points) to the observed subset
// breaks the subtrees apart, so each update re-orders its N_k observations with a kd-tree built
// over them alone: recursive bisection at the median of the widest axis, splits on multiples of
// 128 above 256 points and of 32 below, leaves of <= 32 — every 128-tile is one compact subtree
// (cfg3: evaluated K1 tile-pair fraction 32 % -> ~22 %).  The segment boundaries of every
// level depend on N only; the data decide the split axis; each level is one stable segmented sort
// (CUB), so the order is deterministic.  The permutation only changes which observation sits in
// which row of the inner loop — never a result beyond summation order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/device/device_segmented_sort.cuh>

#include "internal.h"

namespace cakf {

namespace {

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
__global__ void kd_segments_kernel(int N, int level, int nseg, int* __restrict__ beg, int* __restrict__ end) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int b0 = 0, b1 = N;
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
  beg[s] = b0;
  end[s] = b1;
}

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// one block per segment: bounding box, widest axis, keys = that coordinate (0 for leaves)
template <typename T>
__global__ void kd_keys_kernel(const int* __restrict__ beg, const int* __restrict__ end, const int* __restrict__ vals,
                               const int* __restrict__ idx, const V4<T>* __restrict__ coords,
                               uint32_t* __restrict__ keys) {
  __shared__ float red[6][32];
  __shared__ int axis;
  const int b0 = beg[blockIdx.x], b1 = end[blockIdx.x];
  if (b1 - b0 <= 32) {
    for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) keys[i] = 0u;
    return;
  }
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const V4<T> c = coords[idx[vals[i]]];
    const float v[3] = {(float)c.x, (float)c.y, (float)c.z};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], v[d]);
      hi[d] = fmaxf(hi[d], v[d]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      red[d][w] = lo[d];
      red[3 + d][w] = hi[d];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    float L[3] = {INFINITY, INFINITY, INFINITY}, H[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
      for (int d = 0; d < 3; ++d) {
        L[d] = fminf(L[d], red[d][q]);
        H[d] = fmaxf(H[d], red[3 + d][q]);
      }
    int ax = 0;
    for (int d = 1; d < 3; ++d)
      if (H[d] - L[d] > H[ax] - L[ax]) ax = d;
    axis = ax;
  }
  __syncthreads();
  const int ax = axis;
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const V4<T> c = coords[idx[vals[i]]];
    keys[i] = orderable((float)(ax == 0 ? c.x : ax == 1 ? c.y : c.z));
  }
}

__global__ void iota_kernel(int n, int* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void apply_perm_kernel(int N, const int* __restrict__ perm, const int* __restrict__ idx_in,
                                  const int* __restrict__ sig_in, int* __restrict__ idx_out, int* __restrict__ sig_out,
                                  int* __restrict__ sig_inv) {
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
  const int L = kd_levels(std::max(Nmax, 1));
  const int maxseg = 1 << std::max(L - 1, 0);
  size_t cub_bytes = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                            (const int*)nullptr, (int*)nullptr, std::max(Nmax, 1), maxseg,
                                            (const int*)nullptr, (const int*)nullptr);
  return 2 * align256((size_t)Nmax * 4) * 2 + 2 * align256((size_t)maxseg * 4) + align256(cub_bytes) + 1024;
}

template <typename T>
cudaError_t kd_obs_order(int N, const int* idx, const V4<T>* coords, int* sig_io, int* sig_inv, int* idx_out,
                         const int* sig_in_sorted, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const int L = kd_levels(N);
  const int maxseg = 1 << std::max(L - 1, 0);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  auto take = [&](size_t b) { unsigned char* q = p; p += align256(b); return q; };
  uint32_t* kA = reinterpret_cast<uint32_t*>(take((size_t)N * 4));
  uint32_t* kB = reinterpret_cast<uint32_t*>(take((size_t)N * 4));
  int* vA = reinterpret_cast<int*>(take((size_t)N * 4));
  int* vB = reinterpret_cast<int*>(take((size_t)N * 4));
  int* beg = reinterpret_cast<int*>(take((size_t)maxseg * 4));
  int* end = reinterpret_cast<int*>(take((size_t)maxseg * 4));
  size_t cub_bytes = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, cub_bytes, kA, kB, vA, vB, N, maxseg, beg, end, st);
  void* cub_tmp = take(cub_bytes);
  if ((size_t)(p - reinterpret_cast<unsigned char*>(ws)) > ws_bytes) return cudaErrorInvalidValue;
  iota_kernel<<<(N + 255) / 256, 256, 0, st>>>(N, vA);
  cudaError_t e = note_launch_err();
  for (int l = 0; l < L && e == cudaSuccess; ++l) {
    const int nseg = 1 << l;
    kd_segments_kernel<<<(nseg + 255) / 256, 256, 0, st>>>(N, l, nseg, beg, end);
    if ((e = note_launch_err()) != cudaSuccess) break;
    kd_keys_kernel<T><<<nseg, 128, 0, st>>>(beg, end, vA, idx, coords, kA);
    if ((e = note_launch_err()) != cudaSuccess) break;
    size_t tb = cub_bytes;
    e = cub::DeviceSegmentedSort::StableSortPairs(cub_tmp, tb, kA, kB, vA, vB, N, nseg, beg, end, st);
    std::swap(kA, kB);
    std::swap(vA, vB);
  }
  if (e != cudaSuccess) return e;
  apply_perm_kernel<<<(N + 255) / 256, 256, 0, st>>>(N, vA, idx, sig_in_sorted, idx_out, sig_io, sig_inv);
  return note_launch_err();
}

template cudaError_t kd_obs_order<float>(int, const int*, const V4<float>*, int*, int*, int*, const int*, void*, size_t,
                                         cudaStream_t);
template cudaError_t kd_obs_order<double>(int, const int*, const V4<double>*, int*, int*, int*, const int*, void*,
                                          size_t, cudaStream_t);

}  // namespace cakf
