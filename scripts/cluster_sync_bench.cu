// Microbenchmark: cost of cluster.sync() and of an L2 broadcast round trip inside a 16-CTA cluster
// (tridiagonalisation design, kernels_eig.cu).  nvcc -arch=sm_100a -O3 -o cluster_sync_bench cluster_sync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_loop(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void bcast_loop(int iters, double* buf, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = cl.block_rank();
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (q == (i & 15)) buf[(i & 1) * 1024 + threadIdx.x] = i + threadIdx.x;
    cl.sync();
    acc += __ldcg(buf + (i & 1) * 1024 + (threadIdx.x ^ 5));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (acc == -1) out[1] = 0;
}

__global__ void dsmem_loop(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double sbuf[2][1024];
  const int q = cl.block_rank();
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (q == (i & 15)) sbuf[i & 1][threadIdx.x] = i + threadIdx.x;
    cl.sync();
    const double* rem = cl.map_shared_rank(&sbuf[i & 1][0], i & 15);
    acc += rem[threadIdx.x ^ 5];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (acc == -1) out[1] = 0;
}

template <typename K, typename... A>
long long run(K k, int threads, A... a) {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long* d;
  cudaMalloc(&d, 16);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, a..., d);
  cudaDeviceSynchronize();
  long long h = -1;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
  cudaFree(d);
  return h;
}

int main() {
  double* buf;
  cudaMalloc(&buf, 2 * 1024 * 8);
  for (int t : {128, 256, 512, 1024}) {
    printf("threads %4d: cluster.sync %lld cyc, sync + L2 bcast %lld cyc, sync + DSMEM read %lld cyc\n", t,
           run(sync_loop, t, 1000), run(bcast_loop, t, 1000, buf), run(dsmem_loop, t, 1000));
  }
  return 0;
}
