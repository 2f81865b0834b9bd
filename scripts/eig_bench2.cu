// cuSOLVER eigensolver variants for the truncation Gram: Xsyevd, XsyevBatched(batch 1), Xsyevdx (top r),
// syevd eigenvalues-only, at c = 320 (cfg2) and 576 (cfg3), fp64.
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cublas_v2.h>
int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cublasHandle_t b; cublasCreate(&b);
  cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
  for (int n : {320, 576}) {
    const int k = 4 * n;
    std::vector<double> X((size_t)k * n);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    for (auto& v : X) v = nd(g);
    double *dX, *dA, *dA0, *dW; int* info;
    cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dA, (size_t)n * n * 8); cudaMalloc(&dA0, (size_t)n * n * 8);
    cudaMalloc(&dW, n * 8); cudaMalloc(&info, 4);
    cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
    double one = 1, zero = 0;
    cublasDgemm(b, CUBLAS_OP_T, CUBLAS_OP_N, n, n, k, &one, dX, k, dX, k, &zero, dA0, n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    auto timeit = [&](const char* name, auto fn) {
      for (int it = 0; it < 4; ++it) {
        cudaMemcpy(dA, dA0, (size_t)n * n * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        int st = fn();
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        if (it == 3) printf("n=%d %-28s %8.3f ms (status %d)\n", n, name, ms, st);
      }
    };
    size_t wd = 0, wh = 0;
    cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &wd, &wh);
    void* dwk; cudaMalloc(&dwk, wd + 4096); std::vector<char> hw(wh + 4096);
    timeit("Xsyevd vectors", [&] { return (int)cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwk, wd, hw.data(), wh, info); });
    timeit("Xsyevd values only", [&] { return (int)cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwk, wd, hw.data(), wh, info); });
    size_t wd2 = 0, wh2 = 0;
    cusolverStatus_t s2 = cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &wd2, &wh2, 1);
    void* dwk2; cudaMalloc(&dwk2, wd2 + 4096); std::vector<char> hw2(wh2 + 4096);
    printf("n=%d XsyevBatched bufferSize status %d\n", n, (int)s2);
    timeit("XsyevBatched(1)", [&] { return (int)cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwk2, wd2, hw2.data(), wh2, info, 1); });
    int64_t meig = 0; double vl = 0, vu = 0; size_t wd3 = 0, wh3 = 0;
    const int64_t il = 64 + 1, iu = n;   // top n-64
    cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, &vl, &vu, il, iu, &meig, CUDA_R_64F, dW, CUDA_R_64F, &wd3, &wh3);
    void* dwk3; cudaMalloc(&dwk3, wd3 + 4096); std::vector<char> hw3(wh3 + 4096);
    timeit("Xsyevdx top n-64", [&] { return (int)cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, &vl, &vu, il, iu, &meig, CUDA_R_64F, dW, CUDA_R_64F, dwk3, wd3, hw3.data(), wh3, info); });
    // fp32 variants
    float* fA; cudaMalloc(&fA, (size_t)n * n * 4); float* fW; cudaMalloc(&fW, n * 4);
    cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_32F, fA, n, CUDA_R_32F, fW, CUDA_R_32F, &wd, &wh);
    void* dwk4; cudaMalloc(&dwk4, wd + 4096); std::vector<char> hw4(wh + 4096);
    timeit("Xsyevd fp32 vectors", [&] { return (int)cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_32F, fA, n, CUDA_R_32F, fW, CUDA_R_32F, dwk4, wd, hw4.data(), wh, info); });
  }
  return 0;
}
