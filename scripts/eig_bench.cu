// Micro-benchmark: symmetric eigensolvers for the truncation Gram (n = 576 / 1088), fp64.
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cublas_v2.h>
int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cublasHandle_t b; cublasCreate(&b);
  for (int n : {576, 1088}) {
    const int k = 4 * n;
    std::vector<double> X((size_t)k * n);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    for (auto& v : X) v = nd(g);
    double *dX, *dA, *dA0, *dW, *work; int* info;
    cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dA, (size_t)n * n * 8); cudaMalloc(&dA0, (size_t)n * n * 8);
    cudaMalloc(&dW, n * 8); cudaMalloc(&info, 4);
    cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
    double one = 1, zero = 0;
    cublasDgemm(b, CUBLAS_OP_T, CUBLAS_OP_N, n, n, k, &one, dX, k, dX, k, &zero, dA0, n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    // dsyevd
    int lw = 0; cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw);
    cudaMalloc(&work, (size_t)lw * 8 + 1024);
    for (int it = 0; it < 4; ++it) {
      cudaMemcpy(dA, dA0, (size_t)n * n * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d dsyevd %.3f ms\n", n, ms);
    cudaFree(work);
    // dsyevj
    syevjInfo_t pj; cusolverDnCreateSyevjInfo(&pj);
    cusolverDnXsyevjSetTolerance(pj, 1e-14); cusolverDnXsyevjSetMaxSweeps(pj, 20);
    cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw, pj);
    cudaMalloc(&work, (size_t)lw * 8 + 1024);
    for (int it = 0; it < 3; ++it) {
      cudaMemcpy(dA, dA0, (size_t)n * n * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info, pj);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    int sweeps = 0; cusolverDnXsyevjGetSweeps(h, pj, &sweeps);
    printf("n=%d dsyevj %.3f ms (%d sweeps)\n", n, ms, sweeps);
    cudaFree(work);
    // Xsyevd 64-bit API
    cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
    size_t wd = 0, wh = 0;
    cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &wd, &wh);
    void* dwk; cudaMalloc(&dwk, wd + 1024); std::vector<char> hw(wh + 1024);
    for (int it = 0; it < 3; ++it) {
      cudaMemcpy(dA, dA0, (size_t)n * n * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwk, wd, hw.data(), wh, info);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d Xsyevd %.3f ms\n", n, ms);
    // fp32 ssyevd
    float *sA; cudaMalloc(&sA, (size_t)n * n * 4); float* sW; cudaMalloc(&sW, n * 4);
    std::vector<double> hA((size_t)n * n); cudaMemcpy(hA.data(), dA0, hA.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<float> fA(hA.begin(), hA.end());
    cusolverDnSsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, sA, n, sW, &lw);
    float* swk; cudaMalloc(&swk, (size_t)lw * 4 + 1024);
    for (int it = 0; it < 3; ++it) {
      cudaMemcpy(sA, fA.data(), fA.size() * 4, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      cusolverDnSsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, sA, n, sW, swk, lw, info);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d ssyevd %.3f ms\n", n, ms);
    // dsyrk vs dgemm for the Gram of D x n, D = 231360
    const long D = 231360;
    double* F; cudaMalloc(&F, D * n * 8); cudaMemset(F, 0, D * n * 8);
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      cublasDsyrk(b, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n, D, &one, F, D, &zero, dA, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d dsyrk D=%ld %.3f ms\n", n, D, ms);
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      cublasDgemm(b, CUBLAS_OP_T, CUBLAS_OP_N, n, n, D, &one, F, D, F, D, &zero, dA, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d dgemm-gram %.3f ms\n", n, ms);
    float* Ff = (float*)F; float fone = 1, fzero = 0;
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      cublasSgemm(b, CUBLAS_OP_T, CUBLAS_OP_N, n, n, D, &fone, Ff, D, Ff, D, &fzero, sA, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d sgemm-gram %.3f ms\n", n, ms);
    cublasSetMathMode(b, CUBLAS_FP32_EMULATED_BF16X9_MATH);
    cublasStatus_t st = CUBLAS_STATUS_SUCCESS;
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      st = cublasGemmEx(b, CUBLAS_OP_T, CUBLAS_OP_N, n, n, D, &fone, Ff, CUDA_R_32F, D, Ff, CUDA_R_32F, D, &fzero, sA, CUDA_R_32F, n, CUBLAS_COMPUTE_32F_EMULATED_16BFX9, CUBLAS_GEMM_DEFAULT);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("n=%d bf16x9-gram %.3f ms (status %d)\n", n, ms, (int)st);
    cublasSetMathMode(b, CUBLAS_DEFAULT_MATH);
    cudaFree(F);
  }
  int v; cublasGetVersion(b, &v); printf("cublas version %d\n", v);
  return 0;
}
