// c5's large factor pairs: 8 generalised eigenproblems (n = 769, 769, 768, 768, 513, 513, 512,
// 512) from one host thread each, (a) cuSOLVER sygvd vs (b) potrf + trsm (async, one thread)
// followed by syevd per thread.  Wall time for all eight.  Diagnostic.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
using clk = std::chrono::steady_clock;
int main() {
  const int ns[8] = {769, 769, 768, 768, 513, 513, 512, 512};
  const int J = 8;
  std::vector<cusolverDnHandle_t> hs(J);
  std::vector<cublasHandle_t> hb(J);
  std::vector<cudaStream_t> st(J);
  std::vector<double*> A(J), B(J), A0(J), B0(J), W(J), work(J);
  std::vector<int*> info(J);
  std::vector<int> lw(J);
  srand(3);
  for (int j = 0; j < J; ++j) {
    const int n = ns[j];
    cusolverDnCreate(&hs[j]);
    cublasCreate(&hb[j]);
    cudaStreamCreateWithFlags(&st[j], cudaStreamNonBlocking);
    cusolverDnSetStream(hs[j], st[j]);
    cublasSetStream(hb[j], st[j]);
    std::vector<double> a(n * n), b(n * n), g(n * n);
    for (auto& x : g) x = rand() / (double)RAND_MAX - 0.5;
    for (int r = 0; r < n; ++r)
      for (int c = 0; c <= r; ++c) {
        double s1 = 0, s2 = 0;
        for (int k = 0; k < 16; ++k) { s1 += g[r * n + k] * g[c * n + k]; s2 += g[r * n + 16 + k] * g[c * n + 16 + k]; }
        a[r * n + c] = a[c * n + r] = s1 / 16 + (r == c ? 1e-2 : 0);
        b[r * n + c] = b[c * n + r] = s2 / 16 + (r == c ? 1e-2 : 0);
      }
    cudaMalloc(&A[j], 8 * n * n); cudaMalloc(&B[j], 8 * n * n);
    cudaMalloc(&A0[j], 8 * n * n); cudaMalloc(&B0[j], 8 * n * n);
    cudaMalloc(&W[j], 8 * n); cudaMalloc(&info[j], 4 * 2);
    cudaMemcpy(A0[j], a.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(B0[j], b.data(), 8 * n * n, cudaMemcpyHostToDevice);
    int l1 = 0, l2 = 0;
    cusolverDnDsygvd_bufferSize(hs[j], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A[j], n, B[j], n, W[j], &l1);
    cusolverDnDsyevd_bufferSize(hs[j], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A[j], n, W[j], &l2);
    lw[j] = l1 > l2 ? l1 : l2;
    cudaMalloc(&work[j], 8 * (size_t)lw[j]);
  }
  auto reset = [&]() {
    for (int j = 0; j < J; ++j) {
      cudaMemcpy(A[j], A0[j], 8 * ns[j] * ns[j], cudaMemcpyDeviceToDevice);
      cudaMemcpy(B[j], B0[j], 8 * ns[j] * ns[j], cudaMemcpyDeviceToDevice);
    }
    cudaDeviceSynchronize();
  };
  const double one = 1.0;
  for (int rep = 0; rep < 4; ++rep) {
    reset();
    auto t0 = clk::now();
    {
      std::vector<std::thread> th;
      for (int j = 0; j < J; ++j)
        th.emplace_back([&, j] {
          cusolverDnDsygvd(hs[j], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ns[j], A[j], ns[j], B[j], ns[j], W[j], work[j], lw[j], info[j]);
          cudaStreamSynchronize(st[j]);
        });
      for (auto& t : th) t.join();
    }
    auto t1 = clk::now();
    reset();
    auto t2 = clk::now();
    for (int j = 0; j < J; ++j) {  // async reduction, one thread
      const int n = ns[j];
      cusolverDnDpotrf(hs[j], CUBLAS_FILL_MODE_LOWER, n, B[j], n, work[j], lw[j], info[j] + 1);
      cublasDtrsm(hb[j], CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, B[j], n, A[j], n);
      cublasDtrsm(hb[j], CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n, n, &one, B[j], n, A[j], n);
    }
    {
      std::vector<std::thread> th;
      for (int j = 0; j < J; ++j)
        th.emplace_back([&, j] {
          cusolverDnDsyevd(hs[j], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, ns[j], A[j], ns[j], W[j], work[j], lw[j], info[j]);
          cublasDtrsm(hb[j], CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, ns[j], ns[j], &one, B[j], ns[j], A[j], ns[j]);
          cudaStreamSynchronize(st[j]);
        });
      for (auto& t : th) t.join();
    }
    auto t3 = clk::now();
    printf("8 pairs: sygvd threads %.2f ms | potrf+trsm + syevd threads %.2f ms\n",
           std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t3 - t2).count());
  }
  return 0;
}
