// Concurrency of cuSOLVER sygvj (Jacobi, device-only) on several streams from one thread,
// vs sygvd; realistic-ish SPD pairs (diagonal spread + low-rank part). Diagnostic.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <chrono>
#include <cmath>
#include <cuda_runtime.h>
#include <cusolverDn.h>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 257;
  int ns = argc > 2 ? atoi(argv[2]) : 8;
  double tol = argc > 3 ? atof(argv[3]) : 1e-14;
  std::vector<double> a(n * n), b(n * n);
  srand(3);
  // A = G G^T / n + 1e-3 I with G n x n random; B likewise (different seed)
  auto spd = [&](std::vector<double>& m, double scale) {
    std::vector<double> g(n * n);
    for (auto& x : g) x = (rand() / (double)RAND_MAX - 0.5) * scale;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
      double s = 0; for (int k = 0; k < n; ++k) s += g[i * n + k] * g[j * n + k] * (k < n / 4 ? 10.0 : 0.1);
      m[i * n + j] = s / n + (i == j ? 1e-3 : 0.0);
    }
  };
  spd(a, 1.0); spd(b, 1.0);
  std::vector<cusolverDnHandle_t> h(ns); std::vector<cudaStream_t> st(ns);
  std::vector<double*> dA(ns), dB(ns), dW(ns), work(ns); std::vector<int*> info(ns);
  std::vector<syevjInfo_t> jp(ns);
  int lw = 0, lwd = 0;
  for (int t = 0; t < ns; ++t) {
    cusolverDnCreate(&h[t]); cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking); cusolverDnSetStream(h[t], st[t]);
    cudaMalloc(&dA[t], 8 * n * n); cudaMalloc(&dB[t], 8 * n * n); cudaMalloc(&dW[t], 8 * n); cudaMalloc(&info[t], 4);
    cusolverDnCreateSyevjInfo(&jp[t]); cusolverDnXsyevjSetTolerance(jp[t], tol); cusolverDnXsyevjSetMaxSweeps(jp[t], 100);
    cusolverDnDsygvj_bufferSize(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t], &lw, jp[t]);
    cusolverDnDsygvd_bufferSize(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t], &lwd);
    cudaMalloc(&work[t], 8 * (size_t)(lw > lwd ? lw : lwd));
  }
  auto reset = [&]() { for (int t = 0; t < ns; ++t) { cudaMemcpy(dA[t], a.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemcpy(dB[t], b.data(), 8 * n * n, cudaMemcpyHostToDevice); } cudaDeviceSynchronize(); };
  for (int rep = 0; rep < 3; ++rep) {
    reset();
    auto t0 = clk::now();
    for (int t = 0; t < ns; ++t)
      cusolverDnDsygvj(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t], work[t], lw, info[t], jp[t]);
    auto t1 = clk::now();
    cudaDeviceSynchronize();
    auto t2 = clk::now();
    int sw = 0; cusolverDnXsyevjGetSweeps(h[0], jp[0], &sw);
    reset();
    auto t3 = clk::now();
    cusolverDnDsygvj(h[0], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA[0], n, dB[0], n, dW[0], work[0], lw, info[0], jp[0]);
    cudaDeviceSynchronize();
    auto t4 = clk::now();
    reset();
    auto t5 = clk::now();
    for (int t = 0; t < ns; ++t)
      cusolverDnDsygvd(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t], work[t], lwd, info[t]);
    cudaDeviceSynchronize();
    auto t6 = clk::now();
    printf("n=%d x%d: sygvj issue %.2f ms, all done %.2f ms (sweeps %d); one sygvj %.2f ms; %d sygvd serial %.2f ms\n", n, ns, ms(t0, t1), ms(t0, t2), sw, ms(t3, t4), ns, ms(t5, t6));
  }
  return 0;
}
