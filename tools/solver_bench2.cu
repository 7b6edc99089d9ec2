// cusolverDnXsyevBatched vs syevd, and syevd concurrency from host threads (diagnostic).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <thread>
#include <chrono>
#include <cuda_runtime.h>
#include <cusolverDn.h>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 257;
  int batch = argc > 2 ? atoi(argv[2]) : 2;
  int nthr = argc > 3 ? atoi(argv[3]) : 8;
  std::vector<double> a((size_t)n * n * batch);
  srand(1);
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {
      double r = 0.2 * (rand() / (double)RAND_MAX - 0.5);
      a[(size_t)b * n * n + i * n + j] = a[(size_t)b * n * n + j * n + i] = (i == j ? 1.0 + i * 0.01 : 0.0) + r / n;
    }
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cusolverDnSetStream(h, s);
  cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
  double *dA, *dW; int* info;
  cudaMalloc(&dA, 8 * a.size()); cudaMalloc(&dW, 8 * (size_t)n * batch); cudaMalloc(&info, 4 * batch);
  size_t wd = 0, wh = 0;
  cusolverStatus_t st = cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &wd, &wh, batch);
  void* dwork; cudaMalloc(&dwork, wd + 8); std::vector<char> hwork(wh + 8);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dA, a.data(), 8 * a.size(), cudaMemcpyHostToDevice); cudaDeviceSynchronize();
    auto t0 = clk::now();
    st = cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwork, wd, hwork.data(), wh, info, batch);
    auto t1 = clk::now();
    cudaStreamSynchronize(s);
    auto t2 = clk::now();
    printf("n=%d batch=%d syevBatched status=%d: return %.3f ms, done %.3f ms\n", n, batch, (int)st, ms(t0, t1), ms(t0, t2));
  }
  // syevd from nthr threads concurrently (own handle + stream each)
  std::vector<double*> mats(nthr);
  std::vector<double*> ws(nthr);
  std::vector<cusolverDnHandle_t> hs(nthr);
  std::vector<cudaStream_t> ss(nthr);
  int lw = 0;
  for (int t = 0; t < nthr; ++t) {
    cusolverDnCreate(&hs[t]); cudaStreamCreateWithFlags(&ss[t], cudaStreamNonBlocking); cusolverDnSetStream(hs[t], ss[t]);
    cudaMalloc(&mats[t], 8 * (size_t)n * n);
    cusolverDnDsyevd_bufferSize(hs[t], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, mats[t], n, dW, &lw);
    cudaMalloc(&ws[t], 8 * (size_t)lw + 8 * n);
  }
  for (int rep = 0; rep < 3; ++rep) {
    for (int t = 0; t < nthr; ++t) cudaMemcpy(mats[t], a.data(), 8 * (size_t)n * n, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    auto t0 = clk::now();
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) th.emplace_back([&, t]() {
      int* inf; cudaMallocAsync(&inf, 4, ss[t]);
      cusolverDnDsyevd(hs[t], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, mats[t], n, ws[t] + lw, ws[t], lw, inf);
      cudaStreamSynchronize(ss[t]);
    });
    for (auto& x : th) x.join();
    auto t1 = clk::now();
    printf("n=%d syevd x%d threads: %.3f ms\n", n, nthr, ms(t0, t1));
  }
  return 0;
}
