// cuSOLVER generalised-eigensolver variants for mid-size factors (diagnostic).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>
#include <cusolverDn.h>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 257;
  std::vector<double> a(n * n), b(n * n);
  srand(1);
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {
    double r1 = 0.2 * (rand() / (double)RAND_MAX - 0.5), r2 = 0.2 * (rand() / (double)RAND_MAX - 0.5);
    a[i * n + j] = a[j * n + i] = (i == j ? 1.0 + i * 0.01 : 0.0) + r1 / n;
    b[i * n + j] = b[j * n + i] = (i == j ? 1.0 : 0.0) + r2 / n;
  }
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cudaStream_t s; cudaStreamCreate(&s); cusolverDnSetStream(h, s);
  double *dA, *dB, *dW, *work; int *info;
  cudaMalloc(&dA, 8 * n * n); cudaMalloc(&dB, 8 * n * n); cudaMalloc(&dW, 8 * n); cudaMalloc(&info, 4);
  int lw1 = 0, lw2 = 0, lw3 = 0;
  cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dB, n, dW, &lw1);
  syevjInfo_t jp; cusolverDnCreateSyevjInfo(&jp); cusolverDnXsyevjSetTolerance(jp, 1e-14);
  cusolverDnDsygvj_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dB, n, dW, &lw2, jp);
  cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw3);
  int lw = lw1 > lw2 ? lw1 : lw2; lw = lw > lw3 ? lw : lw3;
  cudaMalloc(&work, 8 * (size_t)lw);
  auto reset = [&]() { cudaMemcpy(dA, a.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemcpy(dB, b.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaDeviceSynchronize(); };
  for (int rep = 0; rep < 3; ++rep) {
    reset();
    auto t0 = std::chrono::steady_clock::now();
    cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dB, n, dW, work, lw1, info);
    cudaStreamSynchronize(s);
    auto t1 = std::chrono::steady_clock::now();
    reset();
    auto t2 = std::chrono::steady_clock::now();
    cusolverDnDsygvj(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dB, n, dW, work, lw2, info, jp);
    cudaStreamSynchronize(s);
    auto t3 = std::chrono::steady_clock::now();
    reset();
    auto t4 = std::chrono::steady_clock::now();
    cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw3, info);
    cudaStreamSynchronize(s);
    auto t5 = std::chrono::steady_clock::now();
    int sweeps = 0; cusolverDnXsyevjGetSweeps(h, jp, &sweeps);
    printf("n=%d sygvd %.3f ms  sygvj %.3f ms (sweeps %d)  syevd %.3f ms\n", n,
           std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t3 - t2).count(), sweeps,
           std::chrono::duration<double, std::milli>(t5 - t4).count());
  }
  return 0;
}
