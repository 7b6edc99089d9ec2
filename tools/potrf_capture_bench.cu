// Is cuSOLVER potrf (+ cuBLAS trsm) asynchronous / graph-capturable?  Times n = 129..257.
// Diagnostic:  potrf_capture_bench [n]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 257;
  std::vector<double> a(n * n);
  srand(5);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = (rand() / (double)RAND_MAX - 0.5) * 0.01 + (i == j ? 1.0 : 0.0);
      a[i * n + j] = a[j * n + i] = v;
    }
  cusolverDnHandle_t h;
  cublasHandle_t b;
  cusolverDnCreate(&h);
  cublasCreate(&b);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cusolverDnSetStream(h, s);
  cublasSetStream(b, s);
  double *dA, *dA0, *dX, *work;
  int* info;
  cudaMalloc(&dA, 8 * n * n);
  cudaMalloc(&dA0, 8 * n * n);
  cudaMalloc(&dX, 8 * n * n);
  cudaMalloc(&info, 4);
  cudaMemcpy(dA0, a.data(), 8 * n * n, cudaMemcpyHostToDevice);
  int lw = 0;
  cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, &lw);
  cudaMalloc(&work, 8 * (size_t)lw);
  const double one = 1.0;
  auto seq = [&]() {
    cudaMemcpyAsync(dA, dA0, 8 * n * n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(dX, dA0, 8 * n * n, cudaMemcpyDeviceToDevice, s);
    cusolverStatus_t st = cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, work, lw, info);
    cublasDtrsm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n,
                n, &one, dA, n, dX, n);
    cublasDtrsm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n,
                n, &one, dA, n, dX, n);
    return st;
  };
  for (int rep = 0; rep < 3; ++rep) {
    cudaDeviceSynchronize();
    auto t0 = clk::now();
    seq();
    auto t1 = clk::now();
    cudaStreamSynchronize(s);
    auto t2 = clk::now();
    printf("n=%d potrf+2 trsm: host issue %.3f ms, done %.3f ms\n", n, ms(t0, t1), ms(t0, t2));
  }
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
  cusolverStatus_t st = seq();
  cudaError_t e = cudaStreamEndCapture(s, &g);
  printf("capture: solver %d, %s\n", (int)st, cudaGetErrorString(e));
  if (e == cudaSuccess && st == CUSOLVER_STATUS_SUCCESS) {
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = clk::now();
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      auto t1 = clk::now();
      printf("graph replay %.3f ms\n", ms(t0, t1));
    }
  }
  int hi = -1;
  cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
  printf("info %d\n", hi);
  return 0;
}
