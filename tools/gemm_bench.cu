// Microbenchmark of the FP64 DMMA GEMM variants vs cuBLAS DGEMM on the c5 shapes.
// Build: see tools/Makefile.bench ; run on the GPU box.
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2405_15603_b200/csrc/kp_internal.h"

namespace kp {
void count_launch() {}
int64_t launch_count() { return 0; }
int fail_cuda(cudaError_t e, const char* what, const char* file, int line) { return 5; }
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffffff) / double(0xffffff) - 0.5;
  }
}

__global__ void maxdiff(const double* a, const double* b, size_t n, double* out) {
  double m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[i] - b[i]));
  atomicMax((unsigned long long*)out, __double_as_longlong(m));
}

int main(int argc, char** argv) {
  const long M = argc > 1 ? atol(argv[1]) : 306000;
  struct Shape { int N, K; };
  std::vector<Shape> shapes = {{768, 768}, {512, 768}, {512, 512}, {768, 512}, {64, 64}, {48, 64}};
  double *A, *B, *C, *R, *md;
  size_t maxk = 768, maxn = 768;
  cudaMalloc(&A, M * maxk * 8); cudaMalloc(&B, maxn * maxk * 8);
  cudaMalloc(&C, M * maxn * 8); cudaMalloc(&R, M * maxn * 8); cudaMalloc(&md, 8);
  fill<<<1024, 256>>>(A, M * maxk, 1); fill<<<1024, 256>>>(B, maxn * maxk, 2);
  cublasHandle_t h; cublasCreate(&h);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto sh : shapes) {
    kp::GemmNT g{A, sh.K, B, sh.K, C, sh.N, M, sh.N, sh.K, nullptr, 0, 1};
    double flops = 2.0 * M * sh.N * sh.K;
    // cuBLAS reference: C^T (N x M col-major) = B (N x K) * A^T -> col-major: C_cm(N,M) = B_cm^T? use row-major trick
    const double one = 1, zero = 0;
    auto cublas = [&]() {
      cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, sh.N, (int)M, sh.K, &one, B, sh.K, A, sh.K, &zero, R, sh.N);
    };
    auto timeit = [&](auto fn, int reps) {
      fn(); cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) fn();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      return ms / reps;
    };
    int reps = 5;
    float tc = timeit(cublas, reps);
    printf("M=%ld N=%d K=%d  cuBLAS %.3f ms %.2f TF/s\n", M, sh.N, sh.K, tc, flops / tc / 1e9);
    for (int v = -1; v <= 5; ++v) {
      bool ok = true;
      auto fn = [&]() {
        if (v < 0) kp::launch_gemm_nt_cpasync(g, 0);
        else ok = kp::launch_gemm_nt_tma(g, 0, v);
      };
      cudaMemset(C, 0, M * sh.N * 8);
      fn();
      if (!ok) { printf("   variant %d: n/a\n", v); continue; }
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) { printf("   variant %d: CUDA error %s\n", v, cudaGetErrorString(err)); return 1; }
      cudaMemset(md, 0, 8);
      maxdiff<<<1024, 256>>>(C, R, (size_t)M * sh.N, md);
      double mdh; cudaMemcpy(&mdh, md, 8, cudaMemcpyDeviceToHost);
      float t = timeit(fn, reps);
      printf("   variant %2d: %.3f ms %.2f TF/s  maxdiff vs cuBLAS %.2e\n", v, t, flops / t / 1e9, mdh);
    }
  }
  return 0;
}
