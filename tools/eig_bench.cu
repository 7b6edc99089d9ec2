// Standalone timing of the small on-device generalised eigensolver (kp_eig_small.cu).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2405_15603_b200/csrc/kp_internal.h"
namespace kp {
void count_launch() {}
int64_t launch_count() { return 0; }
int fail_cuda(cudaError_t, const char*, const char*, int) { return 5; }
int small_eig_sweeps_used();
}
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 65;
  int jobs = argc > 2 ? atoi(argv[2]) : 10;
  double eps = argc > 3 ? atof(argv[3]) : 0.05;
  std::vector<double> h1(n * n), h2(n * n);
  srand(1);
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {
    double r1 = eps * (rand() / (double)RAND_MAX - 0.5), r2 = eps * (rand() / (double)RAND_MAX - 0.5);
    h1[i * n + j] = h1[j * n + i] = (i == j ? 1.0 : 0.0) + r1;
    h2[i * n + j] = h2[j * n + i] = (i == j ? 1.0 : 0.0) + r2;
  }
  double *f1, *f2, *t, *lam; int *info, *status;
  cudaMalloc(&f1, 8 * n * n); cudaMalloc(&f2, 8 * n * n); cudaMalloc(&t, 8 * n * n * jobs);
  cudaMalloc(&lam, 8 * n * jobs); cudaMalloc(&info, 4 * 2 * jobs); cudaMalloc(&status, 4);
  cudaMemcpy(f1, h1.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaMemcpy(f2, h2.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaMemset(status, 0, 4);
  kp::SmallEigJobs ej{};
  for (int k = 0; k < jobs; ++k) ej.job[k] = kp::SmallEigJob{n, f1, f2, 1e-3, t + k * n * n, lam + k * n, info + k};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 300; ++w) kp::launch_gen_eig_small(ej, jobs, n, status, 0);  // clocks up
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kp::launch_gen_eig_small(ej, jobs, n, status, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("n=%d jobs=%d eps=%g: %.3f ms  sweeps=%d  err=%s\n", n, jobs, eps, ms, kp::small_eig_sweeps_used(), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
