// Standalone timing / accuracy of the cluster one-sided Jacobi (kp_eig_mid.cu).
//   eig_mid_bench [n] [near_diag_eps]
// C = Q diag(d) Q^T + eps-perturbation (near-diagonal when eps is small), R = chol(C) upper.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2405_15603_b200/csrc/kp_internal.h"
namespace kp { int mid_eig_sweeps_used(); void count_launch() {} }
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 257;
  const double eps = argc > 2 ? atof(argv[2]) : -1.0;  // < 0: random dense SPD
  std::vector<double> C(n * n), R(n * n, 0.0);
  srand(7);
  auto rnd = [] { return rand() / (double)RAND_MAX - 0.5; };
  if (eps < 0) {
    std::vector<double> G(n * n);
    for (auto& x : G) x = rnd();
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < n; ++k) s += G[i * n + k] * G[j * n + k];
        C[i * n + j] = s / n + (i == j ? 1e-2 : 0.0);
      }
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        const double v = i == j ? 1.0 + i * 0.01 : eps * rnd();
        C[i * n + j] = C[j * n + i] = v;
      }
  }
  // Cholesky C = R^T R (R upper), column-major R[col*n + row]
  std::vector<double> L(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s = C[j * n + j];
    for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
    L[j * n + j] = sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double t = C[i * n + j];
      for (int k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = t / L[j * n + j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) R[i * n + j] = L[i * n + j];  // R(row j, col i) = L(i, j)
  double *dR, *dl;
  int *dinfo, *dci;
  long long* dprof;
  cudaMalloc(&dR, 8 * n * n);
  cudaMalloc(&dl, 8 * n);
  cudaMalloc(&dinfo, 4);
  cudaMalloc(&dci, 8);
  cudaMalloc(&dprof, 8 * 512);
  cudaMemset(dprof, 0, 8 * 512);
  cudaMemset(dci, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<double> V(n * n), lam(n);
  for (int w = 0; w < 100; ++w) {  // clocks up
    cudaMemcpy(dR, R.data(), 8 * n * n, cudaMemcpyHostToDevice);
    kp::launch_eig_mid(n, dR, dl, dinfo, dci, 0, nullptr, nullptr);
  }
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dR, R.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    kp::launch_eig_mid(n, dR, dl, dinfo, dci, 0, nullptr, rep == 2 ? dprof : nullptr);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int info = -1;
    cudaMemcpy(&info, dinfo, 4, cudaMemcpyDeviceToHost);
    printf("n=%d eps=%g: %.3f ms info=%d sweeps(max so far)=%d err=%s\n", n, eps, ms, info,
           kp::mid_eig_sweeps_used(), cudaGetErrorString(err));
  }
  long long prof[512];
  cudaMemcpy(prof, dprof, 8 * 512, cudaMemcpyDeviceToHost);
  for (int c = 0; c < 16; ++c)
    printf("cta %d: rot %lld sync %lld xchg %lld upd %lld cycles, sweeps %lld\n", c, prof[5 * c],
           prof[5 * c + 1], prof[5 * c + 2], prof[5 * c + 3], prof[5 * c + 4]);
  cudaMemcpy(V.data(), dR, 8 * n * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(lam.data(), dl, 8 * n, cudaMemcpyDeviceToHost);
  // residual ||C V - V diag(lam)||_max / ||C||_max and orthogonality ||V^T V - I||_max
  double res = 0, cmax = 0, orth = 0;
  for (int i = 0; i < n * n; ++i) cmax = fmax(cmax, fabs(C[i]));
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < n; ++i) {
      double s = 0;
      for (int j = 0; j < n; ++j) s += C[i * n + j] * V[k * n + j];
      res = fmax(res, fabs(s - lam[k] * V[k * n + i]));
    }
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += V[a * n + i] * V[b * n + i];
      orth = fmax(orth, fabs(s - (a == b ? 1.0 : 0.0)));
    }
  printf("residual %.3e (rel), orthogonality %.3e\n", res / cmax, orth);
  return 0;
}
