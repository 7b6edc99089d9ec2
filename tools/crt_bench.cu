// Micro-benchmark of the CRT (INT8 tensor-core) fused Taylor layer against the FP64 DMMA fused
// layer, through the library's internal launchers (linked against libkfac_pinn_b200.so).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_15603_b200/csrc \
//        -o crt_bench crt_bench.cu -L../paper_2405_15603_b200 -lkfac_pinn_b200 -lcuda
//   KP_CRT=1 LD_LIBRARY_PATH=../paper_2405_15603_b200 ./crt_bench [n_samples] [K] [N] [d] [reps]
//
// Prints per-launch times of the state slicing, the weight slicing, the CRT layer (ACT_LOSS and
// ACT_LAST) and the DMMA layer, and the largest difference of the CRT activations from the DMMA
// ones relative to the row's largest |activation|.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kp_internal.h"
#ifdef CRT_INLINE  // compile the CRT kernels into this binary (timing variants)
#include "kp_crt.cu"
#endif

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 16384;
  const int K = argc > 2 ? atoi(argv[2]) : 768;
  const int N = argc > 3 ? atoi(argv[3]) : 768;
  const int d = argc > 4 ? atoi(argv[4]) : 100;
  const int reps = argc > 5 ? atoi(argv[5]) : 5;
  const int S = d + 2;
  const int64_t R = n * S;
  printf("n %lld S %d K %d N %d crt_ok %d\n", (long long)n, S, K, N, (int)kp::crt_act_ok(S, K, N));
  std::mt19937_64 gen(11);
  std::normal_distribution<double> nd;
  std::vector<double> H((size_t)R * K), W((size_t)N * K), bias(N), cd(d), wl(N);
  for (int64_t r = 0; r < R; ++r) {
    const int c = (int)(r % S);
    const double sc = c == 0 ? 1.0 : (c == S - 1 ? 3.0 : 0.3);
    for (int k = 0; k < K; ++k) H[r * K + k] = c == 0 ? std::tanh(nd(gen)) : sc * nd(gen);
  }
  for (auto& v : W) v = nd(gen) / std::sqrt((double)K);
  for (auto& v : bias) v = 0.1 * nd(gen);
  for (auto& v : cd) v = 1.0;
  for (auto& v : wl) v = nd(gen) / std::sqrt((double)N);
  double *dH, *dW, *db, *dcd, *dwl, *o1, *o2, *up1, *up2;
  int8_t *rH, *rW;
  int *eH, *eW;
  const int nm = kp::crt_moduli();
  CK(cudaMalloc(&dH, H.size() * 8));
  CK(cudaMalloc(&dW, W.size() * 8));
  CK(cudaMalloc(&db, N * 8));
  CK(cudaMalloc(&dcd, d * 8));
  CK(cudaMalloc(&dwl, N * 8));
  CK(cudaMalloc(&o1, (size_t)R * N * 8));
  CK(cudaMalloc(&o2, (size_t)R * N * 8));
  CK(cudaMalloc(&up1, (size_t)R * (N / 64 + 1) * 8));
  CK(cudaMalloc(&up2, (size_t)R * (N / 64 + 1) * 8));
  CK(cudaMalloc(&rH, (size_t)nm * R * K));
  CK(cudaMalloc(&rW, (size_t)nm * N * K));
  CK(cudaMalloc(&eH, R * 4));
  CK(cudaMalloc(&eW, N * 4));
  CK(cudaMemcpy(dH, H.data(), H.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bias.data(), N * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcd, cd.data(), d * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dwl, wl.data(), N * 8, cudaMemcpyHostToDevice));
  kp::GemmAct g{};
  g.A = dH;
  g.lda = K;
  g.B = dW;
  g.ldb = K;
  g.bias = db;
  g.bias_stride = 1;
  g.n_samples = n;
  g.S = S;
  g.d = d;
  g.taylor = true;
  g.N = N;
  g.K = K;
  g.cdiag = dcd;
  g.ldo = N;
  g.wlast = dwl;
  int* dcnt;
  CK(cudaMalloc(&dcnt, 64 * sizeof(int)));
  cudaEvent_t ev[6];
  for (auto& ee : ev) CK(cudaEventCreate(&ee));
  float best[5] = {1e30f, 1e30f, 1e30f, 1e30f, 1e30f};
  for (int rep = 0; rep < reps; ++rep) {
    CK(cudaEventRecord(ev[0]));
    kp::launch_crt_slice(dH, R, K, K, rH, eH, false, 0);
    CK(cudaEventRecord(ev[1]));
    kp::launch_crt_slice(dW, N, K, K, rW, eW, true, 0);
    CK(cudaEventRecord(ev[2]));
    g.post = o1;
    if (!kp::launch_crt_act(g, kp::ACT_LOSS, rH, eH, rW, eW, 0, dcnt)) printf("crt LOSS rejected\n");
    CK(cudaEventRecord(ev[3]));
    g.post = nullptr;
    g.upart = up1;
    if (!kp::launch_crt_act(g, kp::ACT_LAST, rH, eH, rW, eW, 0, dcnt + 1)) printf("crt LAST rejected\n");
    CK(cudaEventRecord(ev[4]));
    g.upart = nullptr;
    g.post = o2;
    if (!kp::launch_gemm_act(g, kp::ACT_LOSS, 0)) printf("dmma rejected\n");
    CK(cudaEventRecord(ev[5]));
    CK(cudaEventSynchronize(ev[5]));
    CK(cudaGetLastError());
    for (int i = 0; i < 5; ++i) {
      float t;
      CK(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
      best[i] = std::min(best[i], t);
    }
  }
  const double fl = 2.0 * R * K * N;
  printf("slice states %.3f ms (%.0f GB/s of 21 B/elem)\n", best[0], R * (double)K * 21 / best[0] / 1e6);
  printf("slice weights %.3f ms\n", best[1]);
  printf("crt LOSS %.3f ms = %.1f FP64-equiv TFLOP/s\n", best[2], fl / best[2] / 1e9);
  printf("crt LAST %.3f ms\n", best[3]);
  printf("dmma LOSS %.3f ms = %.1f TFLOP/s\n", best[4], fl / best[4] / 1e9);
#if defined(CRT_INLINE) && defined(CRT_TIMING)
  {  // one more launch per mode, then block 0's cycle counters
    for (int mode = 0; mode < 2; ++mode) {
      g.post = mode == 0 ? o1 : nullptr;
      g.upart = mode == 0 ? nullptr : up1;
      kp::launch_crt_act(g, mode == 0 ? kp::ACT_LOSS : kp::ACT_LAST, rH, eH, rW, eW, 0, dcnt + 2);
      CK(cudaDeviceSynchronize());
      long long h[16];
      CK(cudaMemcpyFromSymbol(h, kp::crt_dbg, sizeof(h)));
      printf("block 0 (%s), kilo-clocks: producer wait-empty %lld of %lld | mma wait-tempty %lld wait-full %lld "
             "of %lld | epilogue warp 4: wait-tfull %lld, tail %lld (cumulative: barrier %lld, reconstruct %lld, "
             "activation %lld, outputs %lld) of %lld\n",
             mode == 0 ? "LOSS" : "LAST", h[0] / 1000, h[1] / 1000, h[2] / 1000, h[3] / 1000, h[4] / 1000,
             h[5] / 1000, h[6] / 1000, h[7] / 1000, h[9] / 1000, h[10] / 1000, h[11] / 1000, h[8] / 1000);
    }
  }
#endif
  // compare activations row by row (relative to the row's max |.|) on a sample of rows
  std::vector<double> a((size_t)N), b((size_t)N);
  double worst = 0;
  for (int64_t r = 0; r < R; r += std::max<int64_t>(1, R / 4096)) {
    CK(cudaMemcpy(a.data(), o1 + r * N, N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), o2 + r * N, N * 8, cudaMemcpyDeviceToHost));
    double m = 0, e = 0;
    for (int u = 0; u < N; ++u) {
      m = std::max(m, std::fabs(b[u]));
      e = std::max(e, std::fabs(a[u] - b[u]));
    }
    if (m > 0) worst = std::max(worst, e / m);
  }
  printf("max |crt - dmma| / row max: %.3e\n", worst);
  return 0;
}
