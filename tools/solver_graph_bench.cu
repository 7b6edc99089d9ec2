// Can cuSOLVER's sygvd be captured into a CUDA graph, and does a graph with one branch per
// factor pair run the generalised eigenproblems concurrently (no per-call host launch cost)?
// Diagnostic:  solver_graph_bench [n] [pairs]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}
#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e), __FILE__, __LINE__, #x); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 257;
  const int ns = argc > 2 ? atoi(argv[2]) : 8;
  std::vector<double> a(n * n), b(n * n);
  srand(3);
  auto spd = [&](std::vector<double>& m) {
    std::vector<double> g(n * n);
    for (auto& x : g) x = (rand() / (double)RAND_MAX - 0.5);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < n; ++k) s += g[i * n + k] * g[j * n + k] * (k < n / 4 ? 10.0 : 0.1);
        m[i * n + j] = s / n + (i == j ? 1e-3 : 0.0);
      }
  };
  spd(a);
  spd(b);
  std::vector<cusolverDnHandle_t> h(ns);
  std::vector<cudaStream_t> st(ns);
  std::vector<cudaEvent_t> ev(ns);
  std::vector<double*> dA(ns), dB(ns), dA0(ns), dB0(ns), dW(ns), work(ns);
  std::vector<int*> info(ns);
  int lwd = 0;
  for (int t = 0; t < ns; ++t) {
    cusolverDnCreate(&h[t]);
    CK(cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev[t], cudaEventDisableTiming));
    cusolverDnSetStream(h[t], st[t]);
    CK(cudaMalloc(&dA[t], 8 * n * n));
    CK(cudaMalloc(&dB[t], 8 * n * n));
    CK(cudaMalloc(&dA0[t], 8 * n * n));
    CK(cudaMalloc(&dB0[t], 8 * n * n));
    CK(cudaMalloc(&dW[t], 8 * n));
    CK(cudaMalloc(&info[t], 4));
    cusolverDnDsygvd_bufferSize(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t], &lwd);
    CK(cudaMalloc(&work[t], 8 * (size_t)lwd));
    CK(cudaMemcpy(dA0[t], a.data(), 8 * n * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB0[t], b.data(), 8 * n * n, cudaMemcpyHostToDevice));
  }
  cudaStream_t s0;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  cudaEvent_t fork;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));

  // reference: plain calls, one after another from this thread
  auto copy_in = [&](int t, cudaStream_t s) {
    cudaMemcpyAsync(dA[t], dA0[t], 8 * n * n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(dB[t], dB0[t], 8 * n * n, cudaMemcpyDeviceToDevice, s);
  };
  std::vector<double> w_ref(n), w_g(n);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = clk::now();
    for (int t = 0; t < ns; ++t) {
      copy_in(t, st[t]);
      cusolverDnDsygvd(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                       n, dA[t], n, dB[t], n, dW[t], work[t], lwd, info[t]);
    }
    CK(cudaDeviceSynchronize());
    auto t1 = clk::now();
    printf("plain: %d x sygvd(n=%d) from one thread: %.3f ms\n", ns, n, ms(t0, t1));
  }
  CK(cudaMemcpy(w_ref.data(), dW[0], 8 * n, cudaMemcpyDeviceToHost));

  // capture: fork from s0 into ns streams, one sygvd each, join back
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  CK(cudaEventRecord(fork, s0));
  int bad = 0;
  for (int t = 0; t < ns; ++t) {
    CK(cudaStreamWaitEvent(st[t], fork, 0));
    copy_in(t, st[t]);
    cusolverStatus_t cs = cusolverDnDsygvd(h[t], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                           CUBLAS_FILL_MODE_LOWER, n, dA[t], n, dB[t], n, dW[t],
                                           work[t], lwd, info[t]);
    if (cs != CUSOLVER_STATUS_SUCCESS) {
      printf("sygvd under capture: cusolver status %d\n", (int)cs);
      bad = 1;
    }
    CK(cudaEventRecord(ev[t], st[t]));
    CK(cudaStreamWaitEvent(s0, ev[t], 0));
  }
  cudaError_t ce = cudaStreamEndCapture(s0, &g);
  printf("capture: %s%s\n", cudaGetErrorString(ce), bad ? " (solver errors)" : "");
  if (ce != cudaSuccess || bad) return 0;
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  printf("graph nodes: %zu\n", nn);
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(dW[0], 0, 8 * n));
    CK(cudaDeviceSynchronize());
    auto t0 = clk::now();
    CK(cudaGraphLaunch(ge, s0));
    CK(cudaStreamSynchronize(s0));
    auto t1 = clk::now();
    printf("graph: %d x sygvd(n=%d) concurrent branches: %.3f ms\n", ns, n, ms(t0, t1));
  }
  CK(cudaMemcpy(w_g.data(), dW[0], 8 * n, cudaMemcpyDeviceToHost));
  double md = 0;
  for (int i = 0; i < n; ++i) md = fmax(md, fabs(w_g[i] - w_ref[i]) / fmax(fabs(w_ref[i]), 1e-300));
  int inf = -1;
  CK(cudaMemcpy(&inf, info[0], 4, cudaMemcpyDeviceToHost));
  printf("graph vs plain eigenvalues: max rel diff %.3e, info %d, lam[0] %.6e lam[n-1] %.6e\n", md,
         inf, w_ref[0], w_ref[n - 1]);
  return 0;
}
