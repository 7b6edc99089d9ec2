// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Register-only inner loops, no memory traffic; measures issue-limited peak.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[i][0]), "+d"(c[i][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16_loop(double* out, int iters, double seed) {
  // m16n8k4: A 2 regs, B 1 reg, C 4 regs
  double a0 = seed + threadIdx.x * 1e-3, a1 = seed * 0.5, b = seed - threadIdx.x * 1e-3;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123.456) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* d;
  CK(cudaMalloc(&d, 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
    for (int threads = 128; threads <= 512; threads *= 2) {
      int grid = sms * blocks_per_sm;
      // DMMA m8n8k4: 256 FMA = 512 flop per warp instr
      for (int rep = 0; rep < 2; ++rep) {
        dmma_loop<8><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e0);
        dmma_loop<8><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * grid * (threads / 32);
        if (rep) printf("DMMA.m8n8k4 grid=%d thr=%d : %.2f TFLOP/s (%.3f ms)\n", grid, threads, flops / ms / 1e9, ms);
      }
      for (int rep = 0; rep < 2; ++rep) {
        dmma16_loop<4><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e0);
        dmma16_loop<4><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 512 * 4 * (double)iters * grid * (threads / 32);
        if (rep) printf("DMMA.m16n8k4 grid=%d thr=%d : %.2f TFLOP/s (%.3f ms)\n", grid, threads, flops / ms / 1e9, ms);
      }
      for (int rep = 0; rep < 2; ++rep) {
        dfma_loop<16><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e0);
        dfma_loop<16><<<grid, threads>>>(d, iters, 1.0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * (double)iters * grid * threads;
        if (rep) printf("DFMA grid=%d thr=%d : %.2f TFLOP/s (%.3f ms)\n", grid, threads, flops / ms / 1e9, ms);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
