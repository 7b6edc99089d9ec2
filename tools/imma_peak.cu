// INT8 warp-MMA (mma.sync m16n8k32 s8 -> s32) issue-limited peak on B200 (sm_100a), to size
// an Ozaki-style FP64 emulation on the legacy tensor-core path.  Register-only
// loops, no memory traffic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_peak imma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void imma_loop(int* out, int iters, int seed) {
  unsigned a0 = seed * 0x01010101u + threadIdx.x, a1 = a0 ^ 0x5a5a5a5a, a2 = a0 + 7, a3 = a0 * 3;
  unsigned b0 = seed ^ threadIdx.x, b1 = b0 * 5;
  int c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123456) out[0] = s;
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    auto run = [&](auto kern, int chains) {
      kern<<<sms * 2, warps * 32>>>(out, 100, 1);
      cudaEventRecord(e0);
      kern<<<sms * 2, warps * 32>>>(out, iters, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 16 * 8 * 32 * (double)chains * iters * warps * sms * 2;
      printf("warps/CTA %2d chains %d: %.1f TOPS (%.3f ms)\n", warps, chains, ops / ms / 1e9,
             ms);
    };
    run(imma_loop<4>, 4);
    run(imma_loop<8>, 8);
  }
  return 0;
}
