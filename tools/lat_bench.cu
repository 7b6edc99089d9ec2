// Latency microbenchmarks (cycles) on one warp / one CTA: dependent DFMA chain, FP64 divide,
// sqrt, dependent 64-bit SHFL, __syncthreads with 1024 threads.  Diagnostic.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int iters) {
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  double d = a;
  for (int i = 0; i < iters; ++i) d = 1.0 / (d + 1.0);
  long long t2 = clock64();
  double e = d + 2.0;
  for (int i = 0; i < iters; ++i) e = sqrt(e + 1.0);
  long long t3 = clock64();
  double f = e;
  for (int i = 0; i < iters; ++i) f = __shfl_xor_sync(0xffffffffu, f, 1) + 1e-3;
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t5 = clock64();
  float g = (float)f;
  for (int i = 0; i < iters; ++i) g = fmaf(g, 1.0000001f, 1e-9f);
  long long t6 = clock64();
  double h = g;
  for (int i = 0; i < iters; ++i) h = rsqrt(h + 1.0);
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters;
    cyc[3] = (t4 - t3) / iters; cyc[4] = (t5 - t4) / iters; cyc[5] = (t6 - t5) / iters;
    cyc[6] = (t7 - t6) / iters;
  }
  out[threadIdx.x] = a + d + e + f + h;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 8);
  for (int bs : {32, 1024}) {
    for (int r = 0; r < 3; ++r) k<<<1, bs>>>(o, c, 1.0, 4096);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("block %4d: DFMA chain %lld, DDIV(+DADD) %lld, DSQRT(+DADD) %lld, SHFL64(+DADD) %lld, "
           "syncthreads %lld, FFMA %lld, DRSQRT(+DADD) %lld cycles\n", bs, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  }
  return 0;
}
