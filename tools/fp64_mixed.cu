// Are the DMMA (mma.sync f64) and DFMA pipes separate on B200?  Warps of one kernel split
// between a DMMA loop and a DFMA loop; if the combined FP64 rate exceeds the DMMA-only peak,
// the pipes run concurrently.  Diagnostic.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mixed(double* out, int iters_mma, int iters_fma, int mma_warps) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < mma_warps) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
    double c[8][2] = {};
    for (int it = 0; it < iters_mma; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = i * 1e-3;
    for (int it = 0; it < iters_fma; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  if (s == 123.456) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  const int threads = 512, warps = threads / 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mw : {16, 0, 8, 12, 4}) {
    // per-warp work so both halves run ~equally long at their standalone rates
    const int im = 20000, ifm = 20000 * 64 / 8 * 37 / 34;  // DMMA: 512 flop/instr/warp... equalise time
    mixed<<<296, threads>>>(o, im, ifm, mw);  // warm
    cudaEventRecord(e0);
    mixed<<<296, threads>>>(o, im, ifm, mw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_mma = 296.0 * mw * (double)im * 8 * 512;             // 8x8x4 x2 per instr
    const double fl_fma = 296.0 * (warps - mw) * 32.0 * (double)ifm * 8 * 2;
    printf("mma warps %2d/%d: %.3f ms, DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", mw, warps, ms,
           fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
  }
  return 0;
}
