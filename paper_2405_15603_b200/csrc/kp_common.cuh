// Shared device helpers for the KFAC-PINN sm_100a kernels (FP64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define KP_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t e__ = (expr);                               \
    if (e__ != cudaSuccess) return kp::fail_cuda(e__, #expr, __FILE__, __LINE__); \
  } while (0)

namespace kp {

int fail_cuda(cudaError_t e, const char* what, const char* file, int line);

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async global->shared copy; zero-fills when !pred (src-size 0).
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr(dst)), "l"(src),
               "r"(pred ? 8 : 0));
}

// 16-byte async copy (cg: bypass L1), zero-fill when !pred.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr(dst)), "l"(src),
               "r"(pred ? 16 : 0));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col); lowers to SASS DMMA.8x8x4.
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c = {C[lane/4][2*(lane%4)], C[lane/4][2*(lane%4)+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- mbarrier + bulk-copy (TMA engine, SASS UBLKCP) helpers --------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}

// Orders this thread's (and, through the preceding mbarrier acquire, the consumers')
// generic-proxy shared-memory accesses before subsequent async-proxy (TMA) accesses: the
// refill of a pipeline stage must not overtake the reads of its previous contents.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// One contiguous global->shared bulk copy (bytes % 16 == 0, both 16 B aligned),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// tanh and its derivatives s1 = 1 - s0^2, s2 = -2 s0 s1, s3 = -2 s1^2 - 2 s0 s2
// (reference src/network.py:54-62; same operation order).
struct TanhD {
  double s0, s1, s2, s3;
};

__device__ __forceinline__ TanhD tanh_derivs(double z, bool third) {
  TanhD t;
  t.s0 = tanh(z);
  t.s1 = 1.0 - t.s0 * t.s0;
  t.s2 = -2.0 * t.s0 * t.s1;
  t.s3 = third ? (-2.0 * t.s1 * t.s1 - 2.0 * t.s0 * t.s2) : 0.0;
  return t;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// 2^-e for the binary exponent e of x > 0 (exact power of two; x normal).
__device__ __forceinline__ double pow2_neg_exponent(double x) {
  const int e = ((__double2hiint(x) >> 20) & 0x7ff) - 1023;
  return __hiloint2double((1023 - e) << 20, 0);
}

// Rotation (cs, sn) that orthogonalises two rows with squared norms a, b and inner product
// g: tan = 2g sign(b - a) / (|b - a| + sqrt((b - a)^2 + 4 g^2)), formed in FP32 after a
// power-of-two rescaling (the angle only steers convergence: an inexact one leaves a tiny
// remainder for the next sweep); cs = (1 + t^2)^-1/2 from an FP32 estimate refined by two
// FP64 Newton steps, sn = cs t, so cs^2 + sn^2 = 1 to FP64 precision.  Branch-free.
__device__ __forceinline__ void jacobi_angle(double a, double b, double g, double& cs,
                                             double& sn) {
  const double d = b - a, g2 = 2.0 * g;
  const double sc = pow2_neg_exponent(fmax(fabs(d), fabs(g2)));
  const float df = (float)(d * sc), gf = (float)(g2 * sc);
  const float den = fabsf(df) + sqrtf(fmaf(df, df, gf * gf));
  const float tf = (df >= 0.0f ? gf : -gf) * __frcp_rn(den);
  const double t = (double)tf;
  const double q1 = fma(t, t, 1.0);
  double y = (double)rsqrtf((float)q1);
  y = y * fma(-0.5 * q1 * y, y, 1.5);
  y = y * fma(-0.5 * q1 * y, y, 1.5);
  cs = y;
  sn = y * t;
}

}  // namespace kp
