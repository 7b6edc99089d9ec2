// FP64 GEMM emulated on the tcgen05 INT8 tensor cores (Ozaki scheme I), sm_100a — the hidden
// layers of the line-search forwards (reference src/taylor.py:134-148, 31 of the 32 forward
// passes of a KFAC step, src/optim.py:195-211) when KP_OZAKI=1.
//
//   Z_out = Z_in W^T + b (bias on value rows), Z_in: M x K, W: N x K, both FP64.
//
// Every row of Z_in and of W is scaled by a power of two into (-1, 1) and split exactly into
// OZ_S signed 7-bit slices: a = 2^e sum_{i=1..S} 2^-7i A_i, |A_i| <= 127 (OZ_S = 8: 56 bits,
// the whole 53-bit mantissa of every element within 3 binades of its row's largest).  Then
//   Z[r][n] = 2^(ea_r + eb_n) sum_{l=2..S+1} 2^-7l sum_{i+j=l} <A_i[r], B_j[n]>
// where the slice products are exact int32 sums (K 127^2 S < 2^31) accumulated level by level
// in tensor memory; products of levels above S + 1 are dropped (below 2^-7(S+2) of the
// leading term).  Error per element <= ~2^-7S max_k|a| sum_k|b_k|: measured 3e-17 of
// sum_k|a_k b_k| (tools/ozaki_gemm.cu), i.e. below DGEMM's own rounding bound.
//
// Kernel layout (one CTA per 128 x 64 output tile, 192 threads): warp 0 lane 0 = TMA
// producer (one 3-D TMA per operand per 64-byte K block brings all S planes, 64-byte swizzle,
// two stages of 96 KB), warp 1 = TMEM allocator (512 columns: one 64-column int32
// accumulator per level) + single-thread MMA issuer (S(S+1)/2 products x 2 k-steps of
// tcgen05.mma.cta_group::1.kind::i8, M 128, N 64, K 32), warps 2-5 = epilogue (tcgen05.ld of
// the levels, FP64 sum from the smallest level, scaling, bias, staged through shared memory
// for coalesced row stores).  The activation follows in k_act_fwd (not fused).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

namespace {

constexpr int OZ_S = 8;
constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 64, OZ_ST = 2;
constexpr int OZ_APL = OZ_BM * OZ_BK, OZ_BPL = OZ_BN * OZ_BK;
constexpr int OZ_ABYTES = OZ_S * OZ_APL, OZ_BBYTES = OZ_S * OZ_BPL;
constexpr int OZ_STAGE = OZ_ABYTES + OZ_BBYTES;
constexpr int OZ_TPITCH = OZ_BN + 1;  // epilogue staging pitch (doubles)
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

__device__ __forceinline__ void oz_tma3d(void* dst, const CUtensorMap* m, int x, int y, int z,
                                         uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(b))
      : "memory");
}

// K-major, 64-byte swizzle UMMA shared-memory descriptor: start >> 4, LBO 16 B (unused),
// SBO 512 B (8 rows x 64 B), version 1, layout SWIZZLE_64B
__device__ __forceinline__ uint64_t oz_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// One warp per row: e = exponent of the row's largest |x| (so |x 2^-e| < 1); slices
// d_i = trunc(frac * 2^7) taken successively (exact in FP64).  Lane l handles 4 consecutive
// columns per step.  planes: OZ_S x rows x K int8 (plane stride ps bytes); ex[row] = e.
__global__ void k_oz_slice(const double* __restrict__ X, int64_t rows, int K, int64_t ldx,
                           int8_t* __restrict__ planes, int64_t ps, int* __restrict__ ex) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* x = X + row * ldx;
  double m = 0.0;
  for (int k = 4 * lane; k < K; k += 128) {
    const double2 v0 = *reinterpret_cast<const double2*>(x + k);
    const double2 v1 = *reinterpret_cast<const double2*>(x + k + 2);
    m = fmax(m, fmax(fmax(fabs(v0.x), fabs(v0.y)), fmax(fabs(v1.x), fabs(v1.y))));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (lane == 0) ex[row] = e;
  for (int k = 4 * lane; k < K; k += 128) {
    const double2 v0 = *reinterpret_cast<const double2*>(x + k);
    const double2 v1 = *reinterpret_cast<const double2*>(x + k + 2);
    double r[4] = {ldexp(v0.x, -e), ldexp(v0.y, -e), ldexp(v1.x, -e), ldexp(v1.y, -e)};
#pragma unroll
    for (int i = 0; i < OZ_S; ++i) {
      char4 d;
      signed char* dd = reinterpret_cast<signed char*>(&d);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        r[t] *= 128.0;
        const double q = trunc(r[t]);
        r[t] -= q;
        dd[t] = (signed char)q;
      }
      *reinterpret_cast<char4*>(planes + i * ps + row * (int64_t)K + k) = d;
    }
  }
}

__global__ void __launch_bounds__(192, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
              const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C,
              int64_t ldc, int64_t M, int K, const double* __restrict__ bias, int64_t bias_stride,
              int rows_per_sample) {
  constexpr int S = OZ_S;
  extern __shared__ __align__(1024) uint8_t oz_sm[];
  uint8_t* base =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[OZ_ST], empty[OZ_ST], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * OZ_BM;
  const int n0 = blockIdx.x * OZ_BN;
  const int KB = K / OZ_BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % OZ_ST;
      if (kb >= OZ_ST) mbar_wait(&empty[s], ((kb / OZ_ST) - 1) & 1);
      uint8_t* a = base + s * OZ_STAGE;
      mbar_arrive_expect_tx(&full[s], OZ_STAGE);
      oz_tma3d(a, &mA, kb * OZ_BK, (int)m0, 0, &full[s]);
      oz_tma3d(a + OZ_ABYTES, &mB, kb * OZ_BK, n0, 0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % OZ_ST;
      mbar_wait(&full[s], (kb / OZ_ST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a = smem_addr(base + s * OZ_STAGE), b = a + OZ_ABYTES;
      for (int i = 0; i < S; ++i)
        for (int j = 0; j + i < S; ++j) {  // level (i+1)+(j+1) -> accumulator i + j
          const uint32_t acc_col = tmem + (uint32_t)((i + j) * OZ_BN);
#pragma unroll
          for (int k = 0; k < OZ_BK / 32; ++k) {
            const uint64_t da = oz_desc(a + i * OZ_APL + 32 * k);
            const uint64_t db = oz_desc(b + j * OZ_BPL + 32 * k);
            const uint32_t accum = (kb | k | i) ? 1u : 0u;  // i = 0 opens every level
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc_col),
                "l"(da), "l"(db), "r"(OZ_IDESC), "r"(accum));
          }
        }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_addr(&empty[s]))
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_addr(&tfull))
        : "memory");
  } else if (warp >= 2) {  // epilogue
    mbar_wait(&tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int q = warp & 3;
    const int rl = 32 * q + lane;  // tile row of this thread (TMEM lane)
    const int64_t row = m0 + rl;
    double acc[OZ_BN];
#pragma unroll
    for (int c = 0; c < OZ_BN; ++c) acc[c] = 0.0;
    for (int lv = S - 1; lv >= 0; --lv) {  // smallest level first
      const double sc = ldexp(1.0, -7 * (lv + 2));
#pragma unroll
      for (int c0 = 0; c0 < OZ_BN; c0 += 32) {
        uint32_t r[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(lv * OZ_BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          acc[c0 + jj] = fma((double)(int32_t)r[jj], sc, acc[c0 + jj]);
      }
    }
    // scale, stage in smem (the operand stages are idle once the last MMA has completed)
    double* tile = reinterpret_cast<double*>(base);
    const int er = row < M ? ea[row] : 0;
#pragma unroll
    for (int c = 0; c < OZ_BN; ++c) tile[rl * OZ_TPITCH + c] = ldexp(acc[c], er + eb[n0 + c]);
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    // coalesced stores (warp q: rows 32q .. 32q + 31, lanes across the 64 columns); the bias
    // is added to the value row of every sample after the product (src/taylor.py:134-148,
    // the same order as the DMMA kernels)
    for (int rr = 32 * q; rr < 32 * q + 32; ++rr) {
      const int64_t grow = m0 + rr;
      if (grow >= M) break;
      const bool add_bias = bias != nullptr && (grow % rows_per_sample) == 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        double v = tile[rr * OZ_TPITCH + c];
        if (add_bias) v += bias[(int64_t)(n0 + c) * bias_stride];
        C[grow * ldc + n0 + c] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

static PFN_cuTensorMapEncodeTiled_v12000 oz_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// planes (OZ_S x rows x K int8, plane stride ps bytes) as a 3-D tensor map: box {64 bytes of
// K, box_rows rows, all OZ_S planes}, 64-byte swizzle; cached by geometry.
bool oz_map(CUtensorMap* m, const int8_t* planes, int64_t rows, int K, int64_t ps,
            uint32_t box_rows) {
  using Key = std::tuple<const int8_t*, int64_t, int, int64_t, uint32_t>;
  static std::map<Key, CUtensorMap> cache;
  static std::mutex mu;
  const Key key{planes, rows, K, ps, box_rows};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  auto fn = oz_encode();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)OZ_S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)ps};
  cuuint32_t box[3] = {OZ_BK, box_rows, (cuuint32_t)OZ_S};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

}  // namespace

bool ozaki_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_OZAKI");
    return e && atoi(e) == 1;
  }();
  return on;
}

int ozaki_slices() { return OZ_S; }

bool ozaki_gemm_ok(int64_t M, int N, int K, int64_t lda, int64_t ldb) {
  return ozaki_enabled() && N % OZ_BN == 0 && K % OZ_BK == 0 && K >= OZ_BK && lda % 2 == 0 &&
         ldb % 2 == 0 && M >= OZ_BM && K <= 16384;
}

// C (M x N, ldc) = A (M x K, lda) B^T (B: N x K, ldb) (+ bias[n * bias_stride] on rows
// r % rows_per_sample == 0), FP64 emulated on INT8 tensor cores.  Scratch: a_planes
// (OZ_S x M x K bytes), a_ex (M ints), b_planes (OZ_S x N x K bytes), b_ex (N ints).
bool launch_ozaki_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                       int64_t ldc, int64_t M, int N, int K, const double* bias,
                       int64_t bias_stride, int rows_per_sample, int8_t* a_planes, int* a_ex,
                       int8_t* b_planes, int* b_ex, cudaStream_t s) {
  if (!ozaki_gemm_ok(M, N, K, lda, ldb)) return false;
  const int64_t psa = M * (int64_t)K, psb = (int64_t)N * K;
  CUtensorMap ma, mb;
  if (!oz_map(&ma, a_planes, M, K, psa, OZ_BM) || !oz_map(&mb, b_planes, N, K, psb, OZ_BN))
    return false;
  static bool attr = false;
  const size_t smem = OZ_ST * OZ_STAGE + 1024;
  if (!attr) {
    cudaFuncSetAttribute(k_oz_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  count_launch();
  k_oz_slice<<<(unsigned)ceil_div(M, 8), 256, 0, s>>>(A, M, K, lda, a_planes, psa, a_ex);
  count_launch();
  k_oz_slice<<<(unsigned)ceil_div(N, 8), 256, 0, s>>>(B, N, K, ldb, b_planes, psb, b_ex);
  count_launch();
  dim3 grid((unsigned)(N / OZ_BN), (unsigned)ceil_div(M, OZ_BM));
  k_oz_gemm<<<grid, 192, smem, s>>>(ma, mb, a_ex, b_ex, C, ldc, M, K, bias, bias_stride,
                                    rows_per_sample);
  return true;
}

}  // namespace kp
