// Standalone probe: FP64 GEMM C = A B^T emulated on the tcgen05 INT8 tensor cores (Ozaki
// scheme I), sm_100a.  Every row of A (M x K) and of B (N x K) is scaled by a power of two
// into (-1, 1) and split exactly into S = 8 signed 7-bit slices (56 bits >= the 53 of a
// double): a = 2^e sum_i 2^-7i A_i.  Then
//   C[r][n] = 2^(ea_r + eb_n) sum_{l = i + j} 2^-7l sum_k A_i[r][k] B_j[n][k],
// with the 36 slice products of levels l = 2 .. S + 1 accumulated exactly in int32 in tensor
// memory (one 64-column accumulator per level: 8 x 64 = 512 columns), K-block by K-block:
// per 64-byte K block the 8 A planes (128 rows) and 8 B planes (64 rows) arrive by one 3-D
// TMA each (64-byte swizzle), and 36 x 2 tcgen05.mma.kind::i8 (M 128, N 64, K 32) consume
// them.  The epilogue drains the eight levels (tcgen05.ld), sums them in FP64 from the
// smallest and writes FP64 C.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ozaki_gemm ozaki_gemm.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int S = 8;                  // slices per operand
constexpr int NLEV = S;               // levels 2 .. S + 1
constexpr int BM = 128, BN = 64, BK = 64, STAGES = 2;
constexpr int A_PLANE = BM * BK, B_PLANE = BN * BK;            // bytes per plane per stage
constexpr int A_BYTES = S * A_PLANE, B_BYTES = S * B_PLANE;   // 64 KB + 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int CN = 4;  // cluster size along N: the A slab of a stage is multicast to all four

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          saddr(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma3d_mc(void* dst, const CUtensorMap* m, int x, int y, int z,
                                         uint64_t* b, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(saddr(b)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, int x, int y, int z,
                                      uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(saddr(b))
      : "memory");
}
// K-major, 64-byte swizzle descriptor: SBO = 8 rows x 64 B, layout SWIZZLE_64B (4), version 1
__device__ __forceinline__ uint64_t sdesc64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

// ---- slicing: one warp per row; x = 2^e sum_i 2^-7i d_i, |d_i| <= 127, e = exponent of the
// row max + 1 (so |x 2^-e| < 1).  planes: S x rows x K int8; ex[row] = e.
__global__ void k_slice(const double* X, int rows, int K, int8_t* planes, int* ex) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* x = X + (size_t)row * K;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = fmax(m, fabs(x[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0) frexp(m, &e);  // m = f 2^e, f in [0.5, 1)  ->  |x 2^-e| < 1
  if (lane == 0) ex[row] = e;
  for (int k = lane; k < K; k += 32) {
    double r = ldexp(x[k], -e);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      r *= 128.0;
      const double d = trunc(r);
      r -= d;
      planes[(size_t)i * rows * K + (size_t)row * K + k] = (int8_t)d;
    }
  }
}

__global__ void __launch_bounds__(192, 1)
    k_ozaki(const __grid_constant__ CUtensorMap mAq, const __grid_constant__ CUtensorMap mB,
            const int* __restrict__ ea, const int* __restrict__ eb, double* C, int M, int N,
            int K) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KB = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CN);  // one MMA commit from every CTA of the cluster
    }
    mbar_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const uint32_t rank = cta_rank();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     saddr(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  cluster_sync_all();  // barrier inits visible cluster-wide before any multicast / remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      uint8_t* a = base + s * STAGE_BYTES;
      mbar_expect(&full[s], STAGE_BYTES);
      // this CTA's share of the A planes goes to every CTA of the cluster (same smem offset)
      constexpr int PPC = S / CN;
      tma3d_mc(a + rank * PPC * A_PLANE, &mAq, kb * BK, m0, (int)rank * PPC, &full[s],
               (uint16_t)((1u << CN) - 1));
      tma3d(a + A_BYTES, &mB, kb * BK, n0, 0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a = saddr(base + s * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
      for (int i = 0; i < S; ++i)
#pragma unroll
        for (int j = 0; j + i < S; ++j) {  // level l = (i + 1) + (j + 1) -> accumulator i + j
          const uint32_t acc_col = tmem + (uint32_t)((i + j) * BN);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            const uint64_t da = sdesc64(a + i * A_PLANE + 32 * k);
            const uint64_t db = sdesc64(b + j * B_PLANE + 32 * k);
            const uint32_t accum = (kb | k | i) ? 1u : 0u;  // first product of each level: i = 0
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc_col),
                "l"(da), "l"(db), "r"(IDESC), "r"(accum));
          }
        }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              saddr(&empty[s])),
          "h"((uint16_t)((1u << CN) - 1))
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     saddr(&tfull))
                 : "memory");
  } else if (warp >= 2) {  // epilogue
    mbar_wait(&tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    double acc[BN];
#pragma unroll
    for (int c = 0; c < BN; ++c) acc[c] = 0.0;
#pragma unroll
    for (int lv = NLEV - 1; lv >= 0; --lv) {  // smallest level first
      const double sc = ldexp(1.0, -7 * (lv + 2));
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(lv * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
              "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
              "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c0 + j] = fma((double)(int32_t)r[j], sc, acc[c0 + j]);
      }
    }
    if (row < M) {
      const int er = ea[row];
      double* out = C + (size_t)row * N + n0;
#pragma unroll
      for (int c = 0; c < BN; ++c) out[c] = ldexp(acc[c], er + eb[n0 + c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

// planes: S x rows x K int8; box {BK bytes, box_rows, S planes}, 64-byte swizzle
static CUtensorMap map_planes(const void* base, uint64_t rows, uint64_t K, uint32_t box_rows,
                              uint32_t box_planes = S) {
  CUtensorMap m;
  cuuint64_t dims[3] = {K, rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {K, rows * K};
  cuuint32_t box[3] = {BK, box_rows, box_planes};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 512, N = argc > 2 ? atoi(argv[2]) : 768,
            K = argc > 3 ? atoi(argv[3]) : 768;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> A((size_t)M * K), B((size_t)N * K);
  for (size_t i = 0; i < A.size(); ++i) A[i] = std::tanh(3.0 * U(g)) * std::pow(10.0, (int)(i / K % 5) - 2);
  for (auto& v : B) v = U(g) / std::sqrt((double)K);
  double *dA, *dB, *dC;
  int8_t *pA, *pB;
  int *eA, *eB;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dB, B.size() * 8));
  CK(cudaMalloc(&dC, (size_t)M * N * 8));
  CK(cudaMalloc(&pA, (size_t)S * M * K));
  CK(cudaMalloc(&pB, (size_t)S * N * K));
  CK(cudaMalloc(&eA, M * 4));
  CK(cudaMalloc(&eB, N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  CUtensorMap mA = map_planes(pA, M, K, BM, S / CN), mB = map_planes(pB, N, K, BN);
  const size_t smem = STAGES * STAGE_BYTES + 1024;
  CK(cudaFuncSetAttribute(k_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  auto gemm = [&]() { CK(cudaLaunchKernelEx(&cfg, k_ozaki, mA, mB, (const int*)eA, (const int*)eB, dC, M, N, K)); };
  auto run = [&]() {
    k_slice<<<(M + 7) / 8, 256>>>(dA, M, K, pA, eA);
    k_slice<<<(N + 7) / 8, 256>>>(dB, N, K, pB, eB);
    gemm();
  };
  run();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<double> C((size_t)M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
  double worst = 0.0, worst_ab = 0.0;
  const int step = M > 4096 ? M / 97 : 1;
  for (int i = 0; i < M; i += step)
    for (int j = 0; j < N; ++j) {
      long double s = 0, sab = 0;
      for (int k = 0; k < K; ++k) {
        s += (long double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
        sab += fabsl((long double)A[(size_t)i * K + k] * B[(size_t)j * K + k]);
      }
      const double err = (double)fabsl((long double)C[(size_t)i * N + j] - s);
      worst = fmax(worst, err / fmax((double)fabsl(s), 1e-300));
      worst_ab = fmax(worst_ab, err / (double)sab);
    }
  printf("M %d N %d K %d: max rel err %.3e, max err / sum|ab| %.3e\n", M, N, K, worst, worst_ab);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_slice<<<(M + 7) / 8, 256>>>(dA, M, K, pA, eA);
  cudaEventRecord(e1);
  for (int r = 0; r < reps; ++r) gemm();
  cudaEventRecord(e2);
  CK(cudaEventSynchronize(e2));
  float ms1 = 0, ms2 = 0;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventElapsedTime(&ms2, e1, e2);
  printf("slice A %.3f ms, ozaki GEMM %.3f ms: %.1f FP64-equivalent TFLOP/s (GEMM only)\n",
         ms1 / reps, ms2 / reps, 2.0 * M * N * K / (ms2 / reps) / 1e9);
  return 0;
}
