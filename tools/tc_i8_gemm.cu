// Standalone tcgen05 (5th-gen tensor core) INT8 GEMM probe for sm_100a: C (s32, M x N) =
// A (s8, M x K) * B (s8, N x K)^T, both K-major.  TMA (128-byte swizzle) -> shared memory ->
// tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 256, K = 32 per instruction) with the
// accumulator in tensor memory, read back by tcgen05.ld.  Warp roles: 0 = TMA producer,
// 1 = TMEM allocator + MMA issuer, 2..5 = epilogue (one TMEM lane quadrant each).
// Purpose: correctness + throughput of the int8 path an Ozaki-style FP64 emulation would
// need.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;

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
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(saddr(b))
      : "memory");
}
// K-major, 128-byte swizzle shared-memory matrix descriptor (tcgen05): start >> 4, LBO 16 B
// (unused for swizzled K-major), SBO 1024 B (8-row groups), version 1, layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// instruction descriptor: D s32, A/B signed int8, both K-major, N >> 3, M >> 4
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(192, 1)
    k_i8_gemm(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
              int32_t* C, int M, int N, int K) {
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
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     saddr(&tmem_base)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      uint8_t* a = base + s * STAGE_BYTES;
      uint8_t* b = a + A_BYTES;
      mbar_expect(&full[s], STAGE_BYTES);
      tma2d(a, &mA, kb * BK, m0, &full[s]);
      tma2d(b, &mB, kb * BK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a = saddr(base + s * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {
        const uint64_t da = sdesc(a + 32 * k), db = sdesc(b + 32 * k);
        const uint32_t acc = (kb | k) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       saddr(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     saddr(&tfull))
                 : "memory");
  } else if (warp >= 2) {  // epilogue: TMEM lane quadrant = warp % 4
    mbar_wait(&tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + c;
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
      if (row < M) {
        int32_t* out = C + (size_t)row * N + n0 + c;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<int4*>(out + j) = make_int4(r[j], r[j + 1], r[j + 2], r[j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap map_i8(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 512, N = argc > 2 ? atoi(argv[2]) : 512,
            K = argc > 3 ? atoi(argv[3]) : 768;
  std::vector<int8_t> A((size_t)M * K), B((size_t)N * K);
  srand(1);
  for (auto& v : A) v = (int8_t)((rand() % 255) - 127);
  for (auto& v : B) v = (int8_t)((rand() % 255) - 127);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CUtensorMap mA = map_i8(dA, M, K, BM), mB = map_i8(dB, N, K, BN);
  const size_t smem = STAGES * STAGE_BYTES + 1024;
  CK(cudaFuncSetAttribute(k_i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  k_i8_gemm<<<grid, 192, smem>>>(mA, mB, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C((size_t)M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; i += (M > 2048 ? M / 61 : 1))
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[(size_t)i * K + k] * B[(size_t)j * K + k];
      if (s != C[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): %ld vs %d\n", i, j, s, C[(size_t)i * N + j]);
        ++bad;
      }
    }
  printf("M %d N %d K %d: %ld mismatches\n", M, N, K, bad);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) k_i8_gemm<<<grid, 192, smem>>>(mA, mB, dC, M, N, K);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%.3f ms per GEMM, %.1f TOPS\n", ms / reps, 2.0 * M * N * K / (ms / reps) / 1e9);
  return 0;
}
