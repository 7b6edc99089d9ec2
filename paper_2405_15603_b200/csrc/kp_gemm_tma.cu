// TMA-fed FP64 DMMA GEMM, C = A B^T (+ value-row bias), for sm_100a.
//
// Operand tiles are moved global->shared by the Tensor Memory Accelerator
// (cp.async.bulk.tensor.2d, SASS UTMALDG): one instruction per 16-column slab
// of the A or B tile, 128-byte swizzle, completion counted on the stage's
// mbarrier.  Warp 0, lane 0 doubles as the producer: it refills a stage once
// every warp has released it (empty mbarrier).  Consumer warps only wait,
// load fragments with 16-byte LDS (two DMMA k-steps per load: lane t holds
// k = 2t, 2t+1 of an 8-wide k chunk, the same permutation in A and B) and
// issue DMMA.8x8x4 (FP64 tensor cores; tcgen05 has no f64 kind).
//
// Swizzle / bank mapping: a 128-byte smem row holds 16 doubles of one operand
// row; 16-byte chunk c of row r sits at chunk (c ^ (r & 7)).  A quarter-warp of
// LDS.128 reads 2 rows x 4 chunks; to keep those 128 bytes conflict-free the
// two rows must differ in bit 2, so MMA row/col g of an 8-block reads smem row
// sigma(g) = (g >> 1) + 4 (g & 1).  The epilogue un-permutes: output row
// sigma(g), output columns sigma(2t) = t and sigma(2t+1) = t + 4.
//
// Requirements (else the cp.async kernel runs): K % BK == 0, lda/ldb even,
// A/B 16-byte aligned.  Out-of-range rows are zero-filled by the TMA unit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ int sigma8(int g) { return (g >> 1) + ((g & 1) << 2); }

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    k_gemm_nt_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  GemmNT g, int tiles_n) {
  constexpr int NW = WM * WN;
  constexpr int SLABS = BK / 16;                 // 16-double (128 B) swizzle slabs per k-tile
  constexpr int A_STAGE = BM * BK, B_STAGE = BN * BK;  // doubles
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int TM = WTM / 8, TN = WTN / 8;
  extern __shared__ __align__(1024) unsigned char smt_raw[];
  // 128-byte swizzle atoms need a 1024-byte aligned destination
  double* smt = reinterpret_cast<double*>(smt_raw + ((1024 - (smem_addr(smt_raw) & 1023)) & 1023));
  double* As = smt;
  double* Bs = smt + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tn = blockIdx.x % tiles_n;
  const int m0 = (int)((blockIdx.x / tiles_n) * BM);
  const int n0 = tn * BN;
  const int KT = g.K / BK;
  constexpr uint32_t kStageBytes = (uint32_t)(A_STAGE + B_STAGE) * sizeof(double);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  auto produce = [&](int kt) {
    const int s = kt % STAGES;
    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
    for (int sl = 0; sl < SLABS; ++sl) {
      tma_load_2d(As + s * A_STAGE + sl * BM * 16, &mapA, kt * BK + sl * 16, m0, &full[s]);
      tma_load_2d(Bs + s * B_STAGE + sl * BN * 16, &mapB, kt * BK + sl * 16, n0, &full[s]);
    }
  };
  if (threadIdx.x == 0)
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) produce(kt);

  const int wm = warp / WN, wn = warp % WN;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int sg = sigma8(g4);
  // byte offsets inside a slab for this lane: row (.. + sigma(g)), chunk (c ^ sigma(g))
  const int a_row = wm * WTM + sg;
  const int b_row = wn * WTN + sg;
  const int ch0 = ((0 + t4) ^ sg) * 2;  // k chunk 0..3 (kk = 0)  -> doubles offset
  const int ch1 = ((4 + t4) ^ sg) * 2;  // k chunk 4..7 (kk = 8)

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    const uint32_t par = (kt / STAGES) & 1;
    mbar_wait(&full[s], par);
#pragma unroll
    for (int sl = 0; sl < SLABS; ++sl) {
      const double* as = As + s * A_STAGE + sl * BM * 16 + a_row * 16;
      const double* bs = Bs + s * B_STAGE + sl * BN * 16 + b_row * 16;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int ch = half ? ch1 : ch0;
        double2 a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = *reinterpret_cast<const double2*>(as + i * 8 * 16 + ch);
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = *reinterpret_cast<const double2*>(bs + j * 8 * 16 + ch);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && kt + STAGES < KT) {
      mbar_wait(&empty[s], par);
      fence_proxy_async_smem();
      produce(kt + STAGES);
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = (int64_t)m0 + wm * WTM + i * 8 + sg;
    if (row >= g.M) continue;
    const bool add_bias = g.bias != nullptr && (row % g.S) == 0;
    double* crow = g.C + row * g.ldc;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c0 = n0 + wn * WTN + j * 8 + t4;
      const int c1 = c0 + 4;
      if (c0 < g.N) crow[c0] = acc[i][j][0] + (add_bias ? g.bias[(int64_t)c0 * g.bias_stride] : 0.0);
      if (c1 < g.N) crow[c1] = acc[i][j][1] + (add_bias ? g.bias[(int64_t)c1 * g.bias_stride] : 0.0);
    }
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (cached by operand geometry) and launch

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2-D FP64 tensor map, 16-column (128 B) boxes of box_rows rows, 128-byte swizzle;
// cached by geometry (encoding is a host call).
bool make_tma_map_2d(CUtensorMap* m, const double* base, uint64_t rows, uint64_t cols, uint64_t ld,
                     uint32_t box_rows) {
  using Key = std::tuple<const double*, uint64_t, uint64_t, uint64_t, uint32_t>;
  static std::map<Key, CUtensorMap> cache;
  static std::mutex mu;
  const Key key{base, rows, cols, ld, box_rows};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * sizeof(double)};
  cuuint32_t box[2] = {16, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
static bool run_tma(const GemmNT& g, cudaStream_t s) {
  CUtensorMap ma, mb;
  if (!make_tma_map_2d(&ma, g.A, (uint64_t)g.M, (uint64_t)g.K, (uint64_t)g.lda, BM)) return false;
  if (!make_tma_map_2d(&mb, g.B, (uint64_t)g.N, (uint64_t)g.K, (uint64_t)g.ldb, BN)) return false;
  const size_t smem = (size_t)STAGES * (BM + BN) * BK * sizeof(double) + 2 * STAGES * 8 + 1024;
  auto kern = k_gemm_nt_tma<BM, BN, WM, WN, BK, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int tiles_n = (int)ceil_div(g.N, BN);
  const int64_t tiles = ceil_div(g.M, BM) * tiles_n;
  count_launch();
  kern<<<(unsigned)tiles, WM * WN * 32, smem, s>>>(ma, mb, g, tiles_n);
  return true;
}

static bool tma_ok(const GemmNT& g) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return g.K % 16 == 0 && g.lda % 2 == 0 && g.ldb % 2 == 0 && al16(g.A) && al16(g.B) &&
         g.M < (int64_t(1) << 31);
}

// variant 0 = auto
bool launch_gemm_nt_tma(const GemmNT& g, cudaStream_t s, int variant) {
  if (g.M <= 0 || g.N <= 0) return true;
  if (!tma_ok(g)) return false;
  const bool k32 = g.K % 32 == 0;
  switch (variant) {
    case 1: return run_tma<128, 128, 2, 4, 16, 6>(g, s);
    case 2: return run_tma<128, 128, 4, 4, 16, 6>(g, s);
    case 3: return k32 && run_tma<128, 128, 2, 4, 32, 3>(g, s);
    case 4: return k32 && run_tma<128, 128, 4, 4, 32, 3>(g, s);
    case 5: return run_tma<128, 64, 4, 2, 16, 8>(g, s);
    default:  // measured on B200 (tools/gemm_bench.cu): 35.6 TFLOP/s at 128x128x32, 4x4 warps
      if (g.N <= 64) return run_tma<128, 64, 4, 2, 16, 8>(g, s);
      if (k32) return run_tma<128, 128, 4, 4, 32, 3>(g, s);
      return run_tma<128, 128, 4, 4, 16, 6>(g, s);
  }
}

}  // namespace kp
