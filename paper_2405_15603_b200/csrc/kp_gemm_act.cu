// Fused Taylor layer: (N*S, K) x (K, N)^T FP64 DMMA GEMM + bias + tanh Taylor
// activation (reference src/taylor.py:140-169) in one kernel, sm_100a.
//
// The activation of sample n mixes its S = d+2 rows (value, d derivatives,
// operator row: L z_out = s1 L z + s2 sum_i c_ii g_i^2), so the M tiles are
// SAMPLE-ALIGNED: a CTA owns nb = floor(128 / S) whole samples (c5: one 102-row
// sample), loaded by a 2-D TMA box of round_up(nb*S, 8) rows starting at row
// tile*nb*S, and 128 output units.  8 warps each own 16 units and all m8
// tiles (up to 16).  After the k loop the pre-activation tile is staged in
// shared memory (reusing the pipeline buffers) and one thread per
// (sample, unit) walks the sample's S rows: computes s0, s1, s2 from the value
// row, the derivative rows and the operator row, and writes them coalesced.
//
// Modes: STORE writes the pre-activation (needed by the reverse pass) and the
// activation output; LOSS writes only the output (line search); LAST does not
// write the output at all but reduces each row against the last layer's weight
// vector (h_out = 1), leaving per-tile partial dot products for
// k_last_from_partials — the line search never materialises the last hidden
// state.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

bool make_tma_map_2d(CUtensorMap* m, const double* base, uint64_t rows, uint64_t cols,
                     uint64_t ld, uint32_t box_rows);  // kp_gemm_tma.cu

namespace {

constexpr int BN_MAX = 128, ROWS_MAX = 128;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ int sigma8(int g) { return (g >> 1) + ((g & 1) << 2); }

// NW warps, each owning BN / NW output units and all TM m8 tiles.  NW = 4 keeps the
// per-CTA footprint small enough for two co-resident CTAs per SM (one's epilogue
// overlaps the other's DMMA loop); NW = 8 serves the 15-16 tile shapes.
template <int BK, int STAGES, int MODE, int TM, int NW, int BN, int MINB = 8 / NW>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_gemm_act(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               GemmAct g, int tiles_n, int box_rows) {
  constexpr int NWARP = NW;
  constexpr int CPITCH = BN + 4;
  constexpr int WCOLS = BN / NW, TNW = WCOLS / 8;  // units and n8 tiles per warp
  constexpr int SLABS = BK / 16;
  constexpr int AROWS = TM * 8;
  constexpr int A_STAGE = AROWS * BK, B_STAGE = BN * BK;
  extern __shared__ __align__(1024) unsigned char act_raw[];
  double* sm = reinterpret_cast<double*>(act_raw + ((1024 - (smem_addr(act_raw) & 1023)) & 1023));
  double* As = sm;
  double* Bs = sm + STAGES * A_STAGE;
  // The pipeline barriers sit after both the pipeline stages and the epilogue's C staging
  // (which reuses the stage smem): overwriting live mbarrier objects (no mbarrier.inval)
  // gave sporadic garbage rows (NaN in ~1 of 10^3 line-search launches at c5 scale).
  // (A static __shared__ array instead costs 2.5% on the line search.)
  constexpr int CS_DOUBLES = AROWS * (BN + 4);
  constexpr int PIPE_DOUBLES = STAGES * (A_STAGE + B_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (CS_DOUBLES > PIPE_DOUBLES ? CS_DOUBLES : PIPE_DOUBLES));
  uint64_t* empty = full + STAGES;
  double* Cs = sm;  // epilogue staging, aliases the (drained) pipeline

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tn = blockIdx.x % tiles_n;
  const int64_t smp0 = (int64_t)(blockIdx.x / tiles_n) * g.nb;
  const int S = g.S;
  const int kk = blockIdx.y;  // candidate batch entry
  const int m0 = (int)(smp0 * S);                             // row inside this entry
  const int ma = (int)(kk * g.n_samples * S + m0);            // row in the stacked A map
  const int n0 = tn * BN;
  const int nb0 = kk * g.N + n0;                              // row in the stacked B map
  if (kk > 0) {
    if (g.bias) g.bias += kk * g.bias_bstride;
    if (g.pre) g.pre += kk * g.out_bstride;
    if (g.post) g.post += kk * g.out_bstride;
    if (g.upart) g.upart += kk * g.upart_bstride;
    if (g.wlast) g.wlast += kk * g.wlast_bstride;
  }
  const int KT = g.K / BK;
  // Two CTAs share each SM (NW = 4).  Launched together they run in lockstep, so both
  // epilogues leave the DMMA pipe idle at the same time.  On long grids, delay the second
  // CTA of each SM in the first wave (blocks 148..295: the scheduler fills SMs breadth-first)
  // by about half a tile so that one CTA's epilogue overlaps the other's k loop
  // (measured: c5 line search -1.1%).
  if (NW == 4 && blockIdx.y == 0 && gridDim.x >= 8 * 296 && blockIdx.x >= 148 && blockIdx.x < 296) {
    const unsigned ns = (unsigned)KT * (BK / 16) * 850u;
    for (unsigned t = 0; t < ns; t += 1000000u) __nanosleep(ns - t < 1000000u ? ns - t : 1000000u);
  }
  const uint32_t stage_bytes = (uint32_t)(box_rows + BN) * BK * sizeof(double);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto produce = [&](int kt) {
    const int s = kt % STAGES;
    mbar_arrive_expect_tx(&full[s], stage_bytes);
#pragma unroll
    for (int sl = 0; sl < SLABS; ++sl) {
      tma2d(As + s * A_STAGE + sl * AROWS * 16, &mapA, kt * BK + sl * 16, ma, &full[s]);
      tma2d(Bs + s * B_STAGE + sl * BN * 16, &mapB, kt * BK + sl * 16, nb0, &full[s]);
    }
  };
  if (threadIdx.x == 0)
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) produce(kt);

  const int g4 = lane >> 2, t4 = lane & 3;
  const int sg = sigma8(g4);
  const int ch0 = ((0 + t4) ^ sg) * 2, ch1 = ((4 + t4) ^ sg) * 2;

  double acc[TM][TNW][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TNW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    const uint32_t par = (kt / STAGES) & 1;
    mbar_wait(&full[s], par);
#pragma unroll
    for (int sl = 0; sl < SLABS; ++sl) {
      const double* as = As + s * A_STAGE + sl * AROWS * 16 + sg * 16;
      const double* bs = Bs + s * B_STAGE + sl * BN * 16 + (warp * WCOLS + sg) * 16;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int ch = half ? ch1 : ch0;
        double2 b[TNW];
#pragma unroll
        for (int j = 0; j < TNW; ++j) b[j] = *reinterpret_cast<const double2*>(bs + j * 8 * 16 + ch);
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const double2 a = *reinterpret_cast<const double2*>(as + i * 8 * 16 + ch);
#pragma unroll
          for (int j = 0; j < TNW; ++j) {
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a.x, b[j].x);
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a.y, b[j].y);
          }
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
  __syncthreads();  // every stage consumed: the pipeline smem becomes the C tile

  // stage pre-activations (+ value-row bias) in smem: row 8i + sigma(g), col 16w + 8j + t (+4)
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = i * 8 + sg;
    const bool vrow = ((row % S) == 0) && g.bias != nullptr;
#pragma unroll
    for (int j = 0; j < TNW; ++j) {
      const int c0 = warp * WCOLS + j * 8 + t4, c1 = c0 + 4;
      double v0 = acc[i][j][0], v1 = acc[i][j][1];
      if (vrow) {
        if (n0 + c0 < g.N) v0 += g.bias[(int64_t)(n0 + c0) * g.bias_stride];
        if (n0 + c1 < g.N) v1 += g.bias[(int64_t)(n0 + c1) * g.bias_stride];
      }
      Cs[row * CPITCH + c0] = v0;
      Cs[row * CPITCH + c1] = v1;
    }
  }
  __syncthreads();

  const int64_t nsmp = (g.n_samples - smp0) < g.nb ? (g.n_samples - smp0) : (int64_t)g.nb;
  const int ncol = min(BN, g.N - n0);
  const int d = g.d;
  for (int idx = threadIdx.x; idx < nsmp * BN; idx += NWARP * 32) {
    const int k = idx / BN, j = idx % BN;
    if (j >= ncol) continue;
    double* cs = Cs + (k * S) * CPITCH + j;
    const int64_t grow = (int64_t)m0 + k * S;
    const TanhD t = tanh_derivs(cs[0], false);
    if (MODE == ACT_STORE) g.pre[grow * g.ldo + n0 + j] = cs[0];
    double o0 = t.s0;
    if (MODE == ACT_LAST) cs[0] = o0;
    else g.post[grow * g.ldo + n0 + j] = o0;
    if (!g.taylor) continue;
    double quad = 0.0;
    for (int i = 1; i <= d; ++i) {
      const double gi = cs[i * CPITCH];
      quad += (gi * g.cdiag[i - 1]) * gi;
      const double o = t.s1 * gi;
      if (MODE == ACT_STORE) g.pre[(grow + i) * g.ldo + n0 + j] = gi;
      if (MODE == ACT_LAST) cs[i * CPITCH] = o;
      else g.post[(grow + i) * g.ldo + n0 + j] = o;
    }
    const double ell = cs[(d + 1) * CPITCH];
    const double o = t.s1 * ell + t.s2 * quad;
    if (MODE == ACT_STORE) g.pre[(grow + d + 1) * g.ldo + n0 + j] = ell;
    if (MODE == ACT_LAST) cs[(d + 1) * CPITCH] = o;
    else g.post[(grow + d + 1) * g.ldo + n0 + j] = o;
  }
  if (MODE == ACT_LAST) {
    // one thread per row: a sequential dot over the tile's units against the last layer's
    // weights (staged in smem), starting at unit (r mod 32) so that the 32 rows of a warp
    // hit distinct banks (row pitch CPITCH + 1 is odd in 8-byte words)
    __shared__ double wl[BN];
    for (int j = threadIdx.x; j < BN; j += NWARP * 32) wl[j] = j < ncol ? g.wlast[n0 + j] : 0.0;
    __syncthreads();
    const int rows = (int)nsmp * S;
    for (int r = threadIdx.x; r < rows; r += NWARP * 32) {
      const double* cr = Cs + r * CPITCH;
      double a = 0.0;
      int j = (r & 31) % ncol;
      for (int jj = 0; jj < ncol; ++jj) {
        a = fma(cr[j], wl[j], a);
        j = (j + 1 == ncol) ? 0 : j + 1;
      }
      g.upart[((int64_t)m0 + r) * tiles_n + tn] = a;
    }
  }
}

template <int MODE, int TM, int NW, int BK, int STAGES, int BN = BN_MAX, int MINB = 8 / NW>
bool run_act(const GemmAct& g, int box_rows, cudaStream_t s) {
  constexpr int CPITCH = BN + 4;
  CUtensorMap ma, mb;
  const int64_t M = g.n_samples * g.S * g.batch;
  if (g.K % BK) return false;
  if (!make_tma_map_2d(&ma, g.A, (uint64_t)M, (uint64_t)g.K, (uint64_t)g.lda, box_rows)) return false;
  if (!make_tma_map_2d(&mb, g.B, (uint64_t)g.N * g.batch, (uint64_t)g.K, (uint64_t)g.ldb, BN))
    return false;
  const size_t pipe = (size_t)STAGES * (TM * 8 + BN) * BK * sizeof(double);
  const size_t cst = (size_t)TM * 8 * CPITCH * sizeof(double);
  const size_t smem = std::max(pipe, cst) + 2 * STAGES * 8 + 1024;
  auto kern = k_gemm_act<BK, STAGES, MODE, TM, NW, BN, MINB>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int tiles_n = (int)ceil_div(g.N, BN);
  const int64_t tiles = ceil_div(g.n_samples, g.nb) * tiles_n;
  count_launch();
  kern<<<dim3((unsigned)tiles, (unsigned)g.batch), NW * 32, smem, s>>>(ma, mb, g, tiles_n, box_rows);
  return true;
}

// Tile shapes up to 13 m8 tiles (one large sample per tile): 4 warps x 128 units, BK 16,
// 3 stages -> ~111 KB, two CTAs per SM.  14-16 tiles (many small samples per tile): 4 warps
// x 64 units, BK 16, 3 stages, three CTAs per SM.
template <int MODE, int TM>
bool run_act_tm(const GemmAct& g, int box_rows, cudaStream_t s) {
  if constexpr (TM <= 8) {
    // 64-row tiles for short K (<= 64: c1-c3): 64-unit tiles, 2 stages, five CTAs per SM
    // (~36 KB each; 3 stages / 4 CTAs: c2 line search 1.03 ms, this 0.95; 6 CTAs spill)
    return run_act<MODE, TM, 4, 16, 2, 64, 5>(g, box_rows, s);
  } else if constexpr (TM <= 13) {
    return run_act<MODE, TM, 4, 16, 3>(g, box_rows, s);
  } else {
    // 64-unit tiles, 4 warps, BK 16, 3 stages, three CTAs per SM (~72 KB each) so that
    // epilogues overlap other CTAs' k loops (vs 8 warps x 128 units: c4 line search -11%;
    // vs BK 32 x 2 stages for short K: c1-c3 line search -7%)
    return run_act<MODE, TM, 4, 16, 3, 64, 3>(g, box_rows, s);
  }
}

}  // namespace

// State rows per tile: 64 for short K (the tiles are latency-bound; smaller ones let four
// CTAs share an SM), else 128.  KP_ACT_SMALL_ROWS=0 keeps 128 (measurements).
static int act_rows(int K) {
  static const bool small = [] {
    const char* e = getenv("KP_ACT_SMALL_ROWS");
    return !(e && atoi(e) == 0);
  }();
  return (small && K <= 64) ? 64 : ROWS_MAX;
}

int gemm_act_samples_per_tile(int S, int K) {
  const int rows = act_rows(K);
  return S <= rows ? rows / S : 0;
}

// Unit width of the fused layer's tiles for this shape (mirrors run_act_tm); the LAST mode
// leaves ceil(N / width) partial dots per row.
int gemm_act_tile_width(int S, int N, int K) {
  const int nb = gemm_act_samples_per_tile(S, K);
  const int tm = nb > 0 ? (nb * S + 7) / 8 : 0;
  return (tm <= 8 || tm > 13) ? 64 : BN_MAX;
}

bool gemm_act_ok(int S, int K, int64_t lda, int64_t ldb) {
  return S <= ROWS_MAX && K % 16 == 0 && lda % 2 == 0 && ldb % 2 == 0;
}

bool launch_gemm_act(GemmAct g, int mode, cudaStream_t s) {
  if (g.n_samples <= 0) return true;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (g.S > ROWS_MAX || g.K % 16 != 0 || g.lda % 2 || g.ldb % 2 || !al16(g.A) || !al16(g.B) ||
      g.n_samples * g.S * g.batch >= (int64_t(1) << 31) || g.N * (int64_t)g.batch >= (int64_t(1) << 31))
    return false;
  g.nb = gemm_act_samples_per_tile(g.S, g.K);
  if (g.nb <= 0) return false;
  const int box_rows = (g.nb * g.S + 7) / 8 * 8;
  // the m8-tile count is a template parameter: predicated-off DMMAs still occupy the
  // tensor pipe, so a runtime guard over a 16-tile array wastes up to 16/tm of it
  switch (box_rows / 8) {
#define KP_ACT_CASE(T)                                                   \
  case T:                                                                \
    if (mode == ACT_STORE) return run_act_tm<ACT_STORE, T>(g, box_rows, s); \
    if (mode == ACT_LOSS) return run_act_tm<ACT_LOSS, T>(g, box_rows, s);   \
    return run_act_tm<ACT_LAST, T>(g, box_rows, s);
    KP_ACT_CASE(5)
    KP_ACT_CASE(6)
    KP_ACT_CASE(7)
    KP_ACT_CASE(8)
    KP_ACT_CASE(9)
    KP_ACT_CASE(10)
    KP_ACT_CASE(11)
    KP_ACT_CASE(12)
    KP_ACT_CASE(13)
    KP_ACT_CASE(14)
    KP_ACT_CASE(15)
    KP_ACT_CASE(16)
#undef KP_ACT_CASE
    default:
      return false;
  }
}

// u_{n,s} = sum_t upart[(n*S+s)*ntn + t] + (s == 0) b;  residual as in k_last_layer.
constexpr int KP_LAST_MAX_S = 130;  // S <= 128 on the fused path
__global__ void k_last_from_partials(const double* __restrict__ upart, int ntn, int64_t n,
                                     TaylorDims td, const double* __restrict__ bias,
                                     const double* __restrict__ r0, const double* __restrict__ seeds,
                                     const double* __restrict__ targets, double* __restrict__ r,
                                     int64_t bias_bstride, int64_t r_bstride,
                                     const double* __restrict__ quad) {
  upart += (int64_t)blockIdx.y * n * td.S * ntn;
  bias += (int64_t)blockIdx.y * bias_bstride;
  r += (int64_t)blockIdx.y * r_bstride;
  for (int64_t smp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; smp < n;
       smp += (int64_t)gridDim.x * blockDim.x) {
    double uu[KP_LAST_MAX_S];
    double v = 0.0;
    for (int s = 0; s < td.S; ++s) {
      const double* up = upart + (smp * td.S + s) * ntn;
      double u = 0.0;
      for (int t = 0; t < ntn; ++t) u += up[t];
      if (s == 0) u += bias[0];
      if (td.taylor) uu[s] = u;
      else v = u - targets[smp];
    }
    if (td.taylor)
      v = point_residual(uu, td.S, r0[smp], seeds + smp * td.S, quad ? quad + smp * td.d : nullptr,
                         nullptr);
    r[smp] = v;
  }
}

void launch_last_from_partials(const double* upart, int ntn, int64_t n, TaylorDims td,
                               const double* bias, const double* r0, const double* seeds,
                               const double* targets, double* r, cudaStream_t s, int batch,
                               int64_t bias_bstride, int64_t r_bstride, const double* quad) {
  if (n <= 0) return;
  count_launch();
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, 128), 148 * 16);
  k_last_from_partials<<<dim3(blocks, (unsigned)batch), 128, 0, s>>>(
      upart, ntn, n, td, bias, r0, seeds, targets, r, bias_bstride, r_bstride, quad);
}

}  // namespace kp
