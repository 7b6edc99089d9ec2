// TMA-fed FP64 DMMA split-row reduction  C[p][q] += sum_r X[r][p] w(r) Y[r][q]
// for the Kronecker factors A_l = sum zhat zhat^T, B_l = sum g g^T
// (reference src/curvature.py:96-137) and the residual-weighted gradient
// sum_n r_n sum_s g zhat^T (src/optim.py:164-177), sm_100a.
//
// The reduction index r (state rows) is the MMA k dimension, so operand tiles
// are [BK rows x 16 columns] slabs, loaded by the TMA unit with 128-byte
// swizzle (16-byte chunk c of smem row r at chunk c ^ (r & 7)).  A lane reads
// one 16-byte chunk = two adjacent columns (p, p+1), which feed two different
// m8 tiles (even / odd columns), so fragment loads are LDS.128; lane t of a
// k-step reads smem row 2t (+1 for the second k-step), which makes every
// quarter-warp hit 8 distinct chunks.  The per-sample residual weight is one
// __shfl per k-step.  Bias-augmentation columns (curvature.py:88-93) are not in
// this kernel: they are value-row column sums (kp_taylor.cu k_colsum).
//
// Each CTA owns one (p-tile, q-tile) pair (lower-triangle pairs only for the
// symmetric factors) and one contiguous row range ("split"); partial tiles go to
// partial[split] and are summed in split order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

bool make_tma_map_2d(CUtensorMap* m, const double* base, uint64_t rows, uint64_t cols,
                     uint64_t ld, uint32_t box_rows);  // kp_gemm_tma.cu

namespace {

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

constexpr int BM = 128, BN = 128, WM = 4, WN = 4, BK = 32, STAGES = 3;
constexpr int NW = WM * WN;
constexpr int TARGET_CTAS = 148;

struct Grid {
  int nx, ny, tiles_p, tiles_q, pairs;
  int64_t splits, rows_per_split, R;
};

Grid make_grid(int64_t R, int nx, int ny, bool sym) {
  Grid t;
  t.nx = nx;
  t.ny = ny;
  t.R = R;
  t.tiles_p = (int)ceil_div(nx, BM);
  t.tiles_q = (int)ceil_div(ny, BN);
  t.pairs = sym ? t.tiles_p * (t.tiles_p + 1) / 2 : t.tiles_p * t.tiles_q;
  int64_t splits = std::max<int64_t>(1, TARGET_CTAS / t.pairs);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, ceil_div(R, 2 * BK)));
  const int64_t rps = ceil_div(ceil_div(std::max<int64_t>(R, 1), splits), BK) * BK;
  t.splits = ceil_div(std::max<int64_t>(R, 1), rps);
  t.rows_per_split = rps;
  return t;
}

struct Args {
  const double* w;
  int Sw;
  bool sym;
};

__global__ void __launch_bounds__(NW * 32, 1)
    k_gemm_tn_tma(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapY,
                  Args a, Grid t, double* __restrict__ partial) {
  constexpr int XS = BM * BK, YS = BN * BK;  // doubles per stage
  extern __shared__ __align__(1024) unsigned char tn_raw[];
  double* sm = reinterpret_cast<double*>(tn_raw + ((1024 - (smem_addr(tn_raw) & 1023)) & 1023));
  double* Xs = sm;
  double* Ys = sm + STAGES * XS;
  uint64_t* full = reinterpret_cast<uint64_t*>(Ys + STAGES * YS);
  uint64_t* empty = full + STAGES;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.x / t.pairs;
  const int pair = blockIdx.x % t.pairs;
  int tp, tq;
  if (a.sym) {
    tp = 0;
    while ((tp + 1) * (tp + 2) / 2 <= pair) ++tp;
    tq = pair - tp * (tp + 1) / 2;
  } else {
    tp = pair / t.tiles_q;
    tq = pair % t.tiles_q;
  }
  const int p0 = tp * BM, q0 = tq * BN;
  const int64_t r_begin = (int64_t)split * t.rows_per_split;
  const int64_t r_end = min(t.R, r_begin + t.rows_per_split);
  const int KT = (int)((r_end - r_begin + BK - 1) / BK);
  constexpr uint32_t kStageBytes = (uint32_t)(XS + YS) * sizeof(double);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  auto produce = [&](int kt) {
    const int s = kt % STAGES;
    const int r = (int)(r_begin + (int64_t)kt * BK);
    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
    for (int sl = 0; sl < BM / 16; ++sl) tma2d(Xs + s * XS + sl * BK * 16, &mapX, p0 + sl * 16, r, &full[s]);
#pragma unroll
    for (int sl = 0; sl < BN / 16; ++sl) tma2d(Ys + s * YS + sl * BK * 16, &mapY, q0 + sl * 16, r, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) produce(kt);

  const int wm = warp / WN, wn = warp % WN;
  const int g4 = lane >> 2, t4 = lane & 3;
  const bool weighted = a.w != nullptr;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    const uint32_t par = (kt / STAGES) & 1;
    double wl = 1.0;
    if (weighted) {
      const int64_t r = r_begin + (int64_t)kt * BK + lane;
      wl = r < r_end ? a.w[r / a.Sw] : 0.0;
    }
    mbar_wait(&full[s], par);
    const double* xs = Xs + s * XS + (wm * 2) * BK * 16;
    const double* ys = Ys + s * YS + (wn * 2) * BK * 16;
#pragma unroll
    for (int s8 = 0; s8 < BK / 8; ++s8) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int row = 8 * s8 + 2 * t4 + half;
        const int off = row * 16 + ((g4 ^ (2 * t4 + half)) << 1);
        double2 xa[2], yb[2];
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) xa[ip] = *reinterpret_cast<const double2*>(xs + ip * BK * 16 + off);
#pragma unroll
        for (int jp = 0; jp < 2; ++jp) yb[jp] = *reinterpret_cast<const double2*>(ys + jp * BK * 16 + off);
        if (weighted) {
          const double wr = __shfl_sync(0xffffffffu, wl, row);
#pragma unroll
          for (int ip = 0; ip < 2; ++ip) {
            xa[ip].x *= wr;
            xa[ip].y *= wr;
          }
        }
#pragma unroll
        for (int ip = 0; ip < 2; ++ip)
#pragma unroll
          for (int jp = 0; jp < 2; ++jp) {
            dmma_8x8x4(acc[2 * ip][2 * jp][0], acc[2 * ip][2 * jp][1], xa[ip].x, yb[jp].x);
            dmma_8x8x4(acc[2 * ip][2 * jp + 1][0], acc[2 * ip][2 * jp + 1][1], xa[ip].x, yb[jp].y);
            dmma_8x8x4(acc[2 * ip + 1][2 * jp][0], acc[2 * ip + 1][2 * jp][1], xa[ip].y, yb[jp].x);
            dmma_8x8x4(acc[2 * ip + 1][2 * jp + 1][0], acc[2 * ip + 1][2 * jp + 1][1], xa[ip].y,
                       yb[jp].y);
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

  double* out = partial + (size_t)split * t.nx * t.ny;
#pragma unroll
  for (int ip = 0; ip < 2; ++ip)
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int p = p0 + (wm * 2 + ip) * 16 + 2 * g4 + f;
      if (p >= t.nx) continue;
#pragma unroll
      for (int jp = 0; jp < 2; ++jp)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int q = q0 + (wn * 2 + jp) * 16 + 4 * t4 + 2 * c + e;
            if (q < t.ny) out[(size_t)p * t.ny + q] = acc[2 * ip + f][2 * jp + e][c];
          }
    }
}

__global__ void k_tn_reduce2(const double* __restrict__ partial, int64_t splits, int nx, int ny,
                             bool sym, double* __restrict__ acc, int64_t ldacc) {
  const int64_t n = (int64_t)nx * ny;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ny), j = (int)(e % ny);
    if (sym && j > i) continue;
    double v = acc[(int64_t)i * ldacc + j];
    for (int64_t s = 0; s < splits; ++s) v += partial[s * n + e];
    acc[(int64_t)i * ldacc + j] = v;
  }
}

// Many splits (small problems: few tiles, many row splits): 8 warps per 32 consecutive
// entries, warp w summing splits w, w+8, ... in order, then the 8 warp sums in order.
__global__ void __launch_bounds__(256) k_tn_reduce2_wide(const double* __restrict__ partial,
                                                         int64_t splits, int nx, int ny, bool sym,
                                                         double* __restrict__ acc, int64_t ldacc) {
  __shared__ double red[8][33];
  const int64_t n = (int64_t)nx * ny;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double v = 0.0;
  if (e < n)
    for (int64_t s = w; s < splits; s += 8) v += partial[s * n + e];
  red[w][lane] = v;
  __syncthreads();
  if (w == 0 && e < n) {
    const int i = (int)(e / ny), j = (int)(e % ny);
    if (!(sym && j > i)) {
      double t = acc[(int64_t)i * ldacc + j];
#pragma unroll
      for (int k = 0; k < 8; ++k) t += red[k][lane];
      acc[(int64_t)i * ldacc + j] = t;
    }
  }
}

}  // namespace

size_t gemm_tn_tma_partial_doubles(int64_t R, int nx, int ny, bool sym) {
  Grid t = make_grid(R, nx, ny, sym);
  return (size_t)t.splits * nx * ny;
}

bool gemm_tn_tma_ok(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t R) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return ldx % 2 == 0 && ldy % 2 == 0 && al16(X) && al16(Y) && R < (int64_t(1) << 31);
}

bool launch_gemm_tn_tma_accumulate(const double* X, int64_t ldx, int nx, const double* Y,
                                   int64_t ldy, int ny, const double* w, int Sw, int64_t R,
                                   bool sym, double* partial, double* acc, int64_t ldacc,
                                   cudaStream_t s) {
  if (R <= 0 || nx <= 0 || ny <= 0) return true;
  if (!gemm_tn_tma_ok(X, ldx, Y, ldy, R)) return false;
  CUtensorMap mx, my;
  if (!make_tma_map_2d(&mx, X, (uint64_t)R, (uint64_t)nx, (uint64_t)ldx, BK)) return false;
  if (!make_tma_map_2d(&my, Y, (uint64_t)R, (uint64_t)ny, (uint64_t)ldy, BK)) return false;
  Grid t = make_grid(R, nx, ny, sym);
  const size_t smem = (size_t)STAGES * (BM + BN) * BK * sizeof(double) + 2 * STAGES * 8 + 1024;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tn_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  Args a{w, Sw, sym};
  count_launch();
  k_gemm_tn_tma<<<(unsigned)(t.splits * t.pairs), NW * 32, smem, s>>>(mx, my, a, t, partial);
  const int64_t n = (int64_t)nx * ny;
  count_launch();
  if (t.splits >= 16) {
    k_tn_reduce2_wide<<<(unsigned)ceil_div(n, 32), 256, 0, s>>>(partial, t.splits, nx, ny, sym, acc,
                                                                 ldacc);
  } else {
    const int rb = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
    k_tn_reduce2<<<rb, 256, 0, s>>>(partial, t.splits, nx, ny, sym, acc, ldacc);
  }
  return true;
}

}  // namespace kp
