// FP64 tensor-core (DMMA) GEMMs for the Taylor-mode KFAC step on sm_100a.
//
// B200 has no FP64 tcgen05/UMMA kind; FP64 tensor math is the warp-level
// mma.sync .f64 path (SASS DMMA.8x8x4), measured at 37.1 TFLOP/s on the pool's
// B200s (profiles/r01_fp64_peaks.txt) vs 34 TFLOP/s for DFMA.  Operands are
// staged global->shared with a multi-stage cp.async (LDGSTS) pipeline.
//
//  * k_gemm_nt : C = A B^T over the flattened (N*S, h) Taylor state — the
//    per-layer contraction of the forward pass (reference src/taylor.py:134-148)
//    and of the reverse pass (src/taylor.py:271, with B = W^T).
//  * k_gemm_tn : split-row reductions sum_r x_r y_r^T — the Kronecker factors
//    A_l, B_l (src/curvature.py:96-137) and the residual-weighted gradient
//    (src/optim.py:164-177).  Bias-augmentation (src/curvature.py:88-93) is a
//    virtual column, never materialised; per-sample residual weights are applied
//    to the fragments.  Partial tiles are reduced in a fixed order, so results
//    are bit-reproducible run to run.
#include <algorithm>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

// ---------------------------------------------------------------------------
// NT GEMM

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(WM* WN * 32, 1) k_gemm_nt(GemmNT g, int tiles_n) {
  constexpr int NT = WM * WN * 32;
  constexpr int LDS = BK + 4;  // row pitch (doubles): 8 rows x 4 k of a fragment hit distinct banks
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int TM = WTM / 8, TN = WTN / 8;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = sm + STAGES * BM * LDS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int tn = blockIdx.x % tiles_n;
  const int64_t m0 = (int64_t)(blockIdx.x / tiles_n) * BM;
  const int n0 = tn * BN;
  const int KT = (g.K + BK - 1) / BK;
  if (blockIdx.y > 0) {  // batch entry
    g.A += blockIdx.y * g.sA;
    g.B += blockIdx.y * g.sB;
    g.C += blockIdx.y * g.sC;
    if (g.bias) g.bias += blockIdx.y * g.sBias;
  }

  auto load = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * BM * LDS;
    double* bs = Bs + stage * BN * LDS;
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      const int r = e / BK, c = e % BK;
      const int64_t gm = m0 + r;
      const int gk = k0 + c;
      const bool p = gm < g.M && gk < g.K;
      cp_async8(as + r * LDS + c, p ? g.A + gm * g.lda + gk : g.A, p);
    }
#pragma unroll
    for (int e = tid; e < BN * BK; e += NT) {
      const int r = e / BK, c = e % BK;
      const int gn = n0 + r, gk = k0 + c;
      const bool p = gn < g.N && gk < g.K;
      cp_async8(bs + r * LDS + c, p ? g.B + (int64_t)gn * g.ldb + gk : g.B, p);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load(nk % STAGES, nk);
    cp_async_commit();
    const int st = kt % STAGES;
    const double* as = As + st * BM * LDS + (wm * WTM + (lane >> 2)) * LDS + (lane & 3);
    const double* bs = Bs + st * BN * LDS + (wn * WTN + (lane >> 2)) * LDS + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = as[i * 8 * LDS + kk];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = bs[j * 8 * LDS + kk];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = m0 + wm * WTM + i * 8 + (lane >> 2);
    if (row >= g.M) continue;
    const bool add_bias = g.bias != nullptr && (row % g.S) == 0;
    double* crow = g.C + row * g.ldc;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = n0 + wn * WTN + j * 8 + 2 * (lane & 3);
      double c0 = acc[i][j][0], c1 = acc[i][j][1];
      if (col < g.N) {
        if (add_bias) c0 += g.bias[(int64_t)col * g.bias_stride];
        crow[col] = c0;
      }
      if (col + 1 < g.N) {
        if (add_bias) c1 += g.bias[(int64_t)(col + 1) * g.bias_stride];
        crow[col + 1] = c1;
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
static void run_nt(const GemmNT& g, cudaStream_t s) {
  constexpr int LDS = BK + 4;
  const size_t smem = (size_t)STAGES * (BM + BN) * LDS * sizeof(double);
  auto kern = k_gemm_nt<BM, BN, WM, WN, BK, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int tiles_n = (int)ceil_div(g.N, BN);
  const int64_t tiles = ceil_div(g.M, BM) * tiles_n;
  count_launch();
  kern<<<dim3((unsigned)tiles, (unsigned)g.batch), WM * WN * 32, smem, s>>>(g, tiles_n);
}

void launch_gemm_nt(const GemmNT& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.batch == 1 && launch_gemm_nt_tma(g, s, 0)) return;
  launch_gemm_nt_cpasync(g, s);
}

void launch_gemm_nt_cpasync(const GemmNT& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.N <= 64)
    run_nt<128, 64, 4, 2, 16, 4>(g, s);
  else
    run_nt<128, 128, 2, 4, 16, 4>(g, s);
}

// ---------------------------------------------------------------------------
// TN split-row reduction

constexpr int TN_BM = 64, TN_BN = 64, TN_WM = 2, TN_WN = 2, TN_BK = 16, TN_STAGES = 3;
constexpr int TN_TARGET_CTAS = 148 * 4;
// grouped passes: two waves of four CTAs per SM (c1 accumulate 0.528 -> 0.519 ms, c2 0.713 ->
// 0.683; one wave 0.53 / 0.71, four waves 0.54 / 0.70)
constexpr int TN_GROUP_TARGET_CTAS = 148 * 8;

struct TnGrid {
  int P, Q, tiles_p, tiles_q, pairs;
  int64_t splits, rows_per_split;
};

static TnGrid tn_grid(int64_t R, int P, int Q, bool sym) {
  TnGrid t;
  t.P = P;
  t.Q = Q;
  t.tiles_p = (int)ceil_div(P, TN_BM);
  t.tiles_q = (int)ceil_div(Q, TN_BN);
  t.pairs = sym ? t.tiles_p * (t.tiles_p + 1) / 2 : t.tiles_p * t.tiles_q;
  int64_t splits = std::max<int64_t>(1, TN_TARGET_CTAS / t.pairs);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, ceil_div(R, 4 * TN_BK)));
  int64_t rps = ceil_div(ceil_div(std::max<int64_t>(R, 1), splits), TN_BK) * TN_BK;
  t.splits = ceil_div(std::max<int64_t>(R, 1), rps);
  t.rows_per_split = rps;
  return t;
}

// One-column contractions (the h_out = 1 output layer's B factor and gradient:
// X = Gbar_L, one column): acc[j] += sum_r x_r w_{r/Sw} y_{r,j} (+ y's bias column) is a
// weighted column sum over the rows of Y, HBM-bound; the 64 x 64 DMMA tiles would compute
// 63 wasted rows of every tile (c5: 9.3 ms for a 6.8 GB read).  Rows are split over about
// eight blocks per SM, one partial row per block, reduced by k_tn_reduce (fixed order).
constexpr int COL1_THREADS = 256, COL1_WIDE = 4, COL1_TINY = 8;
constexpr int64_t COL1_TARGET_BLOCKS = 148 * 8;

static int64_t col1_splits(int64_t R) {
  return std::max<int64_t>(1, std::min<int64_t>(COL1_TARGET_BLOCKS, ceil_div(R, 4 * COL1_THREADS)));
}

size_t gemm_tn_partial_doubles(int64_t R, int P, int Q, bool sym) {
  TnGrid t = tn_grid(R, P, Q, sym);
  size_t need = (size_t)t.splits * P * Q;
  if (P == 1) need = std::max(need, (size_t)col1_splits(R) * Q);
  return need;
}

__device__ __forceinline__ double col1_x(const GemmTN& g, int64_t r) {
  const double x = g.X[r * g.ldx];
  return g.w ? x * g.w[r / g.Sw] : x;
}

// Q > COL1_TINY: thread t owns columns t + 256 k; the block's rows go through shared memory
// 256 at a time (x_r w_r staged once), each row of Y read coalesced.
__global__ void __launch_bounds__(COL1_THREADS) k_tn_col1_wide(GemmTN g, int Q, int64_t rpb,
                                                             double* __restrict__ partial) {
  __shared__ double xs[COL1_THREADS];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = g.R < r0 + rpb ? g.R : r0 + rpb;
  double acc[COL1_WIDE];
#pragma unroll
  for (int k = 0; k < COL1_WIDE; ++k) acc[k] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += COL1_THREADS) {
    const int nr = (int)(r1 - rb < COL1_THREADS ? r1 - rb : COL1_THREADS);
    __syncthreads();
    if (tid < nr) xs[tid] = col1_x(g, rb + tid);
    __syncthreads();
#pragma unroll 8
    for (int i = 0; i < nr; ++i) {
      const double xv = xs[i];
      const int64_t r = rb + i;
      const double* yr = g.Y + r * g.ldy;
      const bool brow = g.y_bias && (r % g.S) == 0;
#pragma unroll
      for (int k = 0; k < COL1_WIDE; ++k) {
        const int j = tid + COL1_THREADS * k;
        if (j < g.ny) acc[k] = fma(xv, yr[j], acc[k]);
        else if (j == g.ny && brow) acc[k] += xv;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < COL1_WIDE; ++k) {
    const int j = tid + COL1_THREADS * k;
    if (j < Q) partial[(int64_t)blockIdx.x * Q + j] = acc[k];
  }
}

// Q <= COL1_TINY (the 1 x 1 B factor of the output layer): thread per row, block reduction.
__global__ void __launch_bounds__(COL1_THREADS) k_tn_col1_tiny(GemmTN g, int Q, int64_t rpb,
                                                             double* __restrict__ partial) {
  __shared__ double red[COL1_THREADS / 32][COL1_TINY];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = g.R < r0 + rpb ? g.R : r0 + rpb;
  double acc[COL1_TINY];
#pragma unroll
  for (int k = 0; k < COL1_TINY; ++k) acc[k] = 0.0;
  for (int64_t r = r0 + tid; r < r1; r += COL1_THREADS) {
    const double xv = col1_x(g, r);
    const double* yr = g.Y + r * g.ldy;
    const bool brow = g.y_bias && (r % g.S) == 0;
#pragma unroll
    for (int k = 0; k < COL1_TINY; ++k) {
      if (k < g.ny) acc[k] = fma(xv, yr[k], acc[k]);
      else if (k == g.ny && brow) acc[k] += xv;
    }
  }
#pragma unroll
  for (int k = 0; k < COL1_TINY; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (tid < Q) {
    double v = 0.0;
    for (int w = 0; w < COL1_THREADS / 32; ++w) v += red[w][tid];
    partial[(int64_t)blockIdx.x * Q + tid] = v;
  }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__device__ __forceinline__ void tn_block(const GemmTN& g, const TnGrid& t, double* partial,
                                         int block) {
  constexpr int NT = WM * WN * 32;
  constexpr int LDX = BM + 4, LDY = BN + 4;  // pitch = 4 mod 16 doubles: conflict-free fragments
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int TM = WTM / 8, TN = WTN / 8;
  extern __shared__ __align__(16) double tsm[];
  double (*Xs)[BK * LDX] = reinterpret_cast<double (*)[BK * LDX]>(tsm);
  double (*Ys)[BK * LDY] = reinterpret_cast<double (*)[BK * LDY]>(tsm + STAGES * BK * LDX);
  double (*Ws)[BK] = reinterpret_cast<double (*)[BK]>(tsm + STAGES * BK * (LDX + LDY));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int split = block / t.pairs;
  const int pair = block % t.pairs;
  int tp, tq;
  if (g.sym) {
    tp = (int)((sqrt(8.0 * pair + 1.0) - 1.0) * 0.5);
    while ((tp + 1) * (tp + 2) / 2 <= pair) ++tp;
    while (tp * (tp + 1) / 2 > pair) --tp;
    tq = pair - tp * (tp + 1) / 2;
  } else {
    tp = pair / t.tiles_q;
    tq = pair % t.tiles_q;
  }
  const int p0 = tp * BM, q0 = tq * BN;
  const int64_t r_begin = (int64_t)split * t.rows_per_split;
  const int64_t r_end = (g.R < r_begin + t.rows_per_split) ? g.R : r_begin + t.rows_per_split;
  const int64_t span = r_end > r_begin ? r_end - r_begin : 0;
  const int KT = (int)((span + BK - 1) / BK);

  auto load = [&](int stage, int kt) {
    const int64_t r0 = r_begin + (int64_t)kt * BK;
    double* xs = Xs[stage];
    double* ys = Ys[stage];
#pragma unroll
    for (int e = tid; e < BK * BM; e += NT) {
      const int row = e / BM, col = e % BM;
      const int64_t r = r0 + row;
      const int p = p0 + col;
      double* dst = xs + row * LDX + col;
      if (r < r_end && p < g.nx) {
        cp_async8(dst, g.X + r * g.ldx + p, true);
      } else {
        *dst = (r < r_end && g.x_bias && p == g.nx && (r % g.S) == 0) ? 1.0 : 0.0;
      }
    }
#pragma unroll
    for (int e = tid; e < BK * BN; e += NT) {
      const int row = e / BN, col = e % BN;
      const int64_t r = r0 + row;
      const int q = q0 + col;
      double* dst = ys + row * LDY + col;
      if (r < r_end && q < g.ny) {
        cp_async8(dst, g.Y + r * g.ldy + q, true);
      } else {
        *dst = (r < r_end && g.y_bias && q == g.ny && (r % g.S) == 0) ? 1.0 : 0.0;
      }
    }
    if (g.w != nullptr && tid < BK) {
      const int64_t r = r0 + tid;
      Ws[stage][tid] = r < r_end ? g.w[r / g.Sw] : 0.0;
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load(s, s);
    cp_async_commit();
  }
  const bool weighted = g.w != nullptr;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load(nk % STAGES, nk);
    cp_async_commit();
    const int st = kt % STAGES;
    const double* xs = Xs[st] + (lane & 3) * LDX + wm * WTM + (lane >> 2);
    const double* ys = Ys[st] + (lane & 3) * LDY + wn * WTN + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[TM], b[TN];
      const double wk = weighted ? Ws[st][kk + (lane & 3)] : 1.0;
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = xs[kk * LDX + i * 8] * wk;
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = ys[kk * LDY + j * 8];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  double* out = partial + (size_t)split * t.P * t.Q;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = p0 + wm * WTM + i * 8 + (lane >> 2);
    if (row >= t.P) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = q0 + wn * WTN + j * 8 + 2 * (lane & 3);
      if (col < t.Q) out[(size_t)row * t.Q + col] = acc[i][j][0];
      if (col + 1 < t.Q) out[(size_t)row * t.Q + col + 1] = acc[i][j][1];
    }
  }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(WM* WN * 32) k_gemm_tn(GemmTN g, TnGrid t, double* partial) {
  tn_block<BM, BN, WM, WN, BK, STAGES>(g, t, partial, blockIdx.x);
}

// Grouped launch: many small contractions (every factor and gradient block of a pass of
// a small network) share one grid; block b belongs to the job j with
// begin[j] <= b < begin[j + 1].  Same arithmetic and split order as the single launch.
constexpr int TN_GROUP_MAX = 40;
struct TnGroup {
  int njobs;
  int begin[TN_GROUP_MAX + 1];
  GemmTN g[TN_GROUP_MAX];
  TnGrid t[TN_GROUP_MAX];
  double* partial[TN_GROUP_MAX];
  double* acc[TN_GROUP_MAX];
  int64_t ebegin[TN_GROUP_MAX + 1];  // output-element prefix for the grouped reduce
};

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(WM* WN * 32) k_gemm_tn_grouped(const __grid_constant__ TnGroup G) {
  int j = 0;
  while (j + 1 < G.njobs && (int)blockIdx.x >= G.begin[j + 1]) ++j;
  tn_block<BM, BN, WM, WN, BK, STAGES>(G.g[j], G.t[j], G.partial[j], blockIdx.x - G.begin[j]);
}

__global__ void k_tn_reduce_grouped(const __grid_constant__ TnGroup G) {
  const int64_t total = G.ebegin[G.njobs];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < G.njobs && e >= G.ebegin[j + 1]) ++j;
    const int64_t le = e - G.ebegin[j];
    const int P = G.t[j].P, Q = G.t[j].Q;
    const int i = (int)(le / Q), c = (int)(le % Q);
    if (G.g[j].sym && c > i) continue;
    const int64_t n = (int64_t)P * Q;
    const double* part = G.partial[j];
    double v = G.acc[j][le];
    for (int64_t sp = 0; sp < G.t[j].splits; ++sp) v += part[sp * n + le];
    G.acc[j][le] = v;
  }
}

__global__ void k_tn_reduce(const double* __restrict__ partial, int64_t splits, int P, int Q,
                            bool sym, double* __restrict__ acc) {
  const int64_t n = (int64_t)P * Q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / Q), j = (int)(e % Q);
    if (sym && j > i) continue;
    double v = acc[e];
    for (int64_t s = 0; s < splits; ++s) v += partial[s * n + e];
    acc[e] = v;
  }
}

void launch_gemm_tn_accumulate(const GemmTN& g, double* partial, double* acc, cudaStream_t s) {
  const int P = g.nx + (g.x_bias ? 1 : 0);
  const int Q = g.ny + (g.y_bias ? 1 : 0);
  if (g.R <= 0 || P <= 0 || Q <= 0) return;
  if (g.nx == 1 && !g.x_bias && Q <= COL1_THREADS * COL1_WIDE) {
    const int64_t splits = col1_splits(g.R);
    const int64_t rpb = ceil_div(ceil_div(g.R, splits), COL1_THREADS) * COL1_THREADS;
    const int64_t blocks = ceil_div(g.R, rpb);
    count_launch();
    if (Q <= COL1_TINY)
      k_tn_col1_tiny<<<(unsigned)blocks, COL1_THREADS, 0, s>>>(g, Q, rpb, partial);
    else
      k_tn_col1_wide<<<(unsigned)blocks, COL1_THREADS, 0, s>>>(g, Q, rpb, partial);
    count_launch();
    k_tn_reduce<<<(int)std::min<int64_t>(ceil_div(Q, 256), 148 * 8), 256, 0, s>>>(
        partial, blocks, 1, Q, false, acc);
    return;
  }
  TnGrid t = tn_grid(g.R, P, Q, g.sym);
  const unsigned blocks = (unsigned)(t.splits * t.pairs);
  auto kern = k_gemm_tn<TN_BM, TN_BN, TN_WM, TN_WN, TN_BK, TN_STAGES>;
  const size_t smem =
      sizeof(double) * TN_STAGES * TN_BK * ((TN_BM + 4) + (TN_BN + 4) + 1);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  count_launch();
  kern<<<blocks, TN_WM * TN_WN * 32, smem, s>>>(g, t, partial);
  const int64_t n = (int64_t)P * Q;
  const int rb = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
  count_launch();
  k_tn_reduce<<<rb, 256, 0, s>>>(partial, t.splits, P, Q, g.sym, acc);
}


// Splits for a grouped pass: about TN_GROUP_TARGET_CTAS CTAs in total, shared by the jobs in
// proportion to their work (rows x tile pairs).
static void tn_group_grids(const GemmTN* jobs, int n, TnGrid* out) {
  double work = 0.0;
  for (int j = 0; j < n; ++j) {
    const int P = jobs[j].nx + (jobs[j].x_bias ? 1 : 0), Q = jobs[j].ny + (jobs[j].y_bias ? 1 : 0);
    TnGrid t = tn_grid(jobs[j].R, P, Q, jobs[j].sym);
    work += (double)std::max<int64_t>(jobs[j].R, 1) * t.pairs;
    out[j] = t;
  }
  for (int j = 0; j < n; ++j) {
    TnGrid& t = out[j];
    const int64_t R = std::max<int64_t>(jobs[j].R, 1);
    const double share = (double)R * t.pairs / std::max(work, 1.0);
    int64_t splits = std::max<int64_t>(1, (int64_t)(share * TN_GROUP_TARGET_CTAS / t.pairs));
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, ceil_div(R, 4 * TN_BK)));
    const int64_t rps = ceil_div(ceil_div(R, splits), TN_BK) * TN_BK;
    t.splits = ceil_div(R, rps);
    t.rows_per_split = rps;
  }
}

size_t gemm_tn_grouped_partial_doubles(const GemmTN* jobs, int n) {
  if (n <= 0 || n > TN_GROUP_MAX) return 0;
  TnGrid t[TN_GROUP_MAX];
  tn_group_grids(jobs, n, t);
  size_t tot = 0;
  for (int j = 0; j < n; ++j) tot += (size_t)t[j].splits * t[j].P * t[j].Q;
  return tot;
}

bool launch_gemm_tn_grouped(const GemmTN* jobs, double* const* accs, int n, double* partial,
                            size_t partial_cap, cudaStream_t s) {
  if (n <= 0) return true;
  if (n > TN_GROUP_MAX) return false;
  TnGroup G{};
  G.njobs = n;
  tn_group_grids(jobs, n, G.t);
  size_t off = 0;
  int blocks = 0;
  int64_t elems = 0;
  for (int j = 0; j < n; ++j) {
    G.g[j] = jobs[j];
    G.acc[j] = accs[j];
    G.partial[j] = partial + off;
    off += (size_t)G.t[j].splits * G.t[j].P * G.t[j].Q;
    G.begin[j] = blocks;
    blocks += (int)(G.t[j].splits * G.t[j].pairs);
    G.ebegin[j] = elems;
    elems += (int64_t)G.t[j].P * G.t[j].Q;
  }
  G.begin[n] = blocks;
  G.ebegin[n] = elems;
  if (off > partial_cap) return false;
  auto kern = k_gemm_tn_grouped<TN_BM, TN_BN, TN_WM, TN_WN, TN_BK, TN_STAGES>;
  const size_t smem = sizeof(double) * TN_STAGES * TN_BK * ((TN_BM + 4) + (TN_BN + 4) + 1);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  count_launch();
  kern<<<(unsigned)blocks, TN_WM * TN_WN * 32, smem, s>>>(G);
  count_launch();
  k_tn_reduce_grouped<<<(unsigned)std::min<int64_t>(ceil_div(elems, 256), 148 * 8), 256, 0, s>>>(G);
  return true;
}

}  // namespace kp
