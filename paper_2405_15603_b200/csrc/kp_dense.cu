// Dense FP64 linear algebra for the damped Kronecker-sum solves, without library calls
// (sm_100a): a DMMA GEMM with transpose flags, a blocked Cholesky factorisation and a
// blocked lower-triangular solve with a matrix right-hand side.  Everything is row-major.
//
// Used by the generalised eigenproblems of the factor pairs too large for the one-CTA solver
// (kp_step.cu gen_eig_pair): reference src/linalg.py:136-174 reached through
// src/curvature.py:140-163.  Sizes are the factor widths (n <= ~1025), so the routines are
// latency-bound sequences of small launches, all asynchronous on the caller's stream and
// graph-capturable; none blocks the host.
#include <algorithm>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

namespace {

// ---------------------------------------------------------------------------
// C (M x N) = alpha op(A) op(B) + beta C.  op(A) is M x K (A stored M x K, or K x M when
// ta), op(B) is K x N (B stored K x N, or N x K when tb).  64 x 64 tiles, four warps of
// 32 x 32 (4 x 4 DMMA 8x8x4 fragments each), K in steps of 16 through a two-stage cp.async
// pipeline.  lower_only: tiles strictly above the diagonal are skipped (symmetric updates
// whose upper triangle is never read).
constexpr int DG_BM = 64, DG_BN = 64, DG_BK = 16, DG_ST = 2, DG_LDS = DG_BK + 4;

__global__ void __launch_bounds__(128) k_dense_gemm(DenseGemm g) {
  __shared__ __align__(16) double As[DG_ST][DG_BM * DG_LDS];
  __shared__ __align__(16) double Bs[DG_ST][DG_BN * DG_LDS];
  const int tiles_n = (g.N + DG_BN - 1) / DG_BN;
  const int bm = blockIdx.x / tiles_n, bn = blockIdx.x % tiles_n;
  if (g.lower_only && bn > bm) return;
  const int m0 = bm * DG_BM, n0 = bn * DG_BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int KT = (g.K + DG_BK - 1) / DG_BK;

  auto load = [&](int st, int kt) {
    const int k0 = kt * DG_BK;
    for (int e = tid; e < DG_BM * DG_BK; e += 128) {
      // transposed operands: consecutive threads walk m (the contiguous index)
      const int r = g.ta ? e % DG_BM : e / DG_BK, c = g.ta ? e / DG_BM : e % DG_BK;
      const int gm = m0 + r, gk = k0 + c;
      const bool p = gm < g.M && gk < g.K;
      const double* src = g.ta ? g.A + (int64_t)gk * g.lda + gm : g.A + (int64_t)gm * g.lda + gk;
      cp_async8(&As[st][r * DG_LDS + c], p ? src : g.A, p);
    }
    for (int e = tid; e < DG_BN * DG_BK; e += 128) {
      const int r = g.tb ? e / DG_BK : e % DG_BN, c = g.tb ? e % DG_BK : e / DG_BN;
      const int gn = n0 + r, gk = k0 + c;
      const bool p = gn < g.N && gk < g.K;
      const double* src = g.tb ? g.B + (int64_t)gn * g.ldb + gk : g.B + (int64_t)gk * g.ldb + gn;
      cp_async8(&Bs[st][r * DG_LDS + c], p ? src : g.B, p);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < DG_ST - 1; ++s) {
    if (s < KT) load(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<DG_ST - 2>();
    __syncthreads();
    if (kt + DG_ST - 1 < KT) load((kt + DG_ST - 1) % DG_ST, kt + DG_ST - 1);
    cp_async_commit();
    const double* as = &As[kt % DG_ST][(wm * 32 + (lane >> 2)) * DG_LDS + (lane & 3)];
    const double* bs = &Bs[kt % DG_ST][(wn * 32 + (lane >> 2)) * DG_LDS + (lane & 3)];
#pragma unroll
    for (int kk = 0; kk < DG_BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[i * 8 * DG_LDS + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * DG_LDS + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (row >= g.M) continue;
    double* crow = g.C + (int64_t)row * g.ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + wn * 32 + j * 8 + 2 * (lane & 3);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (col + h >= g.N) continue;
        const double v = g.alpha * acc[i][j][h];
        crow[col + h] = g.beta == 0.0 ? v : fma(g.beta, crow[col + h], v);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Blocked right-looking Cholesky, A = L L^T (lower, row-major, in place; the strict upper
// triangle is never read, and the diagonal tiles of the trailing updates overwrite parts of
// it with scratch values).  Per panel of CH_NB columns: one CTA factors the diagonal block in
// shared memory and writes L11 back (k_chol_diag); then CH_ROWS rows of the panel below per
// CTA are solved, L21 = A21 L11^-T (k_chol_rows: a separate launch, so no CTA can read the
// diagonal block while it is being overwritten); the trailing lower triangle is updated by
// the GEMM above, A22 -= L21 L21^T.
// info (LAPACK convention): 0, or the 1-based index of the first non-positive pivot; once
// set, the remaining panels are skipped (their values are then meaningless).
constexpr int CH_NB = 64, CH_ROWS = 128;

__global__ void __launch_bounds__(256) k_chol_diag(int n, double* A, int64_t lda, int k0,
                                                   int* info) {
  __shared__ double D[CH_NB][CH_NB + 1];
  __shared__ int bad;
  if (*info != 0) return;
  const int kb = min(CH_NB, n - k0);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < kb * kb; e += nt) {
    const int r = e / kb, c = e % kb;
    D[r][c] = c <= r ? A[(int64_t)(k0 + r) * lda + k0 + c] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < kb; ++j) {  // unblocked right-looking factorisation
    const double djj = D[j][j];
    if (!(djj > 0.0)) {  // not positive definite (or NaN): uniform across the CTA
      if (tid == 0) bad = k0 + j + 1;
      break;
    }
    const double ljj = sqrt(djj);
    __syncthreads();  // every thread has read D[j][j]
    if (tid == 0) D[j][j] = ljj;
    for (int r = j + 1 + tid; r < kb; r += nt) D[r][j] /= ljj;
    __syncthreads();
    const int w = kb - j - 1;
    for (int e = tid; e < w * w; e += nt) {
      const int r = j + 1 + e / w, c = j + 1 + e % w;
      if (c <= r) D[r][c] = fma(-D[r][j], D[c][j], D[r][c]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) *info = bad;
    return;
  }
  for (int e = tid; e < kb * kb; e += nt) {
    const int r = e / kb, c = e % kb;
    if (c <= r) A[(int64_t)(k0 + r) * lda + k0 + c] = D[r][c];
  }
}

__global__ void __launch_bounds__(CH_ROWS) k_chol_rows(int n, double* A, int64_t lda, int k0,
                                                       const int* info) {
  __shared__ double D[CH_NB][CH_NB + 1];
  if (*info != 0) return;
  const int kb = min(CH_NB, n - k0);
  const int tid = threadIdx.x;
  for (int e = tid; e < kb * kb; e += CH_ROWS) {
    const int r = e / kb, c = e % kb;
    D[r][c] = c <= r ? A[(int64_t)(k0 + r) * lda + k0 + c] : 0.0;
  }
  __syncthreads();
  // row below the block: x L11^T = a  ->  L11 x^T = a^T (forward substitution)
  const int row = k0 + kb + blockIdx.x * CH_ROWS + tid;
  if (row >= n) return;
  double* ar = A + (int64_t)row * lda + k0;
  double x[CH_NB];
#pragma unroll
  for (int c = 0; c < CH_NB; ++c) x[c] = c < kb ? ar[c] : 0.0;
#pragma unroll
  for (int c = 0; c < CH_NB; ++c) {
    if (c < kb) {
      double v = x[c];
#pragma unroll
      for (int k = 0; k < c; ++k) v = fma(-D[c][k], x[k], v);
      x[c] = v / D[c][c];
    }
  }
#pragma unroll
  for (int c = 0; c < CH_NB; ++c)
    if (c < kb) ar[c] = x[c];
}

// ---------------------------------------------------------------------------
// X = L^-1 B for lower-triangular L (n x n) and B (n x m), blocked by TS_NB row blocks:
// X_i = L_ii^-1 (B_i - L[i, :i] X[:i]).  The update is a GEMM (into X_i, which first holds
// B_i); this kernel does the triangular solve of one row block, one thread per column.
// b_identity: B = I (X = L^-1; rows of X beyond the diagonal stay zero).
constexpr int TS_NB = 64, TS_COLS = 128;

__global__ void __launch_bounds__(TS_COLS) k_trsm_block(int n, const double* L, int64_t ldl,
                                                        double* X, int64_t ldx, int m, int i0) {
  __shared__ double D[TS_NB][TS_NB + 1];
  const int kb = min(TS_NB, n - i0);
  for (int e = threadIdx.x; e < kb * kb; e += TS_COLS) {
    const int r = e / kb, c = e % kb;
    D[r][c] = c <= r ? L[(int64_t)(i0 + r) * ldl + i0 + c] : 0.0;
  }
  __syncthreads();
  const int col = blockIdx.x * TS_COLS + threadIdx.x;
  if (col >= m) return;
  double x[TS_NB];
#pragma unroll
  for (int r = 0; r < TS_NB; ++r) x[r] = r < kb ? X[(int64_t)(i0 + r) * ldx + col] : 0.0;
#pragma unroll
  for (int r = 0; r < TS_NB; ++r) {
    if (r < kb) {
      double v = x[r];
#pragma unroll
      for (int k = 0; k < r; ++k) v = fma(-D[r][k], x[k], v);
      x[r] = v / D[r][r];
    }
  }
#pragma unroll
  for (int r = 0; r < TS_NB; ++r)
    if (r < kb) X[(int64_t)(i0 + r) * ldx + col] = x[r];
}

__global__ void k_set_identity(double* X, int n, int64_t ldx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    X[(int64_t)r * ldx + c] = r == c ? 1.0 : 0.0;
  }
}

__global__ void k_copy_matrix(const double* S, int64_t lds, int rows, int cols, double* D,
                              int64_t ldd) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    D[(int64_t)r * ldd + c] = S[(int64_t)r * lds + c];
  }
}

__global__ void k_zero_upper(double* A, int n, int64_t lda) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    if (c > r) A[(int64_t)r * lda + c] = 0.0;
  }
}

unsigned grid_for_elems(int64_t n) {
  return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
}

}  // namespace

void launch_dense_gemm(const DenseGemm& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  count_launch();
  const int tiles = (int)(ceil_div(g.M, DG_BM) * ceil_div(g.N, DG_BN));
  k_dense_gemm<<<tiles, 128, 0, s>>>(g);
}

void launch_cholesky(int n, double* A, int64_t lda, int* info, cudaStream_t s) {
  for (int k0 = 0; k0 < n; k0 += CH_NB) {
    const int kb = std::min(CH_NB, n - k0);
    const int below = n - k0 - kb;
    count_launch();
    k_chol_diag<<<1, 256, 0, s>>>(n, A, lda, k0, info);
    if (below > 0) {
      count_launch();
      k_chol_rows<<<(below + CH_ROWS - 1) / CH_ROWS, CH_ROWS, 0, s>>>(n, A, lda, k0, info);
      DenseGemm g{};
      g.M = g.N = below;
      g.K = kb;
      g.A = A + (int64_t)(k0 + kb) * lda + k0;
      g.lda = lda;
      g.B = g.A;
      g.ldb = lda;
      g.tb = true;
      g.C = A + (int64_t)(k0 + kb) * lda + k0 + kb;
      g.ldc = lda;
      g.alpha = -1.0;
      g.beta = 1.0;
      g.lower_only = true;
      launch_dense_gemm(g, s);
    }
  }
}

void launch_trsm_lower(int n, const double* L, int64_t ldl, double* X, int64_t ldx, int m,
                       bool b_identity, cudaStream_t s) {
  if (b_identity) {
    count_launch();
    k_set_identity<<<grid_for_elems((int64_t)n * n), 256, 0, s>>>(X, n, ldx);
  }
  for (int i0 = 0; i0 < n; i0 += TS_NB) {
    const int kb = std::min(TS_NB, n - i0);
    // X_i -= L[i, :i] X[:i]; with B = I only the first i0 + kb columns can be non-zero
    const int cols = b_identity ? std::min(m, i0 + kb) : m;
    if (i0 > 0) {
      DenseGemm g{};
      g.M = kb;
      g.N = b_identity ? std::min(m, i0) : m;
      g.K = i0;
      g.A = L + (int64_t)i0 * ldl;
      g.lda = ldl;
      g.B = X;
      g.ldb = ldx;
      g.C = X + (int64_t)i0 * ldx;
      g.ldc = ldx;
      g.alpha = -1.0;
      g.beta = 1.0;
      launch_dense_gemm(g, s);
    }
    count_launch();
    k_trsm_block<<<(cols + TS_COLS - 1) / TS_COLS, TS_COLS, 0, s>>>(n, L, ldl, X, ldx, cols, i0);
  }
}

void launch_zero_upper(int n, double* A, int64_t lda, cudaStream_t s) {
  count_launch();
  k_zero_upper<<<grid_for_elems((int64_t)n * n), 256, 0, s>>>(A, n, lda);
}

void launch_copy_matrix(const double* src, int64_t lds, int rows, int cols, double* dst,
                        int64_t ldd, cudaStream_t s) {
  count_launch();
  k_copy_matrix<<<grid_for_elems((int64_t)rows * cols), 256, 0, s>>>(src, lds, rows, cols, dst,
                                                                      ldd);
}

}  // namespace kp
