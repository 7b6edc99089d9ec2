// On-device generalised symmetric-definite eigensolver for small factors (n <= 96)
// and the Kronecker-sum combine, FP64, sm_100a.  Used for the layers whose factors
// fit in one CTA's shared memory (every layer of BASELINE configs c1-c3); larger
// layers go through the mid / large device routes (kp_step.cu gen_eig_pair).  Everything
// stays on the device: no host sync,
// one launch for all small factor pairs, one for all small combines.
//
// For a pair (F1, F2) with damping lam (reference src/curvature.py:150-161):
//   M1 = F1 + lam I, M2 = F2 + lam I
//   M2 = L L^T, M1 = K K^T (Cholesky; failure -> not positive definite, src/linalg.py:128-132)
//   L_C = L^-1 K (one forward substitution; C = L^-1 M1 L^-T = L_C L_C^T, R = L_C^T)
//   one-sided Jacobi on the rows of L_C -> U = R V with orthogonal columns, C V = V diag(lam)
//   T  = K^-T U = L^-T V  (so T^T M2 T = I, T^T M1 T = diag(lam)); V is never accumulated
// Combine (src/linalg.py:168-173 restated on the generalised basis):
//   out = -T_B [(T_B^T G T_A) / (lb la^T + 1)] T_A^T.
// One-sided Jacobi is accurate to a few ulps relative to each eigenpair; the solution of the
// Kronecker-sum system is unique, so it matches the reference's LAPACK route to
// roundoff (tests/test_gpu_parity.py).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../../include/kfac_pinn_b200.h"
#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

namespace {

constexpr int EIG_THREADS = 768;  // 24 warps: 48 half-warp pairs (n <= 96)
constexpr int EIG_MAXN = 96;
constexpr int EIG_MAX_SWEEPS = 30;
// Rotate only when |a_pq| > tol * sqrt(|a_pp a_qq|): relative accuracy ~1e-14 per eigenpair
// (the KFAC parity bar is 1e-10); tighter values let roundoff re-trigger rotations forever.
constexpr double kJacobiTol = 1e-14;

// 16k+1 doubles with 16k >= n: column walks hit 32 distinct banks, and a row holds the
// 16 * ceil(n / 16) elements the Jacobi rounds read without bounds checks (zero padded)
__host__ __device__ inline int eig_pitch(int n) { return ((n + 15) / 16) * 16 + 1; }

__device__ int g_eig_sweeps_max = 0;  // diagnostic: most Jacobi sweeps used by any job
// diagnostic (KP_EIG_TRACE=1): per sweep, print the largest |cos| between two rows and the
// number of rotations applied
__device__ int g_eig_trace = 0;

__device__ __forceinline__ void set_status_dev(int32_t* status, int32_t code) {
  atomicCAS(status, 0, code);
}

// One-sided (Hestenes) Jacobi on the ROWS of a lower-triangular factor G (C = G G^T), with
// the same rotations applied to the rows of W (start: W = I).  On return the rows of G are
// mutually orthogonal: row i of W is eigenvector i of C and ||row i of G||^2 its eigenvalue.
// Half-warp k owns pair k of each round (circle-method ordering over m = n rounded up to
// even, index n a dummy when n is odd): it loads the two rows into registers (EPL elements
// per lane; rows zero-padded to 16 EPL, so no bounds checks), forms the three dot products
// with a 4-level shuffle reduction and rotates both rows of G and W.  Rows do not move,
// only the pairing changes, so a round is one CTA barrier.
template <int EPL, bool ACCW>
__device__ __forceinline__ void jacobi_rows(double* G, double* W, int n, int ld, int* flag,
                                            double tol) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int hl = lane & 15;                 // lane inside the half-warp
  const int k = (tid >> 5) * 2 + (lane >> 4);  // pair slot of this half-warp
  const unsigned hmask = (lane & 16) ? 0xffff0000u : 0x0000ffffu;
  const int m = (n + 1) & ~1;
  const int npair = m / 2;
  const bool active = k < npair;
  const double tol2 = tol * tol;
  __shared__ unsigned long long tr_max;
  __shared__ int tr_rot;
  const bool trace = g_eig_trace != 0;
  for (int sweep = 0; sweep < EIG_MAX_SWEEPS; ++sweep) {
    if (tid == 0) {
      *flag = 0;
      tr_max = 0ull;
      tr_rot = 0;
    }
    __syncthreads();
    int ia = k > 0 ? k - 1 : 0, ib = m - 2 - k;
    for (int round = 0; round < m - 1; ++round) {
      if (active) {
        const int a = (k == 0) ? 0 : 1 + ia;
        const int b = 1 + ib;
        const int p = min(a, b), q = max(a, b);
        if (k != 0) ia = (ia + 1 == m - 1) ? 0 : ia + 1;
        ib = (ib + 1 == m - 1) ? 0 : ib + 1;
        if (q < n) {
          double* gp = G + p * ld + hl;
          double* gq = G + q * ld + hl;
          double x[EPL], y[EPL];
          double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
          for (int u = 0; u < EPL; ++u) {
            x[u] = gp[16 * u];
            y[u] = gq[16 * u];
            al = fma(x[u], x[u], al);
            be = fma(y[u], y[u], be);
            ga = fma(x[u], y[u], ga);
          }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) {
            al += __shfl_xor_sync(hmask, al, o);
            be += __shfl_xor_sync(hmask, be, o);
            ga += __shfl_xor_sync(hmask, ga, o);
          }
          if (trace && hl == 0 && al > 0.0 && be > 0.0)
            atomicMax(&tr_max, (unsigned long long)__double_as_longlong(fabs(ga) / sqrt(al * be)));
          if (ga * ga > tol2 * (al * be) && fabs(ga) > 1e-300) {
            double cs, sn;
            jacobi_angle(al, be, ga, cs, sn);
            if (trace && hl == 0) atomicAdd(&tr_rot, 1);
            double* wp = ACCW ? W + p * ld + hl : nullptr;
            double* wq = ACCW ? W + q * ld + hl : nullptr;
#pragma unroll
            for (int u = 0; u < EPL; ++u) {
              gp[16 * u] = cs * x[u] - sn * y[u];
              gq[16 * u] = sn * x[u] + cs * y[u];
              if (ACCW) {
                const double wx = wp[16 * u], wy = wq[16 * u];
                wp[16 * u] = cs * wx - sn * wy;
                wq[16 * u] = sn * wx + cs * wy;
              }
            }
            if (hl == 0) *flag = 1;
          }
        }
      }
      __syncthreads();
    }
    const int rotated = *flag;
    if (trace && tid == 0)
      printf("[kp eig small] block %d n %d sweep %d max|cos| %.3e rotations %d\n", blockIdx.x, n,
             sweep, __longlong_as_double((long long)tr_max), tr_rot);
    __syncthreads();
    if (rotated == 0) {
      if (tid == 0) atomicMax(&g_eig_sweeps_max, sweep + 1);
      return;
    }
  }
  if (tid == 0) atomicMax(&g_eig_sweeps_max, 1000 + EIG_MAX_SWEEPS);
}

// X <- V^T X V for symmetric X (smem, pitch ld), V in smem, through n x n global scratch.
__device__ __forceinline__ void congruence(double* X, const double* V, double* scratch, int n,
                                          int ld) {
  for (int e = threadIdx.x; e < n * n; e += EIG_THREADS) {  // scratch = X V
    const int i = e / n, j = e % n;
    double a = 0.0;
    for (int k = 0; k < n; ++k) a = fma(X[i * ld + k], V[k * ld + j], a);
    scratch[e] = a;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += EIG_THREADS) {  // X = V^T scratch
    const int i = e / n, j = e % n;
    double a = 0.0;
    for (int k = 0; k < n; ++k) a = fma(V[k * ld + i], scratch[k * n + j], a);
    X[i * ld + j] = a;
  }
  __syncthreads();
}

// X = L^-1 B (UPPER = false) or X = L^-T B (UPPER = true) for lower-triangular L (smem,
// pitch ld, invd[k] = 1 / L[k][k]); B read as B[i][j] or, with trans_b, B[j][i].  Warp per
// column j; lane l owns rows l, l + 32, l + 64 in registers.  Right-looking: once x_k is
// known (broadcast from its lane) every lane updates its remaining rows, so a column costs
// n shuffle + FMA steps and no reductions.
template <bool UPPER>
__device__ __forceinline__ void tri_solve_cols(const double* L, const double* invd,
                                               const double* B, bool trans_b, double* X, int n,
                                               int ld) {
  constexpr int R = (EIG_MAXN + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NWARPS = EIG_THREADS / 32;
  for (int j = warp; j < n; j += NWARPS) {
    double b[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int i = lane + 32 * t;
      b[t] = i < n ? (trans_b ? B[j * ld + i] : B[i * ld + j]) : 0.0;
    }
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int sb = UPPER ? R - 1 - s : s;  // register slot of the rows of this block
      for (int kk = 0; kk < 32; ++kk) {
        const int kl = UPPER ? 31 - kk : kk;
        const int k = 32 * sb + kl;
        if (k >= n) continue;
        const double xk = __shfl_sync(0xffffffffu, b[sb], kl) * invd[k];
        if (lane == kl) X[k * ld + j] = xk;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          const int i = lane + 32 * t;
          if (UPPER ? (i < k) : (i > k && i < n))
            b[t] = fma(-(UPPER ? L[k * ld + i] : L[i * ld + k]), xk, b[t]);
        }
      }
    }
  }
}

// Right-looking Cholesky of the symmetric A (lower triangle, smem, pitch ld) in place; warp w
// owns rows w, w+32, ...  On failure at pivot k, *flag = n + k + 1 (LAPACK's info > n
// convention for the second matrix of a pencil).  Ends with a barrier.
__device__ __forceinline__ void chol_lower(double* A, int n, int ld, int* flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARPS = EIG_THREADS / 32;
  for (int k = 0; k < n; ++k) {
    const double a = A[k * ld + k];
    if (!(a > 0.0)) {
      if (tid == 0) *flag = n + k + 1;
      break;
    }
    const double dk = sqrt(a);
    const double inv = 1.0 / dk;
    __syncthreads();  // everyone has read A[k][k]
    if (tid == 0) A[k * ld + k] = dk;
    for (int i = k + 1 + tid; i < n; i += EIG_THREADS) A[i * ld + k] *= inv;
    __syncthreads();
    for (int i = k + 1 + warp; i < n; i += NWARPS) {
      const double lik = A[i * ld + k];
      for (int j = k + 1 + lane; j <= i; j += 32) A[i * ld + j] -= lik * A[j * ld + k];
    }
    __syncthreads();
  }
  __syncthreads();
}

// One CTA (32 warps) per factor pair.  smem: L, C, V (n x n each, row-major).
__global__ void __launch_bounds__(EIG_THREADS) k_gen_eig_small(const SmallEigJobs jobs,
                                                              int32_t* status) {
  extern __shared__ double esm[];
  const SmallEigJob jb = jobs.job[blockIdx.x];
  const int n = jb.n;
  const int ld = eig_pitch(n);  // 16k+1 doubles: column walks hit 32 distinct banks
  double* L = esm;
  double* C = L + n * ld;
  double* V = C + n * ld;
  double* invd = V + n * ld;  // 1 / diag of the Cholesky factors of M2 (n) and M1 (n)
  __shared__ int flag;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWARPS = EIG_THREADS / 32;
  const double lam = jb.damping;

  // load M2 = F2 + lam I into L and M1 = F1 + lam I into C
  for (int e = tid; e < n * n; e += EIG_THREADS) {
    const int i = e / n, j = e % n;
    L[i * ld + j] = jb.f2[e] + (i == j ? lam : 0.0);
    C[i * ld + j] = jb.f1[e] + (i == j ? lam : 0.0);
  }
  if (tid == 0) flag = 0;
  __syncthreads();
  // warm start: congruence by the previous step's T, kept only while T_prev^T M2 T_prev stays
  // near I (its diagonal within [0.5, 2]); otherwise (first step, re-initialised factors)
  // the cold path below runs on the untransformed pair
  __shared__ int warm;
  if (tid == 0) warm = (jb.warm_t != nullptr && *jb.warm_valid != 0) ? 1 : 0;
  __syncthreads();
  if (warm) {
    for (int e2 = tid; e2 < n * n; e2 += EIG_THREADS) V[(e2 / n) * ld + e2 % n] = jb.warm_t[e2];
    __syncthreads();
    congruence(L, V, jb.warm_scratch, n, ld);
    for (int i = tid; i < n; i += EIG_THREADS) {
      const double dgl = L[i * ld + i];
      if (!(dgl > 0.5 && dgl < 2.0)) warm = 0;
    }
    __syncthreads();
    if (warm) {
      congruence(C, V, jb.warm_scratch, n, ld);
    } else {  // reload the untransformed M2
      for (int e2 = tid; e2 < n * n; e2 += EIG_THREADS) {
        const int i = e2 / n, j = e2 % n;
        L[i * ld + j] = jb.f2[e2] + (i == j ? lam : 0.0);
      }
      __syncthreads();
    }
  }

  // M2 = L L^T and M1 = K K^T (Cholesky, lower triangles of L and C); a failure of M2's ->
  // info > n (second matrix not PD), of M1's -> info = n + 1 (not PD either way)
  chol_lower(L, n, ld, &flag);
  if (flag == 0) {
    chol_lower(C, n, ld, &flag);
    if (flag != 0) flag = n + 1;
  }
  if (flag != 0) {
    if (tid == 0) {
      if (jb.info) *jb.info = flag;
      if (jb.warm_valid) *jb.warm_valid = 0;
      set_status_dev(status, KP_ERR_NOT_PSD);
    }
    return;
  }
  // L_C = L^-1 K (lower triangular; C_sym = L^-1 M1 L^-T = L_C L_C^T, R = L_C^T), into V by
  // right-looking warp-per-column triangular solves; one-sided Jacobi on the rows of L_C
  // (the columns of R) leaves U = R V_eig with orthogonal columns, ||u_i||^2 the eigenvalues;
  // then T = K^-T U (= L^-T L_C^-T R V_eig = L^-T V_eig): the eigenvectors are never
  // accumulated (half the rotation work; the same route as the cluster solvers)
  double* invk = invd + n;
  for (int i = tid; i < n; i += EIG_THREADS) {
    invd[i] = 1.0 / L[i * ld + i];
    invk[i] = 1.0 / C[i * ld + i];
  }
  for (int e = tid; e < n * n; e += EIG_THREADS) {  // K's strict upper triangle still holds M1
    const int i = e / n, j = e % n;
    if (j > i) C[i * ld + j] = 0.0;
  }
  __syncthreads();
  tri_solve_cols<false>(L, invd, C, false, V, n, ld);
  __syncthreads();
  const int nr = ((n + 15) / 16) * 16;  // padded row length read by the Jacobi rounds
  for (int e = tid; e < n * nr; e += EIG_THREADS) {
    const int i = e / nr, j = e % nr;
    if (j > i) V[i * ld + j] = 0.0;  // exact zeros already for j < n; the padding too
  }
  __syncthreads();
  {
    const double tol = fmax(jobs.tol_floor, 2.0 * n * 2.220446049250313e-16);
    switch (nr / 16) {
      case 1: jacobi_rows<1, false>(V, nullptr, n, ld, &flag, tol); break;
      case 2: jacobi_rows<2, false>(V, nullptr, n, ld, &flag, tol); break;
      case 3: jacobi_rows<3, false>(V, nullptr, n, ld, &flag, tol); break;
      case 4: jacobi_rows<4, false>(V, nullptr, n, ld, &flag, tol); break;
      case 5: jacobi_rows<5, false>(V, nullptr, n, ld, &flag, tol); break;
      default: jacobi_rows<6, false>(V, nullptr, n, ld, &flag, tol); break;
    }
  }

  // eigenvalues ||u_i||^2; T = K^-T U (U[k][i] = V[i][k]: transposed read) into L
  for (int i = warp; i < n; i += NWARPS) {
    double a = 0.0;
    for (int j = lane; j < n; j += 32) a = fma(V[i * ld + j], V[i * ld + j], a);
    a = warp_sum(a);
    if (lane == 0) jb.lam[i] = a;
  }
  __syncthreads();
  tri_solve_cols<true>(C, invk, V, true, L, n, ld);
  __syncthreads();
  const double* T = L;
  if (warm) {  // T = T_prev T''  (T_prev from global, T'' in L; result in V)
    for (int e2 = tid; e2 < n * n; e2 += EIG_THREADS) {
      const int i = e2 / n, j = e2 % n;
      double a = 0.0;
      for (int k = 0; k < n; ++k) a = fma(jb.warm_t[i * n + k], L[k * ld + j], a);
      V[i * ld + j] = a;
    }
    __syncthreads();
    T = V;
  }
  for (int e = tid; e < n * n; e += EIG_THREADS) {
    const int i = e / n, j = e % n;
    jb.t[jb.col_major ? j * n + i : e] = T[i * ld + j];
    if (jb.warm_t) jb.warm_t[e] = T[i * ld + j];
  }
  if (tid == 0 && jb.warm_valid) *jb.warm_valid = 1;
  if (tid == 0 && jb.info) *jb.info = 0;
  // PSD check on the generalised eigenvalues (src/linalg.py:79-83, 165-166)
  if (tid == 0) {
    double hi = 0.0, mn = INFINITY;
    for (int i = 0; i < n; ++i) {
      const double v = jb.lam[i];
      mn = fmin(mn, v);
      hi = fmax(hi, fabs(v));
    }
    if (mn < -1e-6 * fmax(hi, 1e-300)) set_status_dev(status, KP_ERR_NOT_PSD);
  }
}

// One CTA per layer: out (q x p, row-major) = sign * T_B [(T_B^T G T_A) / (lb la^T + 1)] T_A^T
// with T_A (p x p) and T_B (q x q) row-major (column k = eigenvector k).
__global__ void __launch_bounds__(1024) k_kron_combine_small(const SmallCombineJobs jobs) {
  const SmallCombineJob jb = jobs.job[blockIdx.x];
  const int p = jb.p, q = jb.q;
  const int tid = threadIdx.x;
  // T1 = G T_A (q x p)
  for (int e = tid; e < q * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < p; ++k) v += jb.g[i * p + k] * jb.ta[k * p + j];
    jb.t1[e] = v;
  }
  __syncthreads();
  // W = (T_B^T T1) / (lb_i la_j + 1)
  for (int e = tid; e < q * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < q; ++k) v += jb.tb[k * q + i] * jb.t1[k * p + j];
    jb.t2[e] = v / (jb.lb[i] * jb.la[j] + 1.0);
  }
  __syncthreads();
  // T1 = W T_A^T
  for (int e = tid; e < q * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < p; ++k) v += jb.t2[i * p + k] * jb.ta[j * p + k];
    jb.t1[e] = v;
  }
  __syncthreads();
  // out = sign * T_B T1
  for (int e = tid; e < q * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < q; ++k) v += jb.tb[i * q + k] * jb.t1[k * p + j];
    jb.out[e] = jb.sign * v;
  }
}

// The same with every operand staged in shared memory (odd pitches: conflict-free column
// walks); used when p^2 + q^2 + 2pq doubles fit (every layer up to 64 wide).
__host__ __device__ inline int comb_pitch(int n) { return n | 1; }
__host__ __device__ inline size_t comb_smem_doubles(int p, int q) {
  return (size_t)p * comb_pitch(p) + (size_t)q * comb_pitch(q) + 2 * (size_t)q * comb_pitch(p);
}
constexpr size_t COMB_SMEM_MAX = 200 * 1024;

__global__ void __launch_bounds__(1024) k_kron_combine_small_smem(const SmallCombineJobs jobs) {
  extern __shared__ double csm[];
  const SmallCombineJob jb = jobs.job[blockIdx.x];
  const int p = jb.p, q = jb.q;
  const int lp = comb_pitch(p), lq = comb_pitch(q);
  double* TA = csm;              // p x p
  double* TB = TA + p * lp;      // q x q
  double* X = TB + q * lq;       // q x p
  double* Y = X + q * lp;        // q x p
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < p * p; e += nt) TA[(e / p) * lp + e % p] = jb.ta[e];
  for (int e = tid; e < q * q; e += nt) TB[(e / q) * lq + e % q] = jb.tb[e];
  for (int e = tid; e < q * p; e += nt) X[(e / p) * lp + e % p] = jb.g[e];
  __syncthreads();
  for (int e = tid; e < q * p; e += nt) {  // Y = G T_A
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < p; ++k) v = fma(X[i * lp + k], TA[k * lp + j], v);
    Y[i * lp + j] = v;
  }
  __syncthreads();
  for (int e = tid; e < q * p; e += nt) {  // X = (T_B^T Y) / (lb_i la_j + 1)
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < q; ++k) v = fma(TB[k * lq + i], Y[k * lp + j], v);
    X[i * lp + j] = v / (jb.lb[i] * jb.la[j] + 1.0);
  }
  __syncthreads();
  for (int e = tid; e < q * p; e += nt) {  // Y = X T_A^T
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < p; ++k) v = fma(X[i * lp + k], TA[j * lp + k], v);
    Y[i * lp + j] = v;
  }
  __syncthreads();
  for (int e = tid; e < q * p; e += nt) {  // out = sign T_B Y
    const int i = e / p, j = e % p;
    double v = 0.0;
    for (int k = 0; k < q; ++k) v = fma(TB[i * lq + k], Y[k * lp + j], v);
    jb.out[e] = jb.sign * v;
  }
}

}  // namespace

int small_eig_max_n() { return EIG_MAXN; }

double jacobi_tol_floor() {
  static const double v = [] {
    const char* e = getenv("KP_JACOBI_TOL");
    return e ? atof(e) : 1e-14;
  }();
  return v;
}

int small_eig_sweeps_used(bool reset) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_eig_sweeps_max, sizeof(int));
  if (reset) {
    const int z = 0;
    cudaMemcpyToSymbol(g_eig_sweeps_max, &z, sizeof(int));
  }
  return v;
}

size_t small_eig_smem_bytes(int n) {
  return sizeof(double) * (3 * (size_t)n * eig_pitch(n) + 2 * (size_t)n);
}

void launch_gen_eig_small(const SmallEigJobs& jobs, int njobs, int max_n, int32_t* status,
                          cudaStream_t s) {
  if (njobs <= 0) return;
  const size_t smem = small_eig_smem_bytes(max_n);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gen_eig_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)small_eig_smem_bytes(EIG_MAXN));
    const char* e = getenv("KP_EIG_TRACE");
    if (e && atoi(e) == 1) {
      const int one = 1;
      cudaMemcpyToSymbol(g_eig_trace, &one, sizeof(int));
    }
    attr_set = true;
  }
  count_launch();
  SmallEigJobs j = jobs;
  j.tol_floor = jacobi_tol_floor();
  k_gen_eig_small<<<njobs, EIG_THREADS, smem, s>>>(j, status);
}

void launch_kron_combine_small(const SmallCombineJobs& jobs, int njobs, cudaStream_t s) {
  if (njobs <= 0) return;
  size_t need = 0;
  for (int j = 0; j < njobs; ++j)
    need = std::max(need, sizeof(double) * comb_smem_doubles(jobs.job[j].p, jobs.job[j].q));
  count_launch();
  if (need <= COMB_SMEM_MAX) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_kron_combine_small_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)COMB_SMEM_MAX);
      attr_set = true;
    }
    k_kron_combine_small_smem<<<njobs, 1024, need, s>>>(jobs);
  } else {
    k_kron_combine_small<<<njobs, 1024, 0, s>>>(jobs);
  }
}

}  // namespace kp
