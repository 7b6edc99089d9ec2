// On-device generalised symmetric-definite eigensolver for small factors (n <= 96)
// and the Kronecker-sum combine, FP64, sm_100a.  Used for the layers whose factors
// fit in one CTA's shared memory (every layer of BASELINE configs c1-c3); larger
// layers go through cuSOLVER sygvd.  Everything stays on the device: no host sync,
// one launch for all small factor pairs, one for all small combines.
//
// For a pair (F1, F2) with damping lam (reference src/curvature.py:150-161):
//   M1 = F1 + lam I, M2 = F2 + lam I
//   M2 = L L^T (Cholesky; failure -> not positive definite, src/linalg.py:128-132)
//   C  = L^-1 M1 L^-T (two forward substitutions, C symmetric)
//   C  = V diag(lam) V^T  (parallel cyclic Jacobi, round-robin pairing)
//   T  = L^-T V           (so T^T M2 T = I, T^T M1 T = diag(lam))
// Combine (src/linalg.py:168-173 restated on the generalised basis):
//   out = -T_B [(T_B^T G T_A) / (lb la^T + 1)] T_A^T.
// Jacobi is accurate to a few ulps relative to each eigenpair; the solution of the
// Kronecker-sum system is unique, so it matches the reference's LAPACK route to
// roundoff (tests/test_gpu_parity.py).
#include <algorithm>

#include "../../include/kfac_pinn_b200.h"
#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

namespace {

constexpr int EIG_THREADS = 1024;
constexpr int EIG_MAXN = 96;
constexpr int EIG_MAX_SWEEPS = 30;
// Rotate only when |a_pq| > tol * sqrt(|a_pp a_qq|): relative accuracy ~1e-14 per eigenpair
// (the KFAC parity bar is 1e-10); tighter values let roundoff re-trigger rotations forever.
constexpr double kJacobiTol = 1e-14;

__host__ __device__ inline int eig_pitch(int n) { return ((n - 1 + 15) / 16) * 16 + 1; }

__device__ int g_eig_sweeps_max = 0;  // diagnostic: most Jacobi sweeps used by any job

__device__ __forceinline__ void set_status_dev(int32_t* status, int32_t code) {
  atomicCAS(status, 0, code);
}

// Parallel cyclic Jacobi on the symmetric C (n x n, pitch ld) accumulating V <- V G^T.
// Round-robin ordering over m = n rounded up to even (index n is a dummy when n is odd):
// m - 1 rounds of m/2 disjoint pairs per sweep.  Lane group k (G lanes) owns pair k of
// every round: it computes the rotation redundantly in registers, then rotates rows p, q of
// C, and (after a barrier) columns p, q of C and V.  Pair positions advance incrementally.
template <int G>
__device__ __forceinline__ void jacobi_sweeps(double* C, double* V, int n, int ld, int* flag) {
  constexpr int GPW = 32 / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = warp * GPW + lane / G;  // pair slot of this lane group
  const int gl = lane % G;
  const int m = (n + 1) & ~1;
  const int npair = m / 2;
  const bool active = k < npair;
  for (int sweep = 0; sweep < EIG_MAX_SWEEPS; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    // round 0 positions: a = 0 (k = 0) or 1 + (k - 1); b = 1 + (m - 2 - k)
    int ia = k > 0 ? k - 1 : 0, ib = m - 2 - k;
    for (int round = 0; round < m - 1; ++round) {
      int p = 0, q = n;
      double c = 1.0, sn = 0.0;
      if (active) {
        const int a = (k == 0) ? 0 : 1 + ia;
        const int b = 1 + ib;
        p = min(a, b);
        q = max(a, b);
        if (q < n) {
          const double apq = C[p * ld + q];
          const double app = C[p * ld + p], aqq = C[q * ld + q];
          if (apq * apq > kJacobiTol * kJacobiTol * fabs(app * aqq) && fabs(apq) > 1e-300) {
            // t = sign(theta) / (|theta| + sqrt(theta^2 + 1)), theta = (aqq - app) / (2 apq)
            const double dd = aqq - app;
            const double two_apq = 2.0 * apq;
            const double den = fabs(dd) + sqrt(fma(dd, dd, two_apq * two_apq));
            const double t = ((dd >= 0.0) == (apq >= 0.0) ? 1.0 : -1.0) * fabs(two_apq) / den;
            c = rsqrt(fma(t, t, 1.0));
            sn = t * c;
            if (gl == 0) *flag = 1;
          }
        }
        if (k != 0) ia = (ia + 1 == m - 1) ? 0 : ia + 1;
        ib = (ib + 1 == m - 1) ? 0 : ib + 1;
      }
      __syncthreads();  // all rotation parameters read C before any row update
      const bool rot = active && q < n && sn != 0.0;
      if (rot) {
        for (int col = gl; col < n; col += G) {
          const double x = C[p * ld + col], y = C[q * ld + col];
          C[p * ld + col] = c * x - sn * y;
          C[q * ld + col] = sn * x + c * y;
        }
      }
      __syncthreads();
      if (rot) {
        for (int row = gl; row < n; row += G) {
          const double x = C[row * ld + p], y = C[row * ld + q];
          C[row * ld + p] = c * x - sn * y;
          C[row * ld + q] = sn * x + c * y;
          const double vx = V[row * ld + p], vy = V[row * ld + q];
          V[row * ld + p] = c * vx - sn * vy;
          V[row * ld + q] = sn * vx + c * vy;
        }
      }
      __syncthreads();
    }
    // every thread reads the flag before thread 0 may reset it for the next sweep
    const int rotated = *flag;
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

  // right-looking Cholesky of M2 (lower triangle of L); warp w owns rows w, w+32, ...
  for (int k = 0; k < n; ++k) {
    const double a = L[k * ld + k];
    if (!(a > 0.0)) {
      if (tid == 0) flag = n + k + 1;  // LAPACK convention: info > n -> second matrix not PD
      break;
    }
    const double dk = sqrt(a);
    const double inv = 1.0 / dk;
    __syncthreads();  // everyone has read L[k][k]
    if (tid == 0) L[k * ld + k] = dk;
    for (int i = k + 1 + tid; i < n; i += EIG_THREADS) L[i * ld + k] *= inv;
    __syncthreads();
    for (int i = k + 1 + warp; i < n; i += NWARPS) {
      const double lik = L[i * ld + k];
      for (int j = k + 1 + lane; j <= i; j += 32) L[i * ld + j] -= lik * L[j * ld + k];
    }
    __syncthreads();
  }
  __syncthreads();
  if (flag != 0) {
    if (tid == 0) {
      if (jb.info) *jb.info = flag;
      if (jb.warm_valid) *jb.warm_valid = 0;
      set_status_dev(status, KP_ERR_NOT_PSD);
    }
    return;
  }

  // C <- L^-1 C then C <- L^-1 C^T (C symmetric).  Warp per column, lanes split the dot
  // product of each forward-substitution row.
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = warp; j < n; j += NWARPS) {
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = lane; k < i; k += 32) acc += L[i * ld + k] * V[k * ld + j];
        acc = warp_sum(acc);
        const double rhs = pass == 0 ? C[i * ld + j] : C[j * ld + i];
        if (lane == 0) V[i * ld + j] = (rhs - acc) / L[i * ld + i];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = tid; e < n * ld; e += EIG_THREADS) C[e] = V[e];
    __syncthreads();
  }
  // symmetrise (roundoff) and V = I
  for (int e = tid; e < n * n; e += EIG_THREADS) {
    const int i = e / n, j = e % n;
    if (i < j) {
      const double a = 0.5 * (C[i * ld + j] + C[j * ld + i]);
      C[i * ld + j] = a;
      C[j * ld + i] = a;
    }
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();

  // parallel cyclic Jacobi (jacobi_sweeps): lane groups of 32 when the m/2 pairs fit the
  // 32 warps, of 16 otherwise (n = 65..96), so no group ever handles two pairs per round
  if (((n + 1) & ~1) / 2 <= NWARPS)
    jacobi_sweeps<32>(C, V, n, ld, &flag);
  else
    jacobi_sweeps<16>(C, V, n, ld, &flag);

  // eigenvalues; T = L^-T V (back substitution, warp per column) written to global
  for (int i = tid; i < n; i += EIG_THREADS) jb.lam[i] = C[i * ld + i];
  __syncthreads();
  for (int j = warp; j < n; j += NWARPS) {
    for (int i = n - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int k = i + 1 + lane; k < n; k += 32) acc += L[k * ld + i] * C[k * ld + j];
      acc = warp_sum(acc);
      if (lane == 0) C[i * ld + j] = (V[i * ld + j] - acc) / L[i * ld + i];  // C reused as T
      __syncwarp();
    }
  }
  __syncthreads();
  const double* T = C;
  if (warm) {  // T = T_prev T''  (T_prev from global, T'' in C; result in V)
    for (int e2 = tid; e2 < n * n; e2 += EIG_THREADS) {
      const int i = e2 / n, j = e2 % n;
      double a = 0.0;
      for (int k = 0; k < n; ++k) a = fma(jb.warm_t[i * n + k], C[k * ld + j], a);
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

}  // namespace

int small_eig_max_n() { return EIG_MAXN; }

int small_eig_sweeps_used() {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_eig_sweeps_max, sizeof(int));
  return v;
}

size_t small_eig_smem_bytes(int n) { return sizeof(double) * 3 * (size_t)n * eig_pitch(n); }

void launch_gen_eig_small(const SmallEigJobs& jobs, int njobs, int max_n, int32_t* status,
                          cudaStream_t s) {
  if (njobs <= 0) return;
  const size_t smem = small_eig_smem_bytes(max_n);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gen_eig_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)small_eig_smem_bytes(EIG_MAXN));
    attr_set = true;
  }
  count_launch();
  k_gen_eig_small<<<njobs, EIG_THREADS, smem, s>>>(jobs, status);
}

void launch_kron_combine_small(const SmallCombineJobs& jobs, int njobs, cudaStream_t s) {
  if (njobs <= 0) return;
  count_launch();
  k_kron_combine_small<<<njobs, 1024, 0, s>>>(jobs);
}

}  // namespace kp
