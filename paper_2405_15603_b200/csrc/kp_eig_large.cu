// Large symmetric eigensolver (288 < n <= 1055) for the damped Kronecker-sum solve:
// one-sided (Hestenes) Jacobi on a Cholesky factor with the vectors resident in L2, one
// 16-CTA thread-block cluster per factor pair, FP64, sm_100a.
//
// Used for the factor pairs above the cluster-shared-memory solver of kp_eig_mid.cu
// (BASELINE c5: widths 512-769).  The generalised problem M1 x = l M2 x of one factor pair
// (reference src/linalg.py:136-174 via src/curvature.py:150-161) is reduced on the device
// (kp_step.cu gen_eig_pair): M2 = L L^T, M1 = K K^T (Cholesky), and C = L^-1 M1 L^-T =
// L_C L_C^T with L_C = L^-1 K lower triangular.  The rows of L_C are the columns of
// R = L_C^T (C = R^T R).  This kernel orthogonalises them by plane rotations,
// U = R V with mutually orthogonal columns u_i, so that
//   C V = V diag(||u_i||^2)   and   T = L^-T V = K^-T U
// (K^-T U = L^-T L_C^-T R V = L^-T V): by default the eigenvectors are never accumulated,
// the caller forms T^T = U^T K^-1 with one triangular inverse and a GEMM.  That halves the
// L2 traffic of a rotation (c5 preconditioner 127 -> 47 ms) at no measurable accuracy cost
// on the BASELINE pairs (Delta vs the reference: 1.2e-12 either way, profiles/r02_parity_margins.md);
// KP_LARGE_ACCV=1 applies every rotation to V (the identity at the start) as well and the
// caller uses T^T = V^T L^-1.
//
// U (and V) (n x n doubles: 4.7 MB at n = 769) do not fit a cluster's shared memory, so the
// rows stay in global memory (L2-resident) and never move: a round of the circle method
// (column 0 fixed, the others rotating one position per round) only changes which rows a
// warp pairs, computed in closed form from the round number.  CTA c owns pairs
// [c ppc, (c+1) ppc) of the round; a warp loads its two rows into registers (L2, .cg: the
// other CTAs' writes of the previous round are visible after the cluster barrier's
// release/acquire), forms the three dot products, rotates and stores them back.  One
// cluster barrier per round; the sweep loop ends after a sweep without rotations anywhere.
// A rotation is applied when |<u_p, u_q>| > tol ||u_p|| ||u_q|| (tol = max(1e-14, 2 n eps)),
// as in the mid-size solver.
#include <cooperative_groups.h>

#include <cfloat>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace cg = cooperative_groups;

namespace kp {

namespace {

constexpr int LG_CL = 16;            // cluster size (non-portable)
constexpr int LG_MAX_SWEEPS = 60;
constexpr int LG_MAXN = 1055;

__device__ int g_large_sweeps_max = 0;  // diagnostic: most sweeps used by any solve

__host__ __device__ inline int lg_ppc(int n) { return ((n + 1) / 2 + LG_CL - 1) / LG_CL; }

// Column held at position j (0 <= j < m) in round r of the circle method over m positions.
__device__ __forceinline__ int lg_col(int j, int r, int m) {
  return j == 0 ? 0 : 1 + (j - 1 + r) % (m - 1);
}

// EFM: register slices per lane and vector (n <= 32 EFM + 31); W: warps per CTA;
// ACCV: apply the rotations to V (else V is not touched and the caller recovers it from U).
template <int EFM, int W, bool ACCV>
__global__ void __launch_bounds__(W * 32, 1)
    k_eig_large(int n, double* __restrict__ U, double* __restrict__ V, double* __restrict__ lam,
                int* __restrict__ info, const int* __restrict__ chol_info, double tol,
                int* __restrict__ warm_valid) {
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  if (chol_info[0] != 0 || chol_info[1] != 0) {  // uniform across the cluster
    if (c == 0 && threadIdx.x == 0) {
      *info = n + 1;
      if (warm_valid) *warm_valid = 0;
    }
    return;
  }
  __shared__ int rotated;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ppc = lg_ppc(n);
  const int m = 2 * LG_CL * ppc;  // positions (rows >= n are virtual zero vectors)
  const int ef = n / 32;          // full 32-element slices
  const bool tl = lane < n - 32 * ef;
  const double tol2 = tol * tol;
  if (ACCV)
    for (int i = c * W + warp; i < n; i += W * LG_CL)  // V = I
      for (int e = lane; e < n; e += 32) __stcg(V + (size_t)i * n + e, e == i ? 1.0 : 0.0);
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  int sweep = 0;
  bool converged = false;
  for (; sweep < LG_MAX_SWEEPS; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    int any_local = 0;
    for (int r = 0; r < m - 1; ++r) {
      for (int k = c * ppc + warp; k < (c + 1) * ppc; k += W) {
        const int cp = lg_col(k, r, m), cq = lg_col(m - 1 - k, r, m);
        if (cp >= n || cq >= n) continue;
        double* up = U + (size_t)cp * n;
        double* uq = U + (size_t)cq * n;
        double x[EFM + 1], y[EFM + 1];
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int u = 0; u < EFM; ++u) {
          const bool in = u < ef;
          x[u] = in ? __ldcg(up + lane + 32 * u) : 0.0;
          y[u] = in ? __ldcg(uq + lane + 32 * u) : 0.0;
        }
        x[EFM] = tl ? __ldcg(up + 32 * ef + lane) : 0.0;
        y[EFM] = tl ? __ldcg(uq + 32 * ef + lane) : 0.0;
#pragma unroll
        for (int u = 0; u <= EFM; ++u) {
          a = fma(x[u], x[u], a);
          b = fma(y[u], y[u], b);
          g = fma(x[u], y[u], g);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (g * g > tol2 * (a * b) && fabs(g) > 1e-300) {
          double cs, sn;
          jacobi_angle(a, b, g, cs, sn);
#pragma unroll
          for (int u = 0; u < EFM; ++u) {
            if (u < ef) {
              __stcg(up + lane + 32 * u, cs * x[u] - sn * y[u]);
              __stcg(uq + lane + 32 * u, sn * x[u] + cs * y[u]);
            }
          }
          if (tl) {
            __stcg(up + 32 * ef + lane, cs * x[EFM] - sn * y[EFM]);
            __stcg(uq + 32 * ef + lane, sn * x[EFM] + cs * y[EFM]);
          }
          double* vp = V + (size_t)cp * n;
          double* vq = V + (size_t)cq * n;
#pragma unroll 4
          for (int e = lane; ACCV && e < n; e += 32) {
            const double pv = __ldcg(vp + e), qv = __ldcg(vq + e);
            __stcg(vp + e, cs * pv - sn * qv);
            __stcg(vq + e, sn * pv + cs * qv);
          }
          any_local = 1;
        }
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (any_local && lane == 0) rotated = 1;
    __syncthreads();
    cluster.sync();  // every CTA's flag written
    int any = 0;
    for (int q = 0; q < LG_CL; ++q) any |= *cluster.map_shared_rank(&rotated, q);
    cluster.sync();  // all flags read before any CTA resets its own
    if (!any) {
      converged = true;
      break;
    }
  }
  // eigenvalues ||u_i||^2
  const int nthr_w = W * LG_CL;
  for (int i = c * W + warp; i < n; i += nthr_w) {
    const double* ui = U + (size_t)i * n;
    double a = 0.0;
    for (int e = lane; e < n; e += 32) {
      const double v = __ldcg(ui + e);
      a = fma(v, v, a);
    }
    a = warp_sum(a);
    if (lane == 0) lam[i] = a;
  }
  if (c == 0 && threadIdx.x == 0) {
    *info = converged ? 0 : 1;
    if (warm_valid) *warm_valid = converged ? 1 : 0;
    atomicMax(&g_large_sweeps_max, converged ? sweep + 1 : 1000 + sweep);
  }
}

template <int EFM, int W>
bool lg_attrs() {
  auto set = [](auto k) {
    return cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
           cudaSuccess;
  };
  return set(k_eig_large<EFM, W, true>) && set(k_eig_large<EFM, W, false>);
}

template <int EFM, int W>
void lg_launch(int n, double* U, double* V, double* lam, int* info, const int* chol_info,
               double tol, int* warm_valid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LG_CL);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = LG_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (V) cudaLaunchKernelEx(&cfg, k_eig_large<EFM, W, true>, n, U, V, lam, info, chol_info, tol, warm_valid);
  else cudaLaunchKernelEx(&cfg, k_eig_large<EFM, W, false>, n, U, V, lam, info, chol_info, tol, warm_valid);
}

int g_large_ok = 0;  // 0 unknown, 1 usable, -1 not schedulable

}  // namespace

int large_eig_max_n() {
  if (g_large_ok == 0) {
    bool ok = lg_attrs<12, 16>() && lg_attrs<16, 16>() && lg_attrs<20, 12>() &&
              lg_attrs<24, 12>() && lg_attrs<28, 12>() && lg_attrs<32, 12>();
    if (ok) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(LG_CL);
      cfg.blockDim = dim3(12 * 32);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = LG_CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      ok = cudaOccupancyMaxActiveClusters(&nc, k_eig_large<32, 12, true>, &cfg) == cudaSuccess && nc >= 1;
    }
    if (!ok) cudaGetLastError();
    g_large_ok = ok ? 1 : -1;
  }
  return g_large_ok > 0 ? LG_MAXN : 0;
}

bool large_eig_accumulate_v() {
  static const bool acc = [] {
    const char* e = getenv("KP_LARGE_ACCV");
    return e && atoi(e) == 1;
  }();
  return acc;
}

int large_eig_sweeps_used(bool reset) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_large_sweeps_max, sizeof(int));
  if (reset) {
    const int z = 0;
    cudaMemcpyToSymbol(g_large_sweeps_max, &z, sizeof(int));
  }
  return v;
}

void launch_eig_large(int n, double* U, double* V, double* lam, int* info, const int* chol_info,
                      cudaStream_t s, int* warm_valid) {
  count_launch();
  const double tol = fmax(1e-14, 2.0 * n * DBL_EPSILON);
  const int ef = n / 32;
  if (ef <= 12) lg_launch<12, 16>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 16) lg_launch<16, 16>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 20) lg_launch<20, 12>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 24) lg_launch<24, 12>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 28) lg_launch<28, 12>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
  else lg_launch<32, 12>(n, U, V, lam, info, chol_info, tol, warm_valid, s);
}

}  // namespace kp
