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
constexpr int LG_MAXN = 1087;      // register-cached kernels (k_eig_large)
constexpr int LG_MAXN_ANY = 16383;  // streaming kernel: bounded only by memory

__device__ int g_large_sweeps_max = 0;  // diagnostic: most sweeps used by any solve

__host__ __device__ inline int lg_ppc(int n) { return ((n + 1) / 2 + LG_CL - 1) / LG_CL; }

// Column held at position j (0 <= j < m) in round r of the circle method over m positions.
__device__ __forceinline__ int lg_col(int j, int r, int m) {
  return j == 0 ? 0 : 1 + (j - 1 + r) % (m - 1);
}

// EFM: 16-byte register slices per lane and vector (n <= 64 EFM + 63); W: warps per CTA;
// ACCV: apply the rotations to V (else V is not touched and the caller recovers it from U).
// Rows have pitch ld (even, so every row is 16-byte aligned): lane l owns the double2 at
// elements 2 l + 64 u, the last n - 64 ef elements are a scalar tail.
template <int EFM, int W, bool ACCV>
__global__ void __launch_bounds__(W * 32, 1)
    k_eig_large(int n, int ld, double* __restrict__ U, double* __restrict__ V,
                double* __restrict__ lam, int* __restrict__ info,
                const int* __restrict__ chol_info, double tol, int* __restrict__ warm_valid) {
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
  const int ef = n / 64;          // full 64-element (double2 per lane) slices
  const int t0 = 64 * ef + lane, t1 = t0 + 32;  // scalar tail elements of this lane
  const bool tl0 = t0 < n, tl1 = t1 < n;
  const double tol2 = tol * tol;
  if (ACCV)
    for (int i = c * W + warp; i < n; i += W * LG_CL)  // V = I
      for (int e = lane; e < n; e += 32) __stcg(V + (size_t)i * ld + e, e == i ? 1.0 : 0.0);
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
        double* up = U + (size_t)cp * ld;
        double* uq = U + (size_t)cq * ld;
        const double2* up2 = reinterpret_cast<const double2*>(up);
        const double2* uq2 = reinterpret_cast<const double2*>(uq);
        double2 x[EFM], y[EFM];
        double xt0, xt1, yt0, yt1;
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int u = 0; u < EFM; ++u) {
          const bool in = u < ef;
          x[u] = in ? __ldcg(up2 + lane + 32 * u) : make_double2(0.0, 0.0);
          y[u] = in ? __ldcg(uq2 + lane + 32 * u) : make_double2(0.0, 0.0);
        }
        xt0 = tl0 ? __ldcg(up + t0) : 0.0;
        yt0 = tl0 ? __ldcg(uq + t0) : 0.0;
        xt1 = tl1 ? __ldcg(up + t1) : 0.0;
        yt1 = tl1 ? __ldcg(uq + t1) : 0.0;
#pragma unroll
        for (int u = 0; u < EFM; ++u) {
          a = fma(x[u].x, x[u].x, a);
          a = fma(x[u].y, x[u].y, a);
          b = fma(y[u].x, y[u].x, b);
          b = fma(y[u].y, y[u].y, b);
          g = fma(x[u].x, y[u].x, g);
          g = fma(x[u].y, y[u].y, g);
        }
        a = fma(xt0, xt0, fma(xt1, xt1, a));
        b = fma(yt0, yt0, fma(yt1, yt1, b));
        g = fma(xt0, yt0, fma(xt1, yt1, g));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (g * g > tol2 * (a * b) && fabs(g) > 1e-300) {
          double cs, sn;
          jacobi_angle(a, b, g, cs, sn);
          double2* wp2 = reinterpret_cast<double2*>(up);
          double2* wq2 = reinterpret_cast<double2*>(uq);
#pragma unroll
          for (int u = 0; u < EFM; ++u) {
            if (u < ef) {
              __stcg(wp2 + lane + 32 * u, make_double2(cs * x[u].x - sn * y[u].x,
                                                       cs * x[u].y - sn * y[u].y));
              __stcg(wq2 + lane + 32 * u, make_double2(sn * x[u].x + cs * y[u].x,
                                                       sn * x[u].y + cs * y[u].y));
            }
          }
          if (tl0) {
            __stcg(up + t0, cs * xt0 - sn * yt0);
            __stcg(uq + t0, sn * xt0 + cs * yt0);
          }
          if (tl1) {
            __stcg(up + t1, cs * xt1 - sn * yt1);
            __stcg(uq + t1, sn * xt1 + cs * yt1);
          }
          double* vp = V + (size_t)cp * ld;
          double* vq = V + (size_t)cq * ld;
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
    const double* ui = U + (size_t)i * ld;
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

// ---------------------------------------------------------------------------
// Any n (the fallback above 1087, where two rows no longer fit a warp's registers): the
// same closed-form circle pairing with the rows in L2, two streaming passes per pair
// (dot products, then rotation), 16-byte accesses, 16 warps per CTA.  No width limit other
// than memory.
__global__ void __launch_bounds__(16 * 32, 1)
    k_eig_stream(int n, int ld, double* __restrict__ U, double* __restrict__ lam,
                 int* __restrict__ info, const int* __restrict__ chol_info, double tol,
                 int* __restrict__ warm_valid) {
  constexpr int W = 16;
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  if (chol_info[0] != 0 || chol_info[1] != 0) {
    if (c == 0 && threadIdx.x == 0) {
      *info = n + 1;
      if (warm_valid) *warm_valid = 0;
    }
    return;
  }
  __shared__ int rotated;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ppc = lg_ppc(n);
  const int m = 2 * LG_CL * ppc;
  const int n2 = n / 2;  // full double2 elements; an odd n leaves element n - 1 (lane 0)
  const double tol2 = tol * tol;
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
        double* up = U + (size_t)cp * ld;
        double* uq = U + (size_t)cq * ld;
        double2* up2 = reinterpret_cast<double2*>(up);
        double2* uq2 = reinterpret_cast<double2*>(uq);
        double a = 0.0, b = 0.0, g = 0.0;
        for (int j = lane; j < n2; j += 32) {
          const double2 x = __ldcg(up2 + j), y = __ldcg(uq2 + j);
          a = fma(x.x, x.x, fma(x.y, x.y, a));
          b = fma(y.x, y.x, fma(y.y, y.y, b));
          g = fma(x.x, y.x, fma(x.y, y.y, g));
        }
        if ((n & 1) && lane == 0) {
          const double x = __ldcg(up + n - 1), y = __ldcg(uq + n - 1);
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
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
          for (int j = lane; j < n2; j += 32) {
            const double2 x = __ldcg(up2 + j), y = __ldcg(uq2 + j);
            __stcg(up2 + j, make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y));
            __stcg(uq2 + j, make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y));
          }
          if ((n & 1) && lane == 0) {
            const double x = __ldcg(up + n - 1), y = __ldcg(uq + n - 1);
            __stcg(up + n - 1, cs * x - sn * y);
            __stcg(uq + n - 1, sn * x + cs * y);
          }
          any_local = 1;
        }
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (any_local && lane == 0) rotated = 1;
    __syncthreads();
    cluster.sync();
    int any = 0;
    for (int q = 0; q < LG_CL; ++q) any |= *cluster.map_shared_rank(&rotated, q);
    cluster.sync();
    if (!any) {
      converged = true;
      break;
    }
  }
  for (int i = c * W + warp; i < n; i += W * LG_CL) {
    const double* ui = U + (size_t)i * ld;
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

// ---------------------------------------------------------------------------
// Split-record variant for 544 < n <= 800 (c5's 768 / 769 pairs), U-only: the one-sided
// Jacobi of kp_eig_mid.cu (columns move between the cluster's CTAs by the circle method, a
// CTA owns 2 ppc column records plus 4 landing records, one warp per pair, the two columns a
// CTA hands over per round are stored straight into the neighbours' landing records) with
// each record split: the first SP_H = 512 entries live in shared memory, the remaining
// n - 512 in a per-CTA global (L2) slot.  So only a third of the rotation traffic touches L2
// (vs all of it in k_eig_large), and the dot products read the smem head twice (dots, then
// rotation) instead of caching whole columns in registers: 25 warps of 32 lanes fit the
// register file.  Tails handed to a neighbour go through global memory, made visible by the
// round's cluster barrier (release / acquire).
constexpr int SP_HE = 16;                       // head slices per lane
constexpr int SP_H = 32 * SP_HE;                // head length (smem)
constexpr int SP_MAXPPC = 25;
constexpr int SP_MAXN = 2 * LG_CL * SP_MAXPPC;  // 800

template <int TE>  // tail double2 slices per lane: n - SP_H <= 64 TE
__global__ void __launch_bounds__(SP_MAXPPC * 32, 1)
    k_eig_split(int n, int ld, double* __restrict__ rv, double* __restrict__ lam,
                int* __restrict__ info, const int* __restrict__ chol_info, double tol,
                int* __restrict__ warm_valid, double* __restrict__ gtail) {
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  if (chol_info[0] != 0 || chol_info[1] != 0) {  // uniform across the cluster
    if (c == 0 && threadIdx.x == 0) {
      *info = n + 1;
      if (warm_valid) *warm_valid = 0;
    }
    return;
  }
  extern __shared__ double ssm[];
  const int ppc = lg_ppc(n);
  const int m = 2 * LG_CL * ppc;
  const int T = n - SP_H;
  const int TP = T + (T & 1);  // even tail pitch: 16-byte aligned tail slots
  const int nrec = 2 * ppc + 4;
  double* buf = ssm;  // nrec heads
  __shared__ int top[2][SP_MAXPPC], bot[2][SP_MAXPPC], colid[2 * SP_MAXPPC + 4];
  __shared__ int land[2][2];
  __shared__ int rotated;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = c > 0 ? c - 1 : c, cr = c < LG_CL - 1 ? c + 1 : c;
  double* const buf_left = cluster.map_shared_rank(buf, cl);
  double* const buf_right = cluster.map_shared_rank(buf, cr);
  int* const colid_left = cluster.map_shared_rank(colid, cl);
  int* const colid_right = cluster.map_shared_rank(colid, cr);
  const int* const land_left = cluster.map_shared_rank(&land[0][0], cl);
  const int* const land_right = cluster.map_shared_rank(&land[0][0], cr);
  double* const tail_me = gtail + (size_t)c * nrec * TP;
  double* const tail_left = gtail + (size_t)cl * nrec * TP;
  double* const tail_right = gtail + (size_t)cr * nrec * TP;
  const int nthr = blockDim.x;
  const double tol2 = tol * tol;

  if (tid < ppc) {
    const int g = c * ppc + tid;
    top[0][tid] = tid;
    bot[0][tid] = ppc + tid;
    colid[tid] = 2 * g;
    colid[ppc + tid] = 2 * g + 1;
  }
  if (tid < 4) {
    land[tid >> 1][tid & 1] = 2 * ppc + tid;
    colid[2 * ppc + tid] = -1;
  }
  for (int e = tid; e < 2 * ppc * n; e += nthr) {
    const int b = e / n, i = e % n;
    const int k = b < ppc ? b : b - ppc;
    const int col = 2 * (c * ppc + k) + (b < ppc ? 0 : 1);
    const double v = (col < n && i <= col) ? rv[(size_t)col * ld + i] : 0.0;
    if (i < SP_H) buf[b * SP_H + i] = v;
    else __stcg(tail_me + (size_t)b * TP + (i - SP_H), v);
  }
  cluster.sync();  // every CTA initialised before any remote store

  int sweep = 0, cur = 0, gr = 0;
  bool converged = false;
  for (; sweep < LG_MAX_SWEEPS; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round, ++gr) {
      const int par = gr & 1;
      if (warp < ppc) {
        const int bp = top[cur][warp], bq = bot[cur][warp];
        const int cp = colid[bp], cq = colid[bq];
        double* rp = buf + bp * SP_H;
        double* rq = buf + bq * SP_H;
        double* tp_ = tail_me + (size_t)bp * TP;
        double* tq_ = tail_me + (size_t)bq * TP;
        const bool send_r = warp == ppc - 1 && c < LG_CL - 1;
        const bool send_l = warp == 0 && c > 0;
        const int dst_r = send_r ? land_right[0 * 2 + par] : 0;
        const int dst_l = send_l ? land_left[1 * 2 + par] : 0;
        // lane l owns the double2 at elements 2 l + 64 u of the head and of the tail
        double2 xt[TE], yt[TE];
        const double2* tp2 = reinterpret_cast<const double2*>(tp_);
        const double2* tq2 = reinterpret_cast<const double2*>(tq_);
#pragma unroll
        for (int u = 0; u < TE; ++u) {  // tails first: the L2 latency overlaps the head dots
          const int i = 2 * lane + 64 * u;
          xt[u] = i < T ? __ldcg(tp2 + lane + 32 * u) : make_double2(0.0, 0.0);
          yt[u] = i < T ? __ldcg(tq2 + lane + 32 * u) : make_double2(0.0, 0.0);
          if (i + 1 >= T) {  // odd tail: the pad element is not part of the vector
            xt[u].y = 0.0;
            yt[u].y = 0.0;
          }
        }
        double2* rp2 = reinterpret_cast<double2*>(rp);
        double2* rq2 = reinterpret_cast<double2*>(rq);
        double a = 0.0, b = 0.0, gm = 0.0;
#pragma unroll
        for (int u = 0; u < SP_HE / 2; ++u) {
          const double2 x = rp2[lane + 32 * u], y = rq2[lane + 32 * u];
          a = fma(x.x, x.x, fma(x.y, x.y, a));
          b = fma(y.x, y.x, fma(y.y, y.y, b));
          gm = fma(x.x, y.x, fma(x.y, y.y, gm));
        }
#pragma unroll
        for (int u = 0; u < TE; ++u) {
          a = fma(xt[u].x, xt[u].x, fma(xt[u].y, xt[u].y, a));
          b = fma(yt[u].x, yt[u].x, fma(yt[u].y, yt[u].y, b));
          gm = fma(xt[u].x, yt[u].x, fma(xt[u].y, yt[u].y, gm));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          gm += __shfl_xor_sync(0xffffffffu, gm, o);
        }
        const bool rot = cp < n && cq < n && gm * gm > tol2 * (a * b) && fabs(gm) > 1e-300;
        double2* dr = send_r ? reinterpret_cast<double2*>(buf_right + (size_t)dst_r * SP_H) : nullptr;
        double2* dl = send_l ? reinterpret_cast<double2*>(buf_left + (size_t)dst_l * SP_H) : nullptr;
        double2* trr = send_r ? reinterpret_cast<double2*>(tail_right + (size_t)dst_r * TP) : nullptr;
        double2* tll = send_l ? reinterpret_cast<double2*>(tail_left + (size_t)dst_l * TP) : nullptr;
        double2* tpw = reinterpret_cast<double2*>(tp_);
        double2* tqw = reinterpret_cast<double2*>(tq_);
        if (rot) {
          double cs, sn;
          jacobi_angle(a, b, gm, cs, sn);
#pragma unroll
          for (int u = 0; u < SP_HE / 2; ++u) {
            const int j = lane + 32 * u;
            const double2 x = rp2[j], y = rq2[j];
            const double2 xr = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
            const double2 yr = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
            rp2[j] = xr;
            rq2[j] = yr;
            if (send_r) dr[j] = xr;
            if (send_l) dl[j] = yr;
          }
#pragma unroll
          for (int u = 0; u < TE; ++u) {
            const int j = lane + 32 * u;
            if (2 * j < T) {
              const double2 xr = make_double2(cs * xt[u].x - sn * yt[u].x, cs * xt[u].y - sn * yt[u].y);
              const double2 yr = make_double2(sn * xt[u].x + cs * yt[u].x, sn * xt[u].y + cs * yt[u].y);
              __stcg(tpw + j, xr);
              __stcg(tqw + j, yr);
              if (send_r) __stcg(trr + j, xr);
              if (send_l) __stcg(tll + j, yr);
            }
          }
          if (lane == 0) rotated = 1;
        } else if (send_r || send_l) {
#pragma unroll
          for (int u = 0; u < SP_HE / 2; ++u) {
            const int j = lane + 32 * u;
            if (send_r) dr[j] = rp2[j];
            if (send_l) dl[j] = rq2[j];
          }
#pragma unroll
          for (int u = 0; u < TE; ++u) {
            const int j = lane + 32 * u;
            if (2 * j < T) {
              if (send_r) __stcg(trr + j, xt[u]);
              if (send_l) __stcg(tll + j, yt[u]);
            }
          }
        }
        if (lane == 0) {
          if (send_r) colid_right[dst_r] = cp;
          if (send_l) colid_left[dst_l] = cq;
        }
      }
      // next slot table by the circle method (see kp_eig_mid.cu)
      const int ot = top[cur][ppc - 1], ob = bot[cur][0];
      const int in_l = land[0][par], in_r = land[1][par];
      int ntop = 0, nbot = 0;
      if (tid < ppc) {
        const int k = tid;
        ntop = k == 0 ? (c == 0 ? top[cur][0] : in_l) : ((c == 0 && k == 1) ? ob : top[cur][k - 1]);
        nbot = k == ppc - 1 ? (c == LG_CL - 1 ? ot : in_r) : bot[cur][k + 1];
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      if (tid < ppc) {
        top[cur ^ 1][tid] = ntop;
        bot[cur ^ 1][tid] = nbot;
      }
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      if (tid == 0) {
        if (c > 0) land[0][par] = ob;
        if (c < LG_CL - 1) land[1][par] = ot;
      }
      cur ^= 1;
      __syncthreads();
    }
    int any = 0;
    for (int r = 0; r < LG_CL; ++r) any |= *cluster.map_shared_rank(&rotated, r);
    cluster.sync();
    if (!any) {
      converged = true;
      break;
    }
  }
  // eigenvalues ||u_i||^2 and the orthogonalised rows U (row col of rv)
  for (int sl = warp; sl < 2 * ppc; sl += nthr / 32) {
    const int bidx = sl < ppc ? top[cur][sl] : bot[cur][sl - ppc];
    const int col = colid[bidx];
    if (col < 0 || col >= n) continue;
    const double* r = buf + bidx * SP_H;
    const double* t = tail_me + (size_t)bidx * TP;
    double a = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double v = i < SP_H ? r[i] : __ldcg(t + (i - SP_H));
      a = fma(v, v, a);
      rv[(size_t)col * ld + i] = v;
    }
    a = warp_sum(a);
    if (lane == 0) lam[col] = a;
  }
  if (c == 0 && tid == 0) {
    *info = converged ? 0 : 1;
    if (warm_valid) *warm_valid = converged ? 1 : 0;
    atomicMax(&g_large_sweeps_max, converged ? sweep + 1 : 1000 + sweep);
  }
}

size_t sp_smem(int n) { return (size_t)(2 * lg_ppc(n) + 4) * SP_H * sizeof(double); }

template <int TE>
void sp_launch(int n, int ld, double* U, double* lam, int* info, const int* chol_info, double tol,
               int* warm_valid, double* gtail, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LG_CL);
  cfg.blockDim = dim3(lg_ppc(n) * 32);
  cfg.dynamicSmemBytes = sp_smem(n);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = LG_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_eig_split<TE>, n, ld, U, lam, info, chol_info, tol, warm_valid,
                     gtail);
}

template <int TE>
bool sp_attrs() {
  return cudaFuncSetAttribute(k_eig_split<TE>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                              1) == cudaSuccess &&
         cudaFuncSetAttribute(k_eig_split<TE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sp_smem(SP_MAXN)) == cudaSuccess;
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
void lg_launch(int n, int ld, double* U, double* V, double* lam, int* info,
               const int* chol_info, double tol, int* warm_valid, cudaStream_t s) {
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
  if (V)
    cudaLaunchKernelEx(&cfg, k_eig_large<EFM, W, true>, n, ld, U, V, lam, info, chol_info, tol,
                       warm_valid);
  else
    cudaLaunchKernelEx(&cfg, k_eig_large<EFM, W, false>, n, ld, U, V, lam, info, chol_info, tol,
                       warm_valid);
}

int g_large_ok = 0;  // 0 unknown, 1 usable, -1 not schedulable
bool g_split_ok = false;

}  // namespace

int large_eig_max_n() {
  if (g_large_ok == 0) {
    bool ok = lg_attrs<6, 16>() && lg_attrs<8, 16>() && lg_attrs<10, 12>() &&
              lg_attrs<12, 12>() && lg_attrs<14, 12>() && lg_attrs<16, 12>();
    ok = ok && cudaFuncSetAttribute(k_eig_stream, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                    1) == cudaSuccess;
    g_split_ok = sp_attrs<1>() && sp_attrs<2>() && sp_attrs<3>() && sp_attrs<4>() &&
                 sp_attrs<5>();
    if (g_split_ok) {  // 16 CTAs of 800 threads and ~221 KB smem must be co-schedulable
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(LG_CL);
      cfg.blockDim = dim3(SP_MAXPPC * 32);
      cfg.dynamicSmemBytes = sp_smem(SP_MAXN);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = LG_CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      g_split_ok = cudaOccupancyMaxActiveClusters(&nc, k_eig_split<5>, &cfg) == cudaSuccess && nc >= 1;
    }
    cudaGetLastError();
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
      ok = cudaOccupancyMaxActiveClusters(&nc, k_eig_large<16, 12, true>, &cfg) == cudaSuccess && nc >= 1;
    }
    if (!ok) cudaGetLastError();
    g_large_ok = ok ? 1 : -1;
  }
  return g_large_ok > 0 ? LG_MAXN_ANY : 0;
}

bool large_eig_accumulate_v() {
  static const bool acc = [] {
    const char* e = getenv("KP_LARGE_ACCV");
    return e && atoi(e) == 1;
  }();
  return acc;
}

int large_eig_accv_max_n() { return LG_MAXN; }

int large_eig_sweeps_used(bool reset) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_large_sweeps_max, sizeof(int));
  if (reset) {
    const int z = 0;
    cudaMemcpyToSymbol(g_large_sweeps_max, &z, sizeof(int));
  }
  return v;
}

bool large_eig_split_ok(int n) {
  static const bool enabled = [] {
    const char* e = getenv("KP_LARGE_SPLIT");
    return !(e && atoi(e) == 0);
  }();
  large_eig_max_n();
  return enabled && g_split_ok && n > SP_H && n <= SP_MAXN;
}

void launch_eig_large(int n, int ld, double* U, double* V, double* lam, int* info,
                      const int* chol_info, cudaStream_t s, int* warm_valid, double* gtail) {
  count_launch();
  const double tol = fmax(jacobi_tol_floor(), 2.0 * n * DBL_EPSILON);
  if (!V && gtail && large_eig_split_ok(n)) {
    switch ((n - SP_H + 63) / 64) {
#define KP_SP_CASE(E)                                                                    case E:                                                                                  sp_launch<E>(n, ld, U, lam, info, chol_info, tol, warm_valid, gtail, s);              return;
      KP_SP_CASE(1)
      KP_SP_CASE(2)
      KP_SP_CASE(3)
      KP_SP_CASE(4)
      KP_SP_CASE(5)
#undef KP_SP_CASE
      default:
        break;
    }
  }
  if (n > LG_MAXN) {  // any width: the streaming kernel (U only)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(LG_CL);
    cfg.blockDim = dim3(16 * 32);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = LG_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_eig_stream, n, ld, U, lam, info, chol_info, tol, warm_valid);
    return;
  }
  const int ef = n / 64;
  if (ef <= 6) lg_launch<6, 16>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 8) lg_launch<8, 16>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 10) lg_launch<10, 12>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 12) lg_launch<12, 12>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
  else if (ef <= 14) lg_launch<14, 12>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
  else lg_launch<16, 12>(n, ld, U, V, lam, info, chol_info, tol, warm_valid, s);
}

}  // namespace kp
