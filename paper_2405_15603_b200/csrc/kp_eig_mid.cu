// Mid-size symmetric eigensolver (96 < n <= 288) for the damped Kronecker-sum solve:
// one-sided (Hestenes) Jacobi on a Cholesky factor, the columns resident in the shared
// memory of a thread-block cluster (16 CTAs, or 8 where 16-CTA clusters cannot be
// scheduled), FP64, sm_100a.
//
// Used for the factor pairs that are too large for the one-CTA solver of kp_eig_small.cu
// (BASELINE c4: 128-257; c5 layer 0's A: 101).  The generalised problem M1 x = l M2 x
// (reference src/linalg.py:136-174 via curvature.py:150-161) is reduced with library calls
// that never block the host (kp_step.cu gen_eig_mid): M2 = L L^T (potrf), C = L^-1 M1 L^-T
// (two trsm), C = R^T R (potrf, upper).  This kernel then orthogonalises the columns of R
// by plane rotations, R J1 J2 ... = R V with mutually orthogonal columns, so that
//   C V = V diag(||R v_i||^2)      (eigenpairs of C, V orthogonal),
// and T = L^-T V (trsm) satisfies T^T M2 T = I, T^T M1 T = diag(lambda).
//
// Parallel ordering: the n columns (padded with zero columns to 2 CL ppc for a cluster of
// CL CTAs) form CL ppc disjoint pairs per round; CTA c owns pairs [c ppc, (c+1) ppc), one
// warp per pair.  Between rounds the pairing advances by the circle method (one column
// fixed, the rest rotate one position), so every pair of columns meets once per sweep of
// 2 CL ppc - 1 rounds.  Inside a CTA a column moves by re-indexing only; at a CTA boundary
// the warp that rotated the outgoing column also stores it (R and V parts, 2n doubles)
// straight into a landing record of the neighbour through distributed shared memory.  The
// landing records rotate with the hand-overs (the record a CTA hands over in round t is its
// landing record for round t + 2), so nothing is copied.  One split cluster barrier per
// round; the slot tables are double-buffered by round parity.  Pairs up to 160 use 8-CTA
// clusters, larger ones 16.
//
// A rotation is applied when |<r_p, r_q>| > tol ||r_p|| ||r_q|| (tol = max(1e-14, 2 n eps));
// the sweep loop ends after a sweep without rotations anywhere in the cluster.
#include <cooperative_groups.h>

#include <cfloat>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace cg = cooperative_groups;

namespace kp {

namespace {

constexpr int MID_MAXN = 288;
// Without V (U-only mode) a record is one column, so 16-CTA clusters hold columns up to
// MID_MAXN_WIDE (c5's 512 / 513 pairs): 17 warps per CTA, 38 records of 544 doubles.
constexpr int MID_MAXN_WIDE = 544;
constexpr int MID_MAX_SWEEPS = 40;

__device__ int g_mid_sweeps_max = 0;  // diagnostic: most sweeps used by any solve

__host__ __device__ inline int mid_ppc(int n, int cl) { return ((n + 1) / 2 + cl - 1) / cl; }

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rv: n x n column-major.  In: the upper-triangular Cholesky factor R of C (the strictly
// lower part is ignored).  Out: the eigenvectors V of C = R^T R (column i = vector i).
// lam[i] = eigenvalue i.  info: 0 ok, 1 no convergence in MID_MAX_SWEEPS sweeps, n + 1 when
// one of the two upstream Cholesky factorisations (chol_info[0..1]) failed (not PD).
// warm_valid (optional): set to 1 on success, 0 otherwise (the caller's warm-start flag).
//
// smem: 2 ppc column records + 4 landing records ([from left, from right] x round parity),
// each record R | V (2n doubles).  A round: every pair warp loads its two R columns into
// registers, forms the three dot products and rotates R and V; the warps owning the CTA's
// outgoing columns (last top slot -> right neighbour, first bottom slot -> left neighbour)
// also store them into the neighbour's landing record.  Between the two halves of the
// cluster barrier each CTA writes the next round's slot table.
template <int CL, int EF, bool ACCV, int MAXN = MID_MAXN>
__global__ void __launch_bounds__(((MAXN / 2 + CL - 1) / CL) * 32, 1)
    k_eig_mid(int n, double* __restrict__ rv, double* __restrict__ lam, int* __restrict__ info,
              const int* __restrict__ chol_info, double tol, int* __restrict__ warm_valid,
              long long* prof) {
  constexpr int MAXPPC = (MAXN / 2 + CL - 1) / CL;
  cg::cluster_group cluster = cg::this_cluster();
  long long t_rot = 0, t_sync = 0, t_upd = 0, t0 = 0;
  const int c = (int)cluster.block_rank();
  if (chol_info[0] != 0 || chol_info[1] != 0) {  // uniform across the cluster: no DSMEM yet
    if (c == 0 && threadIdx.x == 0) {
      *info = n + 1;
      if (warm_valid) *warm_valid = 0;
    }
    return;
  }
  extern __shared__ double msm[];
  const int ppc = mid_ppc(n, CL);
  const int m = 2 * CL * ppc;  // padded column count (columns >= n are zero)
  const size_t cs2 = (ACCV ? 2 : 1) * (size_t)n;  // one column record: R (n) [then V (n)]
  double* buf = msm;  // 2 ppc + 4 records: the slots' columns and 4 landing records
  // land[dir][par]: the record a neighbour stores its handed-over column into in rounds of
  // parity par (dir 0: from the left, 1: from the right).  After the round the record joins
  // the slot table and the record this CTA handed over in that direction takes its place.
  __shared__ int top[2][MAXPPC], bot[2][MAXPPC], colid[2 * MAXPPC + 4];
  __shared__ int land[2][2];
  __shared__ int rotated;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* const buf_left = cluster.map_shared_rank(buf, c > 0 ? c - 1 : c);
  double* const buf_right = cluster.map_shared_rank(buf, c < CL - 1 ? c + 1 : c);
  int* const colid_left = cluster.map_shared_rank(colid, c > 0 ? c - 1 : c);
  int* const colid_right = cluster.map_shared_rank(colid, c < CL - 1 ? c + 1 : c);
  const int* const land_left = cluster.map_shared_rank(&land[0][0], c > 0 ? c - 1 : c);
  const int* const land_right = cluster.map_shared_rank(&land[0][0], c < CL - 1 ? c + 1 : c);
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
    buf[b * cs2 + i] = (col < n && i <= col) ? rv[(size_t)col * n + i] : 0.0;
    if (ACCV) buf[b * cs2 + n + i] = (i == col) ? 1.0 : 0.0;
  }
  cluster.sync();  // every CTA initialised before any remote store

  int sweep = 0, cur = 0;  // cur: slot table of the current round (= parity of gr)
  int gr = 0;              // rounds so far, across sweeps
  bool converged = false;
  for (; sweep < MID_MAX_SWEEPS; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round, ++gr) {
      const int par = gr & 1;
      if (prof) t0 = clock64();
      if (warp < ppc) {
        const int bp = top[cur][warp], bq = bot[cur][warp];
        const int cp = colid[bp], cq = colid[bq];
        double* rp = buf + bp * cs2;
        double* rq = buf + bq * cs2;
        // this warp forwards its top column to the right / its bottom column to the left
        const bool send_r = warp == ppc - 1 && c < CL - 1;
        const bool send_l = warp == 0 && c > 0;
        // the neighbour's landing record for this round (set two rounds ago, see land[])
        const int dst_r = send_r ? land_right[0 * 2 + par] : 0;  // their "from the left"
        const int dst_l = send_l ? land_left[1 * 2 + par] : 0;   // their "from the right"
        // EF = n / 32 full 32-element slices per column (no bounds checks) + a tail of
        // n - 32 EF elements (lanes below it)
        const int tail = n - 32 * EF;
        const bool tl = lane < tail;
        double x[EF + 1], y[EF + 1];
        double a = 0.0, b = 0.0, gm = 0.0;
#pragma unroll
        for (int u = 0; u < EF; ++u) {
          x[u] = rp[lane + 32 * u];
          y[u] = rq[lane + 32 * u];
        }
        x[EF] = tl ? rp[32 * EF + lane] : 0.0;
        y[EF] = tl ? rq[32 * EF + lane] : 0.0;
#pragma unroll
        for (int u = 0; u <= EF; ++u) {
          a = fma(x[u], x[u], a);
          b = fma(y[u], y[u], b);
          gm = fma(x[u], y[u], gm);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // three interleaved butterflies: 5 dependent steps
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          gm += __shfl_xor_sync(0xffffffffu, gm, o);
        }
        const bool rot = cp < n && cq < n && gm * gm > tol2 * (a * b) && fabs(gm) > 1e-300;
        double* dr = send_r ? buf_right + (size_t)dst_r * cs2 : nullptr;
        double* dl = send_l ? buf_left + (size_t)dst_l * cs2 : nullptr;
        double* vp = rp + n;
        double* vq = rq + n;
        if (rot) {
          double cs, sn;
          jacobi_angle(a, b, gm, cs, sn);
#pragma unroll
          for (int u = 0; u <= EF; ++u) {
            const int i = lane + 32 * u;
            if (u < EF || tl) {
              const double xr = cs * x[u] - sn * y[u], yr = sn * x[u] + cs * y[u];
              rp[i] = xr;
              rq[i] = yr;
              if (send_r) dr[i] = xr;
              if (send_l) dl[i] = yr;
              if (ACCV) {
                const double pu = vp[i], qu = vq[i];
                const double xv = cs * pu - sn * qu, yv = sn * pu + cs * qu;
                vp[i] = xv;
                vq[i] = yv;
                if (send_r) dr[n + i] = xv;
                if (send_l) dl[n + i] = yv;
              }
            }
          }
          if (lane == 0) rotated = 1;
        } else if (send_r || send_l) {
#pragma unroll
          for (int u = 0; u <= EF; ++u) {
            const int i = lane + 32 * u;
            if (u < EF || tl) {
              if (send_r) {
                dr[i] = x[u];
                if (ACCV) dr[n + i] = vp[i];
              }
              if (send_l) {
                dl[i] = y[u];
                if (ACCV) dl[n + i] = vq[i];
              }
            }
          }
        }
        if (lane == 0) {
          if (send_r) colid_right[dst_r] = cp;
          if (send_l) colid_left[dst_l] = cq;
        }
      }
      if (prof) { __syncthreads(); const long long t1 = clock64(); t_rot += t1 - t0; t0 = t1; }
      // next slot table by the circle method: top[k] <- top[k-1], bot[k] <- bot[k+1];
      // cluster ends: global top[0] stays, global bot[0] -> top[1], global top[last] ->
      // bot[last]; the columns that arrived sit in land[.][par], the records handed over
      // become the landing records of round + 2.  The table is local, so it is written
      // between the two halves of the cluster barrier; land[.][par] (which neighbours read
      // during the rotation phase) is read before the arrive and rewritten after the wait.
      const int ot = top[cur][ppc - 1], ob = bot[cur][0];
      const int in_l = land[0][par], in_r = land[1][par];
      int ntop = 0, nbot = 0;
      if (tid < ppc) {
        const int k = tid;
        ntop = k == 0 ? (c == 0 ? top[cur][0] : in_l) : ((c == 0 && k == 1) ? ob : top[cur][k - 1]);
        nbot = k == ppc - 1 ? (c == CL - 1 ? ot : in_r) : bot[cur][k + 1];
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      if (tid < ppc) {
        top[cur ^ 1][tid] = ntop;
        bot[cur ^ 1][tid] = nbot;
      }
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      if (prof) { const long long t1 = clock64(); t_sync += t1 - t0; t0 = t1; }
      if (tid == 0) {
        if (c > 0) land[0][par] = ob;       // handed to the left this round
        if (c < CL - 1) land[1][par] = ot;  // handed to the right this round
      }
      cur ^= 1;
      __syncthreads();
      if (prof) t_upd += clock64() - t0;
    }
    // every flag of this sweep was set before the last round's cluster barrier
    int any = 0;
    for (int r = 0; r < CL; ++r) any |= *cluster.map_shared_rank(&rotated, r);
    cluster.sync();  // all flags read before any CTA resets its own
    if (!any) {
      converged = true;
      break;
    }
  }
  // eigenvalues ||R v_i||^2 and eigenvectors V (column col of rv)
  for (int sl = warp; sl < 2 * ppc; sl += nthr / 32) {
    const int bidx = sl < ppc ? top[cur][sl] : bot[cur][sl - ppc];
    const int col = colid[bidx];
    if (col < 0 || col >= n) continue;
    const double* r = buf + bidx * cs2;
    double a = 0.0;
    for (int i = lane; i < n; i += 32) {
      a = fma(r[i], r[i], a);
      rv[(size_t)col * n + i] = ACCV ? r[n + i] : r[i];
    }
    a = warp_allsum(a);
    if (lane == 0) lam[col] = a;
  }
  if (prof && tid == 0) {
    prof[5 * c + 0] = t_rot;
    prof[5 * c + 1] = t_sync;
    prof[5 * c + 2] = 0;
    prof[5 * c + 3] = t_upd;
    prof[5 * c + 4] = sweep;
  }
  if (c == 0 && tid == 0) {
    *info = converged ? 0 : 1;
    if (warm_valid) *warm_valid = converged ? 1 : 0;
    atomicMax(&g_mid_sweeps_max, converged ? sweep + 1 : 1000 + sweep);
  }
}

template <int CL>
size_t mid_smem(int n, bool accv) {  // slots + landing records
  return (size_t)(2 * mid_ppc(n, CL) + 4) * (accv ? 2 : 1) * n * sizeof(double);
}

// Cluster size: 16 when the device can co-schedule 16-CTA clusters of this kernel
// (non-portable size), else 8.
template <int CL>
bool mid_setup() {
  bool ok = true;
  auto attrs = [&](auto k, bool accv) {
    ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)mid_smem<CL>(MID_MAXN, accv)) == cudaSuccess;
    if (CL > 8)
      ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                     cudaSuccess;
  };
#define KP_MID_ATTRS(E)               \
  attrs(k_eig_mid<CL, E, true>, true); \
  attrs(k_eig_mid<CL, E, false>, false);
  KP_MID_ATTRS(3)
  KP_MID_ATTRS(4)
  KP_MID_ATTRS(5)
  KP_MID_ATTRS(6)
  KP_MID_ATTRS(7)
  KP_MID_ATTRS(8)
  KP_MID_ATTRS(9)
#undef KP_MID_ATTRS
  if (CL == 16) {  // wide U-only instances
    auto wide = [&](auto k) {
      ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)mid_smem<16>(MID_MAXN_WIDE, false)) == cudaSuccess;
      ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                     cudaSuccess;
    };
    wide(k_eig_mid<16, 9, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 10, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 11, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 12, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 13, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 14, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 15, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 16, false, MID_MAXN_WIDE>);
    wide(k_eig_mid<16, 17, false, MID_MAXN_WIDE>);
  }
  if (!ok) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(mid_ppc(MID_MAXN, CL) * 32);
  cfg.dynamicSmemBytes = mid_smem<CL>(MID_MAXN, true);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, k_eig_mid<CL, MID_MAXN / 32, true>, &cfg) !=
          cudaSuccess ||
      nc < 1) {
    cudaGetLastError();
    return false;
  }
  return true;
}

template <int CL>
void launch_mid(int n, double* rv, double* lam, int* info, const int* chol_info,
                cudaStream_t s, int* warm_valid, long long* prof, bool accv) {
  const double tol = fmax(jacobi_tol_floor(), 2.0 * n * DBL_EPSILON);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(mid_ppc(n, CL) * 32);
  cfg.dynamicSmemBytes = mid_smem<CL>(n, accv);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (n > MID_MAXN) {  // wide U-only instances (CL == 16 and !accv: see mid_eig_max_n)
    switch (n / 32) {
#define KP_MID_WIDE(E)                                                                        \
  case E:                                                                                     \
    cudaLaunchKernelEx(&cfg, k_eig_mid<16, E, false, MID_MAXN_WIDE>, n, rv, lam, info,        \
                       chol_info, tol, warm_valid, prof);                                     \
    break;
      KP_MID_WIDE(9)
      KP_MID_WIDE(10)
      KP_MID_WIDE(11)
      KP_MID_WIDE(12)
      KP_MID_WIDE(13)
      KP_MID_WIDE(14)
      KP_MID_WIDE(15)
      KP_MID_WIDE(16)
      KP_MID_WIDE(17)
#undef KP_MID_WIDE
      default:
        break;
    }
    return;
  }
  switch (n / 32) {
#define KP_MID_CASE(E)                                                                        \
  case E:                                                                                     \
    if (accv)                                                                                 \
      cudaLaunchKernelEx(&cfg, k_eig_mid<CL, E, true>, n, rv, lam, info, chol_info, tol,      \
                         warm_valid, prof);                                                   \
    else                                                                                      \
      cudaLaunchKernelEx(&cfg, k_eig_mid<CL, E, false>, n, rv, lam, info, chol_info, tol,     \
                         warm_valid, prof);                                                   \
    break;
    KP_MID_CASE(3)
    KP_MID_CASE(4)
    KP_MID_CASE(5)
    KP_MID_CASE(6)
    KP_MID_CASE(7)
    KP_MID_CASE(8)
    KP_MID_CASE(9)
#undef KP_MID_CASE
    default:
      break;
  }
}

int g_mid_cl = 0;  // 0: not chosen yet

}  // namespace

bool mid_eig_accumulate_v() {
  static const bool acc = [] {
    const char* e = getenv("KP_MID_ACCV");
    return e && atoi(e) == 1;
  }();
  return acc;
}

int mid_eig_cluster_size() {
  if (g_mid_cl == 0) {
    const char* env = getenv("KP_MID_CLUSTER");
    const int want = env ? atoi(env) : 16;  // 16 (default), 8, or 0 = off (large-pair route)
    g_mid_cl = want == 0 ? -1 : (want == 16 && mid_setup<16>()) ? 16 : (mid_setup<8>() ? 8 : -1);
  }
  return g_mid_cl;
}

// 0 when no cluster launch of the kernel can be scheduled: the pairs then take the large-pair
// route (kp_eig_large.cu).
int mid_eig_max_n() {
  const int cl = mid_eig_cluster_size();
  if (cl <= 0) return 0;
  return (cl == 16 && !mid_eig_accumulate_v()) ? MID_MAXN_WIDE : MID_MAXN;
}

int mid_eig_sweeps_used(bool reset) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_mid_sweeps_max, sizeof(int));
  if (reset) {
    const int z = 0;
    cudaMemcpyToSymbol(g_mid_sweeps_max, &z, sizeof(int));
  }
  return v;
}

void launch_eig_mid(int n, double* rv, double* lam, int* info, const int* chol_info,
                    cudaStream_t s, int* warm_valid, long long* prof) {
  const bool accv = mid_eig_accumulate_v();
  count_launch();
  // 16-CTA clusters for the large pairs (the critical path); pairs up to 160 use 8 CTAs,
  // which leaves SMs (and whole GPCs) free for the large pairs' clusters (c4 precondition
  // 6.41 -> 5.68 ms)
  constexpr int kSmallN = 160;
  if (mid_eig_cluster_size() == 16 && n > kSmallN)
    launch_mid<16>(n, rv, lam, info, chol_info, s, warm_valid, prof, accv);
  else launch_mid<8>(n, rv, lam, info, chol_info, s, warm_valid, prof, accv);
}

}  // namespace kp
