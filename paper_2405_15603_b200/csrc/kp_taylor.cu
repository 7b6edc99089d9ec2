// Taylor-mode (forward-Laplacian) elementwise kernels, FP64, sm_100a.
//
// State layout follows the reference (src/taylor.py:3-16): sample n owns rows
// n*S .. n*S+S-1 of a row-major (N*S, h) matrix — row 0 the value, rows 1..d the
// directional first derivatives, row d+1 the operator (L z) row.  Every kernel
// maps one thread to one (sample, unit) pair and walks that sample's S rows, so
// each row access is a coalesced 32-wide run of consecutive units and the
// per-sample reductions over the d derivative rows stay in registers.
#include <algorithm>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

static inline unsigned grid_for(int64_t n, int threads) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148LL * 64));
}

// ---------------------------------------------------------------------------
// layer 0 + first activation (taylor.py:124-169 specialised: Z0 = [x; I; 0], so the
// pre-activation of sample n is (z_n = x_n W0^T + b0, derivative rows W0[:, i], operator
// row 0)).  z comes from a small GEMM; this kernel only expands the S output rows, with
// W0^T (coalesced across units) and q_j = sum_i (W0[j,i] c_i) W0[j,i] prepared once per
// parameter set (k_prep_layer0).

// Dense coefficients c = Q diag(lambda) Q^T: the derivative rows are taken along the
// eigenvectors, Z0 = [x; Q^T; 0], so the layer-0 derivative rows become (W0 Q)[:, k] and
// every quadratic form sum_ij c_ij g_i g_j is the diagonal sum_k lambda_k g'_k^2.  The
// factors, gradient and Gramian contractions sum over rows and are invariant under this
// orthogonal change of rows; only the seeds (rotated in) and the layer-0 weight gradient
// and output gradient (rotated back) see Q.
__global__ void k_prep_layer0(const double* __restrict__ th0, int d, int h1,
                              const double* __restrict__ cdiag, const double* __restrict__ rot,
                              double* __restrict__ w0t, double* __restrict__ q0, int64_t D) {
  th0 += (int64_t)blockIdx.y * D;
  w0t += (int64_t)blockIdx.y * d * h1;
  q0 += (int64_t)blockIdx.y * h1;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < h1; j += gridDim.x * blockDim.x) {
    const double* w = th0 + (int64_t)j * (d + 1);
    double q = 0.0;
    for (int k = 0; k < d; ++k) {
      double g;
      if (rot) {
        g = 0.0;
        for (int i = 0; i < d; ++i) g = fma(w[i], rot[(int64_t)i * d + k], g);
      } else {
        g = w[k];
      }
      w0t[(int64_t)k * h1 + j] = g;
      q += (g * cdiag[k]) * g;
    }
    q0[j] = q;
  }
}

void launch_prep_layer0(const double* theta0, int d, int h1, const double* cdiag, const double* rot,
                        double* w0t, double* q0, cudaStream_t s, int batch, int64_t D) {
  count_launch();
  k_prep_layer0<<<dim3((unsigned)ceil_div(h1, 128), (unsigned)batch), 128, 0, s>>>(
      theta0, d, h1, cdiag, rot, w0t, q0, D);
}

__global__ void k_rotate_rows(double* __restrict__ X, int64_t stride, int64_t n, int d,
                              const double* __restrict__ Q, int transpose) {
  extern __shared__ double row[];
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    double* x = X + r * stride;
    for (int i = threadIdx.x; i < d; i += blockDim.x) row[i] = x[i];
    __syncthreads();
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
      double acc = 0.0;
      if (transpose)
        for (int i = 0; i < d; ++i) acc = fma(Q[(int64_t)i * d + k], row[i], acc);
      else
        for (int i = 0; i < d; ++i) acc = fma(Q[(int64_t)k * d + i], row[i], acc);
      x[k] = acc;
    }
    __syncthreads();
  }
}

void launch_rotate_rows(double* X, int64_t stride, int64_t n, int d, const double* Q, int transpose,
                        cudaStream_t s) {
  if (n <= 0 || d <= 0) return;
  count_launch();
  const unsigned blocks = (unsigned)std::min<int64_t>(n, 148 * 16);
  k_rotate_rows<<<blocks, 128, sizeof(double) * d, s>>>(X, stride, n, d, Q, transpose);
}

__global__ void k_rot_accum(const double* __restrict__ T, int q, int d, const double* __restrict__ Q,
                            double* __restrict__ out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)q * d) return;
  const int j = (int)(e / d), i = (int)(e % d);
  double acc = 0.0;
  for (int k = 0; k < d; ++k) acc = fma(T[(int64_t)j * d + k], Q[(int64_t)i * d + k], acc);
  out[(int64_t)j * ldo + i] += acc;
}

void launch_rot_accum(const double* T, int q, int d, const double* Q, double* out, int64_t ldo,
                      cudaStream_t s) {
  count_launch();
  k_rot_accum<<<(unsigned)ceil_div((int64_t)q * d, 256), 256, 0, s>>>(T, q, d, Q, out, ldo);
}

// One warp per (sample, 32-unit tile): lane j writes unit j of every one of the sample's
// S rows (256-byte coalesced stores); the W0^T tile and q live in shared memory.
constexpr int EXP_WARPS = 8;

__global__ void __launch_bounds__(EXP_WARPS * 32)
    k_first_expand(const double* __restrict__ zval, int64_t n, int h1, TaylorDims td,
                   const double* __restrict__ w0t, const double* __restrict__ q0,
                   double* __restrict__ post, int64_t samples_per_block) {
  extern __shared__ double wsm[];  // [d][32] W0^T tile, then q[32]
  const int d = td.d;
  {  // candidate batch entry (grid.z)
    const int64_t kk = blockIdx.z;
    zval += kk * n * h1;
    post += kk * n * td.S * h1;
    w0t += kk * (int64_t)d * h1;
    q0 += kk * h1;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.x * 32;
  const int j = j0 + lane;
  const bool valid = j < h1;
  if (td.taylor) {
    for (int e = threadIdx.x; e < d * 32; e += blockDim.x) {
      const int i = e / 32, jj = j0 + e % 32;
      wsm[e] = jj < h1 ? w0t[(int64_t)i * h1 + jj] : 0.0;
    }
    if (threadIdx.x < 32) wsm[d * 32 + threadIdx.x] = valid ? q0[j] : 0.0;
    __syncthreads();
  }
  const double qj = td.taylor ? wsm[d * 32 + lane] : 0.0;
  const int64_t s_begin = (int64_t)blockIdx.y * samples_per_block;
  const int64_t s_end = min(n, s_begin + samples_per_block);
  for (int64_t smp = s_begin + warp; smp < s_end; smp += EXP_WARPS) {
    if (!valid) continue;
    const TanhD t = tanh_derivs(zval[smp * h1 + j], false);
    double* out = post + smp * td.S * h1 + j;
    out[0] = t.s0;
    if (!td.taylor) continue;
#pragma unroll 8
    for (int i = 0; i < d; ++i) out[(int64_t)(i + 1) * h1] = t.s1 * wsm[i * 32 + lane];
    // operator row: s1 * 0 + s2 * quad (taylor.py:168 with L z_in = 0)
    out[(int64_t)(d + 1) * h1] = t.s2 * qj;
  }
}

void launch_first_layer(const double* x, int64_t n, int d, const double* theta0, int h1,
                        TaylorDims td, const double* w0t, const double* q0, double* zval,
                        double* post, cudaStream_t s, int batch, int64_t D) {
  if (n <= 0) return;
  // z = x W0^T + b0 (value rows only; bias on every row of this n x h1 product)
  GemmNT g{x, d, theta0, d + 1, zval, h1, n, h1, d, theta0 + d, d + 1, 1};
  g.batch = batch;
  g.sB = D;
  g.sBias = D;
  g.sC = n * h1;
  launch_gemm_nt(g, s);
  if (post == nullptr) return;  // z only (the caller expands it: kp_crt.cu k_crt_first)
  const unsigned tiles = (unsigned)ceil_div(h1, 32);
  // about 8 blocks per SM over the whole (tiles x groups x candidates) grid
  const int64_t groups = std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(n, EXP_WARPS),
                           std::max<int64_t>(8, (148LL * 8 / tiles + 1) / std::max(batch, 1))));
  const int64_t spb = ceil_div(n, groups);
  const size_t smem = td.taylor ? sizeof(double) * (size_t)(td.d * 32 + 32) : 0;
  count_launch();
  k_first_expand<<<dim3(tiles, (unsigned)ceil_div(n, spb), (unsigned)batch), EXP_WARPS * 32, smem,
                   s>>>(zval, n, h1, td, w0t, q0, post, spb);
}

// ---------------------------------------------------------------------------
// activation forward (taylor.py:151-169)

// pre == post (in-place) is allowed: each thread reads an element before writing it.
__global__ void k_act_fwd(const double* pre, double* post, int64_t n,
                          int h, TaylorDims td, const double* __restrict__ cdiag) {
  const int64_t total = n * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t smp = e / h;
    const int j = (int)(e % h);
    const int64_t base = smp * td.S * h + j;
    const TanhD t = tanh_derivs(pre[base], false);
    post[base] = t.s0;
    if (!td.taylor) continue;
    double quad = 0.0;
    for (int i = 1; i <= td.d; ++i) {
      const double g = pre[base + (int64_t)i * h];
      post[base + (int64_t)i * h] = t.s1 * g;
      quad += (g * cdiag[i - 1]) * g;
    }
    const int64_t o = base + (int64_t)(td.d + 1) * h;
    post[o] = t.s1 * pre[o] + t.s2 * quad;
  }
}

void launch_act_fwd(const double* pre, double* post, int64_t n, int h, TaylorDims td,
                    const double* cdiag, cudaStream_t s) {
  const int64_t total = n * h;
  if (total <= 0) return;
  count_launch();
  k_act_fwd<<<grid_for(total, 256), 256, 0, s>>>(pre, post, n, h, td, cdiag);
}

// ---------------------------------------------------------------------------
// last (h_out = 1) layer + residual (pde.py:344-360 with the affine residual map)

constexpr int LAST_THREADS = 256;
constexpr int LAST_MAX_ROWS = 1024;

__global__ void __launch_bounds__(LAST_THREADS) k_last_layer(
    const double* __restrict__ post, int64_t n, int h, const double* __restrict__ th,
    TaylorDims td, int spb, const double* __restrict__ r0, const double* __restrict__ seeds,
    const double* __restrict__ targets, double* __restrict__ r, double* __restrict__ u_out,
    const double* __restrict__ quad, double* __restrict__ seeds_out) {
  __shared__ double u[LAST_MAX_ROWS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * spb;
  const int ns = (int)((n - s0) < spb ? (n - s0) : spb);
  const int rows = ns * td.S;
  const double b = th[h];
  for (int row = warp; row < rows; row += LAST_THREADS / 32) {
    const double* pr = post + (s0 * td.S + row) * h;
    double acc = 0.0;
    for (int j = lane; j < h; j += 32) acc = fma(pr[j], th[j], acc);
    acc = warp_sum(acc);
    if (row % td.S == 0) acc += b;
    if (lane == 0) {
      u[row] = acc;
      if (u_out) u_out[s0 * td.S + row] = acc;
    }
  }
  __syncthreads();
  if (r == nullptr) return;
  for (int k = threadIdx.x; k < ns; k += LAST_THREADS) {
    const int64_t smp = s0 + k;
    double v;
    if (td.taylor) {
      v = point_residual(u + k * td.S, td.S, r0[smp], seeds + smp * td.S,
                         quad ? quad + smp * td.d : nullptr,
                         seeds_out ? seeds_out + smp * td.S : nullptr);
    } else {
      v = u[k] - targets[smp];
    }
    r[smp] = v;
  }
}

__global__ void k_split_u(const double* __restrict__ u, int64_t n, int d, double* value,
                          double* grad, double* op) {
  const int S = d + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * S;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t smp = e / S;
    const int s = (int)(e % S);
    if (s == 0) value[smp] = u[e];
    else if (s <= d) grad[smp * d + s - 1] = u[e];
    else op[smp] = u[e];
  }
}

void launch_split_u(const double* u, int64_t n, int d, double* value, double* grad, double* op,
                    cudaStream_t s) {
  if (n <= 0) return;
  count_launch();
  k_split_u<<<grid_for(n * (d + 2), 256), 256, 0, s>>>(u, n, d, value, grad, op);
}

__global__ void k_initial_state(const double* __restrict__ x, int64_t n, int d,
                                double* __restrict__ z) {
  const int S = d + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * S * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t smp = e / ((int64_t)S * d);
    const int rem = (int)(e % ((int64_t)S * d));
    const int s = rem / d, k = rem % d;
    z[e] = s == 0 ? x[smp * d + k] : (s == k + 1 ? 1.0 : 0.0);
  }
}

void launch_initial_state(const double* x, int64_t n, int d, double* z, cudaStream_t s) {
  if (n <= 0) return;
  count_launch();
  k_initial_state<<<grid_for(n * (d + 2) * d, 256), 256, 0, s>>>(x, n, d, z);
}

void launch_last_layer(const double* post, int64_t n, int h, const double* theta_last,
                       TaylorDims td, const double* r0, const double* seeds,
                       const double* targets, double* r, double* u_out, cudaStream_t s,
                       const double* quad, double* seeds_out) {
  if (n <= 0) return;
  // enough blocks for ~4 per SM (a warp per row: short rows are latency-bound)
  const int64_t want = std::max<int64_t>(1, ceil_div(n, 148 * 4));
  const int spb = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(LAST_MAX_ROWS / td.S, 64), want));
  const int64_t blocks = ceil_div(n, spb);
  count_launch();
  k_last_layer<<<(unsigned)blocks, LAST_THREADS, 0, s>>>(post, n, h, theta_last, td, spb, r0,
                                                         seeds, targets, r, u_out, quad,
                                                         seeds_out);
}

// ---------------------------------------------------------------------------
// activation backward (taylor.py:206-239)

// One thread per (sample, unit) walks the sample's S rows (coalesced across the warp's units).
// Variants: PRE = stored pre-activation state (else layer 0: value z + W0^T rows);
// GIN = full upstream adjoint (else the rank-1 seed x w_last of the h_out = 1 layer).
// Derivative rows go in batches of 8 loads in flight (memory-level parallelism) through
// running row pointers, two CTAs of 256 per SM.
template <bool PRE, bool GIN>
__global__ void __launch_bounds__(256, 2) k_act_bwd(ActBwd a, int64_t n, int h, TaylorDims td,
                                                    const double* __restrict__ cdiag) {
  const int64_t total = n * h;
  const int d = td.d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t smp = e / h;
    const int j = (int)(e % h);
    const int64_t base = smp * td.S * h + j;
    const double z = PRE ? a.pre[base] : a.zval[e];
    const TanhD t = tanh_derivs(z, td.taylor);
    const double wl = GIN ? 0.0 : a.wlast[j];
    const double* sd = GIN ? nullptr : (a.seeds ? a.seeds + smp * td.S : nullptr);
    const double vb = GIN ? a.gin[base] : (sd ? sd[0] * wl : wl);
    double* go = a.gout + base;
    if (!td.taylor) {
      go[0] = t.s1 * vb;  // network.py:229-231
      continue;
    }
    const int64_t hl = h;
    const double lb = GIN ? a.gin[base + (int64_t)(d + 1) * hl] : (sd ? sd[d + 1] * wl : wl);
    const double ell = PRE ? a.pre[base + (int64_t)(d + 1) * hl] : 0.0;
    double quad = 0.0, ggb = 0.0;
    const double two_s2 = 2.0 * t.s2;
    const double* pg = PRE ? a.pre + base + hl : a.w0t + j;   // derivative row i = 1
    const double* pb = GIN ? a.gin + base + hl : nullptr;
    double* po = go + hl;
    auto row = [&](double g, double gb, int i, double* o) {
      const double cg = g * cdiag[i - 1];
      quad += cg * g;
      ggb += g * gb;
      *o = t.s1 * gb + two_s2 * cg * lb;
    };
    int i0 = 1;
    for (; i0 + 7 <= d; i0 += 8) {  // full batches: 8 loads in flight
      double gv[8], gbv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        gv[u] = pg[u * hl];
        gbv[u] = GIN ? pb[u * hl] : (sd ? sd[i0 + u] * wl : wl);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) row(gv[u], gbv[u], i0 + u, po + u * hl);
      pg += 8 * hl;
      if (GIN) pb += 8 * hl;
      po += 8 * hl;
    }
    for (; i0 <= d; ++i0) {
      row(*pg, GIN ? *pb : (sd ? sd[i0] * wl : wl), i0, po);
      pg += hl;
      if (GIN) pb += hl;
      po += hl;
    }
    go[(int64_t)(d + 1) * hl] = t.s1 * lb;
    go[0] = t.s1 * vb + t.s2 * ggb + t.s2 * ell * lb + t.s3 * quad * lb;
  }
}

void launch_act_bwd(const ActBwd& a, int64_t n, int h, TaylorDims td, const double* cdiag,
                    cudaStream_t s) {
  const int64_t total = n * h;
  if (total <= 0) return;
  count_launch();
  const unsigned g = grid_for(total, 256);
  if (a.pre && a.gin) k_act_bwd<true, true><<<g, 256, 0, s>>>(a, n, h, td, cdiag);
  else if (a.pre) k_act_bwd<true, false><<<g, 256, 0, s>>>(a, n, h, td, cdiag);
  else if (a.gin) k_act_bwd<false, true><<<g, 256, 0, s>>>(a, n, h, td, cdiag);
  else k_act_bwd<false, false><<<g, 256, 0, s>>>(a, n, h, td, cdiag);
}

// ---------------------------------------------------------------------------
// weighted value-row column sums: the bias row/column of the factors and of the
// gradient (the virtual "1" entry of zhat, curvature.py:88-93), two passes with a
// fixed summation order.

constexpr int COLSUM_GROUPS = 64;

__global__ void k_colsum_partial(const double* __restrict__ X, int64_t rs, int64_t n, int ncols,
                                 const double* __restrict__ w, double* __restrict__ part) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int sub = threadIdx.x >> 5;  // 8 row lanes per block
  const int g = blockIdx.y;
  __shared__ double red[8][33];
  double acc = 0.0;
  if (j < ncols) {
    const int64_t per = (n + COLSUM_GROUPS - 1) / COLSUM_GROUPS;
    const int64_t lo = g * per, hi = min(n, lo + per);
    for (int64_t r = lo + sub; r < hi; r += 8) {
      const double v = X[r * rs + j];
      acc += w ? w[r] * v : v;
    }
  }
  red[sub][threadIdx.x & 31] = acc;
  __syncthreads();
  if (sub == 0 && j < ncols) {
    double v = 0.0;
    for (int k = 0; k < 8; ++k) v += red[k][threadIdx.x & 31];
    part[(int64_t)g * ncols + j] = v;
  }
}

__global__ void k_colsum_reduce(const double* __restrict__ part, int ncols, double* out,
                                int64_t os, double add_count, int tr_h) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ncols) {
    double v = 0.0;
    for (int g = 0; g < COLSUM_GROUPS; ++g) v += part[(int64_t)g * ncols + j];
    // tr_h > 0: column jj = i * tr_h + u lands at out[u * os + i] (transposed block)
    const int64_t o = tr_h > 0 ? (int64_t)(j % tr_h) * os + j / tr_h : (int64_t)j * os;
    out[o] += v;
  }
  if (j == 0 && add_count != 0.0) out[(int64_t)ncols * os] += add_count;
}

void launch_colsum(const double* X, int64_t rs, int64_t n, int ncols, const double* w, double* out,
                   int64_t os, double add_count, double* scratch, cudaStream_t s, int tr_h) {
  if (n <= 0 || ncols <= 0) return;
  count_launch();
  k_colsum_partial<<<dim3((unsigned)ceil_div(ncols, 32), COLSUM_GROUPS), 256, 0, s>>>(X, rs, n, ncols,
                                                                                    w, scratch);
  count_launch();
  k_colsum_reduce<<<(unsigned)ceil_div(ncols, 128), 128, 0, s>>>(scratch, ncols, out, os, add_count,
                                                                  tr_h);
}

// ---------------------------------------------------------------------------
// Jacobian-vector products for the exact Gramian-vector product of KFAC*
// (reference src/curvature.py:169-194,253-260 without materialising the rows):
// jv_n += sum_{s} <gbar_{n,s}, y_{n,s}> with y = V zhat (one warp per sample).

__global__ void k_rowdot_accum(const double* __restrict__ G, const double* __restrict__ Y, int q,
                               int64_t n, int S, double* __restrict__ jv) {
  const int lane = threadIdx.x & 31;
  const int64_t smp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (smp >= n) return;
  const int64_t len = (int64_t)S * q;
  const double* g = G + smp * len;
  const double* y = Y + smp * len;
  double acc = 0.0;
  for (int64_t e = lane; e < len; e += 32) acc = fma(g[e], y[e], acc);
  acc = warp_sum(acc);
  if (lane == 0) jv[smp] += acc;
}

void launch_rowdot_accum(const double* G, const double* Y, int q, int64_t n, int S, double* jv,
                         cudaStream_t s) {
  if (n <= 0) return;
  count_launch();
  k_rowdot_accum<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(G, Y, q, n, S, jv);
}

// Output layer with h_out = 1 (q = 1): jv[n] += sum_s G[n,s] (z_{n,s} . v + (s == 0) b) in one
// read of the last hidden state (warp per sample, the K/32 entries of v in registers, one
// reduction per sample) instead of an (n S x 1) GEMM output plus a row-dot pass.
constexpr int JVP_LAST_MAXK = 1024;
__global__ void __launch_bounds__(256) k_jvp_last(const double* __restrict__ G,
                                                  const double* __restrict__ Z, int64_t ldz, int K,
                                                  const double* __restrict__ v, const double* __restrict__ b,
                                                  int64_t n, int S, double* __restrict__ jv) {
  const int lane = threadIdx.x & 31;
  const int64_t smp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (smp >= n) return;
  constexpr int U = JVP_LAST_MAXK / 32;
  double vr[U];
#pragma unroll
  for (int u = 0; u < U; ++u) vr[u] = (lane + 32 * u < K) ? v[lane + 32 * u] : 0.0;
  const double* g = G + smp * S;
  double acc = 0.0;
  for (int s = 0; s < S; ++s) {
    const double* z = Z + (smp * S + s) * ldz;
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (lane + 32 * u < K) t = fma(z[lane + 32 * u], vr[u], t);
    acc = fma(g[s], t, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) jv[smp] += fma(g[0], b[0], acc);
}

bool launch_jvp_last(const double* G, const double* Z, int64_t ldz, int K, const double* v,
                     const double* b, int64_t n, int S, double* jv, cudaStream_t s) {
  if (K > JVP_LAST_MAXK) return false;
  if (n <= 0) return true;
  count_launch();
  k_jvp_last<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(G, Z, ldz, K, v, b, n, S, jv);
  return true;
}

// Layer 0: zhat rows are [x; 1] (value), [e_i; 0] (derivatives), 0 (operator), so
// y_value = V0[:, :d] x + V0[:, d] (y0val, from a GEMM) and y_i = V0[:, i].
__global__ void k_jvp_layer0(const double* __restrict__ G, const double* __restrict__ y0val,
                             const double* __restrict__ v0t, int64_t n, int d, int h1,
                             double* __restrict__ jv) {
  const int lane = threadIdx.x & 31;
  const int64_t smp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (smp >= n) return;
  const int S = d + 2;
  const double* g = G + smp * S * h1;
  double acc = 0.0;
  for (int j = lane; j < h1; j += 32) acc = fma(g[j], y0val[smp * h1 + j], acc);
  for (int64_t e = lane; e < (int64_t)d * h1; e += 32) acc = fma(g[h1 + e], v0t[e], acc);
  acc = warp_sum(acc);
  if (lane == 0) jv[smp] += acc;
}

void launch_jvp_layer0(const double* G, const double* y0val, const double* v0t, int64_t n, int d,
                       int h1, double* jv, cudaStream_t s) {
  if (n <= 0) return;
  count_launch();
  k_jvp_layer0<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(G, y0val, v0t, n, d, h1, jv);
}

// ---------------------------------------------------------------------------
// small utilities

__global__ void k_sumsq(const double* __restrict__ v, int64_t n, int64_t stride,
                        double* __restrict__ out, int64_t out_stride) {
  __shared__ double red[512];
  const double* x = v + (int64_t)blockIdx.x * stride;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = fma(x[i], x[i], acc);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[(int64_t)blockIdx.x * out_stride] = red[0];
}

void launch_sumsq(const double* v, int64_t n, int64_t stride, int nvec, double* out,
                  int64_t out_stride, cudaStream_t s) {
  if (nvec <= 0) return;
  count_launch();
  k_sumsq<<<nvec, 512, 0, s>>>(v, n, stride, out, out_stride);
}

__global__ void k_transpose(const double* __restrict__ src, int64_t lds, int rows, int cols,
                            double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = by + k, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[(int64_t)r * lds + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = bx + k, r = by + threadIdx.x;
    if (r < rows && c < cols) dst[(int64_t)c * rows + r] = tile[threadIdx.x][k];
  }
}

// dst (cols x rows, row-major) = src(rows x cols, pitch lds)^T
void launch_transpose(const double* src, int64_t lds, int rows, int cols, double* dst,
                      cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  count_launch();
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(src, lds, rows, cols, dst);
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = v;
}

void launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n <= 0) return;
  count_launch();
  k_fill<<<grid_for(n, 256), 256, 0, s>>>(p, n, v);
}

}  // namespace kp
