// Internal launcher interfaces shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kp {

// Interior residual of one point from its output triple u[0..S) (S = d + 2):
// r = r0 + seeds . u + sum_i quad_i u_{1+i}^2; optional effective seeds (reverse pass).
__host__ __device__ inline double point_residual(const double* u, int S, double r0,
                                                  const double* seeds, const double* quad,
                                                  double* seeds_out) {
  double v = r0;
  for (int s = 0; s < S; ++s) v += seeds[s] * u[s];
  if (quad) {
    for (int i = 0; i < S - 2; ++i) v += quad[i] * u[1 + i] * u[1 + i];
  }
  if (seeds_out) {
    for (int s = 0; s < S; ++s)
      seeds_out[s] = seeds[s] + ((quad && s >= 1 && s <= S - 2) ? 2.0 * quad[s - 1] * u[s] : 0.0);
  }
  return v;
}

// Host-side count of this library's kernel launches (reported as gpu_launches).
void count_launch();
int64_t launch_count();

// ---- FP64 DMMA GEMMs (kp_gemm.cu) -----------------------------------------

// C[M,N] = A[M,K] * B[N,K]^T  (+ bias[n * bias_stride] on rows m with m % S == 0).
struct GemmNT {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int64_t M;
  int N;
  int K;
  const double* bias;
  int64_t bias_stride;
  int S;
  // optional batch (grid.y): operand / output / bias offsets per batch entry
  int batch = 1;
  int64_t sA = 0, sB = 0, sC = 0, sBias = 0;
};
void launch_gemm_nt(const GemmNT& g, cudaStream_t s);
// TMA-fed variant (kp_gemm_tma.cu); returns false when the operands do not meet
// its alignment/shape requirements (the caller then uses the cp.async kernel).
bool launch_gemm_nt_tma(const GemmNT& g, cudaStream_t s, int variant = 0);
// cp.async variant only (the fallback).
void launch_gemm_nt_cpasync(const GemmNT& g, cudaStream_t s);

// Row reduction C[p,q] = sum_r Xh[r,p] * w(r) * Yh[r,q] over rows [0,R), split into
// `splits` row ranges whose partial tiles go to partial[split][P][Q]; then
// acc[p][q] += sum_split partial (fixed order -> deterministic).
// Xh = [X | bias] where the virtual bias column (index nx) is 1 on rows r % S == 0.
// w(r) = w[r / Sw] when w != nullptr.  sym: X == Y, only lower-triangle tiles are
// computed and acc holds a valid lower triangle.
struct GemmTN {
  const double* X;
  int64_t ldx;
  int nx;
  bool x_bias;
  const double* Y;
  int64_t ldy;
  int ny;
  bool y_bias;
  const double* w;
  int Sw;
  int S;  // bias-row period
  int64_t R;
  bool sym;
};
size_t gemm_tn_partial_doubles(int64_t R, int P, int Q, bool sym);
void launch_gemm_tn_accumulate(const GemmTN& g, double* partial, double* acc, cudaStream_t s);
// All of a pass's small contractions in one launch (+ one reduce): acc[j] += job j's
// P x Q result (P = nx + x_bias, Q = ny + y_bias).  Returns false if the partial space
// (gemm_tn_grouped_partial_doubles) or the job-table size (40) is exceeded.
size_t gemm_tn_grouped_partial_doubles(const GemmTN* jobs, int n);
bool launch_gemm_tn_grouped(const GemmTN* jobs, double* const* accs, int n, double* partial,
                            size_t partial_cap, cudaStream_t s);

// TMA-fed split-row reduction without bias columns (kp_gemm_tn_tma.cu):
// acc[p*ldacc + q] += sum_r X[r,p] w(r) Y[r,q], p < nx, q < ny; w(r) = w[r / Sw].
// Returns false when the operands are not TMA-compatible.
size_t gemm_tn_tma_partial_doubles(int64_t R, int nx, int ny, bool sym);
bool gemm_tn_tma_ok(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t R);
bool launch_gemm_tn_tma_accumulate(const double* X, int64_t ldx, int nx, const double* Y,
                                   int64_t ldy, int ny, const double* w, int Sw, int64_t R,
                                   bool sym, double* partial, double* acc, int64_t ldacc,
                                   cudaStream_t s);

// ---- fused Taylor layer: GEMM + bias + activation (kp_gemm_act.cu) ----------
struct TaylorDims;
enum ActMode { ACT_STORE = 0, ACT_LOSS = 1, ACT_LAST = 2 };
struct GemmAct {
  const double* A;  // (n_samples*S) x K layer input
  int64_t lda;
  const double* B;  // N x K weights (pitch ldb)
  int64_t ldb;
  const double* bias;
  int64_t bias_stride;
  int64_t n_samples;
  int S, d;
  bool taylor;
  int N, K;
  const double* cdiag;
  double* pre;    // ACT_STORE: pre-activation out
  double* post;   // ACT_STORE / ACT_LOSS: activation out
  int64_t ldo;
  const double* wlast;  // ACT_LAST: last-layer weight row (length N)
  double* upart;        // ACT_LAST: (n_samples*S) x ceil(N/128) partial dots
  int nb;               // set by the launcher
  // candidate batch (grid.y): A is the stack of `batch` (n_samples*S) x K states, B the
  // stack of `batch` N x K weight blocks (row-contiguous), outputs/bias offset per entry
  int batch = 1;
  int64_t bias_bstride = 0, out_bstride = 0, upart_bstride = 0, wlast_bstride = 0;
};
// Whether launch_gemm_act can run this layer shape (fused path available).
bool gemm_act_ok(int S, int K, int64_t lda, int64_t ldb);
int gemm_act_samples_per_tile(int S, int K);
int gemm_act_tile_width(int S, int N, int K);
bool launch_gemm_act(GemmAct g, int mode, cudaStream_t s);

// ---- Taylor-mode elementwise kernels (kp_taylor.cu) ------------------------

// out[j*os] += sum_{n} w_n X[n*rs + j] for j < ncols (w == nullptr: 1);
// out[ncols*os] += add_count.  scratch: 64 * ncols doubles.
void launch_colsum(const double* X, int64_t rs, int64_t n, int ncols, const double* w, double* out,
                   int64_t os, double add_count, double* scratch, cudaStream_t s, int tr_h = 0);

struct TaylorDims {
  int S;       // rows per sample: d + 2 (Taylor) or 1 (plain)
  int d;       // derivative rows (0 for plain)
  bool taylor; // operator row present
};

// Layer 0 fused with its activation: pre-activation value z = x W0^T + b0 -> zval,
// post-activation state (n*S x h1) -> post.  Derivative rows of the pre-activation
// are W0[:, i] and its operator row is 0 (reference taylor.py:124-131).
// batch > 1: parameter sets theta0 + kk*D; zval/post/w0t/q0 stacked per entry.
// post == nullptr: zval only.
void launch_first_layer(const double* x, int64_t n, int d, const double* theta0, int h1,
                        TaylorDims td, const double* w0t, const double* q0, double* zval,
                        double* post, cudaStream_t s, int batch = 1, int64_t D = 0);
// Per parameter set: w0t = W0^T (d x h1), q0[j] = sum_i (W0[j,i] c_i) W0[j,i].
// rot (d x d, or NULL): derivative directions Q[:, k] instead of e_k (dense coefficients).
void launch_prep_layer0(const double* theta0, int d, int h1, const double* cdiag, const double* rot,
                        double* w0t,
                        double* q0, cudaStream_t s, int batch = 1, int64_t D = 0);
// Taylor activation (taylor.py:151-169): pre (n*S x h) -> post.
void launch_act_fwd(const double* pre, double* post, int64_t n, int h, TaylorDims td,
                    const double* cdiag, cudaStream_t s);
// Scalar output + residual: u_{n,s} = post[n*S+s,:] . w + (s==0) b;
// taylor: r_n = r0_n + sum_s seeds[n,s] u_{n,s};  plain: r_n = u_n - target_n.
// quad (n x d, optional): residual += sum_i quad_i u_i^2; seeds_out (n x S, optional): the
// reverse-pass seeds at these outputs, seeds + [0, 2 quad_i u_i, 0].
void launch_last_layer(const double* post, int64_t n, int h, const double* theta_last,
                       TaylorDims td, const double* r0, const double* seeds,
                       const double* targets, double* r, double* u_out, cudaStream_t s,
                       const double* quad = nullptr, double* seeds_out = nullptr);
// Adjoint of the Taylor activation (taylor.py:206-239).  Pre-activation either a
// stored state `pre` or (layer 0) zval + W0.  gin either a stored adjoint or the
// rank-1 seeds (x) w_last (first reverse step, taylor.py:262,271).
struct ActBwd {
  const double* pre;      // n*S x h (nullptr -> use zval/theta0)
  const double* zval;     // n x h   (layer-0 pre-activation value rows)
  const double* w0t;      // d x h   (layer-0 derivative rows, W0^T)
  const double* gin;      // n*S x h (nullptr -> rank-1)
  const double* seeds;    // n*S (rank-1; nullptr -> ones)
  const double* wlast;    // h (rank-1)
  double* gout;           // n*S x h
};
void launch_act_bwd(const ActBwd& a, int64_t n, int h, TaylorDims td, const double* cdiag,
                    cudaStream_t s);
// Scalar output from ACT_LAST partials + residual (same semantics as launch_last_layer).
void launch_last_from_partials(const double* upart, int ntn, int64_t n, TaylorDims td,
                               const double* bias, const double* r0, const double* seeds,
                               const double* targets, double* r, cudaStream_t s, int batch = 1,
                               int64_t bias_bstride = 0, int64_t r_bstride = 0,
                               const double* quad = nullptr);
// Batched deterministic sum of squares: out[k] = sum_i v[k*stride + i]^2, i < n.
void launch_sumsq(const double* v, int64_t n, int64_t stride, int nvec, double* out,
                  int64_t out_stride, cudaStream_t s);
void launch_transpose(const double* src, int64_t lds, int rows, int cols, double* dst,
                      cudaStream_t s);
void launch_fill(double* p, int64_t n, double v, cudaStream_t s);
// u (n x S) -> value (n), grad (n x d), op (n)
// Rows of X (n rows of pitch `stride`, d entries each) replaced in place by Q^T x
// (transpose = 1) or Q x (transpose = 0).
void launch_rotate_rows(double* X, int64_t stride, int64_t n, int d, const double* Q, int transpose,
                        cudaStream_t s);
// out[j * ldo + i] += sum_k T[j * d + k] Q[i * d + k]   (q x d times Q^T)
void launch_rot_accum(const double* T, int q, int d, const double* Q, double* out, int64_t ldo,
                      cudaStream_t s);
void launch_split_u(const double* u, int64_t n, int d, double* value, double* grad, double* op,
                    cudaStream_t s);
// initial_state (taylor.py:124-131): z (n*S x d) = [x; I; 0]
void launch_initial_state(const double* x, int64_t n, int d, double* z, cudaStream_t s);

// ---- optimizer bookkeeping (kp_optim.cu) ------------------------------------
struct FinalizeJob {
  const double* acc;
  double* F;
  int n;
  double scale;
  int diag_n;
  double diag_add;
};
struct FinalizeJobs {
  int n;
  FinalizeJob job[64];
  int64_t ebegin[65];
};
// EMA update of every factor of a step in one launch.
void launch_factor_finalize_grouped(FinalizeJobs& J, double ema, cudaStream_t s);
void launch_grad_finalize(const double* gi, const double* gb, double ni, double nb,
                          double* grad, int64_t D, cudaStream_t s);
void launch_axpy_out(const double* x, const double* y, double a, double* out, int64_t n,
                     cudaStream_t s);  // out = x + a*y
void launch_losses(const double* sums, double ni, double nb, double* scalars, cudaStream_t s);
// Layer geometry for packing [W|b] rows (pitch h+1) into W rows (pitch h).
struct WPack {
  int L;
  int h[17];
  int64_t th[16];  // offset of layer l in theta
  int64_t wo[16];  // offset of layer l's block in the padded copy
  int64_t ws[16];  // stride between batch entries inside layer l's block (q_l * h_l)
};
// For kk < batch: out[kk] = theta + 2^(exp2 + kk) dir (dir == nullptr: copy theta);
// wpad (optional): padded W copies, entry kk of layer l at wo[l] + kk * ws[l].
void launch_candidate(const double* theta, const double* dir, int exp2, double* out, int64_t D,
                      const WPack& wp, double* wpad, cudaStream_t s, int batch = 1);
void launch_argmin_update(const double* ls_sums, int ncand, int min_exp, double ni, double nb,
                          double* theta, double* prev, const double* dir, int64_t D,
                          double* scalars, double* ls_losses, int32_t* status, double mu,
                          cudaStream_t s);
void launch_damped_copy(const double* F, double lam, int n, double* out, cudaStream_t s);
void launch_eig_status(const double* la, int p, const double* lb, int q, const int* info,
                       int32_t* status, cudaStream_t s);
void launch_kron_scale(double* W, const double* la, int p, const double* lb, int q,
                       cudaStream_t s);
void launch_set_status(int32_t* status, int32_t code, cudaStream_t s);
void launch_warm_identity(double* T, int n, const int* valid, cudaStream_t s);
void launch_merge_chol_info(const int* chol_info, int* info, int n, cudaStream_t s);
void launch_status_slots(const int32_t* status, double* slots, cudaStream_t s);
void launch_slots_status(const double* slots, int32_t* status, cudaStream_t s);
// KFAC*: batched deterministic dot products, quadratic-model solve and update
struct DotJobs {
  const double* a[8];
  const double* b[8];
};
void launch_dots(const DotJobs& jobs, int n, int64_t D, double* out, cudaStream_t s);
void launch_star_solve_update(const double* dots, double lam, double* theta, double* prev,
                              const double* delta, int64_t D, double* scalars, int32_t* status,
                              cudaStream_t s);
// jv[n] += sum over the sample's S rows of <G_row, Y_row> (both pitch q)
void launch_rowdot_accum(const double* G, const double* Y, int q, int64_t n, int S, double* jv,
                         cudaStream_t s);
// layer-0 Jacobian-vector product (value rows from y0val, derivative rows from V0^T)
bool launch_jvp_last(const double* G, const double* Z, int64_t ldz, int K, const double* v,
                     const double* b, int64_t n, int S, double* jv, cudaStream_t s);
void launch_jvp_layer0(const double* G, const double* y0val, const double* v0t, int64_t n, int d,
                       int h1, double* jv, cudaStream_t s);
void launch_gen_eig_1x1(const double* f1, const double* f2, double lam, double* t, double* eig,
                        int* info, cudaStream_t s);
void launch_identity(double* F, int n, double v, cudaStream_t s);

// ---- dense row-major FP64 linear algebra without library calls (kp_dense.cu) ----
// C (M x N) = alpha op(A) op(B) + beta C; op(A) M x K (A stored K x M when ta), op(B) K x N
// (B stored N x K when tb).  lower_only: tiles strictly above the diagonal are skipped.
struct DenseGemm {
  int M, N, K;
  const double* A;
  int64_t lda;
  bool ta;
  const double* B;
  int64_t ldb;
  bool tb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  bool lower_only;
};
void launch_dense_gemm(const DenseGemm& g, cudaStream_t s);
// In-place lower Cholesky A = L L^T (row-major; the strict upper triangle is overwritten
// with scratch values).  info: 0 or the 1-based index of the first non-positive pivot.
void launch_cholesky(int n, double* A, int64_t lda, int* info, cudaStream_t s);
// X = L^-1 B (lower triangular L; X holds B on entry, or b_identity: B = I).
void launch_trsm_lower(int n, const double* L, int64_t ldl, double* X, int64_t ldx, int m,
                       bool b_identity, cudaStream_t s);
void launch_copy_matrix(const double* src, int64_t lds, int rows, int cols, double* dst,
                        int64_t ldd, cudaStream_t s);
void launch_zero_upper(int n, double* A, int64_t lda, cudaStream_t s);

// ---- FP64 GEMM on the INT8 tensor cores, Ozaki scheme (kp_ozaki.cu; KP_OZAKI=1) ------
bool ozaki_enabled();
int ozaki_slices();
bool ozaki_gemm_ok(int64_t M, int N, int K, int64_t lda, int64_t ldb);
bool launch_ozaki_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                       int64_t ldc, int64_t M, int N, int K, const double* bias,
                       int64_t bias_stride, int rows_per_sample, int8_t* a_planes, int* a_ex,
                       int8_t* b_planes, int* b_ex, cudaStream_t s);

// ---- fused Taylor layer, FP64 product on the INT8 tensor cores by the CRT (kp_crt.cu; KP_CRT=0 disables)
bool crt_enabled();
int crt_moduli();
bool crt_first_enabled();
bool crt_act_ok(int S, int K, int N);
void launch_crt_slice(const double* X, int64_t rows, int K, int64_t ldx, int8_t* planes, int* ex,
                      bool weights, cudaStream_t s);
bool launch_crt_first(const double* zval, int64_t n, int h1, int S, int d, const double* w0t,
                      const double* q0, int8_t* planes, int* ex, cudaStream_t s);
bool launch_crt_act(const GemmAct& g, int mode, const int8_t* resH, const int* exH,
                    const int8_t* resW, const int* exW, cudaStream_t s,
                    int* tile_counter = nullptr);

// ---- small on-device generalised eigensolver + combine (kp_eig_small.cu) ---------
struct SmallEigJob {
  int n;
  const double* f1;  // first factor (M1 = f1 + damping I)
  const double* f2;  // second factor (M2 = f2 + damping I, Cholesky'd)
  double damping;
  double* t;         // n x n row-major, column k = generalised eigenvector k
  double* lam;       // n eigenvalues
  int* info;
  int col_major = 0;  // 1: write t column-major (= T^T row-major, for the DMMA combine)
  // Warm start (optional): the previous step's T (n x n row-major) and a validity flag, kept
  // by the context across steps, plus n x n global scratch.  With a valid T_prev the pair is
  // first congruence-transformed, (T_prev^T M1 T_prev, T_prev^T M2 T_prev), which the EMA
  // keeps close to (diag, I), so Jacobi needs far fewer sweeps; T = T_prev T''.
  double* warm_t = nullptr;
  double* warm_scratch = nullptr;
  int* warm_valid = nullptr;
};
struct SmallEigJobs {
  SmallEigJob job[32];
  double tol_floor = 1e-14;  // set by the launcher (jacobi_tol_floor)
};
// Floor of the Jacobi rotation threshold |cos| > max(floor, 2 n eps) of every device
// eigensolver: 1e-14, or KP_JACOBI_TOL (measurements of the accuracy / sweep trade-off).
double jacobi_tol_floor();
struct SmallCombineJob {
  int p, q;
  const double* g;   // q x p gradient
  const double* ta;  // p x p
  const double* tb;  // q x q
  const double* la;
  const double* lb;
  double* t1;        // q x p scratch
  double* t2;        // q x p scratch
  double* out;       // q x p
  double sign;
};
struct SmallCombineJobs {
  SmallCombineJob job[16];
};
int small_eig_max_n();
// kp_eig_mid.cu: one-sided Jacobi in an 8-CTA cluster for small_eig_max_n() < n <= mid_eig_max_n()
int mid_eig_max_n();
int mid_eig_sweeps_used(bool reset = false);
int small_eig_sweeps_used(bool reset = false);
int mid_eig_cluster_size();  // 16, 8, or -1 when no cluster launch is possible
// Rows out of launch_eig_mid: U = R V (default; the caller forms T'^T = U^T K^-1) or,
// KP_MID_ACCV=1, the eigenvectors V accumulated in the kernel (T'^T = V^T L^-1)
bool mid_eig_accumulate_v();
void launch_eig_mid(int n, double* rv, double* lam, int* info, const int* chol_info,
                    cudaStream_t s, int* warm_valid = nullptr, long long* prof = nullptr);
// kp_eig_large.cu: one-sided Jacobi with the vectors in L2, one 16-CTA cluster per pair, for
// mid_eig_max_n() < n <= large_eig_max_n(); U (n x n row-major, even pitch ld): the rows of L_C in,
// orthogonalised rows out; V (n x n): the eigenvectors of C as rows
int large_eig_max_n();
int large_eig_accv_max_n();  // widest pair the V-accumulating variant handles
// T^T = U^T K^-1 from the orthogonalised rows U (default), or KP_LARGE_ACCV=1: V accumulated
// in the kernel and T^T = V^T L^-1
bool large_eig_accumulate_v();
int large_eig_sweeps_used(bool reset = false);
// gtail (optional, U-only): 16 (2 ceil(ceil(n/2)/16) + 4) (n - 512) doubles of scratch for
// the split-record kernel (544 < n <= 800: record heads in smem, tails in L2)
void launch_eig_large(int n, int ld, double* U, double* V, double* lam, int* info,
                      const int* chol_info, cudaStream_t s, int* warm_valid = nullptr,
                      double* gtail = nullptr);
size_t small_eig_smem_bytes(int n);
void launch_gen_eig_small(const SmallEigJobs& jobs, int njobs, int max_n, int32_t* status,
                          cudaStream_t s);
void launch_kron_combine_small(const SmallCombineJobs& jobs, int njobs, cudaStream_t s);

}  // namespace kp
