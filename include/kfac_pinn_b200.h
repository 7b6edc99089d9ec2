/*
 * kfac_pinn_b200.h — C ABI of the B200-native KFAC step for PINN losses.
 *
 * Drop-in boundary for the reference's KFAC optimizer path
 * (/root/reference/pkg/src/pinnopt, "src/" below).  The reference is pure
 * Python/NumPy; its "FFI" for this path is the Python call surface
 *
 *   OptimizerConfig(kind="kfac", ...)          src/optim.py:41-78
 *   init_train_state(params, config)           src/optim.py:102-117
 *   optimizer_step(state, batch, problem)      src/optim.py:396-402
 *     -> kfac_step                             src/optim.py:251-263
 *
 * and this header is what a binding of that path binds (ctypes stub in
 * INTEGRATION.md; the Python mirror in paper_2405_15603_b200/ uses it).
 * Everything is float64.  All pointers in kp_state / kp_batch / kp_step_out
 * are DEVICE pointers owned by the caller; kernels never allocate.  Scratch
 * comes from one caller-owned device workspace sized by kp_workspace_bytes().
 * Every entry point returns a kp_status; device-side failures (not-PD factor,
 * failed line search, non-finite parameters) are written to *out->status and
 * must be read after the stream completes.
 *
 * Layouts (reference conventions, src/taylor.py:3-16, src/network.py:7-13):
 *   theta / prev_update / grad / delta : per linear layer l the augmented
 *       matrix [W_l | b_l] (q_l x p_l, q_l = h_{l+1}, p_l = h_l + 1) stored
 *       ROW-major, layers concatenated (D = sum q_l p_l doubles).
 *   factors a_* : per layer p_l x p_l, b_* : q_l x q_l, row-major, concatenated.
 *   x_int : N x d, seeds : N x (d+2) ([dr/du, dr/dgrad, dr/dLu] per point),
 *   r0 : N (residual at zero network output), x_bnd : Nb x d, targets : Nb.
 */
#ifndef KFAC_PINN_B200_H
#define KFAC_PINN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_MAX_LAYERS 16
#define KP_ABI_VERSION 5

typedef enum kp_status {
  KP_OK = 0,
  KP_ERR_INVALID = 1,       /* ValueError: shapes, damping <= 0 (src/optim.py:61-75, src/curvature.py:147-149) */
  KP_ERR_NOT_PSD = 2,       /* NotPositiveSemidefiniteError (src/linalg.py:39-44,79-83,128-132) */
  KP_ERR_LINE_SEARCH = 3,   /* LineSearchError (src/optim.py:37-38,209-210) */
  KP_ERR_NONFINITE = 4,     /* FloatingPointError (src/optim.py:398-401) */
  KP_ERR_CUDA = 5,          /* CUDA failure */
  KP_ERR_EIG = 6,           /* numpy.linalg.LinAlgError: eigensolver did not converge */
  KP_ERR_WORKSPACE = 7      /* workspace too small */
} kp_status;

/* MLP shape: n_layers linear layers, widths[0] = d, widths[n_layers] = 1
 * (src/network.py:72-96). */
typedef struct kp_net {
  int32_t n_layers;
  int32_t widths[KP_MAX_LAYERS + 1];
} kp_net;

/* Per-rank problem size.  chunk = interior points per device pass (0 = all);
 * the interior batch is streamed through the Taylor engine in chunks so
 * N = 65536 at d = 100 fits in HBM (all reductions are sums over points). */
typedef struct kp_problem {
  kp_net net;
  int64_t n_interior;
  int64_t n_boundary;
  int64_t chunk;
  int32_t n_candidates;      /* line_search_max_exp - line_search_min_exp + 1 */
  int32_t pad_;
} kp_problem;

/* OptimizerConfig(kind="kfac") fields that reach the device (src/optim.py:41-56).
 * n_*_global are the normalisers N_Omega / N_boundary of the whole batch
 * (equal to the local sizes on one GPU; the global sizes when sharded). */
typedef struct kp_kfac_config {
  double ema;
  double damping;
  double momentum;
  int32_t ls_min_exp;
  int32_t ls_max_exp;
  double n_interior_global;
  double n_boundary_global;
  /* KFAC* only: the damping of the 2x2 quadratic model, OptimizerConfig.damping
   * (src/optim.py:303), while the factor damping above is KfacState.damping
   * (src/curvature.py:150-152).  Equal unless the caller edits one of them; <= 0: use
   * damping. */
  double model_damping;
} kp_kfac_config;

/* Persistent optimizer state (TrainState/KfacState, src/optim.py:81-92,
 * src/curvature.py:43-59), device-resident, caller-owned. */
typedef struct kp_state {
  double* theta;
  double* prev_update;
  double* a_int;
  double* b_int;
  double* a_bnd;
  double* b_bnd;
} kp_state;

/* One collocation batch (src/pde.py:54-60) plus the residual terms.  The interior
 * residual is r = r0 + seeds . [u, grad u, Lu] + sum_i quad_i (d u/d x_i)^2 per point
 * (quad = NULL: affine).  Its reverse-pass seeds [dr/du, dr/dgrad, dr/dLu]
 * (src/optim.py:157-158) are seeds + [0, 2 quad_i grad_i u, 0] at the current outputs —
 * this covers every catalog residual including log-Fokker-Planck (src/pde.py:253-263). */
typedef struct kp_batch {
  const double* x_int;
  const double* r0;
  const double* seeds;
  const double* x_bnd;
  const double* targets;
  const double* coeff_diag;  /* d: diagonal operator coefficients (src/taylor.py:43-87), or
                                the eigenvalues lambda of a dense c (see coeff_rot) */
  const double* quad;        /* N x d quadratic gradient coefficients, or NULL */
  const double* coeff_rot;   /* NULL (c diagonal), or the d x d row-major orthogonal Q of
                                c = Q diag(lambda) Q^T (src/taylor.py:72-75).  The engine then
                                propagates derivatives along the columns of Q; seeds stay in
                                the coordinate basis.  Not combinable with quad. */
} kp_batch;

/* Step outputs (device).  scalars[4] = {loss_interior, loss_boundary, alpha, mu}
 * = StepInfo (src/optim.py:217-226).  Optional arrays may be NULL. */
typedef struct kp_step_out {
  double* scalars;
  int32_t* status;
  double* ls_losses;   /* 2 * n_candidates: (interior, boundary) loss per grid point */
  double* grad;        /* D: grad_mats of evaluate_batch (src/optim.py:164-177) */
  double* delta;       /* D: preconditioned gradient (src/curvature.py:140-163) */
} kp_step_out;

typedef struct kp_context kp_context;

/* Library / context. */
int32_t kp_abi_version(void);
const char* kp_status_string(int32_t status);
int32_t kp_context_create(int32_t device, kp_context** ctx);
int32_t kp_context_destroy(kp_context* ctx);
/* Optional kernel timing (CUDA events around the hidden-layer forward GEMMs). */
int32_t kp_profile_enable(kp_context* ctx, int32_t enable);
int32_t kp_profile_read(kp_context* ctx, double* gemm_ms, double* gemm_flops, int64_t* launches,
                        int64_t* kernel_launches);
/* The same for the HBM-bound activation adjoint (k_act_bwd, src/taylor.py:206-239): summed
 * CUDA-event time, algorithmic DRAM bytes and launches since kp_profile_enable. */
int32_t kp_profile_read_hbm(kp_context* ctx, double* ms, double* bytes, int64_t* launches);
/* Further timed categories since kp_profile_enable.  cat 0: the line search's hidden layers on
 * the INT8 tensor cores (the CRT fused layer, src/taylor.py:134-169 inside
 * src/optim.py:195-211), work = FP64-equivalent flops 2 rows K N; cat 1: the residue slicing
 * that feeds them, work = algorithmic DRAM bytes (8 B read + one byte per modulus written per
 * state element). */
int32_t kp_profile_read_cat(kp_context* ctx, int32_t cat, double* ms, double* work,
                            int64_t* launches);
/* Diagnostics: the most Jacobi sweeps any solve of each device eigensolver route used in this
 * process since the last reset (small: one CTA, mid: cluster shared memory, large:
 * L2-resident cluster); 1000 + s marks a solve that did not converge in s sweeps.  Call after
 * the stream has completed; reset != 0 zeroes the counters. */
int32_t kp_solver_sweeps(int32_t* small_max, int32_t* mid_max, int32_t* large_max,
                         int32_t reset);

/* Sizes. */
int64_t kp_param_count(const kp_net* net);              /* D */
int64_t kp_factor_count(const kp_net* net, int32_t which); /* 0: sum p_l^2, 1: sum q_l^2 */
int32_t kp_workspace_bytes(kp_context* ctx, const kp_problem* prob, size_t* bytes);
/* Bytes of workspace per interior point (used by hosts to pick `chunk`). */
int32_t kp_bytes_per_interior_point(const kp_net* net, size_t* bytes);

/* init_kfac_state (src/curvature.py:62-76): identity (init_mode=1) or zero (0)
 * factors, zero prev_update. */
int32_t kp_init_state(kp_context* ctx, const kp_net* net, kp_state* st, int32_t init_identity,
                      void* stream);

/* Whole KFAC step on one device: kfac_step (src/optim.py:251-263) followed by
 * the non-finite parameter check of optimizer_step (src/optim.py:398-401). */
int32_t kp_kfac_step(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                     kp_state* st, const kp_batch* batch, kp_step_out* out, void* workspace,
                     size_t workspace_bytes, void* stream);

/* The same step split at its two data-parallel exchange points, for sharded
 * multi-GPU use.  After phase 1 the caller all-reduces (sums)
 * the contiguous buffer returned by kp_reduce_buffer; after phase 3 the one
 * returned by kp_linesearch_buffer.  kp_kfac_step == phases 1-4 back to back. */
int32_t kp_reduce_buffer(kp_context* ctx, const kp_problem* prob, void* workspace, double** ptr,
                         int64_t* count);
int32_t kp_linesearch_buffer(kp_context* ctx, const kp_problem* prob, void* workspace,
                             double** ptr, int64_t* count);
int32_t kp_kfac_phase_accumulate(kp_context* ctx, const kp_problem* prob,
                                 const kp_kfac_config* cfg, kp_state* st, const kp_batch* batch,
                                 kp_step_out* out, void* workspace, size_t workspace_bytes,
                                 void* stream);
int32_t kp_kfac_phase_precondition(kp_context* ctx, const kp_problem* prob,
                                   const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                   void* workspace, size_t workspace_bytes, void* stream);
int32_t kp_kfac_phase_linesearch(kp_context* ctx, const kp_problem* prob,
                                 const kp_kfac_config* cfg, kp_state* st, const kp_batch* batch,
                                 kp_step_out* out, void* workspace, size_t workspace_bytes,
                                 void* stream);
int32_t kp_kfac_phase_update(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                             kp_state* st, kp_step_out* out, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Distributed Kronecker solves.  The precondition phase split in
 * two around a third exchange: kp_kfac_phase_precondition_owned normalises + EMAs every
 * factor and the gradient like kp_kfac_phase_precondition, but solves only the layers with
 * owned_layers[l] != 0 (host array, n_layers entries) and writes zeros to the other layers'
 * Delta rows.  The caller then sum-all-reduces the buffer of kp_direction_buffer
 * ([Delta (D) | 8 status slots]); with each layer owned by exactly one rank the sum is the
 * owner's Delta bit for bit.  kp_kfac_phase_direction merges the status slots (every rank
 * adopts the smallest failure code any rank saw) and forms delta^ = Delta + mu prev
 * (src/optim.py:254).  Replaces the solve loop of src/curvature.py:150-163. */
int32_t kp_direction_buffer(kp_context* ctx, const kp_problem* prob, void* workspace,
                            double** ptr, int64_t* count);
int32_t kp_kfac_phase_precondition_owned(kp_context* ctx, const kp_problem* prob,
                                         const kp_kfac_config* cfg, kp_state* st,
                                         kp_step_out* out, const int32_t* owned_layers,
                                         void* workspace, size_t workspace_bytes, void* stream);
int32_t kp_kfac_phase_direction(kp_context* ctx, const kp_problem* prob,
                                const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                void* workspace, size_t workspace_bytes, void* stream);

/* KFAC* step (src/optim.py:266-320): the same factors and preconditioned direction
 * Delta as kp_kfac_step, then the exact Gramian-vector products G Delta and G prev
 * (computed as Jacobian-vector products + a weighted reverse contraction — the N x D
 * residual-Jacobian rows of src/curvature.py:169-194 are never formed), the 2 x 2
 * quadratic model for (alpha, mu) (src/optim.py:266-286) and the update
 * theta += alpha Delta + mu prev.  out->scalars = {loss_int, loss_bnd, alpha, mu}.
 * Sharded use: phases accumulate, precondition, star_gvp, [all-reduce kp_gvp_buffer],
 * star_update. */
int32_t kp_kfac_star_step(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                          kp_state* st, const kp_batch* batch, kp_step_out* out, void* workspace,
                          size_t workspace_bytes, void* stream);
int32_t kp_gvp_buffer(kp_context* ctx, const kp_problem* prob, void* workspace, double** ptr,
                      int64_t* count);
int32_t kp_kfac_star_phase_gvp(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                               kp_state* st, const kp_batch* batch, kp_step_out* out,
                               void* workspace, size_t workspace_bytes, void* stream);
int32_t kp_kfac_star_phase_update(kp_context* ctx, const kp_problem* prob,
                                  const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* kp_kfac_step (star = 0) or kp_kfac_star_step (star = 1) replayed from a CUDA graph
 * captured on first use, when every layer's Kronecker solve runs on the device (factor
 * sizes <= 96, no host-blocking library call) and profiling is off; otherwise the same
 * as the plain call.  Intended for launch-bound small problems (BASELINE c1-c3). */
int32_t kp_kfac_step_graphed(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                             kp_state* st, const kp_batch* batch, kp_step_out* out,
                             void* workspace, size_t workspace_bytes, void* stream, int32_t star);

/* Forward-Laplacian forward (src/taylor.py:172-203) of the parameters `theta`
 * at the interior points of `batch`: writes u (N), grad u (N x d), L u (N).
 * Uses prob->n_interior / chunk; boundary fields of prob/batch are ignored. */
int32_t kp_taylor_forward(kp_context* ctx, const kp_problem* prob, const double* theta,
                          const kp_batch* batch, double* value, double* gradient,
                          double* op, void* workspace, size_t workspace_bytes, void* stream);

/* Plain MLP forward u(x) (src/network.py:200-213) at prob->n_boundary points x
 * (n x d) — the evaluation pass of eval_l2 (src/harness.py:155-166). */
int32_t kp_mlp_forward(kp_context* ctx, const kp_problem* prob, const double* theta,
                       const double* x, double* u, void* workspace, size_t workspace_bytes,
                       void* stream);

/* evaluate_losses (src/optim.py:148-152) at `theta`: losses[0..1]. */
int32_t kp_evaluate_losses(kp_context* ctx, const kp_problem* prob, const double* theta,
                           const kp_batch* batch, double* losses, void* workspace,
                           size_t workspace_bytes, void* stream);

/* kron_sum_solve (src/linalg.py:136-174): X (q x p, row-major) with
 * B1 X A1 + B2 X A2 = G for symmetric PD a1,a2 (p x p) and b1,b2 (q x q).
 * Inputs are not modified.  Workspace from kp_kron_solve_workspace_bytes. */
int32_t kp_kron_solve_workspace_bytes(kp_context* ctx, int32_t p, int32_t q, size_t* bytes);
int32_t kp_kron_sum_solve(kp_context* ctx, int32_t p, int32_t q, const double* a1,
                          const double* b1, const double* a2, const double* b2, const double* g,
                          double* x, int32_t* status, void* workspace, size_t workspace_bytes,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KFAC_PINN_B200_H */
