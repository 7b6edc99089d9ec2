// KFAC step orchestration and the extern "C" boundary (include/kfac_pinn_b200.h).
//
// One KFAC step (reference src/optim.py:251-263) on the device, in four phases:
//   1. accumulate  — chunked forward-Laplacian forward (taylor.py:172-203), affine
//      residual, reverse pass (taylor.py:242-276), boundary plain MLP
//      (network.py:200-232) and the UNNORMALISED sums of the interior/boundary
//      factors (curvature.py:96-137), the residual-weighted gradient
//      (optim.py:164-177) and sum r^2 — all into one contiguous reduce buffer
//      (the only thing multi-GPU ranks must all-reduce).
//   2. precondition — normalise + EMA, damped Kronecker-sum solve per layer
//      (curvature.py:140-163 / linalg.py:136-174), direction = Delta + mu prev.
//   3. line search — 31 forward-only passes at theta + 2^e dir (optim.py:195-211);
//      per-candidate sums of r^2 into a second small buffer (all-reduce #2).
//   4. update — device argmin (ascending grid, finite, strict <), theta += a dir,
//      prev = a dir, non-finite check (optim.py:260-262, 398-401).

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/kfac_pinn_b200.h"
#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

int fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  fprintf(stderr, "[kfac_pinn_b200] CUDA error %s in %s (%s:%d)\n", cudaGetErrorString(e), what,
          file, line);
  return KP_ERR_CUDA;
}

}  // namespace kp

using namespace kp;

struct kp_context {
  int device = 0;
  bool profile = false;
  std::vector<cudaEvent_t> ev;  // pairs
  size_t ev_used = 0;
  double prof_flops = 0.0;
  int64_t prof_launches = 0;
  // the same for the HBM-bound activation adjoint (k_act_bwd): event pairs + algorithmic bytes
  std::vector<cudaEvent_t> ev_hbm;
  size_t ev_hbm_used = 0;
  double prof_hbm_bytes = 0.0;
  int64_t prof_hbm_launches = 0;
  // further categories (kp_profile_read_cat): 0 = the INT8 tensor-core (CRT) fused layers of
  // the line search (work = FP64-equivalent flops), 1 = their residue slicing (work =
  // algorithmic DRAM bytes)
  unsigned crt_seq = 0;  // next slot of the CRT layer's tile-counter ring
  std::vector<cudaEvent_t> ev_cat[2];
  size_t ev_cat_used[2] = {0, 0};
  double prof_cat_work[2] = {0.0, 0.0};
  int64_t prof_cat_launches[2] = {0, 0};
  // side streams for the per-layer Kronecker-sum solves (2 per layer: A and B factor pairs)
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_ev;
  // early preconditioning (single-call steps): layer l's factor contractions done / its factor
  // EMA done, so the layer's eigenproblems start while later layers are still contracted
  std::vector<cudaEvent_t> layer_ev, fin_ev;
  // CUDA-graph replay of whole steps (only when every layer uses the on-device solver)
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t cap_in = nullptr, cap_out = nullptr;
  std::vector<unsigned char> graph_key;
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<unsigned char> graph_failed_key;  // arguments whose capture failed: run plain
  // warm-start cache of the on-device eigensolver (previous T per small factor pair, scratch,
  // validity flags), keyed on the layer shapes and the state's factor buffers
  double* warm_buf = nullptr;
  size_t warm_cap = 0;  // doubles
  int* warm_flags = nullptr;
  cudaEvent_t warm_ev = nullptr;  // the flags' reset on the main stream, for the side streams
  std::vector<unsigned char> warm_key;
  // cache of the last workspace plan (make_plan: host cost)
  kp_problem plan_key{};
  bool plan_valid = false;
  std::vector<unsigned char> plan_blob;
};

static int ensure_side_streams(kp_context* c, int n) {
  while ((int)c->layer_ev.size() < n / 2) {  // per-layer events of the early preconditioning
    cudaEvent_t a, b;
    KP_CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    KP_CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    c->layer_ev.push_back(a);
    c->fin_ev.push_back(b);
  }
  while ((int)c->side.size() < n) {
    cudaStream_t s;
    KP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e;
    KP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->side.push_back(s);
    c->side_ev.push_back(e);
  }
  return KP_OK;
}

#define KP_TRY(expr)          \
  do {                        \
    int r__ = (expr);         \
    if (r__ != KP_OK) return r__; \
  } while (0)

namespace {

constexpr int MAXL = KP_MAX_LAYERS;

// Static description of the step: shapes, parameter/factor packing, workspace carve.
struct Plan {
  int L = 0, d = 0, S = 0, ncand = 0, maxh = 0, maxp = 0, maxq = 0;
  int h[MAXL + 1] = {};
  int p[MAXL] = {}, q[MAXL] = {};
  int64_t N = 0, Nb = 0, Nc = 0;
  int64_t D = 0, FA = 0, FB = 0;
  int64_t th[MAXL] = {}, fa[MAXL] = {}, fb[MAXL] = {};
  // workspace offsets, in doubles
  int64_t o_wT[MAXL] = {}, o_zval0 = 0, o_post[MAXL] = {}, o_pre[MAXL] = {}, o_gout[MAXL] = {};
  int64_t o_ping = 0, o_pong = 0;
  int64_t o_ozEa = 0, o_ozB = 0, o_ozEb = 0;  // Ozaki line-search scratch (KP_OZAKI=1)
  int64_t o_crtH = 0, o_crtEH = 0, o_crtW = 0, o_crtEW = 0;  // CRT line-search residues
  int64_t o_crtCnt = 0;                                      // ring of 64 tile counters
  int64_t o_bzval0 = 0, o_bpost[MAXL] = {}, o_bpre[MAXL] = {}, o_bg[MAXL] = {};
  int64_t o_bping = 0, o_bpong = 0, o_ones = 0;
  int64_t o_r = 0, o_rb = 0, o_rls = 0, o_rbls = 0, o_u = 0, o_upart = 0;
  bool tn_grouped = false;  // small network: grouped TN contractions (accumulate)
  bool tn_grouped_bnd = false;  // boundary pass (few rows): grouped TN contractions
  size_t partial_cap = 0;   // doubles at o_partial
  int64_t o_partial = 0, o_red = 0, o_grad = 0, o_delta = 0, o_dslot = 0, o_dir = 0, o_thc = 0, o_ls = 0;
  int64_t o_A1 = 0, o_A2 = 0, o_B1 = 0, o_B2 = 0, o_la = 0, o_lb = 0, o_T1 = 0, o_T2 = 0;
  int64_t o_work = 0, o_info = 0;
  // per-layer Kronecker-solve scratch (layers solve concurrently on side streams)
  int64_t k_A1[MAXL] = {}, k_A2[MAXL] = {}, k_B1[MAXL] = {}, k_B2[MAXL] = {}, k_la[MAXL] = {},
          k_lb[MAXL] = {}, k_T1[MAXL] = {}, k_T2[MAXL] = {}, k_wa[MAXL] = {}, k_wb[MAXL] = {},
          k_info[MAXL] = {};
  int64_t o_wpad = 0, o_wpadc = 0, wo[MAXL] = {};
  int64_t o_w0t = 0, o_q0 = 0, o_w0tc = 0, o_q0c = 0;
  WPack wp{};   // layout of the padded copy of theta
  WPack wpc{};  // layout of the Bc line-search candidates' padded copies (layer-major)
  // KFAC*: Gramian-vector products
  int64_t o_gv = 0, o_gvd = 0, o_gvp = 0, o_jv = 0, o_jvb = 0, o_wpadv = 0, o_v0t = 0, o_vq0 = 0,
          o_dots = 0;
  int64_t o_seeds_eff = 0;  // per-point reverse-pass seeds of a non-affine residual
                            // (or the rotated seeds of dense coefficients)
  int64_t o_rotg = 0;       // layer-0 derivative-row gradient in the rotated basis (h1 x d)
  int Bc = 1;   // line-search candidates evaluated per batched launch
  int64_t total = 0;  // doubles
  // reduce-buffer sub-offsets (relative to o_red)
  int64_t r_aint = 0, r_bint = 0, r_abnd = 0, r_bbnd = 0, r_gint = 0, r_gbnd = 0, r_ss = 0,
          r_count = 0;
};

// Scratch of the device generalised eigensolver per factor pair (gen_eig_pair): M1 / K, and
// two n x n work matrices (n x (n + 1) each: the large-pair Jacobi wants an even row pitch).
inline int64_t pair_scratch_doubles(int n) { return 3LL * n * (n + 1); }

// Largest factor size the device solvers handle (small / mid / large route).
inline int max_pair_n() {
  return std::max(small_eig_max_n(), std::max(mid_eig_max_n(), large_eig_max_n()));
}

int check_net(const kp_net* net) {
  if (!net || net->n_layers < 1 || net->n_layers > MAXL) return KP_ERR_INVALID;
  for (int l = 0; l <= net->n_layers; ++l)
    if (net->widths[l] < 1) return KP_ERR_INVALID;
  if (net->widths[net->n_layers] != 1) return KP_ERR_INVALID;
  return KP_OK;
}

// Bytes of chunk-dependent workspace per interior point.
int64_t per_point_doubles(const kp_net* net) {
  const int L = net->n_layers, d = net->widths[0], S = d + 2;
  int maxh = d;
  for (int l = 1; l < L; ++l) maxh = std::max(maxh, net->widths[l]);
  int64_t v = net->widths[1];  // zval0
  for (int l = 1; l < L; ++l) v += (int64_t)S * net->widths[l];           // post
  for (int l = 1; l + 1 < L; ++l) v += (int64_t)S * net->widths[l + 1];   // pre
  for (int l = 0; l + 1 < L; ++l) v += (int64_t)S * net->widths[l + 1];   // gout
  v += 2LL * S * maxh;                                                   // ping/pong
  v += (int64_t)S;                                                       // u
  return v;
}

struct Plan;
struct StateBufs;
int tn_pass_jobs(const Plan& P, const double* x, int64_t n, const TaylorDims& td,
                 const StateBufs* b, const double* gl_last, const double* w, double* accA,
                 double* accB, double* accG, GemmTN* jobs, double** accs);

// Boundary passes with at most this much contraction work (points x widest layer^2) use
// the grouped TN launch (c4: 1000 x 256^2; c5's 768-wide layers stay on the TMA kernel,
// where the grouped cp.async kernel measured slower).
constexpr double kBndGroupMaxWork = 134217728.0;  // 2^27

int make_plan(kp_context* ctx, const kp_problem* pr, Plan& P) {
  KP_TRY(check_net(&pr->net));
  for (int l = 0; l <= pr->net.n_layers; ++l)  // factor sizes h + 1 (A) and h (B)
    if (pr->net.widths[l] + (l < pr->net.n_layers ? 1 : 0) > max_pair_n()) return KP_ERR_INVALID;
  if (pr->n_interior < 1 || pr->n_boundary < 1 || pr->n_candidates < 1) return KP_ERR_INVALID;
  P.L = pr->net.n_layers;
  for (int l = 0; l <= P.L; ++l) P.h[l] = pr->net.widths[l];
  P.d = P.h[0];
  P.S = P.d + 2;
  P.ncand = pr->n_candidates;
  P.N = pr->n_interior;
  P.Nb = pr->n_boundary;
  P.Nc = (pr->chunk > 0 && pr->chunk < P.N) ? pr->chunk : P.N;
  P.maxh = P.d;
  for (int l = 1; l < P.L; ++l) P.maxh = std::max(P.maxh, P.h[l]);
  int64_t off = 0;
  for (int l = 0; l < P.L; ++l) {
    P.p[l] = P.h[l] + 1;
    P.q[l] = P.h[l + 1];
    P.maxp = std::max(P.maxp, P.p[l]);
    P.maxq = std::max(P.maxq, P.q[l]);
    P.th[l] = off;
    off += (int64_t)P.p[l] * P.q[l];
  }
  P.D = off;
  int64_t woff = 0;
  P.wp.L = P.L;
  for (int l = 0; l < P.L; ++l) {
    P.wo[l] = woff;
    P.wp.h[l] = P.h[l];
    P.wp.th[l] = P.th[l];
    P.wp.wo[l] = woff;
    woff += ((int64_t)P.q[l] * P.h[l] + 1) / 2 * 2;  // keep every layer 16-byte aligned
  }
  // candidate batching: small problems evaluate all grid points per launch
  {
    bool fused_ok = P.L >= 3;
    for (int l = 1; l + 1 < P.L; ++l) fused_ok = fused_ok && gemm_act_ok(P.S, P.h[l], P.h[l], P.h[l]);
    const int64_t per = std::max<int64_t>(P.Nc * P.S, P.Nb) * P.maxh;
    const int64_t cap = 300000000;  // doubles per stacked state buffer
    P.Bc = fused_ok ? (int)std::max<int64_t>(1, std::min<int64_t>(P.ncand, cap / std::max<int64_t>(per, 1))) : 1;
  }
  int64_t wcoff = 0;
  P.wpc = P.wp;
  for (int l = 0; l < P.L; ++l) {
    P.wpc.wo[l] = wcoff;
    P.wpc.ws[l] = (int64_t)P.q[l] * P.h[l];
    wcoff += ((int64_t)P.Bc * P.q[l] * P.h[l] + 1) / 2 * 2;
  }
  for (int l = 0; l < P.L; ++l) {
    P.fa[l] = P.FA;
    P.FA += (int64_t)P.p[l] * P.p[l];
    P.fb[l] = P.FB;
    P.FB += (int64_t)P.q[l] * P.q[l];
  }
  const int64_t Mc = P.Nc * P.S;
  int64_t o = 0;
  auto take = [&](int64_t n) {
    const int64_t at = o;
    o += (n + 31) / 32 * 32;  // 256-byte alignment
    return at;
  };
  for (int l = 1; l < P.L; ++l) P.o_wT[l] = take((int64_t)P.h[l] * P.q[l]);
  P.o_zval0 = take(P.Bc * P.Nc * P.h[1]);
  for (int l = 1; l < P.L; ++l) P.o_post[l] = take(Mc * P.h[l]);
  for (int l = 1; l + 1 < P.L; ++l) P.o_pre[l] = take(Mc * P.h[l + 1]);
  for (int l = 0; l + 1 < P.L; ++l) P.o_gout[l] = take(Mc * P.h[l + 1]);
  P.o_ping = take(P.Bc * Mc * P.maxh);
  P.o_pong = take(P.Bc * Mc * P.maxh);
  P.o_u = take(Mc);
  P.o_upart = take(P.Bc * std::max(Mc, P.Nb) * ceil_div(std::max(P.maxh, 1), 64));
  P.o_bzval0 = take(P.Bc * P.Nb * P.h[1]);
  for (int l = 1; l < P.L; ++l) P.o_bpost[l] = take(P.Nb * P.h[l]);
  for (int l = 1; l + 1 < P.L; ++l) P.o_bpre[l] = take(P.Nb * P.h[l + 1]);
  for (int l = 0; l + 1 < P.L; ++l) P.o_bg[l] = take(P.Nb * P.h[l + 1]);
  P.o_bping = take(P.Bc * P.Nb * P.maxh);
  if (ozaki_enabled()) {  // A planes alias the layer's stored-state buffer (idle in the line search)
    P.o_ozEa = take(Mc / 2 + 1);
    P.o_ozB = take((int64_t)P.maxh * P.maxh);
    P.o_ozEb = take(P.maxh);
  }
  if (crt_enabled()) {  // residue planes of one layer's states and weights (int8) + exponents
    P.o_crtH = take(ceil_div((int64_t)crt_moduli() * Mc * P.maxh, 8));
    P.o_crtEH = take(Mc / 2 + 1);
    P.o_crtW = take(ceil_div((int64_t)crt_moduli() * P.maxh * P.maxh, 8));
    P.o_crtEW = take(P.maxh / 2 + 1);
    P.o_crtCnt = take(32);
  }
  P.o_bpong = take(P.Bc * P.Nb * P.maxh);
  P.o_ones = take(P.Nb);
  P.o_r = take(P.N);
  P.o_rb = take(P.Nb);
  P.o_rls = take(P.N * P.ncand);
  P.o_rbls = take(P.Nb * P.ncand);
  // TN partial buffer: max over every contraction of a step
  size_t part = 1;
  auto upd = [&](int64_t R, int Pp, int Qq, bool sym) {
    part = std::max(part, gemm_tn_partial_doubles(R, Pp, Qq, sym));
    part = std::max(part, gemm_tn_tma_partial_doubles(R, Pp, Qq, sym));
  };
  part = std::max(part, (size_t)64 * (P.maxh + P.maxq + 1));  // colsum scratch
  part = std::max(part, (size_t)64 * P.d * P.h[1]);             // layer-0 derivative colsum
  for (int64_t R : {P.Nc, P.Nb}) {
    const bool interior = (R == P.Nc);
    const int64_t rows = interior ? R * P.S : R;
    for (int l = 0; l < P.L; ++l) {
      const int64_t Rz = l == 0 ? R : rows;
      upd(Rz, P.p[l], P.p[l], true);
      upd(rows, P.q[l], P.q[l], true);
      upd(Rz, P.q[l], P.p[l], false);
      upd(Rz, P.h[l], P.h[l], true);    // TMA kernel: no bias column
      upd(Rz, P.q[l], P.h[l], false);
    }
  }
  if (P.maxh <= 128 && 3 * P.L <= 40) {
    GemmTN jobs[3 * MAXL];
    double* accs[3 * MAXL];
    const TaylorDims tdi{P.S, P.d, true}, tdb{1, 0, false};
    const int ki = tn_pass_jobs(P, nullptr, P.Nc, tdi, nullptr, nullptr, nullptr, nullptr, nullptr,
                                nullptr, jobs, accs);
    part = std::max(part, gemm_tn_grouped_partial_doubles(jobs, ki));
    const int kb = tn_pass_jobs(P, nullptr, P.Nb, tdb, nullptr, nullptr, nullptr, nullptr, nullptr,
                                nullptr, jobs, accs);
    part = std::max(part, gemm_tn_grouped_partial_doubles(jobs, kb));
    P.tn_grouped = true;
  }
  // Wider networks: the boundary pass alone (S = 1, few rows: one launch per contraction
  // would be launch-latency bound) still goes through the grouped launch.
  if (!P.tn_grouped && 3 * P.L <= 40 && (double)P.Nb * P.maxh * P.maxh <= kBndGroupMaxWork) {
    GemmTN jobs[3 * MAXL];
    double* accs[3 * MAXL];
    const TaylorDims tdb{1, 0, false};
    const int kb = tn_pass_jobs(P, nullptr, P.Nb, tdb, nullptr, nullptr, nullptr, nullptr, nullptr,
                                nullptr, jobs, accs);
    part = std::max(part, gemm_tn_grouped_partial_doubles(jobs, kb));
    P.tn_grouped_bnd = true;
  }
  P.partial_cap = part;
  P.o_partial = take((int64_t)part);
  P.r_aint = 0;
  P.r_bint = P.r_aint + P.FA;
  P.r_abnd = P.r_bint + P.FB;
  P.r_bbnd = P.r_abnd + P.FA;
  P.r_gint = P.r_bbnd + P.FB;
  P.r_gbnd = P.r_gint + P.D;
  P.r_ss = P.r_gbnd + P.D;
  P.r_count = P.r_ss + 2;
  P.o_red = take(P.r_count);
  P.o_grad = take(P.D);
  P.o_delta = take(P.D + 8);  // delta, then 8 status slots: the direction exchange buffer
  P.o_dslot = P.o_delta + P.D;
  P.o_dir = take(P.D);
  P.o_thc = take(P.Bc * P.D);
  P.o_wpad = take(woff);
  P.o_wpadc = take(wcoff);
  P.o_w0t = take((int64_t)P.d * P.h[1]);
  P.o_q0 = take(P.h[1]);
  P.o_w0tc = take((int64_t)P.Bc * P.d * P.h[1]);
  P.o_q0c = take((int64_t)P.Bc * P.h[1]);
  P.o_gv = take(4 * P.D);  // reduce buffer #3: G.Delta (int, bnd), G.prev (int, bnd), raw sums
  P.o_gvd = take(P.D);
  P.o_gvp = take(P.D);
  P.o_jv = take(P.Nc);
  P.o_jvb = take(P.Nb);
  P.o_wpadv = take(woff);
  P.o_v0t = take((int64_t)P.d * P.h[1]);
  P.o_vq0 = take(P.h[1]);
  P.o_dots = take(8);
  P.o_seeds_eff = take(P.N * P.S);
  P.o_rotg = take((int64_t)P.h[1] * P.d);
  P.o_ls = take(2 * (int64_t)P.ncand);
  P.o_A1 = take((int64_t)P.maxp * P.maxp);
  P.o_A2 = take((int64_t)P.maxp * P.maxp);
  P.o_B1 = take((int64_t)P.maxq * P.maxq);
  P.o_B2 = take((int64_t)P.maxq * P.maxq);
  P.o_la = take(P.maxp);
  P.o_lb = take(P.maxq);
  P.o_T1 = take((int64_t)P.maxp * P.maxq);
  P.o_T2 = take((int64_t)P.maxp * P.maxq);
  for (int l = 0; l < P.L; ++l) {
    const int64_t p = P.p[l], q = P.q[l];
    P.k_A1[l] = take(p * p);
    P.k_A2[l] = take(p * p);
    P.k_B1[l] = take(q * q);
    P.k_B2[l] = take(q * q);
    P.k_la[l] = take(p);
    P.k_lb[l] = take(q);
    P.k_T1[l] = take(p * q);
    P.k_T2[l] = take(p * q);
    P.k_wa[l] = take(pair_scratch_doubles(P.p[l]));  // device generalised eigensolver scratch
    P.k_wb[l] = take(pair_scratch_doubles(P.q[l]));
    P.k_info[l] = take(4);  // 8 ints: eig info (A, B), Cholesky infos (A: M2, C; B: M2, C)
  }
  P.total = o;
  return KP_OK;
}

struct Ctx {
  kp_context* ctx;
  const Plan& P;
  double* W;  // workspace base
  cudaStream_t s;
  const double* rot = nullptr;  // Q of dense operator coefficients (kp_batch.coeff_rot)
  // single-call step with per-layer contractions and off-launch (mid-size / large) factor
  // pairs: the accumulate phase records ctx->layer_ev and the precondition phase starts each
  // such layer's EMA and eigenproblems as soon as its factors are complete
  bool early = false;
  double* at(int64_t off) const { return W + off; }
};

// Optional CUDA-event timing of the hidden-layer forward GEMMs (fused or not).
template <typename F>
void prof_launch(const Ctx& c, double flops, F&& launch) {
  kp_context* ctx = c.ctx;
  if (!ctx->profile) {
    launch();
    return;
  }
  if (ctx->ev_used + 2 > ctx->ev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->ev.push_back(e);
    }
  }
  cudaEventRecord(ctx->ev[ctx->ev_used], c.s);
  launch();
  cudaEventRecord(ctx->ev[ctx->ev_used + 1], c.s);
  ctx->ev_used += 2;
  ctx->prof_flops += flops;
  ctx->prof_launches += 1;
}

// Optional CUDA-event timing of the HBM-bound activation adjoint; ``bytes`` = algorithmic
// DRAM bytes of the launch (every operand read once, the output written once).
template <typename F>
void prof_hbm_launch(const Ctx& c, double bytes, F&& launch) {
  kp_context* ctx = c.ctx;
  if (!ctx->profile) {
    launch();
    return;
  }
  if (ctx->ev_hbm_used + 2 > ctx->ev_hbm.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->ev_hbm.push_back(e);
    }
  }
  cudaEventRecord(ctx->ev_hbm[ctx->ev_hbm_used], c.s);
  launch();
  cudaEventRecord(ctx->ev_hbm[ctx->ev_hbm_used + 1], c.s);
  ctx->ev_hbm_used += 2;
  ctx->prof_hbm_bytes += bytes;
  ctx->prof_hbm_launches += 1;
}

// CUDA-event timing of category `cat` (kp_context::ev_cat): CRT layers / residue slicing.
template <typename F>
void prof_cat_launch(const Ctx& c, int cat, double work, F&& launch) {
  kp_context* ctx = c.ctx;
  if (!ctx->profile) {
    launch();
    return;
  }
  auto& ev = ctx->ev_cat[cat];
  size_t& used = ctx->ev_cat_used[cat];
  if (used + 2 > ev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
  }
  cudaEventRecord(ev[used], c.s);
  launch();
  cudaEventRecord(ev[used + 1], c.s);
  used += 2;
  ctx->prof_cat_work[cat] += work;
  ctx->prof_cat_launches[cat] += 1;
}

// Algorithmic bytes of one k_act_bwd launch per (sample, unit): the stored pre-activation
// state (S rows, or the one value row of layer 0), the incoming adjoint (S rows, or the
// per-sample rank-1 seed, negligible) and the outgoing adjoint (S rows).
double act_bwd_bytes(const ActBwd& a, int64_t n, int h, const TaylorDims& td) {
  const double S = td.S;
  const double per = 8.0 * ((a.pre ? S : 1.0) + (a.gin ? S : 0.0) + S);
  return per * (double)n * h;
}

void prof_gemm(const Ctx& c, const GemmNT& g) {
  prof_launch(c, 2.0 * (double)g.M * g.N * g.K, [&] { launch_gemm_nt(g, c.s); });
}

// Hidden layer l forward: fused GEMM + bias + activation when possible, else GEMM then
// the elementwise activation kernel.  mode: ACT_STORE (pre + post), ACT_LOSS (post).
// wl = padded W_l (h_{l+1} x h_l, pitch h_l).
void hidden_layer(const Ctx& c, const double* theta, const double* wl, int l, const double* in,
                  int64_t n, const TaylorDims& td, const double* cdiag, double* pre, double* post,
                  int mode) {
  const Plan& P = c.P;
  GemmAct ga{};
  ga.A = in;
  ga.lda = P.h[l];
  ga.B = wl;
  ga.ldb = P.h[l];
  ga.bias = theta + P.th[l] + P.h[l];
  ga.bias_stride = P.p[l];
  ga.n_samples = n;
  ga.S = td.S;
  ga.d = td.d;
  ga.taylor = td.taylor;
  ga.N = P.h[l + 1];
  ga.K = P.h[l];
  ga.cdiag = cdiag;
  ga.pre = pre;
  ga.post = post;
  ga.ldo = P.h[l + 1];
  bool done = false;
  prof_launch(c, 2.0 * (double)n * td.S * P.h[l] * P.h[l + 1],
              [&] { done = launch_gemm_act(ga, mode, c.s); });
  if (done) return;
  double* out = mode == ACT_STORE ? pre : post;
  GemmNT g{in, P.h[l], wl, P.h[l], out, P.h[l + 1], n * td.S, P.h[l + 1], P.h[l],
           theta + P.th[l] + P.h[l], P.p[l], td.S};
  prof_gemm(c, g);
  launch_act_fwd(out, post, n, P.h[l + 1], td, cdiag, c.s);
}

struct StateBufs {
  double* zval0;
  double* post[MAXL];
  double* pre[MAXL];
  double* gout[MAXL];
  double* ping;
  double* pong;
};

StateBufs interior_bufs(const Ctx& c) {
  const Plan& P = c.P;
  StateBufs b{};
  b.zval0 = c.at(P.o_zval0);
  for (int l = 1; l < P.L; ++l) b.post[l] = c.at(P.o_post[l]);
  for (int l = 1; l + 1 < P.L; ++l) b.pre[l] = c.at(P.o_pre[l]);
  for (int l = 0; l + 1 < P.L; ++l) b.gout[l] = c.at(P.o_gout[l]);
  b.ping = c.at(P.o_ping);
  b.pong = c.at(P.o_pong);
  return b;
}

StateBufs boundary_bufs(const Ctx& c) {
  const Plan& P = c.P;
  StateBufs b{};
  b.zval0 = c.at(P.o_bzval0);
  for (int l = 1; l < P.L; ++l) b.post[l] = c.at(P.o_bpost[l]);
  for (int l = 1; l + 1 < P.L; ++l) b.pre[l] = c.at(P.o_bpre[l]);
  for (int l = 0; l + 1 < P.L; ++l) b.gout[l] = c.at(P.o_bg[l]);
  b.ping = c.at(P.o_bping);
  b.pong = c.at(P.o_bpong);
  return b;
}

// Residual definition for one pass (interior: affine residual; boundary: u - target).
struct ResidualIn {
  const double* r0;
  const double* seeds;
  const double* targets;
  const double* quad = nullptr;  // interior: quadratic gradient coefficients (n x d)
  double* seeds_out = nullptr;   // interior: effective reverse-pass seeds (n x S)
};

// Forward pass storing every state needed by the reverse pass (taylor.py:172-203;
// boundary: network.py:200-213).  Writes residuals r[0..n).
// `cand` selects the prepared copies of this parameter set: false = theta (o_wpad, o_w0t,
// o_q0), true = the line-search candidate (o_wpadc, o_w0tc, o_q0c).
void forward_store(const Ctx& c, const double* theta, const double* wpad, const double* x, int64_t n,
                   const TaylorDims& td, const double* cdiag, const StateBufs& b,
                   const ResidualIn& ri, double* r, double* u_out) {
  const Plan& P = c.P;
  const int L = P.L;
  const double* last_in;
  if (L == 1) {
    if (td.taylor) {
      launch_initial_state(x, n, P.d, b.ping, c.s);
      last_in = b.ping;
    } else {
      last_in = x;
    }
  } else {
    launch_first_layer(x, n, P.d, theta + P.th[0], P.h[1], td, c.at(P.o_w0t), c.at(P.o_q0),
                       b.zval0, b.post[1], c.s);
    for (int l = 1; l + 1 < L; ++l)
      hidden_layer(c, theta, wpad + P.wo[l], l, b.post[l], n, td, cdiag, b.pre[l], b.post[l + 1],
                   ACT_STORE);
    last_in = b.post[L - 1];
  }
  launch_last_layer(last_in, n, P.h[L - 1], theta + P.th[L - 1], td, ri.r0, ri.seeds, ri.targets,
                    r, u_out, c.s, ri.quad, ri.seeds_out);
}

// Forward pass for losses only (no stored states): ping-pong buffers.  `batch` parameter
// sets are evaluated per launch (theta + kk*D, padded weights per `wp`, states stacked in
// ping/pong, residuals r + kk*r_bstride); batch > 1 requires the fused layer path.
void forward_loss(const Ctx& c, const double* theta, const double* wpad, const double* x, int64_t n,
                  const TaylorDims& td, const double* cdiag, double* ping, double* pong,
                  const ResidualIn& ri, double* r, double* u_out, bool cand = false,
                  int batch = 1, int64_t r_bstride = 0) {
  const Plan& P = c.P;
  const int L = P.L;
  const WPack& wp = cand ? P.wpc : P.wp;
  const double* cur;
  if (L == 1) {
    if (td.taylor) {
      launch_initial_state(x, n, P.d, ping, c.s);
      cur = ping;
    } else {
      cur = x;
    }
  } else {
    double* zs = td.taylor ? c.at(P.o_zval0) : c.at(P.o_bzval0);
    const double* w0t = c.at(cand ? P.o_w0tc : P.o_w0t);
    const double* q0 = c.at(cand ? P.o_q0c : P.o_q0);
    // When the first hidden layer runs on the INT8 tensor cores, layer 0 goes straight to its
    // residue planes (k_crt_first): the FP64 state is neither written nor read back.
    bool first_sliced = false;
    if (L > 2 && batch == 1 && td.taylor && crt_act_ok(td.S, P.h[1], P.h[2]) && crt_first_enabled()) {
      launch_first_layer(x, n, P.d, theta + P.th[0], P.h[1], td, w0t, q0, zs, nullptr, c.s, 1, P.D);
      prof_cat_launch(c, 1, (double)crt_moduli() * (double)n * td.S * P.h[1], [&] {
        first_sliced = launch_crt_first(zs, n, P.h[1], td.S, td.d, w0t, q0,
                                        reinterpret_cast<int8_t*>(c.at(P.o_crtH)),
                                        reinterpret_cast<int*>(c.at(P.o_crtEH)), c.s);
      });
      if (!first_sliced)  // shape outside the fused kernel: expand z the usual way
        launch_first_layer(x, n, P.d, theta + P.th[0], P.h[1], td, w0t, q0, zs, ping, c.s, 1, P.D);
    } else {
      launch_first_layer(x, n, P.d, theta + P.th[0], P.h[1], td, w0t, q0, zs, ping, c.s, batch, P.D);
    }
    double* a = ping;
    double* b = pong;
    for (int l = 1; l + 1 < L; ++l) {
      // FP64 product emulated on the INT8 tensor cores by the CRT construction (kp_crt.cu):
      // slice the states and the candidate's weights into residue planes, then the fused
      // layer (c5's one-sample tiles; the output layer folded in as in ACT_LAST below).
      if (batch == 1 && td.taylor && crt_act_ok(td.S, P.h[l], P.h[l + 1])) {
        int8_t* resH = reinterpret_cast<int8_t*>(c.at(P.o_crtH));
        int* exH = reinterpret_cast<int*>(c.at(P.o_crtEH));
        int8_t* resW = reinterpret_cast<int8_t*>(c.at(P.o_crtW));
        int* exW = reinterpret_cast<int*>(c.at(P.o_crtEW));
        // slicing: 8 B read + one byte per modulus written per state element
        if (!(l == 1 && first_sliced))
          prof_cat_launch(c, 1, (8.0 + crt_moduli()) * (double)n * td.S * P.h[l], [&] {
            launch_crt_slice(a, n * td.S, P.h[l], P.h[l], resH, exH, false, c.s);
          });
        launch_crt_slice(wpad + wp.wo[l], P.h[l + 1], P.h[l], P.h[l], resW, exW, true, c.s);
        GemmAct ga{};
        ga.bias = theta + P.th[l] + P.h[l];
        ga.bias_stride = P.p[l];
        ga.n_samples = n;
        ga.S = td.S;
        ga.d = td.d;
        ga.taylor = true;
        ga.N = P.h[l + 1];
        ga.K = P.h[l];
        ga.cdiag = cdiag;
        const bool last = (l == L - 2 && u_out == nullptr);
        if (last) {
          ga.wlast = theta + P.th[L - 1];
          ga.upart = c.at(P.o_upart);
        } else {
          ga.post = b;
          ga.ldo = P.h[l + 1];
        }
        bool done = false;
        prof_cat_launch(c, 0, 2.0 * (double)n * td.S * P.h[l] * P.h[l + 1], [&] {
          int* cnt = reinterpret_cast<int*>(c.at(P.o_crtCnt)) + (c.ctx->crt_seq++ % 64);
          done = launch_crt_act(ga, last ? ACT_LAST : ACT_LOSS, resH, exH, resW, exW, c.s, cnt);
        });
        if (!done && l == 1 && first_sliced) {  // the DMMA layer below needs layer 0's FP64 state
          launch_first_layer(x, n, P.d, theta + P.th[0], P.h[1], td, w0t, q0, zs, ping, c.s, 1, P.D);
          first_sliced = false;
        }
        if (done) {  // (a rejected launch falls through to the FP64 DMMA layer below)
          if (last) {
            launch_last_from_partials(c.at(P.o_upart), P.h[l + 1] / 128, n, td,
                                      theta + P.th[L - 1] + P.h[L - 1], ri.r0, ri.seeds,
                                      ri.targets, r, c.s, batch, P.D, r_bstride, ri.quad);
            return;
          }
          std::swap(a, b);
          continue;
        }
      }
      // FP64 emulated on the INT8 tensor cores (KP_OZAKI=1): GEMM + bias, then the Taylor
      // activation in place; the layer's stored-state buffer (idle during the line search)
      // holds the input's slices.  The h_out = 1 output layer then runs unfused below.
      if (batch == 1 && ozaki_gemm_ok(n * td.S, P.h[l + 1], P.h[l], P.h[l], P.h[l])) {
        bool done = false;
        prof_launch(c, 2.0 * (double)n * td.S * P.h[l] * P.h[l + 1], [&] {
          done = launch_ozaki_gemm(a, P.h[l], wpad + wp.wo[l], P.h[l], b, P.h[l + 1], n * td.S,
                                   P.h[l + 1], P.h[l], theta + P.th[l] + P.h[l], P.p[l], td.S,
                                   reinterpret_cast<int8_t*>(c.at(P.o_post[l])),
                                   reinterpret_cast<int*>(c.at(P.o_ozEa)),
                                   reinterpret_cast<int8_t*>(c.at(P.o_ozB)),
                                   reinterpret_cast<int*>(c.at(P.o_ozEb)), c.s);
        });
        if (done) {
          launch_act_fwd(b, b, n, P.h[l + 1], td, cdiag, c.s);
          std::swap(a, b);
          continue;
        }
      }
      GemmAct ga{};
      ga.A = a;
      ga.lda = P.h[l];
      ga.B = wpad + wp.wo[l];
      ga.ldb = P.h[l];
      ga.bias = theta + P.th[l] + P.h[l];
      ga.bias_stride = P.p[l];
      ga.n_samples = n;
      ga.S = td.S;
      ga.d = td.d;
      ga.taylor = td.taylor;
      ga.N = P.h[l + 1];
      ga.K = P.h[l];
      ga.cdiag = cdiag;
      ga.batch = batch;
      ga.bias_bstride = P.D;
      if (l == L - 2 && u_out == nullptr) {
        // last hidden layer: fuse the h_out = 1 output layer, never store this state
        const int ntn = (int)ceil_div(P.h[l + 1], gemm_act_tile_width(td.S, P.h[l + 1], P.h[l]));
        ga.wlast = theta + P.th[L - 1];
        ga.wlast_bstride = P.D;
        ga.upart = c.at(P.o_upart);
        ga.upart_bstride = n * td.S * ntn;
        bool done = false;
        prof_launch(c, 2.0 * (double)batch * n * td.S * P.h[l] * P.h[l + 1],
                    [&] { done = launch_gemm_act(ga, ACT_LAST, c.s); });
        if (done) {
          launch_last_from_partials(c.at(P.o_upart), ntn, n, td, theta + P.th[L - 1] + P.h[L - 1],
                                    ri.r0, ri.seeds, ri.targets, r, c.s, batch, P.D, r_bstride,
                                    ri.quad);
          return;
        }
      } else {
        ga.post = b;
        ga.ldo = P.h[l + 1];
        ga.out_bstride = n * td.S * P.h[l + 1];
        bool done = false;
        prof_launch(c, 2.0 * (double)batch * n * td.S * P.h[l] * P.h[l + 1],
                    [&] { done = launch_gemm_act(ga, ACT_LOSS, c.s); });
        if (done) {
          std::swap(a, b);
          continue;
        }
      }
      // unfused fallback (only reachable with batch == 1, see make_plan)
      hidden_layer(c, theta, wpad + wp.wo[l], l, a, n, td, cdiag, b, b, ACT_LOSS);
      std::swap(a, b);
    }
    cur = a;
  }
  for (int kk = 0; kk < batch; ++kk)
    launch_last_layer(cur + (int64_t)kk * n * td.S * P.h[L - 1], n, P.h[L - 1],
                      theta + kk * P.D + P.th[L - 1], td, ri.r0, ri.seeds, ri.targets,
                      r ? r + kk * r_bstride : nullptr, u_out, c.s, ri.quad);
}

// Reverse pass (taylor.py:242-276 / network.py:216-232): gout[l] for l < L-1.
void backward(const Ctx& c, const double* theta, int64_t n, const TaylorDims& td,
              const double* cdiag, const StateBufs& b, const double* seeds) {
  const Plan& P = c.P;
  const int L = P.L;
  if (L < 2) return;
  {
    ActBwd a{};
    a.pre = (L - 2 == 0) ? nullptr : b.pre[L - 2];
    a.zval = b.zval0;
    a.w0t = c.at(P.o_w0t);
    a.gin = nullptr;
    a.seeds = seeds;
    a.wlast = theta + P.th[L - 1];
    a.gout = b.gout[L - 2];
    prof_hbm_launch(c, act_bwd_bytes(a, n, P.h[L - 1], td),
                    [&] { launch_act_bwd(a, n, P.h[L - 1], td, cdiag, c.s); });
  }
  for (int l = L - 2; l >= 1; --l) {
    GemmNT g{b.gout[l], P.h[l + 1], c.at(P.o_wT[l]), P.h[l + 1], b.ping, P.h[l],
             n * td.S, P.h[l], P.h[l + 1], nullptr, 0, td.S};
    launch_gemm_nt(g, c.s);
    ActBwd a{};
    a.pre = (l - 1 == 0) ? nullptr : b.pre[l - 1];
    a.zval = b.zval0;
    a.w0t = c.at(P.o_w0t);
    a.gin = b.ping;
    a.gout = b.gout[l - 1];
    prof_hbm_launch(c, act_bwd_bytes(a, n, P.h[l], td),
                    [&] { launch_act_bwd(a, n, P.h[l], td, cdiag, c.s); });
  }
}

// One layer of  acc += sum_n w_n sum_s g_{n,s} zhat_{n,s}^T  — the residual-weighted gradient
// (optim.py:170-176, w = r) and, with w = J v, the exact Gramian-vector product of KFAC*
// (curvature.py:253-260).  For layer 0 only the value rows of Z0 = [x; I; 0] are dense; the
// derivative rows e_i contribute a weighted column sum.
void contract_grad_deriv0(const Ctx& c, int64_t n, const TaylorDims& td, const double* G,
                          const double* w, double* out);

// The factor and gradient contractions of one pass (an interior chunk of n points or the
// boundary) as cp.async TN jobs with synthesised bias columns, for the grouped launch of
// small networks.  Null buffers give shape-only jobs (workspace sizing).
int tn_pass_jobs(const Plan& P, const double* x, int64_t n, const TaylorDims& td,
                 const StateBufs* b, const double* gl_last, const double* w, double* accA,
                 double* accB, double* accG, GemmTN* jobs, double** accs) {
  int k = 0;
  const int64_t rows = n * td.S;
  for (int l = 0; l < P.L; ++l) {
    const int q = P.q[l], hz = P.h[l];
    const double* G = (l == P.L - 1) ? gl_last : (b ? b->gout[l] : nullptr);
    const double* Z = (l == 0) ? x : (b ? b->post[l] : nullptr);
    const int64_t ldz = (l == 0) ? P.d : P.h[l];
    const int64_t Rz = (l == 0) ? n : rows;
    const int Sz = (l == 0) ? 1 : td.S;
    const int64_t ldg = (l == 0) ? (int64_t)td.S * q : q;
    const int Sw = (l == 0) ? 1 : td.S;
    jobs[k] = GemmTN{Z, ldz, hz, true, Z, ldz, hz, true, nullptr, 1, Sz, Rz, true};
    accs[k++] = accA ? accA + P.fa[l] : nullptr;
    jobs[k] = GemmTN{G, q, q, false, G, q, q, false, nullptr, 1, 1, rows, true};
    accs[k++] = accB ? accB + P.fb[l] : nullptr;
    jobs[k] = GemmTN{G, ldg, q, false, Z, ldz, hz, true, w, Sw, Sz, Rz, false};
    accs[k++] = accG ? accG + P.th[l] : nullptr;
  }
  return k;
}

void contract_grad_layer(const Ctx& c, const double* x, int64_t n, const TaylorDims& td,
                         const StateBufs& b, const double* gl_last, const double* w,
                         double* accG, int l) {
  const Plan& P = c.P;
  double* part = c.at(P.o_partial);
  const int64_t rows = n * td.S;
  const int q = P.q[l], hz = P.h[l], p = P.p[l];
  const double* G = (l == P.L - 1) ? gl_last : b.gout[l];
  const double* Z = (l == 0) ? x : b.post[l];
  const int64_t ldz = (l == 0) ? P.d : P.h[l];
  const int64_t Rz = (l == 0) ? n : rows;
  const int Sz = (l == 0) ? 1 : td.S;
  double* out = accG + P.th[l];
  const int64_t ldg = (l == 0) ? (int64_t)td.S * q : q;
  const int Sw = (l == 0) ? 1 : td.S;
  if (launch_gemm_tn_tma_accumulate(G, ldg, q, Z, ldz, hz, w, Sw, Rz, false, part, out, p, c.s)) {
    launch_colsum(G, (int64_t)td.S * q, n, q, w, out + hz, p, 0.0, part, c.s);
  } else {
    GemmTN gg{G, ldg, q, false, Z, ldz, hz, true, w, Sw, Sz, Rz, false};
    launch_gemm_tn_accumulate(gg, part, out, c.s);
  }
  if (l == 0 && td.taylor) contract_grad_deriv0(c, n, td, G, w, out);
}

// Layer-0 gradient, derivative rows e_i: out[j][i] += sum_n w_n Gbar0[n, 1+i, j] (the
// contiguous d x q block after each sample's value row).
void contract_grad_deriv0(const Ctx& c, int64_t n, const TaylorDims& td, const double* G,
                          const double* w, double* out) {
  const Plan& P = c.P;
  double* part = c.at(P.o_partial);
  const int q = P.q[0], p = P.p[0];
  {
    if (!c.rot) {
      launch_colsum(G + q, (int64_t)td.S * q, n, P.d * q, w, out, p, 0.0, part, c.s, q);
    } else {  // rows along Q[:, k]: out[j][i] += sum_k (sum_n w_n Gbar0[n, 1+k, j]) Q[i][k]
      double* t = c.at(P.o_rotg);
      cudaMemsetAsync(t, 0, sizeof(double) * q * P.d, c.s);
      launch_colsum(G + q, (int64_t)td.S * q, n, P.d * q, w, t, P.d, 0.0, part, c.s, q);
      launch_rot_accum(t, q, P.d, c.rot, out, p, c.s);
    }
  }
}

// Factor and gradient contractions of one pass into the reduce buffer.  The bulk of
// every contraction runs in the TMA-fed DMMA kernel; the bias-augmentation row /
// column (the virtual 1 on value rows, curvature.py:88-93) are value-row column
// sums.  Operands that are not TMA-compatible (odd pitch) use the cp.async kernel,
// which synthesises the bias column itself.
void accumulate(const Ctx& c, const double* x, int64_t n, const TaylorDims& td,
                const StateBufs& b, const double* gl_last, const double* r, double* accA,
                double* accB, double* accG, bool record_layers = false) {
  const Plan& P = c.P;
  const int L = P.L;
  double* part = c.at(P.o_partial);
  const int64_t rows = n * td.S;
  if (P.tn_grouped || (P.tn_grouped_bnd && td.S == 1)) {  // every contraction in one launch
    GemmTN jobs[3 * MAXL];
    double* accs[3 * MAXL];
    const int k = tn_pass_jobs(P, x, n, td, &b, gl_last, r, accA, accB, accG, jobs, accs);
    if (launch_gemm_tn_grouped(jobs, accs, k, part, P.partial_cap, c.s)) {
      if (td.taylor) contract_grad_deriv0(c, n, td, L == 1 ? gl_last : b.gout[0], r, accG);
      return;
    }
  }
  for (int l = 0; l < L; ++l) {
    const int q = P.q[l], hz = P.h[l], p = P.p[l];
    const double* G = (l == L - 1) ? gl_last : b.gout[l];
    const double* Z = (l == 0) ? x : b.post[l];
    const int64_t ldz = (l == 0) ? P.d : P.h[l];
    const int64_t Rz = (l == 0) ? n : rows;  // rows of the layer input matrix
    const int Sz = (l == 0) ? 1 : td.S;      // its value-row period
    // A_l = sum zhat zhat^T over the bias-augmented layer inputs (curvature.py:112-114)
    {
      double* out = accA + P.fa[l];
      if (launch_gemm_tn_tma_accumulate(Z, ldz, hz, Z, ldz, hz, nullptr, 1, Rz, true, part, out, p,
                                        c.s)) {
        launch_colsum(Z, (int64_t)Sz * ldz, n, hz, nullptr, out + (int64_t)hz * p, 1, (double)n,
                      part, c.s);
      } else {
        GemmTN a{Z, ldz, hz, true, Z, ldz, hz, true, nullptr, 1, Sz, Rz, true};
        launch_gemm_tn_accumulate(a, part, out, c.s);
      }
    }
    // B_l = sum g g^T over all rows (curvature.py:113,115)
    if (!launch_gemm_tn_tma_accumulate(G, q, q, G, q, q, nullptr, 1, rows, true, part,
                                       accB + P.fb[l], q, c.s)) {
      GemmTN bb{G, q, q, false, G, q, q, false, nullptr, 1, 1, rows, true};
      launch_gemm_tn_accumulate(bb, part, accB + P.fb[l], c.s);
    }
    if (record_layers) cudaEventRecord(c.ctx->layer_ev[l], c.s);  // A_l, B_l complete
    contract_grad_layer(c, x, n, td, b, gl_last, r, accG, l);
  }
}

int phase_accumulate(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, const kp_batch* bt) {
  const Plan& P = c.P;
  double* red = c.at(P.o_red);
  KP_CUDA_TRY(cudaMemsetAsync(red, 0, sizeof(double) * P.r_count, c.s));
  for (int l = 1; l < P.L; ++l)
    launch_transpose(st->theta + P.th[l], P.p[l], P.q[l], P.h[l], c.at(P.o_wT[l]), c.s);
  launch_candidate(st->theta, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpad), c.s);
  if (P.L >= 2)
    launch_prep_layer0(st->theta, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_w0t), c.at(P.o_q0), c.s);
  const TaylorDims tdi{P.S, P.d, true};
  const TaylorDims tdb{1, 0, false};
  auto boundary_pass = [&]() {
    const StateBufs bb = boundary_bufs(c);
    double* ones = c.at(P.o_ones);
    launch_fill(ones, P.Nb, 1.0, c.s);
    ResidualIn rb{nullptr, nullptr, bt->targets};
    forward_store(c, st->theta, c.at(P.o_wpad), bt->x_bnd, P.Nb, tdb, bt->coeff_diag, bb, rb,
                  c.at(P.o_rb), nullptr);
    backward(c, st->theta, P.Nb, tdb, bt->coeff_diag, bb, nullptr);
    accumulate(c, bt->x_bnd, P.Nb, tdb, bb, ones, c.at(P.o_rb), red + P.r_abnd, red + P.r_bbnd,
               red + P.r_gbnd);
  };
  // early preconditioning: the boundary sums first, so that each layer's factors are
  // complete right after its interior contractions (last chunk)
  if (c.early) boundary_pass();
  const StateBufs bi = interior_bufs(c);
  for (int64_t n0 = 0; n0 < P.N; n0 += P.Nc) {
    const int64_t nc = std::min(P.Nc, P.N - n0);
    const double* x = bt->x_int + n0 * P.d;
    const double* seeds = bt->seeds + n0 * P.S;
    double* r = c.at(P.o_r) + n0;
    ResidualIn ri{bt->r0 + n0, seeds, nullptr};
    if (bt->quad) {  // seeds depend on the outputs (optim.py:157-158): computed by the forward
      ri.quad = bt->quad + n0 * P.d;
      ri.seeds_out = c.at(P.o_seeds_eff) + n0 * P.S;
      seeds = ri.seeds_out;
    }
    forward_store(c, st->theta, c.at(P.o_wpad), x, nc, tdi, bt->coeff_diag, bi, ri, r, nullptr);
    backward(c, st->theta, nc, tdi, bt->coeff_diag, bi, seeds);
    accumulate(c, x, nc, tdi, bi, seeds, r, red + P.r_aint, red + P.r_bint, red + P.r_gint,
               c.early && n0 + nc >= P.N);
  }
  if (!c.early) boundary_pass();
  launch_sumsq(c.at(P.o_r), P.N, 0, 1, red + P.r_ss, 1, c.s);
  launch_sumsq(c.at(P.o_rb), P.Nb, 0, 1, red + P.r_ss + 1, 1, c.s);
  return KP_OK;
}

// Generalised eigenproblem M1 x = lam M2 x of one factor pair (M_i = F_i + damping I) with
// small_eig_max_n() < n, entirely on the device and asynchronous on stream s (no library
// call, nothing blocks the host, graph-capturable).  Warm start as in the small solver: the
// pair is first congruence-transformed by the previous step's T (tp holds T^T row-major, the
// identity until a solve of this pair has succeeded, decided on the device by *valid, so the
// same launches serve cold and warm steps):
//   M_i' = T_p^T M_i T_p,  M2' = L L^T,  M1' = K K^T  (blocked Cholesky, kp_dense.cu),
//   L_C = L^-1 K  (lower triangular: C = L^-1 M1' L^-T = L_C L_C^T, R = L_C^T),
// then one-sided Jacobi on the rows of L_C (= the columns of R), U = R V with orthogonal
// columns (C V = V diag(||u_i||^2)):
//   n <= mid_eig_max_n(): R in a thread-block cluster's shared memory (kp_eig_mid.cu),
//   larger:               R in L2, one 16-CTA cluster (kp_eig_large.cu);
// T' = L^-T V = K^-T U (K^-T U = L^-T L_C^-T R V), i.e. T'^T = U^T K^-1, so V is never
// accumulated (KP_MID_ACCV=1 / KP_LARGE_ACCV=1: the kernels rotate V too, T'^T = V^T L^-1);
// and T = T_p T'.  Out: tout = T^T row-major (= T column-major), lam = eigenvalues; the same
// T^T is kept in tp for the next step.  chol_info[0..1]: Cholesky infos of M2', M1' (a failure
// makes the eigensolver report info = n + 1: not positive definite).
// scratch: pair_scratch_doubles(n) = 3 n^2; m2: n^2.
int gen_eig_pair(cudaStream_t s, int n, const double* f1, const double* f2, double lam,
                 double* tout, double* m2, double* ev, double* scratch, int* info, int* chol_info,
                 double* tp, int* valid) {
  const size_t region = (size_t)n * (n + 1);
  const int ld2 = n + (n & 1);  // even row pitch of the Jacobi rows (16-byte aligned)
  double* m1 = scratch;
  double* s1 = scratch + region;
  double* s2 = scratch + 2 * region;
  KP_CUDA_TRY(cudaMemsetAsync(chol_info, 0, 2 * sizeof(int), s));
  launch_damped_copy(f1, lam, n, m1, s);
  launch_damped_copy(f2, lam, n, m2, s);
  launch_warm_identity(tp, n, valid, s);
  for (double* m : {m2, m1}) {  // M' = Tp^T M Tp = tp M tp^T
    launch_dense_gemm(DenseGemm{n, n, n, tp, n, false, m, n, false, s1, n, 1.0, 0.0, false}, s);
    launch_dense_gemm(DenseGemm{n, n, n, s1, n, false, tp, n, true, m, n, 1.0, 0.0, false}, s);
  }
  launch_cholesky(n, m2, n, chol_info, s);      // L
  launch_cholesky(n, m1, n, chol_info + 1, s);  // K
  launch_zero_upper(n, m1, n, s);
  launch_trsm_lower(n, m2, n, s1, n, n, true, s);  // s1 = L^-1
  const bool mid = n <= mid_eig_max_n();
  const int lu = mid ? n : ld2;  // pitch of the Jacobi rows
  launch_dense_gemm(DenseGemm{n, n, n, s1, n, false, m1, n, false, s2, lu, 1.0, 0.0, false}, s);
  const double* vt = s2;  // rows: V^T (eigenvectors accumulated) or U^T
  int lv = lu;
  bool u_rows = true;
  if (mid) {
    launch_eig_mid(n, s2, ev, info, chol_info, s, valid);
    u_rows = !mid_eig_accumulate_v();
  } else if (large_eig_accumulate_v() && n <= large_eig_accv_max_n()) {
    launch_eig_large(n, ld2, s2, m1, ev, info, chol_info, s, valid);  // m1 <- V^T (pitch ld2)
    vt = m1;
    u_rows = false;
  } else {
    // s1 (L^-1) is dead until K^-1 is formed below: the split-record tails live there
    launch_eig_large(n, ld2, s2, nullptr, ev, info, chol_info, s, valid, s1);
  }
  // T'^T = U^T K^-1 (K^-T U = L^-T V) or V^T L^-1
  if (u_rows) launch_trsm_lower(n, m1, n, s1, n, n, true, s);  // s1 = K^-1
  launch_dense_gemm(DenseGemm{n, n, n, vt, lv, false, s1, n, false, m2, n, 1.0, 0.0, false}, s);
  // T^T = T'^T T_p^T
  launch_dense_gemm(DenseGemm{n, n, n, m2, n, false, tp, n, false, tout, n, 1.0, 0.0, false}, s);
  launch_copy_matrix(tout, n, n, n, tp, n, s);
  return KP_OK;
}

// out (q x p row-major) = sign * T_B [(T_B^T G T_A) / (lb la^T + 1)] T_A^T  (the
// two-term Kronecker-sum solution, linalg.py:168-173) from TtA = T_A^T (p x p) and
// TtB = T_B^T (q x q), both row-major, and the q x p gradient G; t1, t2: q x p scratch.
void kron_combine(cudaStream_t s, int p, int q, const double* TtA, const double* la,
                  const double* TtB, const double* lb, const double* G, double* out, double sign,
                  double* t1, double* t2) {
  launch_dense_gemm(DenseGemm{q, p, q, TtB, q, false, G, p, false, t1, p, 1.0, 0.0, false}, s);
  launch_dense_gemm(DenseGemm{q, p, p, t1, p, false, TtA, p, true, t2, p, 1.0, 0.0, false}, s);
  launch_kron_scale(t2, la, p, lb, q, s);
  launch_dense_gemm(DenseGemm{q, p, q, TtB, q, true, t2, p, false, t1, p, 1.0, 0.0, false}, s);
  launch_dense_gemm(DenseGemm{q, p, p, t1, p, false, TtA, p, false, out, p, sign, 0.0, false}, s);
}

// `owned` (host, L flags) = nullptr: every layer's Kronecker solve runs here and the phase
// ends with the momentum direction (phase_direction).  Otherwise only the flagged layers are
// solved; the others' Delta rows are zeroed and the phase stops at the direction exchange
// buffer [Delta | status slots] (kp_direction_buffer), which the ranks sum-all-reduce —
// every layer is owned by exactly one rank, so the sum is that rank's Delta bit for bit —
// before phase_direction.
int phase_direction(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                    bool merge_slots);

int phase_precondition(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                       const int32_t* owned) {
  const Plan& P = c.P;
  double* red = c.at(P.o_red);
  const double Ng = cfg->n_interior_global, Nbg = cfg->n_boundary_global;
  const double ema = cfg->ema;
  kp_context* ctx = c.ctx;
  auto pair_small = [&](int l, int k) { return (k == 0 ? P.p[l] : P.q[l]) <= small_eig_max_n(); };
  // early layers: their factors were completed (c.early: ctx->layer_ev) before the end of the
  // accumulate phase; their EMA and eigenproblems start on the side streams right then
  std::vector<char> early(P.L, 0);
  if (c.early && !owned) {
    KP_TRY(ensure_side_streams(ctx, 2 * P.L + 2));
    for (int l = 0; l < P.L; ++l) early[l] = !pair_small(l, 0) || !pair_small(l, 1);
  }
  {  // EMA of the normalised factor sums (curvature.py:79-85, 112-115, 133-134), one launch
    FinalizeJobs fj{};
    for (int l = 0; l < P.L; ++l) {
      FinalizeJobs lj{};
      FinalizeJobs& j = early[l] ? lj : fj;
      j.job[j.n++] = FinalizeJob{red + P.r_aint + P.fa[l], st->a_int + P.fa[l], P.p[l], Ng * P.S,
                                 l == 0 ? P.d : 0, Ng};
      j.job[j.n++] = FinalizeJob{red + P.r_bint + P.fb[l], st->b_int + P.fb[l], P.q[l], Ng, 0, 0.0};
      j.job[j.n++] = FinalizeJob{red + P.r_abnd + P.fa[l], st->a_bnd + P.fa[l], P.p[l], Nbg, 0, 0.0};
      j.job[j.n++] = FinalizeJob{red + P.r_bbnd + P.fb[l], st->b_bnd + P.fb[l], P.q[l], Nbg, 0, 0.0};
      if (early[l]) {  // this layer's EMA on its A-side stream, after its contractions
        cudaStream_t s2 = ctx->side[2 * l];
        KP_CUDA_TRY(cudaStreamWaitEvent(s2, ctx->layer_ev[l], 0));
        launch_factor_finalize_grouped(lj, ema, s2);
        KP_CUDA_TRY(cudaEventRecord(ctx->fin_ev[l], s2));
      }
    }
    if (fj.n > 0) launch_factor_finalize_grouped(fj, ema, c.s);
    for (int l = 0; l < P.L; ++l)  // the one-launch small solver reads every layer's factors
      if (early[l]) KP_CUDA_TRY(cudaStreamWaitEvent(c.s, ctx->fin_ev[l], 0));
  }
  double* grad = c.at(P.o_grad);
  launch_grad_finalize(red + P.r_gint, red + P.r_gbnd, Ng, Nbg, grad, P.D, c.s);
  launch_losses(red + P.r_ss, Ng, Nbg, out->scalars, c.s);
  double* delta = c.at(P.o_delta);
  const double lam = cfg->damping;
  // The 2L generalised eigenproblems are independent: fan out over side streams (A and B
  // factor pair of layer l on streams 2l and 2l+1), combine on 2l, join back.
  // Factor pairs up to small_eig_max_n(): on-device Cholesky + Jacobi solver, all of them in
  // one launch on the main stream (plus one combine launch for the layers whose two pairs are
  // both small).  Larger pairs: the device route of gen_eig_pair on the pair's own side
  // stream (blocked Cholesky / triangular solves / DMMA GEMMs and a cluster Jacobi), all
  // pairs concurrently; a layer with a larger pair is combined by DMMA GEMMs on its side
  // stream.
  bool any_big = false;
  for (int l = 0; l < P.L; ++l)
    any_big |= (!owned || owned[l]) && (!pair_small(l, 0) || !pair_small(l, 1));
  cudaEvent_t ready = nullptr, small_done = nullptr;
  if (any_big) {
    KP_TRY(ensure_side_streams(ctx, 2 * P.L + 2));
    ready = ctx->side_ev[2 * P.L];
    small_done = ctx->side_ev[2 * P.L + 1];
    KP_CUDA_TRY(cudaEventRecord(ready, c.s));
  }
  std::vector<int> big;  // layers with at least one pair outside the one-launch small solver
  struct PairWarm {
    double* t;
    int* valid;
  };
  std::vector<PairWarm> pair_warm(2 * P.L, PairWarm{nullptr, nullptr});
  // warm-start cache for the small pairs (re-keyed when shapes or factor buffers change)
  bool warm_reset = false;
  {
    std::vector<unsigned char> key;
    auto put = [&](const void* p, size_t n) {
      const unsigned char* b = static_cast<const unsigned char*>(p);
      key.insert(key.end(), b, b + n);
    };
    size_t need = 0;
    for (int l = 0; l < P.L; ++l) {
      put(&P.p[l], sizeof(int));
      put(&P.q[l], sizeof(int));
      for (int k = 0; k < 2; ++k) {
        const size_t nn = (size_t)(k == 0 ? P.p[l] : P.q[l]);
        // small pairs keep T and a scratch matrix, the others their previous T^T
        need += (pair_small(l, k) ? 2 : 1) * nn * nn;
      }
    }
    put(&st->a_int, sizeof(double*));
    put(&st->b_int, sizeof(double*));
    put(&st->a_bnd, sizeof(double*));
    put(&st->b_bnd, sizeof(double*));
    if (key != ctx->warm_key) {
      if (need + 32 > ctx->warm_cap) {
        if (ctx->warm_buf) {
          KP_CUDA_TRY(cudaDeviceSynchronize());
          KP_CUDA_TRY(cudaFree(ctx->warm_buf));
        }
        ctx->warm_buf = nullptr;
        ctx->warm_cap = 0;
        ctx->warm_flags = nullptr;
        KP_CUDA_TRY(cudaMalloc(&ctx->warm_buf, sizeof(double) * (need + 32)));
        ctx->warm_cap = need + 32;
        ctx->warm_flags = reinterpret_cast<int*>(ctx->warm_buf + need);
      }
      KP_CUDA_TRY(cudaMemsetAsync(ctx->warm_flags, 0, sizeof(int) * 64, c.s));
      ctx->warm_key = key;
      // the larger pairs read their flags on side streams that (for early layers) wait
      // only on their own factors: order them after this reset
      if (!ctx->warm_ev) KP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->warm_ev, cudaEventDisableTiming));
      KP_CUDA_TRY(cudaEventRecord(ctx->warm_ev, c.s));
      warm_reset = true;
    }
  }
  {
    size_t woff = 0;
    int wjob = 0;
    auto warm = [&](SmallEigJob& j) {
      j.warm_t = ctx->warm_buf + woff;
      j.warm_scratch = ctx->warm_buf + woff + (size_t)j.n * j.n;
      j.warm_valid = ctx->warm_flags + wjob++;
      woff += 2 * (size_t)j.n * j.n;
    };
    SmallEigJobs ej{};
    SmallCombineJobs cj{};
    int ne = 0, nc = 0, maxn = 1;
    for (int l = 0; l < P.L; ++l) {
      int* info = reinterpret_cast<int*>(c.at(P.k_info[l]));
      const bool sa = pair_small(l, 0), sb = pair_small(l, 1);
      if (owned && !owned[l]) {  // another rank solves this layer; keep warm slots stable
        SmallEigJob skip{};
        if (sa) {
          skip.n = P.p[l];
          warm(skip);
        }
        if (sb) {
          skip.n = P.q[l];
          warm(skip);
        }
        KP_CUDA_TRY(cudaMemsetAsync(delta + P.th[l], 0, sizeof(double) * P.p[l] * P.q[l], c.s));
        continue;
      }
      if (sa) {
        ej.job[ne++] = SmallEigJob{P.p[l], st->a_int + P.fa[l], st->a_bnd + P.fa[l], lam,
                                   c.at(P.k_A1[l]), c.at(P.k_la[l]), info, sb ? 0 : 1};
        warm(ej.job[ne - 1]);
        maxn = std::max(maxn, P.p[l]);
      }
      if (sb) {
        ej.job[ne++] = SmallEigJob{P.q[l], st->b_int + P.fb[l], st->b_bnd + P.fb[l], lam,
                                   c.at(P.k_B1[l]), c.at(P.k_lb[l]), info + 1, sa ? 0 : 1};
        warm(ej.job[ne - 1]);
        maxn = std::max(maxn, P.q[l]);
      }
      if (sa && sb)
        cj.job[nc++] = SmallCombineJob{P.p[l], P.q[l], grad + P.th[l], c.at(P.k_A1[l]),
                                       c.at(P.k_B1[l]), c.at(P.k_la[l]), c.at(P.k_lb[l]),
                                       c.at(P.k_T1[l]), c.at(P.k_T2[l]), delta + P.th[l], -1.0};
      else
        big.push_back(l);
    }
    // warm-start slots of the larger pairs follow the small ones (owned or not: stable)
    for (int l = 0; l < P.L; ++l)
      for (int k = 0; k < 2; ++k) {
        if (pair_small(l, k)) continue;
        const size_t n = (size_t)(k == 0 ? P.p[l] : P.q[l]);
        pair_warm[2 * l + k] = PairWarm{ctx->warm_buf + woff, ctx->warm_flags + wjob++};
        woff += n * n;
      }
    launch_gen_eig_small(ej, ne, maxn, out->status, c.s);
    if (any_big) KP_CUDA_TRY(cudaEventRecord(small_done, c.s));
    launch_kron_combine_small(cj, nc, c.s);
  }
  // pairs above the one-launch small solver: the device route (gen_eig_pair) on the pair's
  // side stream, then each such layer is combined on its A-side stream
  for (int l : big)
    for (int k = 0; k < 2; ++k) {
      if (pair_small(l, k)) continue;
      cudaStream_t s = ctx->side[2 * l + k];
      KP_CUDA_TRY(cudaStreamWaitEvent(s, early[l] ? ctx->fin_ev[l] : ready, 0));
      if (warm_reset) KP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->warm_ev, 0));
      int* info = reinterpret_cast<int*>(c.at(P.k_info[l])) + k;
      KP_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int), s));
      KP_TRY(gen_eig_pair(s, k == 0 ? P.p[l] : P.q[l],
                          k == 0 ? st->a_int + P.fa[l] : st->b_int + P.fb[l],
                          k == 0 ? st->a_bnd + P.fa[l] : st->b_bnd + P.fb[l], lam,
                          c.at(k == 0 ? P.k_A1[l] : P.k_B1[l]), c.at(k == 0 ? P.k_A2[l] : P.k_B2[l]),
                          c.at(k == 0 ? P.k_la[l] : P.k_lb[l]), c.at(k == 0 ? P.k_wa[l] : P.k_wb[l]),
                          info, reinterpret_cast<int*>(c.at(P.k_info[l])) + 2 + 2 * k,
                          pair_warm[2 * l + k].t, pair_warm[2 * l + k].valid));
      KP_CUDA_TRY(cudaEventRecord(ctx->side_ev[2 * l + k], s));
    }
  for (int l : big) {
    cudaStream_t s = ctx->side[2 * l];
    if (!pair_small(l, 1)) KP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->side_ev[2 * l + 1], 0));
    if (pair_small(l, 0) || pair_small(l, 1)) KP_CUDA_TRY(cudaStreamWaitEvent(s, small_done, 0));
    if (early[l]) KP_CUDA_TRY(cudaStreamWaitEvent(s, ready, 0));  // the finalized gradient
    launch_eig_status(c.at(P.k_la[l]), P.p[l], c.at(P.k_lb[l]), P.q[l],
                      reinterpret_cast<int*>(c.at(P.k_info[l])), out->status, s);
    kron_combine(s, P.p[l], P.q[l], c.at(P.k_A1[l]), c.at(P.k_la[l]), c.at(P.k_B1[l]),
                 c.at(P.k_lb[l]), grad + P.th[l], delta + P.th[l], -1.0, c.at(P.k_T1[l]),
                 c.at(P.k_T2[l]));
    KP_CUDA_TRY(cudaEventRecord(ctx->side_ev[2 * l], s));
  }
  for (int l : big) KP_CUDA_TRY(cudaStreamWaitEvent(c.s, ctx->side_ev[2 * l], 0));
  if (owned) {
    launch_status_slots(out->status, c.at(P.o_dslot), c.s);
    return KP_OK;
  }
  return phase_direction(c, cfg, st, out, false);
}

// delta^ = Delta + mu prev (optim.py:254) and the optional grad / Delta outputs; after a
// distributed solve the status slots summed over ranks are merged into *out->status first.
int phase_direction(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                    bool merge_slots) {
  const Plan& P = c.P;
  double* grad = c.at(P.o_grad);
  double* delta = c.at(P.o_delta);
  if (merge_slots) launch_slots_status(c.at(P.o_dslot), out->status, c.s);
  launch_axpy_out(delta, st->prev_update, cfg->momentum, c.at(P.o_dir), P.D, c.s);
  if (out->grad) KP_CUDA_TRY(cudaMemcpyAsync(out->grad, grad, sizeof(double) * P.D,
                                             cudaMemcpyDeviceToDevice, c.s));
  if (out->delta) KP_CUDA_TRY(cudaMemcpyAsync(out->delta, delta, sizeof(double) * P.D,
                                              cudaMemcpyDeviceToDevice, c.s));
  return KP_OK;
}

int phase_linesearch(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, const kp_batch* bt) {
  const Plan& P = c.P;
  const TaylorDims tdi{P.S, P.d, true};
  const TaylorDims tdb{1, 0, false};
  double* thc = c.at(P.o_thc);
  double* dir = c.at(P.o_dir);
  for (int k0 = 0; k0 < P.ncand; k0 += P.Bc) {
    const int nb = std::min(P.Bc, P.ncand - k0);
    launch_candidate(st->theta, dir, cfg->ls_min_exp + k0, thc, P.D, P.wpc, c.at(P.o_wpadc), c.s,
                     nb);
    if (P.L >= 2)
      launch_prep_layer0(thc, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_w0tc), c.at(P.o_q0c), c.s, nb,
                         P.D);
    for (int64_t n0 = 0; n0 < P.N; n0 += P.Nc) {
      const int64_t nc = std::min(P.Nc, P.N - n0);
      ResidualIn ri{bt->r0 + n0, bt->seeds + n0 * P.S, nullptr};
      if (bt->quad) ri.quad = bt->quad + n0 * P.d;
      forward_loss(c, thc, c.at(P.o_wpadc), bt->x_int + n0 * P.d, nc, tdi, bt->coeff_diag,
                   c.at(P.o_ping), c.at(P.o_pong), ri, c.at(P.o_rls) + k0 * P.N + n0, nullptr, true,
                   nb, P.N);
    }
    ResidualIn rb{nullptr, nullptr, bt->targets};
    forward_loss(c, thc, c.at(P.o_wpadc), bt->x_bnd, P.Nb, tdb, bt->coeff_diag, c.at(P.o_bping),
                 c.at(P.o_bpong), rb, c.at(P.o_rbls) + k0 * P.Nb, nullptr, true, nb, P.Nb);
  }
  double* ls = c.at(P.o_ls);
  launch_sumsq(c.at(P.o_rls), P.N, P.N, P.ncand, ls, 2, c.s);
  launch_sumsq(c.at(P.o_rbls), P.Nb, P.Nb, P.ncand, ls + 1, 2, c.s);
  return KP_OK;
}

int phase_update(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, kp_step_out* out) {
  const Plan& P = c.P;
  launch_argmin_update(c.at(P.o_ls), P.ncand, cfg->ls_min_exp, cfg->n_interior_global,
                       cfg->n_boundary_global, st->theta, st->prev_update, c.at(P.o_dir), P.D,
                       out->scalars, out->ls_losses, out->status, cfg->momentum, c.s);
  return KP_OK;
}


// ---------------------------------------------------------------------------
// KFAC* (reference src/optim.py:266-320): Gramian-vector products G v for v in {Delta,
// prev} without the per-sample Jacobian rows.  With J_n the residual Jacobian of point n,
// (J v)_n = sum_l sum_s <gbar_{n,s,l}, V_l zhat_{n,s,l}> and G v = sum_n (J v)_n J_n^T / N
// (+ the boundary term), i.e. the gradient contraction with weights (J v)_n.

// jv[n] = (J v)_n for the points of one pass (states in b, seeds/ones in gl_last); V's padded
// weights and V0^T must be prepared in o_wpadv / o_v0t.
void jvp_pass(const Ctx& c, const double* x, int64_t n, const TaylorDims& td, const StateBufs& b,
              const double* gl_last, const double* V, double* jv) {
  const Plan& P = c.P;
  const int L = P.L;
  cudaMemsetAsync(jv, 0, sizeof(double) * n, c.s);
  const double* wv = c.at(P.o_wpadv);
  for (int l = 0; l < L; ++l) {
    const int q = P.q[l];
    const double* G = (l == L - 1) ? gl_last : b.gout[l];
    if (l == 0) {
      // value rows: y = V0[:, :d] x + V0[:, d]   (n x q)
      double* y0 = c.at(P.o_pong);
      GemmNT g{x, P.d, V + P.th[0], P.p[0], y0, q, n, q, P.d, V + P.th[0] + P.d, P.p[0], 1};
      launch_gemm_nt(g, c.s);
      if (td.taylor) launch_jvp_layer0(G, y0, c.at(P.o_v0t), n, P.d, q, jv, c.s);
      else launch_rowdot_accum(G, y0, q, n, 1, jv, c.s);
    } else {
      if (q == 1 && launch_jvp_last(G, b.post[l], P.h[l], P.h[l], wv + P.wo[l],
                                    V + P.th[l] + P.h[l], n, td.S, jv, c.s))
        continue;
      double* y = c.at(P.o_ping);
      GemmNT g{b.post[l], P.h[l], wv + P.wo[l], P.h[l], y, q, n * td.S, q, P.h[l],
               V + P.th[l] + P.h[l], P.p[l], td.S};
      launch_gemm_nt(g, c.s);
      launch_rowdot_accum(G, y, q, n, td.S, jv, c.s);
    }
  }
}

// Gramian-vector products of vectors [v0, v1) of {Delta, prev}: each vector owns its two
// slots of o_gv (interior, boundary), so the vectors can be computed in either order.
static int star_gvp_range(const Ctx& c, const kp_kfac_config* cfg, kp_state* st,
                          const kp_batch* bt, int v0, int v1) {
  const Plan& P = c.P;
  double* gv = c.at(P.o_gv);
  KP_CUDA_TRY(cudaMemsetAsync(gv + 2 * v0 * P.D, 0, sizeof(double) * 2 * (v1 - v0) * P.D, c.s));
  const TaylorDims tdi{P.S, P.d, true};
  const TaylorDims tdb{1, 0, false};
  const bool single = P.Nc >= P.N;  // else the interior states are recomputed per chunk
  const double* vecs[2] = {c.at(P.o_delta), st->prev_update};
  const StateBufs bi = interior_bufs(c);
  auto prep = [&](const double* v) {
    launch_candidate(v, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpadv), c.s);
    if (P.L >= 2)
      launch_prep_layer0(v, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_v0t), c.at(P.o_vq0), c.s);
  };
  for (int64_t n0 = 0; n0 < P.N; n0 += P.Nc) {
    const int64_t nc = std::min(P.Nc, P.N - n0);
    const double* x = bt->x_int + n0 * P.d;
    const double* seeds = bt->quad ? c.at(P.o_seeds_eff) + n0 * P.S : bt->seeds + n0 * P.S;
    if (!single) {
      launch_candidate(st->theta, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpad), c.s);
      if (P.L >= 2)
        launch_prep_layer0(st->theta, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_w0t), c.at(P.o_q0),
                           c.s);
      ResidualIn ri{bt->r0 + n0, bt->seeds + n0 * P.S, nullptr};
      if (bt->quad) {
        ri.quad = bt->quad + n0 * P.d;
        ri.seeds_out = c.at(P.o_seeds_eff) + n0 * P.S;
      }
      forward_store(c, st->theta, c.at(P.o_wpad), x, nc, tdi, bt->coeff_diag, bi, ri,
                    c.at(P.o_r) + n0, nullptr);
      backward(c, st->theta, nc, tdi, bt->coeff_diag, bi, seeds);
    }
    for (int v = v0; v < v1; ++v) {
      prep(vecs[v]);
      jvp_pass(c, x, nc, tdi, bi, seeds, vecs[v], c.at(P.o_jv));
      for (int l = 0; l < P.L; ++l)
        contract_grad_layer(c, x, nc, tdi, bi, seeds, c.at(P.o_jv), gv + (2 * v) * P.D, l);
    }
  }
  const StateBufs bb = boundary_bufs(c);
  for (int v = v0; v < v1; ++v) {
    prep(vecs[v]);
    jvp_pass(c, bt->x_bnd, P.Nb, tdb, bb, c.at(P.o_ones), vecs[v], c.at(P.o_jvb));
    for (int l = 0; l < P.L; ++l)
      contract_grad_layer(c, bt->x_bnd, P.Nb, tdb, bb, c.at(P.o_ones), c.at(P.o_jvb),
                          gv + (2 * v + 1) * P.D, l);
  }
  return KP_OK;
}

int phase_star_gvp(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, const kp_batch* bt) {
  return star_gvp_range(c, cfg, st, bt, 0, 2);
}

int phase_star_update(const Ctx& c, const kp_kfac_config* cfg, kp_state* st, kp_step_out* out) {
  const Plan& P = c.P;
  const double Ng = cfg->n_interior_global, Nbg = cfg->n_boundary_global;
  double* gv = c.at(P.o_gv);
  // G v = J_int^T J_int v / N + J_bnd^T J_bnd v / Nb   (curvature.py:253-260)
  launch_grad_finalize(gv, gv + P.D, Ng, Nbg, c.at(P.o_gvd), P.D, c.s);
  launch_grad_finalize(gv + 2 * P.D, gv + 3 * P.D, Ng, Nbg, c.at(P.o_gvp), P.D, c.s);
  const double* d = c.at(P.o_delta);
  const double* p = st->prev_update;
  const double* g = c.at(P.o_grad);
  DotJobs dj{{d, d, d, p, d, d, p, p}, {c.at(P.o_gvd), d, g, p, c.at(P.o_gvp), p, c.at(P.o_gvp), g}};
  launch_dots(dj, 8, P.D, c.at(P.o_dots), c.s);
  launch_star_solve_update(c.at(P.o_dots), cfg->model_damping > 0.0 ? cfg->model_damping : cfg->damping, st->theta, st->prev_update, d, P.D,
                           out->scalars, out->status, c.s);
  return KP_OK;
}

int validate_cfg(const kp_problem* pr, const kp_kfac_config* cfg) {
  if (!cfg) return KP_ERR_INVALID;
  if (!(cfg->ema >= 0.0 && cfg->ema < 1.0)) return KP_ERR_INVALID;
  if (!(cfg->damping > 0.0)) return KP_ERR_INVALID;
  if (!(cfg->momentum >= 0.0)) return KP_ERR_INVALID;
  if (cfg->ls_max_exp - cfg->ls_min_exp + 1 != pr->n_candidates) return KP_ERR_INVALID;
  if (!(cfg->n_interior_global >= 1.0) || !(cfg->n_boundary_global >= 1.0)) return KP_ERR_INVALID;
  return KP_OK;
}

int cached_plan(kp_context* ctx, const kp_problem* pr, Plan& P) {
  if (ctx->plan_valid && std::memcmp(&ctx->plan_key, pr, sizeof(kp_problem)) == 0 &&
      ctx->plan_blob.size() == sizeof(Plan)) {
    std::memcpy(&P, ctx->plan_blob.data(), sizeof(Plan));
    return KP_OK;
  }
  KP_TRY(make_plan(ctx, pr, P));
  ctx->plan_key = *pr;
  ctx->plan_blob.resize(sizeof(Plan));
  std::memcpy(ctx->plan_blob.data(), &P, sizeof(Plan));
  ctx->plan_valid = true;
  return KP_OK;
}

int prepare(kp_context* ctx, const kp_problem* pr, Plan& P, size_t ws_bytes) {
  if (!ctx || !pr) return KP_ERR_INVALID;
  KP_TRY(cached_plan(ctx, pr, P));
  if ((size_t)P.total * sizeof(double) > ws_bytes) return KP_ERR_WORKSPACE;
  return KP_OK;
}

}  // namespace

// ===========================================================================
// extern "C"

extern "C" {

int32_t kp_abi_version(void) { return KP_ABI_VERSION; }

const char* kp_status_string(int32_t s) {
  switch (s) {
    case KP_OK: return "ok";
    case KP_ERR_INVALID: return "invalid argument";
    case KP_ERR_NOT_PSD: return "matrix not positive (semi)definite";
    case KP_ERR_LINE_SEARCH: return "loss is non-finite at every line-search step size";
    case KP_ERR_NONFINITE: return "parameters became non-finite during the step";
    case KP_ERR_CUDA: return "CUDA failure";
    case KP_ERR_EIG: return "eigensolver did not converge";
    case KP_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int32_t kp_context_create(int32_t device, kp_context** out) {
  if (!out) return KP_ERR_INVALID;
  KP_CUDA_TRY(cudaSetDevice(device));
  kp_context* c = new kp_context();
  c->device = device;
  *out = c;
  return KP_OK;
}

int32_t kp_context_destroy(kp_context* c) {
  if (!c) return KP_OK;
  if (c->warm_buf) {
    cudaDeviceSynchronize();
    cudaFree(c->warm_buf);
  }
  if (c->warm_ev) cudaEventDestroy(c->warm_ev);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->cap_stream) {
    cudaStreamSynchronize(c->cap_stream);
    cudaStreamDestroy(c->cap_stream);
  }
  if (c->cap_in) cudaEventDestroy(c->cap_in);
  if (c->cap_out) cudaEventDestroy(c->cap_out);
  for (size_t k = 0; k < c->side.size(); ++k) {
    cudaStreamSynchronize(c->side[k]);
    cudaEventDestroy(c->side_ev[k]);
    cudaStreamDestroy(c->side[k]);
  }
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->layer_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->fin_ev) cudaEventDestroy(e);
  delete c;
  return KP_OK;
}

int32_t kp_profile_enable(kp_context* c, int32_t enable) {
  if (!c) return KP_ERR_INVALID;
  c->profile = enable != 0;
  c->ev_used = 0;
  c->prof_flops = 0.0;
  c->prof_launches = 0;
  c->ev_hbm_used = 0;
  c->prof_hbm_bytes = 0.0;
  c->prof_hbm_launches = 0;
  for (int k = 0; k < 2; ++k) {
    c->ev_cat_used[k] = 0;
    c->prof_cat_work[k] = 0.0;
    c->prof_cat_launches[k] = 0;
  }
  return KP_OK;
}

int32_t kp_profile_read_cat(kp_context* c, int32_t cat, double* ms_out, double* work,
                            int64_t* launches) {
  if (!c || cat < 0 || cat > 1) return KP_ERR_INVALID;
  double ms = 0.0;
  for (size_t k = 0; k + 1 < c->ev_cat_used[cat]; k += 2) {
    KP_CUDA_TRY(cudaEventSynchronize(c->ev_cat[cat][k + 1]));
    float t = 0.f;
    KP_CUDA_TRY(cudaEventElapsedTime(&t, c->ev_cat[cat][k], c->ev_cat[cat][k + 1]));
    ms += t;
  }
  if (ms_out) *ms_out = ms;
  if (work) *work = c->prof_cat_work[cat];
  if (launches) *launches = c->prof_cat_launches[cat];
  c->ev_cat_used[cat] = 0;
  c->prof_cat_work[cat] = 0.0;
  c->prof_cat_launches[cat] = 0;
  return KP_OK;
}

int32_t kp_solver_sweeps(int32_t* small_max, int32_t* mid_max, int32_t* large_max,
                         int32_t reset) {
  if (small_max) *small_max = small_eig_sweeps_used(reset != 0);
  if (mid_max) *mid_max = mid_eig_sweeps_used(reset != 0);
  if (large_max) *large_max = large_eig_sweeps_used(reset != 0);
  return KP_OK;
}

int32_t kp_profile_read_hbm(kp_context* c, double* ms_out, double* bytes, int64_t* launches) {
  if (!c) return KP_ERR_INVALID;
  double ms = 0.0;
  for (size_t k = 0; k + 1 < c->ev_hbm_used; k += 2) {
    KP_CUDA_TRY(cudaEventSynchronize(c->ev_hbm[k + 1]));
    float t = 0.f;
    KP_CUDA_TRY(cudaEventElapsedTime(&t, c->ev_hbm[k], c->ev_hbm[k + 1]));
    ms += t;
  }
  if (ms_out) *ms_out = ms;
  if (bytes) *bytes = c->prof_hbm_bytes;
  if (launches) *launches = c->prof_hbm_launches;
  c->ev_hbm_used = 0;
  c->prof_hbm_bytes = 0.0;
  c->prof_hbm_launches = 0;
  return KP_OK;
}

int32_t kp_profile_read(kp_context* c, double* gemm_ms, double* gemm_flops, int64_t* launches,
                        int64_t* kernel_launches) {
  if (!c) return KP_ERR_INVALID;
  double ms = 0.0;
  for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
    KP_CUDA_TRY(cudaEventSynchronize(c->ev[k + 1]));
    float t = 0.f;
    KP_CUDA_TRY(cudaEventElapsedTime(&t, c->ev[k], c->ev[k + 1]));
    ms += t;
  }
  if (gemm_ms) *gemm_ms = ms;
  if (gemm_flops) *gemm_flops = c->prof_flops;
  if (launches) *launches = c->prof_launches;
  if (kernel_launches) *kernel_launches = kp::launch_count();
  c->ev_used = 0;
  c->prof_flops = 0.0;
  c->prof_launches = 0;
  return KP_OK;
}

int64_t kp_param_count(const kp_net* net) {
  if (check_net(net) != KP_OK) return -1;
  int64_t D = 0;
  for (int l = 0; l < net->n_layers; ++l) D += (int64_t)(net->widths[l] + 1) * net->widths[l + 1];
  return D;
}

int64_t kp_factor_count(const kp_net* net, int32_t which) {
  if (check_net(net) != KP_OK) return -1;
  int64_t n = 0;
  for (int l = 0; l < net->n_layers; ++l) {
    const int64_t k = which == 0 ? net->widths[l] + 1 : net->widths[l + 1];
    n += k * k;
  }
  return n;
}

int32_t kp_workspace_bytes(kp_context* ctx, const kp_problem* pr, size_t* bytes) {
  if (!ctx || !pr || !bytes) return KP_ERR_INVALID;
  Plan P;
  KP_TRY(cached_plan(ctx, pr, P));
  *bytes = (size_t)P.total * sizeof(double);
  return KP_OK;
}

int32_t kp_bytes_per_interior_point(const kp_net* net, size_t* bytes) {
  if (!bytes) return KP_ERR_INVALID;
  KP_TRY(check_net(net));
  *bytes = (size_t)per_point_doubles(net) * sizeof(double);
  return KP_OK;
}

int32_t kp_init_state(kp_context* ctx, const kp_net* net, kp_state* st, int32_t init_identity,
                      void* stream) {
  if (!ctx || !st) return KP_ERR_INVALID;
  KP_TRY(check_net(net));
  cudaStream_t s = (cudaStream_t)stream;
  const double v = init_identity ? 1.0 : 0.0;
  int64_t oa = 0, ob = 0, D = 0;
  for (int l = 0; l < net->n_layers; ++l) {
    const int p = net->widths[l] + 1, q = net->widths[l + 1];
    launch_identity(st->a_int + oa, p, v, s);
    launch_identity(st->a_bnd + oa, p, v, s);
    launch_identity(st->b_int + ob, q, v, s);
    launch_identity(st->b_bnd + ob, q, v, s);
    oa += (int64_t)p * p;
    ob += (int64_t)q * q;
    D += (int64_t)p * q;
  }
  KP_CUDA_TRY(cudaMemsetAsync(st->prev_update, 0, sizeof(double) * D, s));
  if (ctx->warm_flags)  // re-initialised factors: cold-start the eigensolver
    KP_CUDA_TRY(cudaMemsetAsync(ctx->warm_flags, 0, sizeof(int) * 64, s));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_reduce_buffer(kp_context* ctx, const kp_problem* pr, void* ws, double** ptr,
                         int64_t* count) {
  Plan P;
  KP_TRY(cached_plan(ctx, pr, P));
  *ptr = static_cast<double*>(ws) + P.o_red;
  *count = P.r_count;
  return KP_OK;
}

int32_t kp_direction_buffer(kp_context* ctx, const kp_problem* pr, void* ws, double** ptr,
                            int64_t* count) {
  Plan P;
  KP_TRY(cached_plan(ctx, pr, P));
  *ptr = static_cast<double*>(ws) + P.o_delta;
  *count = P.D + 8;
  return KP_OK;
}

int32_t kp_linesearch_buffer(kp_context* ctx, const kp_problem* pr, void* ws, double** ptr,
                             int64_t* count) {
  Plan P;
  KP_TRY(cached_plan(ctx, pr, P));
  *ptr = static_cast<double*>(ws) + P.o_ls;
  *count = 2LL * P.ncand;
  return KP_OK;
}


// Dense operator coefficients (kp_batch.coeff_rot != NULL): the engine works in the
// eigenbasis of c, so the gradient part of the seeds is rotated in once per call,
// seeds'[1..d] = Q^T seeds[1..d] (into the workspace), and the rotated batch is used.
int rotated_batch(Ctx& c, const kp_batch* bt, kp_batch& tmp, const kp_batch*& use) {
  use = bt;
  if (!bt || !bt->coeff_rot) return KP_OK;
  if (bt->quad) return KP_ERR_INVALID;  // quadratic-in-grad residuals need coordinate rows
  const Plan& P = c.P;
  c.rot = bt->coeff_rot;
  tmp = *bt;
  if (P.N > 0 && bt->seeds) {
    double* s = c.at(P.o_seeds_eff);
    KP_CUDA_TRY(cudaMemcpyAsync(s, bt->seeds, sizeof(double) * P.N * P.S, cudaMemcpyDeviceToDevice,
                                c.s));
    launch_rotate_rows(s + 1, P.S, P.N, P.d, bt->coeff_rot, 1, c.s);
    tmp.seeds = s;
  }
  use = &tmp;
  return KP_OK;
}

#define KP_PHASE_PROLOGUE                                            \
  Plan P;                                                            \
  KP_TRY(prepare(ctx, prob, P, ws_bytes));                           \
  KP_TRY(validate_cfg(prob, cfg));                                   \
  if (!st || !out || !out->scalars || !out->status) return KP_ERR_INVALID; \
  Ctx c{ctx, P, static_cast<double*>(ws), (cudaStream_t)stream};

int32_t kp_kfac_phase_accumulate(kp_context* ctx, const kp_problem* prob,
                                 const kp_kfac_config* cfg, kp_state* st, const kp_batch* bt,
                                 kp_step_out* out, void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!bt) return KP_ERR_INVALID;
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  KP_CUDA_TRY(cudaMemsetAsync(out->status, 0, sizeof(int32_t), c.s));
  KP_TRY(phase_accumulate(c, cfg, st, bt));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_phase_precondition(kp_context* ctx, const kp_problem* prob,
                                   const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                   void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  KP_TRY(phase_precondition(c, cfg, st, out, nullptr));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_phase_precondition_owned(kp_context* ctx, const kp_problem* prob,
                                         const kp_kfac_config* cfg, kp_state* st,
                                         kp_step_out* out, const int32_t* owned_layers,
                                         void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!owned_layers) return KP_ERR_INVALID;
  KP_TRY(phase_precondition(c, cfg, st, out, owned_layers));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_phase_direction(kp_context* ctx, const kp_problem* prob,
                                const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  KP_TRY(phase_direction(c, cfg, st, out, true));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_phase_linesearch(kp_context* ctx, const kp_problem* prob,
                                 const kp_kfac_config* cfg, kp_state* st, const kp_batch* bt,
                                 kp_step_out* out, void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!bt) return KP_ERR_INVALID;
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  KP_TRY(phase_linesearch(c, cfg, st, bt));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_phase_update(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                             kp_state* st, kp_step_out* out, void* ws, size_t ws_bytes,
                             void* stream) {
  KP_PHASE_PROLOGUE
  KP_TRY(phase_update(c, cfg, st, out));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

// Early preconditioning for single-call steps (Ctx::early): per-layer contractions (not the
// grouped small-network launch), at least one factor pair outside the one-launch small
// solver and none above 288 (c4).  KP_EARLY_PRECOND=0 turns it off (measurements).
static int setup_early(Ctx& c) {
  static const bool enabled = [] {
    const char* e = getenv("KP_EARLY_PRECOND");
    return !(e && atoi(e) == 0);
  }();
  const Plan& P = c.P;
  if (!enabled || P.tn_grouped) return KP_OK;
  bool any = false;
  int maxn = 0;
  for (int l = 0; l < P.L; ++l) {
    any |= std::max(P.p[l], P.q[l]) > small_eig_max_n();
    maxn = std::max(maxn, std::max(P.p[l], P.q[l]));
  }
  // Pairs above 288 run 16-CTA clusters for tens of milliseconds (c5: 512-769); started
  // during the accumulate phase they take SMs from its contractions and the step gets
  // slower (c5 N = 16384: 4523 vs 4483 ms per step), so they wait for the phase to end.
  static const bool force = [] {  // KP_EARLY_PRECOND=2: also for pairs above 288
    const char* e = getenv("KP_EARLY_PRECOND");
    return e && atoi(e) == 2;
  }();
  if (!any || (maxn > 288 && !force)) return KP_OK;
  KP_TRY(ensure_side_streams(c.ctx, 2 * P.L + 2));
  c.early = true;
  return KP_OK;
}

int32_t kp_kfac_step(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                     kp_state* st, const kp_batch* bt, kp_step_out* out, void* ws,
                     size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!bt) return KP_ERR_INVALID;
  KP_TRY(setup_early(c));
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  KP_CUDA_TRY(cudaMemsetAsync(out->status, 0, sizeof(int32_t), c.s));
  KP_TRY(phase_accumulate(c, cfg, st, bt));
  KP_TRY(phase_precondition(c, cfg, st, out, nullptr));
  KP_TRY(phase_linesearch(c, cfg, st, bt));
  KP_TRY(phase_update(c, cfg, st, out));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}


int32_t kp_gvp_buffer(kp_context* ctx, const kp_problem* pr, void* ws, double** ptr,
                      int64_t* count) {
  Plan P;
  KP_TRY(cached_plan(ctx, pr, P));
  *ptr = static_cast<double*>(ws) + P.o_gv;
  *count = 4 * P.D;
  return KP_OK;
}

int32_t kp_kfac_star_phase_gvp(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                               kp_state* st, const kp_batch* bt, kp_step_out* out, void* ws,
                               size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!bt) return KP_ERR_INVALID;
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  KP_TRY(phase_star_gvp(c, cfg, st, bt));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_star_phase_update(kp_context* ctx, const kp_problem* prob,
                                  const kp_kfac_config* cfg, kp_state* st, kp_step_out* out,
                                  void* ws, size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  KP_TRY(phase_star_update(c, cfg, st, out));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kfac_star_step(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                          kp_state* st, const kp_batch* bt, kp_step_out* out, void* ws,
                          size_t ws_bytes, void* stream) {
  KP_PHASE_PROLOGUE
  if (!bt) return KP_ERR_INVALID;
  KP_TRY(setup_early(c));
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  KP_CUDA_TRY(cudaMemsetAsync(out->status, 0, sizeof(int32_t), c.s));
  KP_TRY(phase_accumulate(c, cfg, st, bt));
  // G prev needs no Delta: with early preconditioning (the large eigenproblems on side
  // streams / host threads) and the states of a single pass still resident, it is issued
  // before the preconditioner so that the GPU computes it while the solves run
  static const bool ahead_on = [] {  // KP_STAR_AHEAD=0: Delta first (measurements)
    const char* e = getenv("KP_STAR_AHEAD");
    return !(e && atoi(e) == 0);
  }();
  const bool ahead = ahead_on && c.early && c.P.Nc >= c.P.N;
  if (ahead) KP_TRY(star_gvp_range(c, cfg, st, bt, 1, 2));
  KP_TRY(phase_precondition(c, cfg, st, out, nullptr));
  KP_TRY(star_gvp_range(c, cfg, st, bt, 0, ahead ? 1 : 2));
  KP_TRY(phase_star_update(c, cfg, st, out));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}


// Whole step (KFAC or KFAC*) replayed from a CUDA graph captured on first use.  Only when
// every factor pair is within the device solvers' range (max_pair_n) and profiling is off; otherwise identical to kp_kfac_step / kp_kfac_star_step.  The graph is
// keyed on every argument (pointers and configuration values are baked into the nodes).
int32_t kp_kfac_step_graphed(kp_context* ctx, const kp_problem* prob, const kp_kfac_config* cfg,
                             kp_state* st, const kp_batch* bt, kp_step_out* out, void* ws,
                             size_t ws_bytes, void* stream, int32_t star) {
  auto plain = [&]() {
    return star ? kp_kfac_star_step(ctx, prob, cfg, st, bt, out, ws, ws_bytes, stream)
                : kp_kfac_step(ctx, prob, cfg, st, bt, out, ws, ws_bytes, stream);
  };
  if (!ctx || !prob || !cfg || !st || !bt || !out) return KP_ERR_INVALID;
  Plan P;
  KP_TRY(prepare(ctx, prob, P, ws_bytes));
  bool capturable = !ctx->profile;
  for (int l = 0; l < P.L; ++l) capturable &= std::max(P.p[l], P.q[l]) <= max_pair_n();
  if (!capturable) return plain();
  std::vector<unsigned char> key;
  auto put = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    key.insert(key.end(), b, b + n);
  };
  put(prob, sizeof(*prob));
  put(cfg, sizeof(*cfg));
  put(st, sizeof(*st));
  put(bt, sizeof(*bt));
  put(out, sizeof(*out));
  put(&ws, sizeof(ws));
  put(&ws_bytes, sizeof(ws_bytes));
  put(&star, sizeof(star));
  cudaStream_t caller = (cudaStream_t)stream;
  if (!ctx->cap_stream) {
    KP_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    KP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->cap_in, cudaEventDisableTiming));
    KP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->cap_out, cudaEventDisableTiming));
  }
  if (key == ctx->graph_failed_key) return plain();
  if (!ctx->graph_exec || key != ctx->graph_key) {
    if (ctx->graph_exec) {
      cudaGraphExecDestroy(ctx->graph_exec);
      ctx->graph_exec = nullptr;
    }
    // one uncaptured step first: lazy one-time setup (function attributes, tensor maps)
    // must not happen inside the capture
    KP_TRY(plain());
    KP_CUDA_TRY(cudaEventRecord(ctx->cap_in, caller));
    KP_CUDA_TRY(cudaStreamWaitEvent(ctx->cap_stream, ctx->cap_in, 0));
    KP_CUDA_TRY(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    const int rc = star ? kp_kfac_star_step(ctx, prob, cfg, st, bt, out, ws, ws_bytes, ctx->cap_stream)
                        : kp_kfac_step(ctx, prob, cfg, st, bt, out, ws, ws_bytes, ctx->cap_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (rc != KP_OK || ce != cudaSuccess || !graph) {
      // not capturable (a library call refused the capture): this call's step already ran
      // uncaptured above; later calls with these arguments run plain
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      ctx->graph_failed_key = key;
      return KP_OK;
    }
    const cudaError_t ie = cudaGraphInstantiate(&ctx->graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      ctx->graph_exec = nullptr;
      cudaGetLastError();
      ctx->graph_failed_key = key;
      return KP_OK;
    }
    ctx->graph_key = key;
    KP_CUDA_TRY(cudaEventRecord(ctx->cap_out, ctx->cap_stream));
    KP_CUDA_TRY(cudaStreamWaitEvent(caller, ctx->cap_out, 0));
    return KP_OK;  // the uncaptured step above was this call's step
  }
  KP_CUDA_TRY(cudaEventRecord(ctx->cap_in, caller));
  KP_CUDA_TRY(cudaStreamWaitEvent(ctx->cap_stream, ctx->cap_in, 0));
  KP_CUDA_TRY(cudaGraphLaunch(ctx->graph_exec, ctx->cap_stream));
  KP_CUDA_TRY(cudaEventRecord(ctx->cap_out, ctx->cap_stream));
  KP_CUDA_TRY(cudaStreamWaitEvent(caller, ctx->cap_out, 0));
  return KP_OK;
}

int32_t kp_taylor_forward(kp_context* ctx, const kp_problem* prob, const double* theta,
                          const kp_batch* bt, double* value, double* gradient, double* op,
                          void* ws, size_t ws_bytes, void* stream) {
  Plan P;
  KP_TRY(prepare(ctx, prob, P, ws_bytes));
  if (!theta || !bt || !value || !gradient || !op) return KP_ERR_INVALID;
  Ctx c{ctx, P, static_cast<double*>(ws), (cudaStream_t)stream};
  const TaylorDims tdi{P.S, P.d, true};
  launch_candidate(theta, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpad), c.s);
  if (P.L >= 2)
    launch_prep_layer0(theta, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_w0t), c.at(P.o_q0), c.s);
  for (int64_t n0 = 0; n0 < P.N; n0 += P.Nc) {
    const int64_t nc = std::min(P.Nc, P.N - n0);
    ResidualIn ri{nullptr, nullptr, nullptr};
    double* u = c.at(P.o_u);
    forward_loss(c, theta, c.at(P.o_wpad), bt->x_int + n0 * P.d, nc, tdi, bt->coeff_diag, c.at(P.o_ping),
                 c.at(P.o_pong), ri, nullptr, u);
    launch_split_u(u, nc, P.d, value + n0, gradient + n0 * P.d, op + n0, c.s);
    // dense coefficients: the derivative rows are along Q[:, k]; grad u = Q g'
    if (bt->coeff_rot) launch_rotate_rows(gradient + n0 * P.d, P.d, nc, P.d, bt->coeff_rot, 0, c.s);
  }
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}


int32_t kp_mlp_forward(kp_context* ctx, const kp_problem* prob, const double* theta,
                       const double* x, double* u, void* ws, size_t ws_bytes, void* stream) {
  Plan P;
  KP_TRY(prepare(ctx, prob, P, ws_bytes));
  if (!theta || !x || !u) return KP_ERR_INVALID;
  Ctx c{ctx, P, static_cast<double*>(ws), (cudaStream_t)stream};
  const TaylorDims tdb{1, 0, false};
  launch_candidate(theta, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpad), c.s);
  ResidualIn rb{nullptr, nullptr, nullptr};
  forward_loss(c, theta, c.at(P.o_wpad), x, P.Nb, tdb, nullptr, c.at(P.o_bping), c.at(P.o_bpong),
               rb, nullptr, u);
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_evaluate_losses(kp_context* ctx, const kp_problem* prob, const double* theta,
                           const kp_batch* bt, double* losses, void* ws, size_t ws_bytes,
                           void* stream) {
  Plan P;
  KP_TRY(prepare(ctx, prob, P, ws_bytes));
  if (!theta || !bt || !losses) return KP_ERR_INVALID;
  Ctx c{ctx, P, static_cast<double*>(ws), (cudaStream_t)stream};
  kp_batch bt_rot;
  const kp_batch* bt_in = bt;
  KP_TRY(rotated_batch(c, bt_in, bt_rot, bt));
  const TaylorDims tdi{P.S, P.d, true};
  const TaylorDims tdb{1, 0, false};
  launch_candidate(theta, nullptr, 0, nullptr, P.D, P.wp, c.at(P.o_wpad), c.s);
  if (P.L >= 2)
    launch_prep_layer0(theta, P.d, P.h[1], bt->coeff_diag, bt->coeff_rot, c.at(P.o_w0t), c.at(P.o_q0), c.s);
  for (int64_t n0 = 0; n0 < P.N; n0 += P.Nc) {
    const int64_t nc = std::min(P.Nc, P.N - n0);
    ResidualIn ri{bt->r0 + n0, bt->seeds + n0 * P.S, nullptr};
    if (bt->quad) ri.quad = bt->quad + n0 * P.d;
    forward_loss(c, theta, c.at(P.o_wpad), bt->x_int + n0 * P.d, nc, tdi, bt->coeff_diag, c.at(P.o_ping),
                 c.at(P.o_pong), ri, c.at(P.o_r) + n0, nullptr);
  }
  ResidualIn rb{nullptr, nullptr, bt->targets};
  forward_loss(c, theta, c.at(P.o_wpad), bt->x_bnd, P.Nb, tdb, bt->coeff_diag, c.at(P.o_bping), c.at(P.o_bpong),
               rb, c.at(P.o_rb), nullptr);
  double* ss = c.at(P.o_ls);
  launch_sumsq(c.at(P.o_r), P.N, 0, 1, ss, 1, c.s);
  launch_sumsq(c.at(P.o_rb), P.Nb, 0, 1, ss + 1, 1, c.s);
  launch_losses(ss, (double)P.N, (double)P.Nb, losses, c.s);
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

int32_t kp_kron_solve_workspace_bytes(kp_context* ctx, int32_t p, int32_t q, size_t* bytes) {
  if (!ctx || p < 1 || q < 1 || !bytes) return KP_ERR_INVALID;
  // T^T (A, B), M2 (A, B), eigenvalues, two q x p combine buffers, infos, and per larger pair
  // the solver scratch plus a warm-start T (identity: a standalone solve is cold)
  int64_t doubles = 2LL * p * p + 2LL * q * q + p + q + 2LL * p * q + 8 + 16 * 32;
  for (int n : {p, q})
    if (n > small_eig_max_n()) doubles += pair_scratch_doubles(n) + (int64_t)n * n + 32 + 96;
  *bytes = (size_t)doubles * sizeof(double);
  return KP_OK;
}

int32_t kp_kron_sum_solve(kp_context* ctx, int32_t p, int32_t q, const double* a1,
                          const double* b1, const double* a2, const double* b2, const double* g,
                          double* x, int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  size_t need = 0;
  KP_TRY(kp_kron_solve_workspace_bytes(ctx, p, q, &need));
  if (ws_bytes < need) return KP_ERR_WORKSPACE;
  if (!a1 || !b1 || !a2 || !b2 || !g || !x || !status) return KP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  Plan P;
  int64_t o = 0;
  auto take = [&](int64_t n) {
    const int64_t at = o;
    o += (n + 31) / 32 * 32;
    return at;
  };
  P.o_A1 = take((int64_t)p * p);
  P.o_A2 = take((int64_t)p * p);
  P.o_B1 = take((int64_t)q * q);
  P.o_B2 = take((int64_t)q * q);
  P.o_la = take(p);
  P.o_lb = take(q);
  P.o_T1 = take((int64_t)p * q);
  P.o_T2 = take((int64_t)p * q);
  P.o_info = take(8);
  Ctx c{ctx, P, static_cast<double*>(ws), s};
  KP_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
  if (std::max(p, q) <= small_eig_max_n()) {
    SmallEigJobs ej{};
    SmallCombineJobs cj{};
    int* info = reinterpret_cast<int*>(c.at(P.o_info));
    ej.job[0] = SmallEigJob{p, a1, a2, 0.0, c.at(P.o_A1), c.at(P.o_la), info};
    ej.job[1] = SmallEigJob{q, b1, b2, 0.0, c.at(P.o_B1), c.at(P.o_lb), info + 1};
    cj.job[0] = SmallCombineJob{p, q, g, c.at(P.o_A1), c.at(P.o_B1), c.at(P.o_la), c.at(P.o_lb),
                                c.at(P.o_T1), c.at(P.o_T2), x, 1.0};
    launch_gen_eig_small(ej, 2, std::max(p, q), status, s);
    launch_kron_combine_small(cj, 1, s);
    KP_CUDA_TRY(cudaGetLastError());
    return KP_OK;
  }
  // at least one larger pair: device route per larger pair, the small solver for a small
  // one (T written column-major = T^T row-major), then the DMMA combine
  int* info = reinterpret_cast<int*>(c.at(P.o_info));
  KP_CUDA_TRY(cudaMemsetAsync(info, 0, 8 * sizeof(int), s));
  SmallEigJobs ej{};
  int ne = 0;
  int64_t o2 = o;
  for (int k = 0; k < 2; ++k) {
    const int n = k == 0 ? p : q;
    const double* f1 = k == 0 ? a1 : b1;
    const double* f2 = k == 0 ? a2 : b2;
    double* t = c.at(k == 0 ? P.o_A1 : P.o_B1);
    double* ev = c.at(k == 0 ? P.o_la : P.o_lb);
    if (n <= small_eig_max_n()) {
      ej.job[ne++] = SmallEigJob{n, f1, f2, 0.0, t, ev, info + k, 1};
      continue;
    }
    auto take2 = [&](int64_t k) {  // 32-double (256-byte) aligned sub-allocations
      double* at = c.at(o2);
      o2 += (k + 31) / 32 * 32;
      return at;
    };
    double* scratch = take2(pair_scratch_doubles(n));
    double* tp = take2((int64_t)n * n);
    int* valid = reinterpret_cast<int*>(take2(32));
    KP_CUDA_TRY(cudaMemsetAsync(valid, 0, sizeof(int), s));
    KP_TRY(gen_eig_pair(s, n, f1, f2, 0.0, t, c.at(k == 0 ? P.o_A2 : P.o_B2), ev, scratch,
                        info + k, info + 2 + 2 * k, tp, valid));
  }
  if (ne > 0) launch_gen_eig_small(ej, ne, ej.job[0].n, status, s);
  launch_eig_status(c.at(P.o_la), p, c.at(P.o_lb), q, info, status, s);
  kron_combine(s, p, q, c.at(P.o_A1), c.at(P.o_la), c.at(P.o_B1), c.at(P.o_lb), g, x, 1.0,
               c.at(P.o_T1), c.at(P.o_T2));
  KP_CUDA_TRY(cudaGetLastError());
  return KP_OK;
}

}  // extern "C"
