// Fused Taylor layer with the FP64 product emulated on the tcgen05 INT8 tensor cores by the
// Chinese-remainder construction (Ozaki scheme II), sm_100a — the hidden layers of the
// line-search forwards (reference src/taylor.py:134-169 inside src/optim.py:195-211: 31 of the
// 32 forward passes of a KFAC step) for one-sample tiles (57 <= S <= 112: c5's S = 102).
//
// Exactness argument.  Every row of the states H (n*S x K) and of W (N x K) is scaled by a
// power of two to a BETA-bit integer, a = rint(h 2^(BETA - e_r)) with max|h_r| < 2^e_r, so
// |a| <= 2^BETA (and likewise b for W, exponent f_u).  The integer product P = sum_k a_k b_k
// (|P| <= K 2^(2 BETA) < M / 2) is computed exactly modulo NMOD pairwise-coprime moduli
// p_i <= 256 (M = prod p_i; 13 moduli: M ~ 2^102.5, BETA = 45): one int8 x int8 -> int32
// tcgen05 GEMM of the symmetric residues per modulus, exact since K 128^2 <= 2^24.  With
// q_i = M / p_i and s_i = q_i^-1 mod p_i folded into W's residues, t_i = acc_i mod p_i =
// (s_i P) mod p_i and P = sum_i q_i t_i - k M for the integer k = round(sum / M).  The sum is
// carried as an exact FP64 high part (q_i rounded down to a multiple of 2^E) plus an FP32 low
// part (the rest of q_i, accurate to 2^(BETA-1), far below the 2^(BETA+5) input rounding);
// z = P 2^(e_r + f_u - 2 BETA).  The only approximation is the rounding of h and w to BETA bits:
// about 2e-14 of sum_k |h_k w_k| (DGEMM: ~2e-16; 12 moduli, BETA = 41: 16x larger for 6% less
// time, not taken); the line search consumes these losses only
// through the argmin over the step-size grid (tools/crt_check.py: candidate losses within
// 2e-14 relative of the DMMA path, runner-up gaps >= 6e-3).  Constants and the proof
// obligations of the fold: tools/crt_constants.py (tests/test_crt_constants.py).
//
// Kernel (one persistent CTA per SM, 384 threads): warp 0 lane 0 = TMA producer (per modulus,
// K in 128-byte chunks: W residues 128 units x 128 B, H residues 112 rows x 128 B, 128-byte
// swizzle, six stages), warp 1 = TMEM allocator + MMA issuer (tcgen05.mma kind::i8, M 128
// units, N 112 rows, K 32; four int32 accumulators of 112 columns: the MMAs run up to four
// moduli ahead of the fold, which covers the end-of-tile activation), warps 4..11 = epilogue
// (two per TMEM lane quadrant, 56 rows each; setmaxnreg 232).  The fold of one modulus is
// all FP32 / one DFMA per term (measured, tools/fold_bench.cu: integer multiply-high
// reduction + DADD + DFMA with uniform-register constants 2278 clk per modulus and SM, this
// form 2-3x less): t = f - p rint(f / p) on packed f32x2 pipes (FFMA2 / FADD2), the low CRT
// part an FP32 FMA, the high part one DFMA against D = 1.5 +- t / 256, whose high word is the
// bit pattern of an FP32 FMA result and whose low word is a register that stays zero; the
// per-modulus constants are kept in vector registers (an FP64 instruction with a
// uniform-register operand issues at a fraction of the rate).  Then reconstruct, add the
// bias and apply the Taylor activation (s0 on the value row, s1 g_i on the derivative rows,
// s1 l + s2 sum c_i g_i^2 on the operator row; the two halves of a sample exchange s1, s2 and
// the partial quadratic form through shared memory), branch-free over a thread's 56 rows.
// ACT_LOSS writes the activations, ACT_LAST reduces them against the output layer's weights
// into per-(row, unit tile) partial dots (k_last_from_partials).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "kp_common.cuh"
#include "kp_internal.h"

namespace kp {

namespace {

// 13 moduli, log2 M = 102.525, BETA = 45, E = 53  (tools/crt_constants.py 13)
constexpr int NMOD = 13;
constexpr int BETA = 45;
__constant__ double cr_pd[NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211};
__constant__ double cr_ipd[NMOD] = {1.0 / 256, 1.0 / 255, 1.0 / 253, 1.0 / 251, 1.0 / 247, 1.0 / 241, 1.0 / 239, 1.0 / 233, 1.0 / 229, 1.0 / 227, 1.0 / 223, 1.0 / 217, 1.0 / 211};
__constant__ double cr_s[NMOD] = {195, 1, 238, 224, 245, 161, 24, 60, 112, 29, 185, 156, 46};
__constant__ float cr_npf[NMOD] = {-256.0f, -255.0f, -253.0f, -251.0f, -247.0f, -241.0f, -239.0f, -233.0f, -229.0f, -227.0f, -223.0f, -217.0f, -211.0f};
__constant__ float cr_ipf[NMOD] = {0x1.0000000000000p-8f, 0x1.0101020000000p-8f, 0x1.03091c0000000p-8f, 0x1.0519800000000p-8f, 0x1.0953f40000000p-8f, 0x1.0fef020000000p-8f, 0x1.12358e0000000p-8f, 0x1.1945380000000p-8f, 0x1.1e2ef40000000p-8f, 0x1.20b4700000000p-8f, 0x1.25e2280000000p-8f, 0x1.2e025c0000000p-8f, 0x1.3698e00000000p-8f};
__constant__ float cr_cl[NMOD] = {0x1.3db41a0000000p+50f, 0x1.9502080000000p+52f, 0x1.22d5880000000p+52f, 0x1.5585aa0000000p+51f, 0x1.73ed660000000p+51f, 0x1.d22a8c0000000p+51f, 0x1.b28fa40000000p+50f, 0x1.bb3fc00000000p+52f, 0x1.25d7d00000000p+51f, 0x1.9557fe0000000p+52f, 0x1.50d9000000000p+52f, 0x1.e9690e0000000p+51f, 0x1.133b840000000p+51f};
__constant__ float cr_sg[NMOD] = {0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f, -0x1.0000000000000p-11f, 0x1.0000000000000p-11f};
__constant__ double cr_sq[NMOD] = {0x1.703d73109e800p+102, -0x1.71af2232d1000p+102, 0x1.749b44df3c000p+102, -0x1.779353b31e000p+102, 0x1.7da85e6211000p+102, -0x1.8728d7b42d000p+102, 0x1.8a6ececc2d800p+102, -0x1.9497047757000p+102, 0x1.9ba8302477000p+102, -0x1.9f48aedffe000p+102, 0x1.a6bba31685800p+102, -0x1.b26be29560000p+102, 0x1.bec64ef0fa800p+102};
constexpr double CR_C1 = 0x1.318a5ad26f400p+103;  // 384 sum sg_i q1_i
constexpr double CR_M1 = 0x1.703d73109e938p+102, CR_M2 = 0x1.6d0683e4deb00p+52, CR_IM = 0x1.63f115f5d0b38p-103;

#ifndef CRT_KB
#define CRT_KB 128
#endif
#ifndef CRT_ST
#define CRT_ST 6
#endif
// K bytes per pipeline stage (128: 128-byte swizzle, 29 KB stages; 64: 64-byte swizzle) and
// stage count (measured, tools/crt_bench.cu: 64-byte stages x 13 are 15% slower than 128 x 6,
// 128 x 7 no faster)
constexpr int CM = 128, CN = 112, CKB = CRT_KB, CST = CRT_ST;
constexpr int A_BYTES = CM * CKB, B_BYTES = CN * CKB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EWQ = 2, NEW = 4 * EWQ, CPW = CN / EWQ;  // 56 rows per epilogue thread
constexpr int THREADS = 32 * (4 + NEW);
constexpr int NACC = 4, ACC_STRIDE = 128, TM_COLS = NACC * ACC_STRIDE;  // all of TMEM
constexpr int ND = 4;  // zero-low FP64 scratch pairs of the fold
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(CN >> 3) << 17) |
                           ((uint32_t)(CM >> 4) << 24);
constexpr size_t SMEM_BYTES = (size_t)CST * STAGE_BYTES + 1024;
// CTA pair (CL = 2, tcgen05 cta_group::2): one MMA of M 256 units x N 112 rows spans the two
// SMs of a TPC; each CTA stages its own 128 units of W and HALF of the sample's rows (the pair
// shares B), so a stage is 23 KB and eight of them fit.
constexpr int B2_BYTES = (CN / 2) * CKB, STAGE2_BYTES = A_BYTES + B2_BYTES, CST2 = 8;
constexpr size_t SMEM2_BYTES = (size_t)CST2 * STAGE2_BYTES + 1024;
constexpr uint32_t IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(CN >> 3) << 17) |
                            ((uint32_t)((2 * CM) >> 4) << 24);
constexpr int CST_MAX = CST2 > CST ? CST2 : CST;

constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer by addition
constexpr float MAGICF = 12582912.0f;         // 1.5 * 2^23

__device__ __forceinline__ double pow2i(int e) { return __hiloint2double((e + 1023) << 20, 0); }

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, int x, int y, int z,
                                      uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(b))
      : "memory");
}

// K-major swizzled UMMA shared-memory descriptor: start >> 4, LBO 16 B (unused), SBO = 8 rows
// x CKB bytes, version 1, layout SWIZZLE_128B (2) or SWIZZLE_64B (4)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * CKB) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(CKB == 128 ? 2 : 4) << 61;
  return d;
}

template <int N>
__device__ __forceinline__ void tm_ld(uint32_t ta, uint32_t* r);
template <>
__device__ __forceinline__ void tm_ld<32>(uint32_t ta, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t ta, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t ta, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
}
__device__ __forceinline__ void tm_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Packed FP32 pairs (sm_100 f32x2 instructions: SASS FFMA2 / FADD2).
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void unpk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// high word of the FP64 pair D <- bit pattern of fmaf(t, s, b); the low word (zero) stays
__device__ __forceinline__ void set_hi(double& D, float t, float s, float b) {
  asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %0;\nfma.rn.f32 hi, %1, %2, %3;\nmov.b64 %0, {lo, hi};\n}"
      : "+d"(D)
      : "f"(t), "f"(s), "f"(b));
}

// Per-modulus constants of the fold, in vector registers (`tz` is a zero the compiler cannot
// prove uniform: constants it can prove uniform go to uniform registers, and FP64 / packed
// instructions reading those issue far below their rate).
struct FoldC {
  float ip, np, cl, sg;
  double sq;
};
__device__ __forceinline__ FoldC fold_consts(int i, uint32_t tz) {
  FoldC c;
  c.ip = __uint_as_float(__float_as_uint(cr_ipf[i]) | tz);
  c.np = __uint_as_float(__float_as_uint(cr_npf[i]) | tz);
  c.cl = __uint_as_float(__float_as_uint(cr_cl[i]) | tz);
  c.sg = __uint_as_float(__float_as_uint(cr_sg[i]) | tz);
  const double q = cr_sq[i];
  c.sq = __hiloint2double(__double2hiint(q) | (int)tz, __double2loint(q) | (int)tz);
  return c;
}

// Fold NC accumulator columns of one modulus into the CRT sums (tools/crt_constants.py):
// f = float(acc) (exact), t = f - p rint(f / p) in [-128, 128] (magic-number rounding inside
// the FMA), x2 += t cl (FP32 low part, packed pairs), x1 += (1.5 + sg t / 256) (sg 256 q1)
// (exact FP64 high part; the constant 384 sg q1 is removed at the end).
template <int NC>
__device__ __forceinline__ void fold(const uint32_t* r, double* x1, uint64_t* x2, const FoldC& c,
                                     double* D, float bc) {
  const uint64_t ip2 = pk2(c.ip, c.ip), np2 = pk2(c.np, c.np), cl2 = pk2(c.cl, c.cl);
  const uint64_t mg = pk2(MAGICF, MAGICF), nmg = pk2(-MAGICF, -MAGICF);
#pragma unroll
  for (int j = 0; j < NC; j += 2) {
    const uint64_t f2 = pk2(__int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]));
    const uint64_t q2 = fadd2(ffma2(f2, ip2, mg), nmg);
    const uint64_t t2 = ffma2(q2, np2, f2);
    x2[j / 2] = ffma2(t2, cl2, x2[j / 2]);
    float ta, tb;
    unpk2(t2, ta, tb);
    set_hi(D[j % ND], ta, c.sg, bc);
    x1[j] = fma(D[j % ND], c.sq, x1[j]);
    set_hi(D[(j + 1) % ND], tb, c.sg, bc);
    x1[j + 1] = fma(D[(j + 1) % ND], c.sq, x1[j + 1]);
  }
}

// Moduli as compile-time constants for the state slicing: c1 = 2^15 mod p, c2 = 2^30 mod p
// (centred), so that a = a2 2^30 + a1 2^15 + a0 reduces as y = a2 c2 + a1 c1 + a0, |y| < 2^23.
__host__ __device__ constexpr int modulus(int i) {
  return i == 0 ? 256 : i == 1 ? 255 : i == 2 ? 253 : i == 3 ? 251 : i == 4 ? 247 : i == 5 ? 241
       : i == 6 ? 239 : i == 7 ? 233 : i == 8 ? 229 : i == 9 ? 227 : i == 10 ? 223 : i == 11 ? 217
       : 211;
}
__host__ __device__ constexpr int cmod(long long v, int p) {
  return (int)(v % p) > p / 2 ? (int)(v % p) - p : (int)(v % p);
}

// Weight rows (once per layer and candidate): one warp per row, FP64 residue arithmetic with
// s_i folded in, t_i = s_i a mod p_i.
__global__ void __launch_bounds__(256)
    k_crt_slice_w(const double* __restrict__ X, int64_t rows, int K, int64_t ldx,
                  int8_t* __restrict__ planes, int64_t ps, int* __restrict__ ex) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* x = X + row * ldx;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = fmax(m, fabs(x[k]));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (lane == 0) ex[row] = e;
  const double sc = pow2i(BETA - e);
  for (int k = lane; k < K; k += 32) {
    const double a = (x[k] * sc + MAGIC) - MAGIC;  // rint, |a| <= 2^45
#pragma unroll
    for (int i = 0; i < NMOD; ++i) {
      const double p = cr_pd[i], ip = cr_ipd[i];
      double r = fma(-(fma(a, ip, MAGIC) - MAGIC), p, a);  // exact, |r| <= p/2 + 1
      r *= cr_s[i];
      r = fma(-(fma(r, ip, MAGIC) - MAGIC), p, r);
      int ri = __double2loint(r + MAGIC);
      if (ri > 127) ri -= (int)p;
      planes[i * ps + row * (int64_t)K + k] = (int8_t)ri;
    }
  }
}

// Residues of NE = 4 or 8 consecutive elements of one row: a = rint(x sc) read from the bits
// of x sc + 1.5 2^52 (|a| <= 2^45), split into 15-bit pieces held exactly in FP32; per modulus
// y = a2 c2 + a1 c1 + a0 (exact, |y| < 2^23), r = y - p rint(y / p) (exact, |r| <= p/2 + 1;
// p = 255 folds r = 128 to -127), stored as the low byte of r + 1.5 2^23 (packed f32x2
// arithmetic: two elements per instruction; eight elements per call amortise the per-modulus
// constants, which the compiler rematerialises per use).  p = 256 is the low byte of a.
template <int NE>
__device__ __forceinline__ void slice_n(const double (&xv)[NE], double sc, int8_t* dst, int64_t ps) {
  constexpr int NP = NE / 2;
  const long long mb = __double_as_longlong(MAGIC);
  const uint64_t n23 = pk2(-8388608.0f, -8388608.0f), nmg = pk2(-MAGICF, -MAGICF),
                 mg = pk2(MAGICF, MAGICF);
  uint64_t g0[NP], g1[NP], g2[NP];
  uint32_t low[NE];
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    float f0[2], f1[2], f2[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const long long a = __double_as_longlong(fma(xv[2 * u + t], sc, MAGIC)) - mb;
      const uint32_t lo = (uint32_t)a;
      low[2 * u + t] = lo;
      f0[t] = __int_as_float(0x4B000000 | (lo & 0x7fffu));
      f1[t] = __int_as_float(0x4B000000 | ((lo >> 15) & 0x7fffu));
      f2[t] = __int_as_float(0x4B400000 + (int)(a >> 30));
    }
    g0[u] = fadd2(pk2(f0[0], f0[1]), n23);
    g1[u] = fadd2(pk2(f1[0], f1[1]), n23);
    g2[u] = fadd2(pk2(f2[0], f2[1]), nmg);
  }
  auto store = [&](int8_t* d, const uint32_t (&w)[NE]) {
    uint32_t q[NE / 4];
#pragma unroll
    for (int v = 0; v < NE / 4; ++v)
      q[v] = __byte_perm(__byte_perm(w[4 * v], w[4 * v + 1], 0x0040),
                         __byte_perm(w[4 * v + 2], w[4 * v + 3], 0x0040), 0x5410);
    if (NE == 8) *reinterpret_cast<uint2*>(d) = make_uint2(q[0], q[NE / 4 - 1]);
    else *reinterpret_cast<uint32_t*>(d) = q[0];
  };
  store(dst, low);
#pragma unroll
  for (int i = 1; i < NMOD; ++i) {
    const float p = (float)modulus(i), ip = 1.0f / (float)modulus(i);
    const float c1 = (float)cmod(1LL << 15, modulus(i)), c2 = (float)cmod(1LL << 30, modulus(i));
    const uint64_t c1p = pk2(c1, c1), c2p = pk2(c2, c2), ipp = pk2(ip, ip), npp = pk2(-p, -p);
    uint32_t bb[NE];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const uint64_t y = ffma2(g2[u], c2p, ffma2(g1[u], c1p, g0[u]));
      uint64_t r = ffma2(fadd2(ffma2(y, ipp, mg), nmg), npp, y);
      if (modulus(i) == 255) {  // r = 128 does not fit a byte: 128 = -127 (mod 255)
        float ra, rb;
        unpk2(r, ra, rb);
        ra = ra > 127.5f ? ra - p : ra;
        rb = rb > 127.5f ? rb - p : rb;
        r = pk2(ra, rb);
      }
      const uint64_t bq = fadd2(r, mg);
      bb[2 * u] = (uint32_t)bq;
      bb[2 * u + 1] = (uint32_t)(bq >> 32);
    }
    store(dst + i * ps, bb);
  }
}
__device__ __forceinline__ void slice4(const double (&xv)[4], double sc, int8_t* dst, int64_t ps) {
  slice_n<4>(xv, sc, dst, ps);
}

// State rows: one warp per row, lane = 4 consecutive K entries per 128-wide chunk.  max|x| <
// 2^e; a = rint(x 2^(BETA - e)) read from the bits of x 2^(BETA-e) + 1.5 2^52 (|a| <= 2^45),
// split into 15-bit pieces held exactly in FP32; per modulus y = a2 c2 + a1 c1 + a0 (exact,
// |y| < 2^23), r = y - p rint(y / p) (exact, |r| <= p/2 + 1; p = 255 folds r = 128 to -127),
// stored as the low byte of r + 1.5 2^23.  p = 256 is the low byte of a.
__global__ void __launch_bounds__(256)
    k_crt_slice_h(const double* __restrict__ X, int64_t rows, int K, int64_t ldx,
                  int8_t* __restrict__ planes, int64_t ps, int* __restrict__ ex) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* x = X + row * ldx;
  double m = 0.0;
  for (int k = 4 * lane; k < K; k += 128) {
    const double2 v0 = *reinterpret_cast<const double2*>(x + k);
    const double2 v1 = *reinterpret_cast<const double2*>(x + k + 2);
    m = fmax(m, fmax(fmax(fabs(v0.x), fabs(v0.y)), fmax(fabs(v1.x), fabs(v1.y))));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (lane == 0) ex[row] = e;
  const double sc = pow2i(BETA - e);
  const int K8 = K & ~255;
  for (int k = 8 * lane; k < K8; k += 256) {
    double xv[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double2 v = *reinterpret_cast<const double2*>(x + k + 2 * t);
      xv[2 * t] = v.x;
      xv[2 * t + 1] = v.y;
    }
    slice_n<8>(xv, sc, planes + row * (int64_t)K + k, ps);
  }
  if (K8 < K) {  // K = 128 (mod 256): one 128-wide chunk, four elements per lane
    const int k = K8 + 4 * lane;
    const double2 v0 = *reinterpret_cast<const double2*>(x + k);
    const double2 v1 = *reinterpret_cast<const double2*>(x + k + 2);
    const double xv[4] = {v0.x, v0.y, v1.x, v1.y};
    slice4(xv, sc, planes + row * (int64_t)K + k, ps);
  }
}

// Layer 0 straight to residue planes (no FP64 states written or re-read): the activations of
// the first layer are rank-one in the sample (src/taylor.py:124-169 with the linear input:
// value row tanh(z_u), derivative row i: s1(z_u) W0[u, i], operator row: s2(z_u) q_u with
// q_u = sum_i c_i W0[u, i]^2).  One CTA per sample at a time: tanh and its derivatives of the
// sample's h1 pre-activations go to shared memory, then each warp takes rows of the sample and
// treats them like k_crt_slice_h (lane = 4 consecutive units per 128-wide chunk; maximum,
// then slicing), forming the row's entries on the fly from W0^T (d x h1, L2-resident) and q.
constexpr int FIRST_WARPS = 8, FIRST_MAXH = 1024;
__global__ void __launch_bounds__(FIRST_WARPS * 32)
    k_crt_first(const double* __restrict__ zval, int64_t n, int h1, int S, int d,
                const double* __restrict__ w0t, const double* __restrict__ q0,
                int8_t* __restrict__ planes, int64_t ps, int* __restrict__ ex) {
  __shared__ double sv[3][FIRST_MAXH];  // s0, s1, s2 of the current sample
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t smp = blockIdx.x; smp < n; smp += gridDim.x) {
    for (int u = threadIdx.x; u < h1; u += blockDim.x) {
      const TanhD td = tanh_derivs(zval[smp * h1 + u], false);
      sv[0][u] = td.s0;
      sv[1][u] = td.s1;
      sv[2][u] = td.s2;
    }
    __syncthreads();
    for (int i = warp; i < S; i += FIRST_WARPS) {
      const double* coef = i == 0 ? sv[0] : (i <= d ? sv[1] : sv[2]);
      const double* data = i == 0 ? nullptr : (i <= d ? w0t + (int64_t)(i - 1) * h1 : q0);
      auto load4 = [&](int k, double (&xv)[4]) {
        const double2 c0 = *reinterpret_cast<const double2*>(coef + k);
        const double2 c1 = *reinterpret_cast<const double2*>(coef + k + 2);
        if (data == nullptr) {
          xv[0] = c0.x;
          xv[1] = c0.y;
          xv[2] = c1.x;
          xv[3] = c1.y;
        } else {
          const double2 w0 = *reinterpret_cast<const double2*>(data + k);
          const double2 w1 = *reinterpret_cast<const double2*>(data + k + 2);
          xv[0] = c0.x * w0.x;
          xv[1] = c0.y * w0.y;
          xv[2] = c1.x * w1.x;
          xv[3] = c1.y * w1.y;
        }
      };
      double m = 0.0;
      for (int k = 4 * lane; k < h1; k += 128) {
        double xv[4];
        load4(k, xv);
        m = fmax(m, fmax(fmax(fabs(xv[0]), fabs(xv[1])), fmax(fabs(xv[2]), fabs(xv[3]))));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      int e = 0;
      if (m > 0.0) frexp(m, &e);
      const int64_t row = smp * S + i;
      if (lane == 0) ex[row] = e;
      const double sc = pow2i(BETA - e);
      const int h8 = h1 & ~255;
      for (int k = 8 * lane; k < h8; k += 256) {
        double xa[4], xb[4];
        load4(k, xa);
        load4(k + 4, xb);
        const double xv[8] = {xa[0], xa[1], xa[2], xa[3], xb[0], xb[1], xb[2], xb[3]};
        slice_n<8>(xv, sc, planes + row * (int64_t)h1 + k, ps);
      }
      if (h8 < h1) {
        double xv[4];
        load4(h8 + 4 * lane, xv);
        slice4(xv, sc, planes + row * (int64_t)h1 + h8 + 4 * lane, ps);
      }
    }
    __syncthreads();  // sv is rewritten for the next sample
  }
}

// Tile schedule.  CL = 1: tile t -> unit tile t % UT, sample t / UT, CTAs striding by the grid.
// CL = 4: 2 x 2 clusters; cluster tile ct -> unit tiles 2 (ct % (UT/2)) + cu and samples
// 2 (ct / (UT/2)) + cs for the CTA of rank cu + 2 cs; the two CTAs of a unit tile share its
// weight residues and the two CTAs of a sample its state residues, each loading one half with a
// cluster multicast (half the L2 operand traffic).
template <int CL>
struct Sched {
  int first, step, count;  // tile indices < 2^31 (n_samples * UT checked by the launcher)
  int cu, cs, UT;
  __device__ Sched(int64_t n_samples, int ut_count) : UT(ut_count) {
    if (CL == 1) {
      first = blockIdx.x;
      step = gridDim.x;
      count = (int)(n_samples * UT);
      cu = cs = 0;
    } else {
      uint32_t rank, cid, ncl;
      asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
      asm("mov.u32 %0, %%clusterid.x;\n" : "=r"(cid));
      asm("mov.u32 %0, %%nclusterid.x;\n" : "=r"(ncl));
      first = cid;
      step = ncl;
      if (CL == 2) {  // pair tile: unit tiles 2 (t % (UT/2)) + rank of sample t / (UT/2)
        count = (int)(n_samples * (UT / 2));
        cu = (int)rank;
        cs = 0;
      } else {
        count = (int)((n_samples + 1) / 2 * (UT / 2));
        cu = (int)(rank & 1);
        cs = (int)(rank >> 1);
      }
    }
  }
  __device__ int ut(int t) const { return CL == 1 ? t % UT : 2 * (t % (UT / 2)) + cu; }
  __device__ int64_t smp(int t) const {
    return CL == 1 ? t / UT : CL == 2 ? t / (UT / 2) : 2 * (int64_t)(t / (UT / 2)) + cs;
  }
};

__device__ __forceinline__ void tma3d_mc(void* dst, const CUtensorMap* m, int x, int y, int z,
                                         uint64_t* b, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(b)), "h"(mask)
      : "memory");
}

// CTA-pair load: the bytes are counted on the LEADER CTA's mbarrier (`lbar`: its
// shared::cluster address)
__device__ __forceinline__ void tma3d_2sm(void* dst, const CUtensorMap* m, int x, int y, int z,
                                          uint32_t lbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(lbar)
      : "memory");
}
// shared::cluster address of `p` in the CTA of rank `rank`
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

#ifdef CRT_TIMING  // (tools/crt_bench.cu: where block 0's roles spend their cycles)
__device__ long long crt_dbg[16];
#define CRT_T0(v) const long long v = clock64()
#define CRT_ACC(slot, v) dbg_acc[slot] += clock64() - (v)
#else
#define CRT_T0(v)
#define CRT_ACC(slot, v)
#endif

template <int MODE, int CL>
__global__ void __launch_bounds__(THREADS, 1)
    k_crt_act(const __grid_constant__ CUtensorMap mW, const __grid_constant__ CUtensorMap mH,
              const int* __restrict__ exw, const int* __restrict__ exh, GemmAct g, int UT,
              int* __restrict__ tile_counter) {
  extern __shared__ __align__(1024) uint8_t crt_sm[];
  uint8_t* base =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(crt_sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[CST_MAX], empty[CST_MAX], tfull[NACC], tempty[NACC];
  constexpr int NST = CL == 2 ? CST2 : CST;
  constexpr int STB = CL == 2 ? STAGE2_BYTES : STAGE_BYTES;
  __shared__ uint32_t tmem_base;
  __shared__ double xs1[2][CM], xs2[2][CM], xq[2][CM];  // value-row s1, s2 and half-0 quadratic form (by tile parity)
  __shared__ double red[4][CN];                // ACT_LAST: per-quadrant row partials
  __shared__ double sc_s[2][CN];               // row scales 2^(e_r - BETA) of the current / next tile
  __shared__ double cw_s[CN];                  // c_i on derivative row i, 0 elsewhere
  __shared__ uint32_t zero_s[32];
  // tile queue: the producer announces tile k (or -1: no more) in slot k % 8; with a tile
  // counter (independent CTAs) tiles are handed out in order, so the CTAs working on one
  // sample's unit tiles stay within a tile of each other and its residues are read from HBM once
  __shared__ int tq[8];
  __shared__ uint64_t tready[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = g.S;
  const Sched<CL> sch(g.n_samples, UT);
  const int KC = g.K / CKB;
  // multicast groups: same unit tile (weights) and same sample (states); the stage's consumers
  // release it to every CTA that writes into it
  const uint16_t mask_w = (uint16_t)((1u << sch.cu) | (1u << (sch.cu + 2)));
  const uint16_t mask_h = (uint16_t)(3u << (2 * sch.cs));
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL == 4 ? 3 : 1);
    }
    for (int b = 0; b < 8; ++b) mbar_init(&tready[b], 1);
    for (int b = 0; b < NACC; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], CL == 2 ? 2 * NEW : NEW);  // pair: both CTAs' epilogues release
    }
    mbar_fence_init();
  }
  if (threadIdx.x < 32) zero_s[threadIdx.x] = 0u;
  for (int i = threadIdx.x; i < CN; i += THREADS) cw_s[i] = (i >= 1 && i <= g.d) ? g.cdiag[i - 1] : 0.0;
  if (warp == 1) {
    if (CL == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_addr(&tmem_base)),
                   "r"(TM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_addr(&tmem_base)),
                   "r"(TM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    if (warp == 0 && lane == 0) {  // TMA producer
      uint32_t it = 0;
#ifdef CRT_TIMING
      long long dbg_acc[2] = {0, 0};
      const long long dbg_t0 = clock64();
#endif
      const uint32_t lfull0 = CL == 2 ? mapa(&full[0], 0) : 0u;  // the leader's full[0]
      const uint32_t hrows = (uint32_t)((S + 7) & ~7);
      for (uint32_t tk = 0;; ++tk) {
        int tile = (CL == 1 && tile_counter) ? atomicAdd(tile_counter, 1)
                                              : sch.first + (int)tk * sch.step;
        if (tile >= sch.count) tile = -1;
        tq[tk & 7] = tile;
        mbar_arrive(&tready[tk & 7]);
        if (tile < 0) break;
        const int ut = sch.ut(tile);
        const int row0 = (int)(sch.smp(tile) * S);
        for (int i = 0; i < NMOD; ++i)
          for (int kc = 0; kc < KC; ++kc, ++it) {
            const uint32_t s = it % NST;
            {
              CRT_T0(tw);
              if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
              CRT_ACC(0, tw);
            }
            uint8_t* a = base + s * STB;
            if (CL == 2) {  // both CTAs' bytes are counted on the leader's barrier
              if (sch.cu == 0) mbar_arrive_expect_tx(&full[s], 2 * STB);
              const uint32_t lbar = lfull0 + s * (uint32_t)sizeof(uint64_t);
              tma3d_2sm(a, &mW, kc * CKB, ut * CM, i, lbar);
              tma3d_2sm(a + A_BYTES, &mH, kc * CKB, row0 + sch.cu * (CN / 2), i, lbar);
              continue;
            }
            if (CL == 1) {  // only the sample's rows (to a multiple of 8): the rest of the
                            // 112-row operand is stale shared memory feeding unused columns
              mbar_arrive_expect_tx(&full[s], A_BYTES + hrows * CKB);
              tma3d(a, &mW, kc * CKB, ut * CM, i, &full[s]);
              tma3d(a + A_BYTES, &mH, kc * CKB, row0, i, &full[s]);
            } else {
              mbar_arrive_expect_tx(&full[s], STB);  // my half of the unit tile's weights and of the sample's states
              tma3d_mc(a + sch.cs * (CM / 2) * CKB, &mW, kc * CKB, ut * CM + sch.cs * (CM / 2), i,
                       &full[s], mask_w);
              tma3d_mc(a + A_BYTES + sch.cu * (CN / 2) * CKB, &mH, kc * CKB, row0 + sch.cu * (CN / 2),
                       i, &full[s], mask_h);
            }
          }
      }
#ifdef CRT_TIMING
      if (blockIdx.x == 0) {
        crt_dbg[0] = dbg_acc[0];
        crt_dbg[1] = clock64() - dbg_t0;
      }
#endif
    } else if (warp == 1 && lane == 0 && (CL != 2 || sch.cu == 0)) {  // MMA issuer (pair: leader)
      uint32_t it = 0, gm = 0;
#ifdef CRT_TIMING
      long long dbg_acc[2] = {0, 0};
      const long long dbg_t0 = clock64();
#endif
      for (uint32_t tk = 0;; ++tk) {
        mbar_wait(&tready[tk & 7], (tk >> 3) & 1);
        if (tq[tk & 7] < 0) break;
        for (int i = 0; i < NMOD; ++i, ++gm) {
          const uint32_t b = gm % NACC;
          {
            CRT_T0(tw);
            if (gm >= NACC) mbar_wait(&tempty[b], ((gm / NACC) - 1) & 1);
            CRT_ACC(0, tw);
          }
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t acc_col = tmem + b * ACC_STRIDE;
          for (int kc = 0; kc < KC; ++kc, ++it) {
            const uint32_t s = it % NST;
            {
              CRT_T0(tw);
              mbar_wait(&full[s], (it / NST) & 1);
              CRT_ACC(1, tw);
            }
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t a = smem_addr(base + s * STB), bb = a + A_BYTES;
#pragma unroll
            for (int k = 0; k < CKB / 32; ++k) {
              const uint64_t da = sdesc(a + 32 * k), db = sdesc(bb + 32 * k);
              const uint32_t acc = (kc | k) ? 1u : 0u;
#ifndef CRT_DBG_NOMMA  // (tools/crt_bench.cu timing variants)
              if (CL == 2)
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc_col),
                    "l"(da), "l"(db), "r"(IDESC2), "r"(acc));
              else
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc_col),
                    "l"(da), "l"(db), "r"(IDESC), "r"(acc));
#else
              (void)da, (void)db, (void)acc, (void)acc_col;
#endif
            }
            if (CL == 1)
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                      smem_addr(&empty[s]))
                  : "memory");
            else if (CL == 2)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
                  "cluster.b64 [%0], %1;\n" ::"r"(smem_addr(&empty[s])),
                  "h"((uint16_t)3)
                  : "memory");
            else
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::"
                  "cluster.b64 [%0], %1;\n" ::"r"(smem_addr(&empty[s])),
                  "h"((uint16_t)(mask_w | mask_h))
                  : "memory");
          }
          if (CL == 2)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
                "cluster.b64 [%0], %1;\n" ::"r"(smem_addr(&tfull[b])),
                "h"((uint16_t)3)
                : "memory");
          else
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_addr(&tfull[b]))
                : "memory");
        }
      }
#ifdef CRT_TIMING
      if (blockIdx.x == 0) {
        crt_dbg[2] = dbg_acc[0];
        crt_dbg[3] = dbg_acc[1];
        crt_dbg[4] = clock64() - dbg_t0;
      }
#endif
    }
  } else {  // epilogue: quadrant q = TMEM lanes 32q..32q+31 = units, half h = rows 56h..56h+55
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int c0 = h * CPW;
    const int ul = 32 * q + lane;  // unit within the tile
    const int te = threadIdx.x - 128;  // epilogue thread index
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const int d = g.d;
    const int64_t rows_total = g.n_samples * S;
    // a zero the compiler cannot prove uniform (volatile: not rematerialised)
    uint32_t tz;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(tz) : "r"(smem_addr(&zero_s[lane])));
    double D[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) D[j] = __hiloint2double((int)tz, (int)tz);
    const float bc = __uint_as_float(0x3FF80000u | tz);  // 1.9375f: the high word of 1.5
    auto vreg = [tz](double v) {  // the constant in a vector register pair (see FoldC)
      return __hiloint2double(__double2hiint(v) | (int)tz, __double2loint(v) | (int)tz);
    };
    const double c1 = vreg(CR_C1);
    const double v_im = CR_IM, v_mg = MAGIC, v_m1 = CR_M1, v_m2 = CR_M2;
    const uint32_t ltempty0 = CL == 2 ? mapa(&tempty[0], 0) : 0u;  // the leader's tempty[0]
    uint32_t gm = 0, tcount = 0;
#ifdef CRT_TIMING
    long long dbg_acc[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long dbg_t0 = clock64();
#endif
    for (;; ++tcount) {
      mbar_wait(&tready[tcount & 7], (tcount >> 3) & 1);
      const int tile = tq[tcount & 7];
      if (tile < 0) break;
      const int ut = sch.ut(tile);
      const int64_t smp = sch.smp(tile);
      const bool live = smp < g.n_samples;  // (CL = 4, odd n: the last pair's second sample)
      const int64_t row0 = smp * S;
      const int unit = ut * CM + ul;
      double* sc = sc_s[tcount & 1];
      if (te < CN) {  // this tile's row scales 2^(e_r - BETA) (rows past the end: clamped, never stored)
        const int64_t r = row0 + te;
        sc[te] = pow2i(exh[r < rows_total ? r : rows_total - 1] - BETA);
      }
      double x1[CPW];
      uint64_t x2[CPW / 2];
#pragma unroll
      for (int j = 0; j < CPW; ++j) x1[j] = -c1;  // the fold adds C1 = 384 sum sg_i q1_i
#pragma unroll
      for (int j = 0; j < CPW / 2; ++j) x2[j] = 0ull;
#pragma unroll 1
      for (int i = 0; i < NMOD; ++i, ++gm) {
        const uint32_t b = gm % NACC;
        const FoldC fc = fold_consts(i, tz);
        {
          CRT_T0(tw);
          mbar_wait(&tfull[b], (gm / NACC) & 1);
          CRT_ACC(0, tw);
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t ta = lane_base + b * ACC_STRIDE;
        uint32_t ra[16], rb[16];
        tm_ld<16>(ta, ra);
        tm_wait();
        tm_ld<16>(ta + 16, rb);
#ifndef CRT_DBG_NOFOLD
        fold<16>(ra, x1, x2, fc, D, bc);
#endif
        tm_wait();
        tm_ld<16>(ta + 32, ra);
#ifndef CRT_DBG_NOFOLD
        fold<16>(rb, x1 + 16, x2 + 8, fc, D, bc);
#endif
        tm_wait();
        tm_ld<8>(ta + 48, rb);
#ifndef CRT_DBG_NOFOLD
        fold<16>(ra, x1 + 32, x2 + 16, fc, D, bc);
#endif
        tm_wait();
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) {
          if (CL == 2) mbar_arrive_cluster(ltempty0 + b * (uint32_t)sizeof(uint64_t));
          else mbar_arrive(&tempty[b]);
        }
#ifndef CRT_DBG_NOFOLD
        fold<8>(rb, x1 + 48, x2 + 24, fc, D, bc);
#endif
      }
      CRT_T0(ttail);
      asm volatile("bar.sync 5, 256;\n" ::: "memory");  // sc of this tile written
      CRT_ACC(2, ttail);
      // reconstruct y = P 2^(e_r - BETA) (z = y su, su = 2^(f_u - BETA): folded into the
      // activation's factors) in x1, branch-free (rows past S: 0).  x1 started at -C1.
      const double su = pow2i(exw[unit] - BETA);
      auto recon = [&](int j) {
        float lo, hi;
        unpk2(x2[j / 2], lo, hi);
        const double X2 = (double)((j & 1) ? hi : lo);
        // (|low| < 2^65 cannot move the rounding: |P| < M / 2.4 keeps high / M off the ties)
        const double k = fma(x1[j], v_im, v_mg) - v_mg;
        const double P = fma(-k, v_m1, x1[j]) + fma(-k, v_m2, X2);
        const double y = P * sc[c0 + j];
        return (c0 + j < S) ? y : 0.0;
      };
      // Taylor activation (src/taylor.py:140-169): half 0 owns the value row and derivative
      // rows 1..55, half 1 the remaining derivative rows and the operator row S - 1 (S > 56).
      // Half 0 never waits: it publishes s1, s2 as soon as the value row is reconstructed
      // (named barrier 1 + q, arrive only) and its part of the quadratic form after its rows
      // (barrier 6 + q); half 1 needs the first for every row and the second for the operator
      // row only.  xs1 / xs2 / xq are double-buffered by tile parity (half 0 can be at most
      // the accumulators' depth, less than a tile, ahead of half 1).
      const int par = (int)(tcount & 1);
      double s0 = 0.0, s1, s2, quad = 0.0;
      if (h == 0) {
        x1[0] = recon(0);
        const TanhD t = tanh_derivs(fma(x1[0], su, g.bias[(int64_t)unit * g.bias_stride]), false);
        s0 = t.s0;
        s1 = t.s1;
        s2 = t.s2;
        xs1[par][ul] = s1;
        xs2[par][ul] = s2;
        asm volatile("bar.arrive %0, 64;\n" ::"r"(1 + q) : "memory");
#pragma unroll
        for (int j = 1; j < CPW; ++j) x1[j] = recon(j);
        CRT_ACC(3, ttail);
        // quadratic form over this half's derivative rows (cw = 0 on every other row), in
        // units of su^2; the two halves' parts are summed in a fixed order (half 0 + half 1)
#pragma unroll
        for (int j = 1; j < CPW; ++j) quad += (x1[j] * cw_s[c0 + j]) * x1[j];
        xq[par][ul] = quad;
        asm volatile("bar.arrive %0, 64;\n" ::"r"(6 + q) : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < CPW; ++j) x1[j] = recon(j);
        CRT_ACC(3, ttail);
#pragma unroll
        for (int j = 0; j < CPW; ++j) quad += (x1[j] * cw_s[c0 + j]) * x1[j];
        asm volatile("bar.sync %0, 64;\n" ::"r"(1 + q) : "memory");
        s1 = xs1[par][ul];
        s2 = xs2[par][ul];
      }
      CRT_ACC(4, ttail);
      // outputs in x1 (the operator row's s2 term: below, once half 0's quadratic form is in)
      const double s1u = s1 * su;
#pragma unroll
      for (int j = 0; j < CPW; ++j) x1[j] = s1u * x1[j];
      if (h == 0) x1[0] = s0;
      double s2q = 0.0;
      if (MODE == ACT_LAST && h == 1) {  // (the row reduction below needs the complete row)
        asm volatile("bar.sync %0, 64;\n" ::"r"(6 + q) : "memory");
        s2q = s2 * ((xq[par][ul] + quad) * (su * su));
#pragma unroll
        for (int j = 0; j < CPW; ++j) x1[j] = (c0 + j == S - 1) ? x1[j] + s2q : x1[j];
      }
      CRT_ACC(5, ttail);
      if (MODE == ACT_LOSS) {
        double* out = g.post + row0 * g.ldo + unit;
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          const uint32_t ok = (c0 + j < S) && live && !(h == 1 && c0 + j == S - 1);
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\n@p st.global.f64 [%0], %1;\n}\n" ::"l"(
                  out + (int64_t)(c0 + j) * g.ldo),
              "d"(x1[j]), "r"(ok)
              : "memory");
        }
        if (h == 1) {  // the operator row, with half 0's part of the quadratic form
          asm volatile("bar.sync %0, 64;\n" ::"r"(6 + q) : "memory");
          s2q = s2 * ((xq[par][ul] + quad) * (su * su));
          double op = 0.0;
#pragma unroll
          for (int j = 0; j < CPW; ++j) op = (c0 + j == S - 1) ? x1[j] : op;
          if (live) out[(int64_t)(S - 1) * g.ldo] = op + s2q;
        }
      } else {  // ACT_LAST: row partials over this tile's 128 units
        const double wl = g.wlast[unit];
        // sums over the warp's 32 units of all 56 rows by recursive halving: at distance 16
        // a lane keeps one half of the rows and hands the other half to its partner, and so
        // on (28, 14, 7 -> 8, 4, 2 rows: 55 exchanges instead of 56 five-step butterflies);
        // lane l ends with rows 28 b4 + 14 b3 + 7 b2 + 4 b1 + 2 b0 + {0, 1} (b = bits of l)
        double v[CPW];
#pragma unroll
        for (int j = 0; j < CPW; ++j) v[j] = x1[j] * wl;
        auto halve = [&](int len, int off) {  // v[0..len) -> v[0..len/2)
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < CPW / 2; ++i) {
            if (i < len / 2) {
              const double send = up ? v[i] : v[i + len / 2];
              const double keep = up ? v[i + len / 2] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
        };
        halve(56, 16);
        halve(28, 8);
        v[7] = 0.0;  // 14 -> 7 + 7: pad each half to 8 with a zero (slot 7 of the kept half)
        {
          const bool up = (lane & 4) != 0;
#pragma unroll
          for (int i = 0; i < 7; ++i) {
            const double send = up ? v[i] : v[i + 7];
            const double keep = up ? v[i + 7] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
          }
          v[7] = 0.0;
        }
        halve(8, 2);
        halve(4, 1);
        {
          const int sub = ((lane & 2) ? 4 : 0) + ((lane & 1) ? 2 : 0);  // within the 7-row group
          const int base = ((lane & 16) ? 28 : 0) + ((lane & 8) ? 14 : 0) + ((lane & 4) ? 7 : 0) + sub;
          if (sub < 7) red[q][c0 + base] = v[0];
          if (sub + 1 < 7) red[q][c0 + base + 1] = v[1];
        }
        asm volatile("bar.sync 5, 256;\n" ::: "memory");
        for (int col = te; live && col < S; col += 256)
          g.upart[(row0 + col) * UT + ut] = ((red[0][col] + red[1][col]) + red[2][col]) + red[3][col];
        asm volatile("bar.sync 5, 256;\n" ::: "memory");
      }
      CRT_ACC(1, ttail);
    }
#ifdef CRT_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 128) {
      crt_dbg[5] = dbg_acc[0];
      crt_dbg[6] = dbg_acc[1];
      crt_dbg[7] = dbg_acc[2];
      crt_dbg[8] = clock64() - dbg_t0;
      crt_dbg[9] = dbg_acc[3];
      crt_dbg[10] = dbg_acc[4];
      crt_dbg[11] = dbg_acc[5];
    }
#endif
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // no peer still multicasts into this CTA's stages
  if (warp == 1) {
    if (CL == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                   "r"(TM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                   "r"(TM_COLS));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 crt_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// residue planes (NMOD x rows x K int8) as a 3-D tensor map: box {128 bytes of K, box_rows,
// one plane}, 128-byte swizzle; cached by geometry
bool crt_map(CUtensorMap* m, const int8_t* planes, int64_t rows, int K, uint32_t box_rows) {
  using Key = std::tuple<const int8_t*, int64_t, int, uint32_t>;
  static std::map<Key, CUtensorMap> cache;
  static std::mutex mu;
  const Key key{planes, rows, K, box_rows};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  auto fn = crt_encode();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)NMOD};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * (cuuint64_t)rows};
  cuuint32_t box[3] = {CKB, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE,
         CKB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

// On by default; KP_CRT=0 keeps every line-search layer on the FP64 DMMA kernel.
bool crt_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_CRT");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

int crt_moduli() { return NMOD; }

// Layer 0 straight to residue planes (k_crt_first); KP_CRT_FIRST=0 writes the FP64 state and
// slices it like the other layers.
bool crt_first_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_CRT_FIRST");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

bool crt_act_ok(int S, int K, int N) {
  return crt_enabled() && S > CPW && S <= CN && K % CKB == 0 && K >= CKB && K <= 1024 &&
         N % CM == 0;
}

void launch_crt_slice(const double* X, int64_t rows, int K, int64_t ldx, int8_t* planes, int* ex,
                      bool weights, cudaStream_t s) {
  if (rows <= 0) return;
  count_launch();
  const unsigned blocks = (unsigned)ceil_div(rows, 8);
  if (weights)
    k_crt_slice_w<<<blocks, 256, 0, s>>>(X, rows, K, ldx, planes, rows * (int64_t)K, ex);
  else
    k_crt_slice_h<<<blocks, 256, 0, s>>>(X, rows, K, ldx, planes, rows * (int64_t)K, ex);
}

// Layer 0 (given z = x W0^T + b0) straight to the residue planes the first hidden CRT layer
// reads; false when the shape is outside the kernel's (h1 a multiple of 128 up to 1024).
bool launch_crt_first(const double* zval, int64_t n, int h1, int S, int d, const double* w0t,
                      const double* q0, int8_t* planes, int* ex, cudaStream_t s) {
  if (n <= 0) return true;
  if (h1 % 128 != 0 || h1 > FIRST_MAXH || S != d + 2) return false;
  count_launch();
  const unsigned blocks = (unsigned)std::min<int64_t>(n, (int64_t)sm_count() * 8);
  k_crt_first<<<blocks, FIRST_WARPS * 32, 0, s>>>(zval, n, h1, S, d, w0t, q0, planes,
                                                   n * S * (int64_t)h1, ex);
  return true;
}

// Fused layer from residue planes: resH (NMOD x n*S x K, exponents exH), resW (NMOD x N x K,
// exponents exW, sliced with weights = true).  ACT_LOSS: g.post / g.ldo; ACT_LAST: g.wlast,
// g.upart ((n*S) x N/128 partial dots).  tile_counter: one device int owned by the caller for
// the in-order tile schedule (nullptr: static striding); not shared by concurrent launches.
bool launch_crt_act(const GemmAct& g, int mode, const int8_t* resH, const int* exH,
                    const int8_t* resW, const int* exW, cudaStream_t s, int* tile_counter) {
  if (g.n_samples <= 0) return true;
  if (!crt_act_ok(g.S, g.K, g.N) || g.batch != 1 || !g.taylor || (mode != ACT_LOSS && mode != ACT_LAST) ||
      g.n_samples * (g.N / CM) >= (int64_t(1) << 31) || g.n_samples * g.S >= (int64_t(1) << 31))
    return false;
  const int64_t rows = g.n_samples * g.S;
  const int UT = g.N / CM;
  // KP_CRT_CLUSTER: 1 = independent CTAs (the default: fastest, 5649 pts/s on c5), 2 = CTA
  // pairs (tcgen05 cta_group::2 MMA of 256 units, the pair sharing the sample's rows: 23% less
  // L2 and shared-memory fill traffic, but 5483 pts/s), 4 = 2 x 2 clusters of single-CTA MMAs
  // with multicast loads (half the L2 traffic, 5646 pts/s).  Both cluster forms lose to the
  // lock-step of their CTAs what they save in traffic.
  static const int cl_env = [] {
    const char* e = getenv("KP_CRT_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  int CL = 1;
  if (cl_env == 2 && UT % 2 == 0) CL = 2;
  if (cl_env == 4 && UT % 2 == 0 && g.n_samples >= 2) CL = 4;
  CUtensorMap mw, mh;
  if (!crt_map(&mw, resW, g.N, g.K, CL == 4 ? CM / 2 : CM) ||
      !crt_map(&mh, resH, rows, g.K, CL == 1 ? (uint32_t)((g.S + 7) & ~7) : CN / 2))
    return false;
  void (*kern)(const CUtensorMap, const CUtensorMap, const int*, const int*, GemmAct, int, int*);
  if (mode == ACT_LAST)
    kern = CL == 4 ? k_crt_act<ACT_LAST, 4> : CL == 2 ? k_crt_act<ACT_LAST, 2> : k_crt_act<ACT_LAST, 1>;
  else
    kern = CL == 4 ? k_crt_act<ACT_LOSS, 4> : CL == 2 ? k_crt_act<ACT_LOSS, 2> : k_crt_act<ACT_LOSS, 1>;
  const size_t smem = CL == 2 ? SMEM2_BYTES : SMEM_BYTES;
  static std::map<void*, int> max_clusters;  // co-resident clusters (persistent grid)
  static std::mutex mu;
  int grid_ctas;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = max_clusters.find((void*)kern);
    if (it == max_clusters.end()) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int mc = sm_count();
      if (CL > 1) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(CL * sm_count());
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, (const void*)kern, &cfg) != cudaSuccess || mc <= 0)
          mc = 0;
      }
      it = max_clusters.emplace((void*)kern, mc).first;
    }
    grid_ctas = CL * it->second;
  }
  if (grid_ctas <= 0) return false;
  const int64_t work = CL == 4   ? 4 * ((g.n_samples + 1) / 2 * (UT / 2))
                       : CL == 2 ? 2 * (g.n_samples * (UT / 2))
                                 : g.n_samples * UT;
  grid_ctas = (int)std::min<int64_t>(grid_ctas, work);
  count_launch();
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)grid_ctas);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // tile counter of the in-order schedule (independent CTAs): caller-owned (workspace), zeroed
  // here on the launch's stream; KP_CRT_DYNAMIC=0 keeps the static striding
  int* counter = nullptr;
  if (CL == 1 && tile_counter) {
    static const bool dyn = [] {
      const char* e = getenv("KP_CRT_DYNAMIC");
      return !(e && atoi(e) == 0);
    }();
    if (dyn) counter = tile_counter;
    if (counter && cudaMemsetAsync(counter, 0, sizeof(int), s) != cudaSuccess) return false;
  }
  return cudaLaunchKernelEx(&cfg, kern, mw, mh, exW, exH, g, UT, counter) == cudaSuccess;
}

}  // namespace kp
