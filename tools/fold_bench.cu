// Issue-rate probe of the CRT fold (kp_crt.cu epilogue) in isolation: 8 warps per SM (two per
// scheduler, 232 registers as in k_crt_act), each thread folding 56 accumulator columns per
// modulus into the CRT sums; the int32 "accumulators" come from shared memory (LDS.128 stands
// in for tcgen05.ld).  Variants:
//   0  the two-FP64 fold (DADD + DFMA per term), constants in uniform registers
//   1  the same with the constants laundered into vector registers
//   2  one-DFMA fold: D = 1.5 +- t/256 built in the high word, alternating signs
//   3  variant 2 with laundered constants
//   4  integer part only (no FP64)
//   5  FP64 part only (no modular reduction)
//   6  FP32 modular reduction (I2FP, FFMA magic rounding) + one-DFMA fold, uniform constants
//   7  variant 6 with laundered constants
//   8  packed FP32 (f32x2) reduction, FP32 low part, persistent zero-low D pairs, one DFMA
// Prints clocks per modulus step per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fold_bench fold_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int NMOD = 13, CPW = 56;
__constant__ uint32_t c_add[NMOD], c_m[NMOD], c_pu[NMOD], c_c2[NMOD];
__constant__ double c_hd[NMOD], c_q1[NMOD];
__constant__ uint32_t c_hib[NMOD], c_him[NMOD];
__constant__ double c_sq[NMOD];
__constant__ float c_pf[NMOD], c_ipf[NMOD];
__constant__ uint32_t c_hib6[NMOD];

template <bool LAUNDER>
__device__ __forceinline__ uint32_t lu(uint32_t v) {
  if (LAUNDER) asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
template <bool LAUNDER>
__device__ __forceinline__ float lf(float v) {
  if (LAUNDER) asm volatile("mov.b32 %0, %0;" : "+f"(v));
  return v;
}
template <bool LAUNDER>
__device__ __forceinline__ double ld(double v) {
  if (LAUNDER) asm volatile("mov.b64 %0, %0;" : "+d"(v));
  return v;
}

__device__ __forceinline__ uint64_t pk(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t pk_launder(float lo, float hi) {
  uint64_t d;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
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
// hi word of the zero-low pair D <- bits of fmaf(t, s, B)
__device__ __forceinline__ void set_hi(double& D, float t, float s, float B) {
  asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %0;\nfma.rn.f32 hi, %1, %2, %3;\nmov.b64 %0, {lo, hi};\n}"
      : "+d"(D)
      : "f"(t), "f"(s), "f"(B));
}

// variant 8: state x1 (FP64) and the low part as packed FP32 pairs
template <int F>
__global__ void __launch_bounds__(256, 1) k_fold8(int iters, double* out, long long* cyc) {
  __shared__ uint32_t acc[CPW * 32 + 64];
  for (int i = threadIdx.x; i < CPW * 32 + 64; i += blockDim.x) acc[i] = (i * 2654435761u) >> 9;
  __syncthreads();
  double x1[CPW];
  uint64_t x2[CPW / 2];
#pragma unroll
  for (int j = 0; j < CPW; ++j) x1[j] = 0.0;
#pragma unroll
  for (int j = 0; j < CPW / 2; ++j) x2[j] = 0ull;
  constexpr int ND = 8;
  double D[ND];
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    D[j] = 0.0;
    asm volatile("mov.b64 %0, %0;" : "+d"(D[j]));
  }
  const float MAGICF = 12582912.0f;
  const uint64_t magic2 = pk_launder(MAGICF, MAGICF), nmagic2 = pk_launder(-MAGICF, -MAGICF);
  float Bc = 1.9375f;
  asm volatile("mov.b32 %0, %0;" : "+f"(Bc));
  const int lane = threadIdx.x & 31;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int i = 0; i < NMOD; ++i) {
      const float pf = c_pf[i], ipf = c_ipf[i];
      const uint64_t ip2 = pk_launder(ipf, ipf), np2 = pk_launder(-pf, -pf);
      float clf = (float)c_c2[i];
      const uint64_t cl2 = pk_launder(clf, clf);
      float sg = (i & 1) ? -0x1p-11f : 0x1p-11f;
      asm volatile("mov.b32 %0, %0;" : "+f"(sg));
      double sq = c_sq[i];
      asm volatile("mov.b64 %0, %0;" : "+d"(sq));
      uint32_t r[CPW];
#pragma unroll
      for (int j = 0; j < CPW; j += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(&acc[((j * 8 + lane * 4 + it) & 1023) & ~3]);
        r[j] = v.x;
        r[j + 1] = v.y;
        r[j + 2] = v.z;
        r[j + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < CPW; j += 2) {
        const float fa = (F & 1) ? __int_as_float(r[j] & 0x4affffff) : __int2float_rn((int)r[j]);
        const float fb = (F & 1) ? __int_as_float(r[j + 1] & 0x4affffff) : __int2float_rn((int)r[j + 1]);
        const uint64_t f2 = pk(fa, fb);
        const uint64_t q2 = fadd2(ffma2(f2, ip2, magic2), nmagic2);
        const uint64_t t2 = ffma2(q2, np2, f2);
        if (!(F & 4)) x2[j / 2] = ffma2(t2, cl2, x2[j / 2]);
        float ta, tb;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(ta), "=f"(tb) : "l"(t2));
        if (F & 2) {
          x2[(j / 2 + 1) % (CPW / 2)] = ffma2(t2, ip2, x2[(j / 2 + 1) % (CPW / 2)]);
        } else if (F & 8) {
          x1[j] = fma(D[j % ND], sq, x1[j]);
          x1[j + 1] = fma(D[(j + 1) % ND], sq, x1[j + 1]);
          x2[(j / 2 + 1) % (CPW / 2)] = ffma2(t2, ip2, x2[(j / 2 + 1) % (CPW / 2)]);
        } else {
          set_hi(D[j % ND], ta, sg, Bc);
          set_hi(D[(j + 1) % ND], tb, sg, Bc);
          x1[j] = fma(D[j % ND], sq, x1[j]);
          x1[j + 1] = fma(D[(j + 1) % ND], sq, x1[j + 1]);
        }
      }
    }
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) s += x1[j];
#pragma unroll
  for (int j = 0; j < CPW / 2; ++j) s += (double)(x2[j] >> 32) + (double)(uint32_t)x2[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
__global__ void __launch_bounds__(256, 1) k_fold(int iters, double* out, long long* cyc) {
  __shared__ uint32_t acc[CPW * 32 + 64];
  for (int i = threadIdx.x; i < CPW * 32 + 64; i += blockDim.x) acc[i] = (i * 2654435761u) >> 9;
  __syncthreads();
  constexpr bool L = (V == 1 || V == 3 || V == 7);
  double x1[CPW];
  uint32_t x2[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    x1[j] = 0.0;
    x2[j] = 0u;
  }
  const int lane = threadIdx.x & 31;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int i = 0; i < NMOD; ++i) {
      const uint32_t add = lu<L>(c_add[i]), m = lu<L>(c_m[i]), negp = lu<L>(0u - c_pu[i]),
                     c2 = lu<L>(c_c2[i]);
      const double hd = ld<L>(c_hd[i]), q1 = ld<L>(c_q1[i]);
      const uint32_t hib = lu<L>(c_hib[i]), him = lu<L>(c_him[i]);
      const double sq = ld<L>(c_sq[i]);
      const float pf = lf<L>(c_pf[i]), ipf = lf<L>(c_ipf[i]);
      const uint32_t hib6 = lu<L>(c_hib6[i]);
      uint32_t r[CPW];
#pragma unroll
      for (int j = 0; j < CPW; j += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(&acc[((j * 8 + lane * 4 + it) & 1023) & ~3]);
        r[j] = v.x;
        r[j + 1] = v.y;
        r[j + 2] = v.z;
        r[j + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < CPW; ++j) {
        if (V == 5) {
          x1[j] = fma(__hiloint2double(0x43300000, (int)r[j]) - hd, q1, x1[j]);
          continue;
        }
        if (V == 6 || V == 7) {
          const float MAGICF = 12582912.0f;
          const float f = __int2float_rn((int)r[j]);
          const float q = fmaf(f, ipf, MAGICF) - MAGICF;
          const float t = fmaf(-q, pf, f);
          const uint32_t bits = (uint32_t)__float_as_int(t + MAGICF);
          x2[j] += bits * c2;
          x1[j] = fma(__hiloint2double((int)(bits * him + hib6), 0), sq, x1[j]);
          continue;
        }
        const uint32_t w = r[j] + add;
        const uint32_t t = w + (__umulhi(w, m) >> 7) * negp;
        x2[j] += t * c2;
        if (V == 0 || V == 1) {
          x1[j] = fma(__hiloint2double(0x43300000, (int)t) - hd, q1, x1[j]);
        } else if (V == 2 || V == 3) {
          x1[j] = fma(__hiloint2double((int)(t * him + hib), 0), sq, x1[j]);
        }
      }
    }
  }
  const long long t1 = clock64();
  double s = 0.0;
  uint32_t u = 0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    s += x1[j];
    u += x2[j];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (double)u;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int iters, double* out, long long* cyc) {
  k_fold<V><<<148, 256>>>(2, out, cyc);
  cudaDeviceSynchronize();
  k_fold<V><<<148, 256>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  avg /= 148.0;
  printf("%-44s %8.0f clk per modulus step per SM (8 warps x 56 columns)  [%s]\n", name,
         avg / ((double)iters * NMOD), cudaGetErrorString(e));
}

// variant 12: 64-bit fixed-point fold: acc64 += bits * round(2^64 / p) (IMAD.WIDE.U32 + IMAD),
// bits = 0x4B400000 + t from the packed FP32 reduction; no FP64, two registers per column
__global__ void __launch_bounds__(256, 1) k_fold12(int iters, double* out, long long* cyc) {
  __shared__ uint32_t acc[CPW * 32 + 64];
  __shared__ uint32_t zs[32];
  for (int i = threadIdx.x; i < CPW * 32 + 64; i += blockDim.x) acc[i] = (i * 2654435761u) >> 9;
  if (threadIdx.x < 32) zs[threadIdx.x] = 0;
  __syncthreads();
  uint64_t x[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) x[j] = 0ull;
  const int lane = threadIdx.x & 31;
  uint32_t tz;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tz) : "r"((uint32_t)__cvta_generic_to_shared(&zs[lane])));
  const float MAGICF = 12582912.0f;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int i = 0; i < NMOD; ++i) {
      const float ipf = __uint_as_float(__float_as_uint(c_ipf[i]) | tz);
      const float npf = __uint_as_float(__float_as_uint(-c_pf[i]) | tz);
      const uint64_t ip2 = pk(ipf, ipf), np2 = pk(npf, npf);
      const uint64_t mg = pk(MAGICF, MAGICF), nmg = pk(-MAGICF, -MAGICF);
      const uint32_t clo = c_m[i] | tz, chi = c_add[i] | tz;
      uint32_t r[CPW];
#pragma unroll
      for (int j = 0; j < CPW; j += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(&acc[((j * 8 + lane * 4 + it) & 1023) & ~3]);
        r[j] = v.x;
        r[j + 1] = v.y;
        r[j + 2] = v.z;
        r[j + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < CPW; j += 2) {
        const uint64_t f2 = pk(__int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]));
        const uint64_t q2 = fadd2(ffma2(f2, ip2, mg), nmg);
        const uint64_t b2 = fadd2(ffma2(q2, np2, f2), mg);
        const uint32_t ba = (uint32_t)b2, bb = (uint32_t)(b2 >> 32);
        asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[j]) : "r"(ba), "r"(clo));
        asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %0;\nmad.lo.u32 hi, %1, %2, hi;\nmov.b64 %0, {lo, hi};\n}" : "+l"(x[j]) : "r"(ba), "r"(chi));
        asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[j + 1]) : "r"(bb), "r"(clo));
        asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %0;\nmad.lo.u32 hi, %1, %2, hi;\nmov.b64 %0, {lo, hi};\n}" : "+l"(x[j + 1]) : "r"(bb), "r"(chi));
      }
    }
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) s += (double)(long long)x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// reconstruction tail of kp_crt.cu in isolation: 56 columns per thread, 8 warps per SM.
// CV = 0: F2F.F64.F32 for the FP32 low part, 1: integer bit manipulation, 2: no conversion
template <int CV>
__global__ void __launch_bounds__(256, 1) k_tail(int iters, double* out, long long* cyc) {
  __shared__ double sc[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) sc[i] = 1.0 + i * 0x1p-20;
  __syncthreads();
  double x1[CPW];
  float x2[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    x1[j] = 0x1p+100 * (1 + j + threadIdx.x);
    x2[j] = 0x1p+60f * (1 + j);
  }
  const double IM = 0x1.63f115f5d0b38p-103, MG = 6755399441055744.0, M1 = 0x1.703d73109e938p+102,
               M2 = 0x1.6d0683e4deb00p+52;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      double X2;
      if (CV == 0) {
        X2 = (double)x2[j];
      } else if (CV == 1) {
        const uint32_t b = __float_as_uint(x2[j]);
        const uint32_t mag = b & 0x7fffffffu;
        const uint32_t hi = (b & 0x80000000u) | ((mag >> 3) + (mag ? 0x38000000u : 0u));
        X2 = __hiloint2double((int)hi, (int)(b << 29));
      } else {
        X2 = __hiloint2double(__float_as_int(x2[j]), 0);
      }
      const double k = fma(x1[j] + X2, IM, MG) - MG;
      const double P = fma(-k, M1, x1[j]) + fma(-k, M2, X2);
      const double y = P * sc[(j + it) & 127];
      x1[j] = y * 0x1p+40 + 0x1p+100;
      x2[j] = x2[j] * 1.0000001f;
    }
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) s += x1[j] + x2[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CV>
void run_tail(const char* name, int iters, double* out, long long* cyc) {
  k_tail<CV><<<148, 256>>>(2, out, cyc);
  cudaDeviceSynchronize();
  k_tail<CV><<<148, 256>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  printf("%-50s %8.0f clk per 56-column reconstruction per SM  [%s]\n", name, avg / 148.0 / iters, cudaGetErrorString(e));
}

template <int F>
void run8(const char* name, int iters, double* out, long long* cyc) {
  k_fold8<F><<<148, 256>>>(2, out, cyc);
  cudaDeviceSynchronize();
  k_fold8<F><<<148, 256>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  printf("%-50s %8.0f clk per modulus step per SM  [%s]\n", name, avg / 148.0 / ((double)iters * NMOD), cudaGetErrorString(e));
}

int main() {
  uint32_t add[NMOD], m[NMOD], pu[NMOD], c2[NMOD], hib[NMOD], him[NMOD];
  double hd[NMOD], q1[NMOD], sq[NMOD];
  float pf[NMOD], ipf[NMOD];
  uint32_t hib6[NMOD];
  const int p[NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211};
  for (int i = 0; i < NMOD; ++i) {
    pu[i] = p[i];
    add[i] = (1u << 24) / p[i] * p[i] + p[i] / 2;
    m[i] = (uint32_t)(((1ull << 39) + p[i] - 1) / p[i]);
    c2[i] = 100000 + 1000 * i;
    hd[i] = 4503599627370496.0 + p[i] / 2;
    q1[i] = 0x1.7p+94 + i * 0x1p+80;
    const int sign = (i & 1) ? -1 : 1;
    hib[i] = 0x3FF80000u - (uint32_t)(sign * ((p[i] / 2) << 12));
    him[i] = (uint32_t)(sign * 4096);
    sq[i] = sign * 256.0 * q1[i];
    pf[i] = (float)p[i];
    ipf[i] = 1.0f / (float)p[i];
    hib6[i] = 0x3FF80000u - 0x4B400000u * him[i];
  }
  cudaMemcpyToSymbol(c_add, add, sizeof(add));
  cudaMemcpyToSymbol(c_m, m, sizeof(m));
  cudaMemcpyToSymbol(c_pu, pu, sizeof(pu));
  cudaMemcpyToSymbol(c_c2, c2, sizeof(c2));
  cudaMemcpyToSymbol(c_hd, hd, sizeof(hd));
  cudaMemcpyToSymbol(c_q1, q1, sizeof(q1));
  cudaMemcpyToSymbol(c_hib, hib, sizeof(hib));
  cudaMemcpyToSymbol(c_him, him, sizeof(him));
  cudaMemcpyToSymbol(c_sq, sq, sizeof(sq));
  cudaMemcpyToSymbol(c_pf, pf, sizeof(pf));
  cudaMemcpyToSymbol(c_ipf, ipf, sizeof(ipf));
  cudaMemcpyToSymbol(c_hib6, hib6, sizeof(hib6));
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 200;
  run<0>("0 two-FP64 fold, uniform constants", iters, out, cyc);
  run<1>("1 two-FP64 fold, vector-register constants", iters, out, cyc);
  run<2>("2 one-DFMA fold, uniform constants", iters, out, cyc);
  run<3>("3 one-DFMA fold, vector-register constants", iters, out, cyc);
  run<4>("4 integer part only", iters, out, cyc);
  run<5>("5 FP64 part only (DADD + DFMA)", iters, out, cyc);
  run<6>("6 FP32 reduction + one-DFMA, uniform constants", iters, out, cyc);
  run<7>("7 FP32 reduction + one-DFMA, vector constants", iters, out, cyc);
  run8<0>("8 packed f32x2 fold", iters, out, cyc);
  run8<1>("8 ... without I2FP", iters, out, cyc);
  run8<2>("8 ... without the D construction and DFMA", iters, out, cyc);
  run8<3>("8 ... without I2FP, D, DFMA", iters, out, cyc);
  run8<8>("8 ... DFMA on stale D (no scalar FFMA)", iters, out, cyc);
  {
    k_fold12<<<148, 256>>>(2, out, cyc);
    cudaDeviceSynchronize();
    k_fold12<<<148, 256>>>(iters, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += (double)h[i];
    printf("%-50s %8.0f clk per modulus step per SM  [%s]\n", "12 fixed-point 64-bit fold (no FP64)", avg / 148.0 / ((double)iters * NMOD), cudaGetErrorString(e));
  }
  run_tail<0>("tail, F2F.F64.F32 conversion", 400, out, cyc);
  run_tail<1>("tail, integer conversion", 400, out, cyc);
  run_tail<2>("tail, no conversion", 400, out, cyc);
  return 0;
}
