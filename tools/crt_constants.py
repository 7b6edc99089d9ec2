"""Derive the moduli and CRT constants of paper_2405_15603_b200/csrc/kp_crt.cu.

    python tools/crt_constants.py [n_moduli]      # prints the C++ constant block

Moduli: the largest pairwise-coprime integers <= 256 (int8 symmetric residues).  M = prod p_i,
q_i = M / p_i, s_i = q_i^-1 mod p_i (folded into the weight residues), BETA the largest bit
count with 2 K 2^(2 BETA) < M / 2^0.25 for K <= 1024.

Fold of one int32 accumulator acc (|acc| <= 2^24, exact in FP32) of modulus i, as the kernel's
epilogue does it:
    f = float(acc);  q = rint(f * ipf_i) (magic-number rounding inside one FMA);  t = f - q p_i
    (exact; t = acc mod p_i up to the tie, |t| <= 128 -- `reduce_f32` below, checked here)
    low  += t * cl_i                      FP32, cl_i = float(q_i mod 2^E)
    D     = 1.5 + sg_i t / 256            (the FP64 whose high word is the bit pattern of the
                                           FP32 1.9375 + sg_i t 2^-11, low word 0)
    high += D * (sg_i 256 q1_i)           FP64, q1_i = q_i - (q_i mod 2^E); adds q1_i t +
                                           384 sg_i q1_i, sg_i = +-1 alternating
so, started at -C1 (C1 = 384 sum sg_i q1_i), high = sum q1_i t_i exactly: every partial sum is a multiple
of 2^E below 2^(E+53) (`derive` picks E for that; the alternating signs keep the 384 q1_i
offsets from piling up).  P = high + low - k M with k = rint((high + low) / M).  The
FP32 low part is accurate to 2^(BETA - 1), far below the 2^(BETA + 5) rounding of the inputs.
"""
import math
import sys
from fractions import Fraction

import numpy as np

ALL = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199]
MAGICF = 12582912.0  # 1.5 * 2^23


def reduce_f32(acc, p):
    """The kernel's FP32 modular reduction of int32 accumulators (vectorised, exact emulation:
    a 24-bit by 24-bit product is exact in FP64 and the FMA's single rounding lands on the
    integer grid of [2^23, 2^24), ties to even)."""
    f = np.asarray(acc, dtype=np.float64)
    ip = float(np.float32(1.0) / np.float32(p))
    q = np.rint(f * ip)
    return f - q * p


def derive(n):
    mods = ALL[:n]
    for i in range(n):
        for j in range(i):
            assert math.gcd(mods[i], mods[j]) == 1
    M = math.prod(mods)
    log2m = math.log2(M)
    beta = int(math.floor((log2m - 0.25 - math.log2(2 * 1024)) / 2))
    q = [M // p for p in mods]
    s = [pow(x % p, -1, p) for x, p in zip(q, mods)]
    sg = [1 if i % 2 == 0 else -1 for i in range(n)]

    def worst_partial(E):
        q1 = [(x >> E) << E for x in q]
        c1 = 384 * sum(a * b for a, b in zip(sg, q1))
        worst, const, mag = abs(c1), -c1, 0  # the kernel starts the high part at -C1
        for a, b in zip(sg, q1):
            const += 384 * a * b
            mag += 128 * b
            worst = max(worst, abs(const) + mag)
        return worst

    E = max(x.bit_length() for x in q) - 44
    while worst_partial(E) >= 2 ** (E + 53):
        E += 1
    q1 = [(x >> E) << E for x in q]
    lo = [x - y for x, y in zip(q, q1)]
    cl = [float(np.float32(v)) for v in lo]
    sq = [a * 256 * b for a, b in zip(sg, q1)]
    C1 = 384 * sum(a * b for a, b in zip(sg, q1))
    for v in sq + [C1] + q1:
        assert int(float(v)) == v  # exactly representable
    # FP32 low part: representation error of cl_i plus 13 roundings of the running sum
    low_max = sum(128 * c for c in cl)
    low_err = sum(128 * abs(c - v) for c, v in zip(cl, lo)) + n * 2.0 ** (math.ceil(math.log2(low_max)) - 24)
    assert low_err < 2.0 ** (beta - 1), math.log2(low_err)
    M1 = (M >> E) << E
    M2 = M - M1
    # the FP32 reduction: congruent and |t| <= 128 near every rounding boundary and on a sweep
    for p in mods:
        edge = np.arange(-4, 5)
        mult = np.arange(-(2 ** 24) // p - 1, 2 ** 24 // p + 2, 257)
        acc = np.concatenate([(mult[:, None] * p + p // 2 + edge[None, :]).ravel(),
                              (mult[:, None] * p + edge[None, :]).ravel(),
                              np.arange(-2 ** 24, 2 ** 24 + 1, 1009),
                              np.arange(2 ** 24 - 70000, 2 ** 24 + 1), np.arange(-2 ** 24, -2 ** 24 + 70000)])
        acc = acc[np.abs(acc) <= 2 ** 24]
        t = reduce_f32(acc, p)
        assert np.all(np.abs(t) <= 128) and np.all((acc - t.astype(np.int64)) % p == 0)
    return dict(mods=mods, M=M, log2m=log2m, beta=beta, s=s, E=E, q1=q1, lo=lo, cl=cl, sg=sg, sq=sq,
                C1=C1, M1=M1, M2=M2)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 13
    d = derive(n)
    f = lambda v: float(v).hex()
    ff = lambda v: float(np.float32(v)).hex() + "f"
    print(f"// {n} moduli, log2 M = {d['log2m']:.3f}, BETA = {d['beta']}, E = {d['E']}"
          f"  (tools/crt_constants.py {n})")
    print(f"constexpr int NMOD = {n};")
    print(f"constexpr int BETA = {d['beta']};")
    print("__constant__ double cr_pd[NMOD] = {" + ", ".join(str(p) for p in d["mods"]) + "};")
    print("__constant__ double cr_ipd[NMOD] = {" + ", ".join(f"1.0 / {p}" for p in d["mods"]) + "};")
    print("__constant__ double cr_s[NMOD] = {" + ", ".join(str(v) for v in d["s"]) + "};")
    print("__constant__ float cr_npf[NMOD] = {" + ", ".join(f"-{p}.0f" for p in d["mods"]) + "};")
    print("__constant__ float cr_ipf[NMOD] = {" + ", ".join(ff(np.float32(1.0) / np.float32(p)) for p in d["mods"]) + "};")
    print("__constant__ float cr_cl[NMOD] = {" + ", ".join(ff(v) for v in d["cl"]) + "};")
    print("__constant__ float cr_sg[NMOD] = {" + ", ".join(ff(a * 2.0 ** -11) for a in d["sg"]) + "};")
    print("__constant__ double cr_sq[NMOD] = {" + ", ".join(f(v) for v in d["sq"]) + "};")
    print(f"constexpr double CR_C1 = {f(d['C1'])};  // 384 sum sg_i q1_i")
    print(f"constexpr double CR_M1 = {f(d['M1'])}, CR_M2 = {f(d['M2'])}, CR_IM = {f(1.0 / d['M'])};")


if __name__ == "__main__":
    main()
