"""Derive the moduli and CRT constants of paper_2405_15603_b200/csrc/kp_crt.cu.

    python tools/crt_constants.py [n_moduli]      # prints the C++ constant block

Moduli: the largest pairwise-coprime integers <= 256 (int8 symmetric residues).  M = prod p_i,
q_i = M / p_i, s_i = q_i^-1 mod p_i.  The CRT sum sum_i q_i t_i (|t_i| <= 128) is carried as an
exact FP64 high part (q_i rounded down to a multiple of 2^E, E chosen so that 12-13 terms of
(q_i >> E) * 128 stay below 2^53) plus an int32 low part c2_i ~ (q_i mod 2^E) / 2^k with
c2_i < 2^18.  BETA is the largest bit count with 2 K 2^(2 BETA) < M / 2^0.25 for K <= 1024.
Integer reduction of the int32 accumulators: w = acc + add_i >= 0 (add_i = p_i ceil(2^24 / p_i)
+ floor(p_i / 2)), w mod p_i = w - p_i ((w * m_i) >> 39), m_i = ceil(2^39 / p_i); verified here
for every w the kernel can produce.
"""
import math
import sys

ALL = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199]


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
    E = max(x.bit_length() for x in q) - 42
    while max((x >> E) for x in q) * 128 * n >= 2 ** 53:
        E += 1
    q1 = [(x >> E) << E for x in q]
    lo = [x - y for x, y in zip(q, q1)]
    k = max(0, max(v.bit_length() for v in lo) - 18)
    c2 = [round(v / 2 ** k) for v in lo]
    while max(c2) >= 2 ** 18:
        k += 1
        c2 = [round(v / 2 ** k) for v in lo]
    assert sum(c * 255 for c in c2) < 2 ** 31
    M1 = (M >> E) << E
    M2 = M - M1
    m = [-(-(1 << 39) // p) for p in mods]
    add = [p * (-(-(1 << 24) // p)) + p // 2 for p in mods]
    for p, mm, a in zip(mods, m, add):
        assert mm < 2 ** 32
        hi = (1 << 24) + a  # largest w: acc <= 2^24
        for w in list(range(0, 4096)) + list(range(hi - 4096, hi + 1)) + list(range(0, hi, 997)):
            assert (w * mm) >> 39 == w // p
    return dict(mods=mods, M=M, log2m=log2m, beta=beta, s=s, E=E, q1=q1, k=k, c2=c2, M1=M1,
                M2=M2, m=m, add=add)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    d = derive(n)
    f = lambda v: float(v).hex()
    print(f"// {n} moduli, log2 M = {d['log2m']:.3f}, BETA = {d['beta']}, E = {d['E']}, "
          f"low part c2 * 2^{d['k']}  (tools/crt_constants.py {n})")
    print(f"constexpr int NMOD = {n};")
    print(f"constexpr int BETA = {d['beta']};")
    print(f"constexpr double CR_LOW_SCALE = {f(2.0 ** d['k'])};")
    print("__constant__ double cr_pd[NMOD] = {" + ", ".join(str(p) for p in d["mods"]) + "};")
    print("__constant__ double cr_ipd[NMOD] = {" + ", ".join(f"1.0 / {p}" for p in d["mods"]) + "};")
    print("__constant__ double cr_s[NMOD] = {" + ", ".join(str(v) for v in d["s"]) + "};")
    print("__constant__ double cr_q1[NMOD] = {" + ", ".join(f(v) for v in d["q1"]) + "};")
    print("__constant__ uint32_t cr_c2[NMOD] = {" + ", ".join(f"{v}u" for v in d["c2"]) + "};")
    c2h = sum(c * (p // 2) for c, p in zip(d["c2"], d["mods"]))
    print(f"constexpr uint32_t CR_C2H = {c2h}u;  // sum c2_i floor(p_i / 2)")
    print(f"constexpr double CR_M1 = {f(d['M1'])}, CR_M2 = {f(d['M2'])}, CR_IM = {f(1.0 / d['M'])};")
    print("__constant__ uint32_t cr_m[NMOD] = {" + ", ".join(f"{v}u" for v in d["m"]) + "};")
    print("__constant__ uint32_t cr_add[NMOD] = {" + ", ".join(f"{v}u" for v in d["add"]) + "};")
    print("__constant__ uint32_t cr_pu[NMOD] = {" + ", ".join(str(p) for p in d["mods"]) + "};")
    print("__constant__ double cr_hd[NMOD] = {" + ", ".join(f"0x1p52 + {p // 2}" for p in d["mods"]) + "};")


if __name__ == "__main__":
    main()
