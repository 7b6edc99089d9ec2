"""The CRT (INT8 tensor-core) line-search layer's constants (csrc/kp_crt.cu) are the ones
tools/crt_constants.py derives, and the derivation's exactness conditions hold (CPU test)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_kernel_constants_match_generator():
    src = open(os.path.join(ROOT, "paper_2405_15603_b200", "csrc", "kp_crt.cu")).read()
    n = int(re.search(r"constexpr int NMOD = (\d+);", src).group(1))
    gen = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "crt_constants.py"), str(n)],
                         capture_output=True, text=True, check=True).stdout
    for line in gen.strip().splitlines():
        assert line in src, line


@pytest.mark.parametrize("n", [12, 13])
def test_crt_reconstruction_is_exact(n):
    import crt_constants as cc
    import numpy as np

    d = cc.derive(n)
    mods, M = d["mods"], d["M"]
    rng = np.random.default_rng(n)
    K = 768
    lim = 2 ** d["beta"]
    for _ in range(200):
        a = [int(v) for v in rng.integers(-lim, lim + 1, K)]
        b = [int(v) for v in rng.integers(-lim, lim + 1, K)]
        P = sum(x * y for x, y in zip(a, b))
        assert 2 * abs(P) < M
        # per modulus: W residues premultiplied by s_i, t' = acc mod p in [0, p)
        x1 = 0.0
        x2 = 0
        for p, s, q1, c2 in zip(mods, d["s"], d["q1"], d["c2"]):
            acc = sum(((x + p // 2) % p - p // 2) * (((y * s) + p // 2) % p - p // 2)
                      for x, y in zip(a, b))
            assert abs(acc) <= 2 ** 24
            t = (acc + p // 2) % p  # t' of the kernel: (acc + add_i) mod p_i
            x1 += float(q1) * float(t - p // 2)  # exact: q1 multiple of 2^E, small t
            x2 += c2 * t
        c2h = sum(c * (p // 2) for c, p in zip(d["c2"], mods))
        X2 = float(x2 - c2h) * 2.0 ** d["k"]
        k = round((x1 + X2) / float(M))
        Prec = (x1 - k * float(d["M1"])) + (X2 - k * float(d["M2"]))
        assert abs(Prec - P) <= 2.0 ** (d["beta"] + 4), (Prec, P)
