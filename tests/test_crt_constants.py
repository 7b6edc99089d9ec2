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
    """The epilogue's fold and reconstruction, operation by operation (FP32 reduction, FP32 low
    part, exact FP64 high part against D = 1.5 +- t / 256), recover P = sum a_k b_k to far
    below the 2^(BETA+5) rounding of the inputs."""
    import crt_constants as cc
    import numpy as np

    d = cc.derive(n)
    mods, M = d["mods"], d["M"]
    rng = np.random.default_rng(n)
    K = 768
    lim = 2 ** d["beta"]
    f32 = np.float32
    for trial in range(200):
        a = [int(v) for v in rng.integers(-lim, lim + 1, K)]
        b = [int(v) for v in rng.integers(-lim, lim + 1, K)]
        if trial == 0:  # extreme accumulators: every residue product at its bound
            a = [lim] * K
            b = [lim] * K
        P = sum(x * y for x, y in zip(a, b))
        assert 2 * abs(P) < M
        high = -float(d["C1"])   # FP64, must stay exact (the kernel starts at -C1)
        high_exact = -d["C1"]   # the same sum in integers
        low = f32(0.0)
        for p, s, sg, sq, cl, q1 in zip(mods, d["s"], d["sg"], d["sq"], d["cl"], d["q1"]):
            # symmetric int8 residues; W's premultiplied by s_i
            acc = sum(((x + p // 2) % p - p // 2) * (((y * s) + p // 2) % p - p // 2)
                      for x, y in zip(a, b))
            assert abs(acc) <= 2 ** 24
            t = float(cc.reduce_f32(np.array([acc]), p)[0])
            assert abs(t) <= 128 and (acc - int(t)) % p == 0
            low = f32(np.float64(f32(t)) * np.float64(f32(cl)) + np.float64(low))  # FP32 FMA (product exact in FP64)
            g = f32(1.9375) + f32(t) * f32(sg * 2.0 ** -11)  # exact in FP32
            hi_word = int(np.array([g], dtype=np.float32).view(np.uint32)[0])
            D = np.array([hi_word << 32], dtype=np.uint64).view(np.float64)[0]
            assert D == 1.5 + sg * t / 256
            high_exact += int(D * 256) * (sq // 256)
            high = high + D * float(sq)  # FMA: product and sum are exact (checked next line)
            assert int(high) == high_exact
        X1 = high
        X2 = float(low)
        k = float(np.rint((X1 + X2) / float(M)))
        Prec = (X1 - k * float(d["M1"])) + (X2 - k * float(d["M2"]))
        assert abs(Prec - P) <= 2.0 ** (d["beta"] + 1), (Prec, P)


def test_fp32_reduction_full_range():
    """t = f - p rint(f / p) as the kernel computes it: congruent to acc and within [-128, 128]
    for every accumulator value |acc| <= 2^24 (strided sweep here; crt_constants.derive checks
    the neighbourhood of every rounding boundary)."""
    import crt_constants as cc
    import numpy as np

    for p in cc.ALL[:13]:
        acc = np.arange(-2 ** 24, 2 ** 24 + 1, 7, dtype=np.int64)
        t = cc.reduce_f32(acc, p)
        assert np.all(np.abs(t) <= 128)
        assert np.all((acc - t.astype(np.int64)) % p == 0)
