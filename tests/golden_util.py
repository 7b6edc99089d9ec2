"""Helpers to compare arrays against the golden fixtures (full arrays or summaries)."""

import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ("c1", "c2", "c3", "c4", "c5", "c1_momentum", "lfp", "dense")
STAR_NAMES = ("c1_star", "c3_star", "c5_star", "lfp_star", "dense_star")
# ten-step runs of the five BASELINE configs (arrays recorded at steps 1 and 10)
NAMES10 = ("c1_10", "c2_10", "c3_10", "c4_10", "c5_10", "lfp_10", "dense_10", "c1_momentum_10", "c4_zero_10")
STAR10 = ("c1_star_10", "lfp_star_10", "c3_star_10", "c5_star_10")
# the BASELINE sizes themselves (tests/golden/make_golden_full.py): c2-c4 at N_Omega = 3000,
# ten steps; c5 at 3000 / 1000, three steps (the benched code path); c5 KFAC* at 1000 / 333
NAMES_FULL = ("c2_full10", "c3_full10", "c4_full10", "c5_full3")
STAR_FULL = ("c5_star_n1000",)
FULL_WL = {"c2_full10": "c2", "c3_full10": "c3", "c4_full10": "c4", "c5_full3": "c5",
           "c5_star_n1000": "c5"}


def load(name):
    return dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")))


def has(g, key):
    return key in g or f"{key}#sum" in g


def max_rel(a, b):
    """||a - b||_max / max(||b||_max, tiny) (SURVEY.md §8c parity measure)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    assert a.shape == b.shape, (a.shape, b.shape)
    den = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / den if a.size else 0.0


def compare(g, key, arr, rtol):
    """Return the relative discrepancy of ``arr`` vs the golden entry ``key``."""
    arr = np.asarray(arr, dtype=np.float64).ravel()
    if key in g:
        return max_rel(arr, g[key])
    size = int(g[f"{key}#size"])
    assert arr.size == size, (key, arr.size, size)
    idx = g[f"{key}#idx"]
    errs = [max_rel(arr[idx], g[f"{key}#vals"])]
    for stat, val in (("abssum", np.abs(arr).sum()), ("sqsum", (arr * arr).sum())):
        ref = float(g[f"{key}#{stat}"])
        errs.append(abs(val - ref) / max(abs(ref), 1e-300))
    scale = float(g[f"{key}#abssum"])
    errs.append(abs(arr.sum() - float(g[f"{key}#sum"])) / max(scale, 1e-300))
    return max(errs)


def pack_factors(mats):
    return np.concatenate([np.asarray(m, dtype=np.float64).ravel() for m in mats])


def line_search_rel(ls, ref):
    """Worst relative discrepancy of the 31 line-search (interior, boundary) losses.

    Candidates whose total loss exceeds 1e3 x the smallest one are excluded: there the
    tanh network is saturated and the loss (up to ~1e31 for the zero-initialised c4 case)
    is dominated by roundoff — two NumPy runs of the same formulas already differ at 1e-8
    while the direction agrees to 1e-16.  The argmin is decided among the others; a finite /
    non-finite mismatch anywhere still fails."""
    ls = np.asarray(ls, dtype=np.float64).reshape(-1, 2)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1, 2)
    assert np.array_equal(np.isfinite(ls), np.isfinite(ref))
    tot = ref.sum(axis=1)
    fin = np.isfinite(tot)
    keep = fin & (tot <= 1e3 * np.min(tot[fin])) if fin.any() else fin
    if not keep.any():
        return 0.0
    return float(np.max(np.abs(ls[keep] - ref[keep]) / np.maximum(np.abs(ref[keep]), 1e-300)))
