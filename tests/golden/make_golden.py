"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs ``/root/reference``; the GPU box does
not have it):

    python tests/golden/make_golden.py

For every BASELINE workload (c1..c5, reduced N for c2..c5 so the reference
finishes in seconds) it builds inputs with the reference's own seeding recipe
(``init_params`` / ``sample_batch`` seeded through ``_stream_seed``, reference
src/harness.py:64-66,249,284-286), runs the reference ``optimizer_step``
(src/optim.py:396-402) for a few steps, and records losses, alpha, the 31
line-search losses, ``grad_mats``, the preconditioned direction, the four factor
lists and the parameters.  Problems c3/c4/c5 are not in the reference catalog
verbatim; they are reference ``PdeProblem`` objects whose callables come from
this package's ``pde`` module (the rigged-problem pattern of the reference's
pkg/tests/test_harness.py:42-56).

Large arrays are stored as summaries (sum, sum|x|, sum x^2 and 512 entries at
fixed indices) so the fixtures stay small.
"""

from __future__ import annotations

import copy
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from pinnopt import curvature, network, optim, pde  # noqa: E402  (the reference)
from pinnopt.harness import _stream_seed  # noqa: E402

from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200 import pde as my_pde  # noqa: E402

FULL_LIMIT = 20000  # arrays up to this many entries are stored in full

PLAN = {
    # name: (workload key, n_interior, n_boundary, steps)
    "c1": ("c1", 3000, 500, 3),
    "c2": ("c2", 400, 100, 3),
    "c3": ("c3", 400, 200, 3),
    "c4": ("c4", 150, 50, 2),
    "c5": ("c5", 24, 8, 2),
    "c1_momentum": ("c1", 200, 60, 3),
    # KFAC* (src/optim.py:266-320): same inputs, exact Gramian-vector products + 2x2 model
    "c1_star": ("c1", 300, 80, 3),
    "c3_star": ("c3", 200, 100, 3),
    "c5_star": ("c5", 24, 8, 2),
    # reference catalog log-Fokker-Planck (non-affine residual, per-point seeds)
    "lfp": ("lfp", 300, 100, 3),
    "lfp_star": ("lfp", 300, 100, 3),
    # dense (non-diagonal) operator coefficients (src/taylor.py:72-75)
    "dense": ("dense", 400, 100, 3),
    "dense_star": ("dense", 300, 100, 3),
}

# Ten-step runs of the five BASELINE configs (north star: 1e-10 after one step, 1e-8 after
# ten).  c1 at its full size; c2-c5 reduced so the reference finishes in seconds.  Arrays are
# recorded at steps 1 and 10 only; every step records losses, alpha and the line search.
PLAN10 = {
    "c1_10": ("c1", 3000, 500, 10),
    "c2_10": ("c2", 1000, 200, 10),
    "c3_10": ("c3", 1000, 400, 10),
    "c4_10": ("c4", 400, 130, 10),
    "c5_10": ("c5", 24, 8, 10),
    # the section-8(f) paths over ten steps: KFAC* (c1 at full size), the log-Fokker-Planck
    # residual (KFAC and KFAC*) and dense operator coefficients
    "c1_star_10": ("c1", 3000, 500, 10),
    "lfp_10": ("lfp", 300, 100, 10),
    "lfp_star_10": ("lfp", 300, 100, 10),
    "dense_10": ("dense", 400, 100, 10),
    "c3_star_10": ("c3", 400, 200, 10),
    "c5_star_10": ("c5", 24, 8, 10),
    "c1_momentum_10": ("c1", 600, 150, 10),
    "c4_zero_10": ("c4", 400, 130, 10),  # init_mode="zero" (src/curvature.py:62-76)
}
FULL_RECORD_STEPS = {1, 10}


def ref_problem(wl):
    """Reference PdeProblem for a workload (catalog where it exists, else rigged)."""
    if wl.problem in ("poisson2d_sin", "log_fokker_planck"):
        return pde.make_problem(wl.problem)
    if (wl.problem == "poisson_cos_sum" and dict(wl.problem_params).get("dim", 5) == 5
            and wl.dense_coeffs_seed is None):
        return pde.make_problem("poisson_cos_sum")
    mine = wl.make_problem()
    coeffs = pde.OperatorCoeffs(np.asarray(mine.coeffs.c))
    return pde.PdeProblem(
        name=mine.name, dim=mine.dim, coeffs=coeffs, lower=mine.lower, upper=mine.upper,
        boundary_kind=mine.boundary_kind, residual=mine.residual,
        residual_grads=mine.residual_grads, boundary_target=mine.boundary_target,
        true_solution=mine.true_solution,
    )


def summary(a):
    a = np.asarray(a, dtype=np.float64).ravel()
    k = min(512, a.size)
    idx = np.sort(np.random.default_rng(a.size).choice(a.size, size=k, replace=False))
    return {"sum": a.sum(), "abssum": np.abs(a).sum(), "sqsum": (a * a).sum(),
            "idx": idx, "vals": a[idx], "size": np.array(a.size)}


def put(out, key, arr):
    arr = np.asarray(arr, dtype=np.float64)
    if arr.size <= FULL_LIMIT:
        out[key] = arr
    else:
        for k, v in summary(arr).items():
            out[f"{key}#{k}"] = v


def main():
    only = set(sys.argv[1:])
    for name, (wkey, n_int, n_bnd, steps) in {**PLAN, **PLAN10}.items():
        ten = name in PLAN10
        if only and name not in only:
            continue
        wl = cfgs.WORKLOADS[wkey]
        prob = ref_problem(wl)
        arch = network.Architecture(wl.widths)
        params = network.init_params(arch, _stream_seed(0, 0))
        batch = pde.sample_batch(prob, n_int, n_bnd, _stream_seed(0, 1, 0))
        momentum = 0.9 if "momentum" in name else wl.momentum
        kind = "kfac_star" if "_star" in name else "kfac"
        cfg = optim.OptimizerConfig(kind=kind, damping=wl.damping, ema=wl.ema,
                                    momentum=momentum,
                                    init_mode="zero" if "zero" in name else "identity")
        state = optim.init_train_state(params, cfg)
        out = {"widths": np.array(wl.widths), "n_interior": np.array(n_int),
               "init_zero": np.array(1 if "zero" in name else 0),
               "n_boundary": np.array(n_bnd), "momentum": np.array(momentum),
               "damping": np.array(wl.damping), "ema": np.array(wl.ema)}
        put(out, "in/interior", batch.interior)
        put(out, "in/boundary", batch.boundary)
        put(out, "in/targets", batch.boundary_targets)
        put(out, "in/theta", network.params_to_vec(params))
        if wl.dense_coeffs_seed is not None:
            from pinnopt import taylor as ref_taylor
            out["in/coeffs"] = np.asarray(prob.coeffs.c)
            _, tout = ref_taylor.taylor_forward(params, batch.interior, prob.coeffs)
            put(out, "taylor/value", tout.value)
            put(out, "taylor/gradient", tout.gradient)
            put(out, "taylor/operator", tout.operator)
        for t in range(1, steps + 1):
            # intermediates of this step, recomputed exactly as kfac_step does (optim.py:237-263)
            ev = optim.evaluate_batch(state.params, batch, prob)
            kf = copy.deepcopy(state.kfac)
            n_lin = state.params.n_linear
            lin_in = [ev.states[2 * l] for l in range(n_lin)]
            lin_gr = [ev.taylor_grads.layer_grads[2 * l + 1] for l in range(n_lin)]
            curvature.interior_factor_update(kf, lin_in, lin_gr)
            curvature.boundary_factor_update(kf, ev.boundary_trace.linear_inputs, ev.boundary_grads)
            delta = curvature.precondition_gradient(kf, ev.grad_mats)
            direction = [d + momentum * p for d, p in zip(delta, state.prev_update)]
            pre = f"s{t}/"
            if kind == "kfac":
                grid = cfg.line_search_grid()
                ls = np.array([optim.evaluate_losses(network.add_scaled(state.params, direction, a),
                                                     batch, prob) for a in grid])
                out[pre + "ls_losses"] = ls
            info = optim.optimizer_step(state, batch, prob)
            out[pre + "loss_interior"] = np.array(info.loss_interior)
            out[pre + "loss_boundary"] = np.array(info.loss_boundary)
            out[pre + "alpha"] = np.array(info.alpha)
            out[pre + "mu"] = np.array(info.mu)
            if ten and t not in FULL_RECORD_STEPS:
                print(f"{name} step {t}: loss={info.loss_total:.6e} alpha={info.alpha:.10g}",
                      flush=True)
                continue
            put(out, pre + "grad", network.mats_to_vec(ev.grad_mats))
            put(out, pre + "delta", network.mats_to_vec(delta))
            put(out, pre + "theta", network.params_to_vec(state.params))
            put(out, pre + "prev_update", network.mats_to_vec(state.prev_update))
            for fname in ("a_interior", "b_interior", "a_boundary", "b_boundary"):
                mats = getattr(state.kfac, fname)
                put(out, pre + fname, np.concatenate([m.ravel() for m in mats]))
            print(f"{name} step {t}: loss={info.loss_total:.6e} alpha={info.alpha:.10g} "
                  f"mu={info.mu:.10g}", flush=True)
        out["numpy_version"] = np.array(np.__version__)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


if __name__ == "__main__":
    main()
