"""Golden fixtures at the BASELINE sizes, produced by running the REFERENCE itself.

Run in the build container only (needs ``/root/reference``):

    python tests/golden/make_golden_full.py [name ...]

``make_golden.py`` cut c2..c5 to a few hundred points so the reference finishes in
seconds.  This script runs the reference ``optimizer_step`` (src/optim.py:396-402) on the
BASELINE.json sizes themselves:

* c2, c3, c4 at N_Omega = 3000 (N_b 500 / 1000 / 1000), ten KFAC steps each;
* c5 (100d Poisson) at N_Omega = 3000, N_b = 1000, three KFAC steps (the benched code path:
  one-candidate line search, early preconditioning, the large factor pairs); about 10 min
  and 39 GB RSS per reference step;
* c5 KFAC* at N_Omega = 1000, N_b = 333, two steps (the reference materialises the
  N x D residual Jacobian, src/curvature.py:169-194: 10.6 GB at N = 1000).

Unlike ``make_golden.py`` the step's intermediates are not recomputed (that would double
the c5 cost and memory): ``curvature.precondition_gradient`` and ``optim.evaluate_losses``
are wrapped for the duration of the step so the gradient, the direction and the 31
line-search losses the reference step itself computed are recorded
(src/optim.py:237-263, 195-211).  Inputs use the reference seeding recipe
(src/harness.py:64-66,249,284-286).  Arrays are summaries (sum, sum|x|, sum x^2 and 512
fixed entries) above ``FULL_LIMIT`` entries, as in ``make_golden.py``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import put, ref_problem  # noqa: E402  (also puts the reference on sys.path)
from pinnopt import curvature, network, optim, pde  # noqa: E402  (the reference)
from pinnopt.harness import _stream_seed  # noqa: E402

from paper_2405_15603_b200 import configs as cfgs  # noqa: E402

PLAN_FULL = {
    # name: (workload, n_interior, n_boundary, steps, kind, steps with full array records)
    "c2_full10": ("c2", 3000, 500, 10, "kfac", {1, 10}),
    "c3_full10": ("c3", 3000, 1000, 10, "kfac", {1, 10}),
    "c4_full10": ("c4", 3000, 1000, 10, "kfac", {1, 10}),
    "c5_star_n1000": ("c5", 1000, 333, 2, "kfac_star", {1, 2}),
    "c5_full3": ("c5", 3000, 1000, 3, "kfac", {1, 2, 3}),
}


class _Capture:
    """Record what the reference step computes, without changing it."""

    def __init__(self):
        self.grad = self.delta = None
        self.ls = []
        self._pg = curvature.precondition_gradient
        self._el = optim.evaluate_losses

    def __enter__(self):
        def pg(kfac, grads, *a, **k):
            out = self._pg(kfac, grads, *a, **k)
            self.grad, self.delta = network.mats_to_vec(grads), network.mats_to_vec(out)
            return out

        def el(params, batch, problem):
            out = self._el(params, batch, problem)
            self.ls.append(out)
            return out

        curvature.precondition_gradient = pg
        optim.evaluate_losses = el
        return self

    def __exit__(self, *exc):
        curvature.precondition_gradient = self._pg
        optim.evaluate_losses = self._el


def main():
    only = set(sys.argv[1:])
    for name, (wkey, n_int, n_bnd, steps, kind, full_steps) in PLAN_FULL.items():
        if only and name not in only:
            continue
        wl = cfgs.WORKLOADS[wkey]
        prob = ref_problem(wl)
        params = network.init_params(network.Architecture(wl.widths), _stream_seed(0, 0))
        batch = pde.sample_batch(prob, n_int, n_bnd, _stream_seed(0, 1, 0))
        cfg = optim.OptimizerConfig(kind=kind, damping=wl.damping, ema=wl.ema,
                                    momentum=wl.momentum, init_mode="identity")
        state = optim.init_train_state(params, cfg)
        out = {"widths": np.array(wl.widths), "n_interior": np.array(n_int),
               "init_zero": np.array(0), "n_boundary": np.array(n_bnd),
               "momentum": np.array(wl.momentum), "damping": np.array(wl.damping),
               "ema": np.array(wl.ema)}
        put(out, "in/interior", batch.interior)
        put(out, "in/boundary", batch.boundary)
        put(out, "in/targets", batch.boundary_targets)
        put(out, "in/theta", network.params_to_vec(params))
        for t in range(1, steps + 1):
            t0 = time.time()
            with _Capture() as cap:
                info = optim.optimizer_step(state, batch, prob)
            pre = f"s{t}/"
            if kind == "kfac":
                assert len(cap.ls) == 31, len(cap.ls)
                out[pre + "ls_losses"] = np.array(cap.ls, dtype=np.float64)
            out[pre + "loss_interior"] = np.array(info.loss_interior)
            out[pre + "loss_boundary"] = np.array(info.loss_boundary)
            out[pre + "alpha"] = np.array(info.alpha)
            out[pre + "mu"] = np.array(info.mu)
            if t in full_steps:
                put(out, pre + "grad", cap.grad)
                put(out, pre + "delta", cap.delta)
                put(out, pre + "theta", network.params_to_vec(state.params))
                put(out, pre + "prev_update", network.mats_to_vec(state.prev_update))
                for fname in ("a_interior", "b_interior", "a_boundary", "b_boundary"):
                    mats = getattr(state.kfac, fname)
                    put(out, pre + fname, np.concatenate([m.ravel() for m in mats]))
            print(f"{name} step {t}: loss={info.loss_total:.6e} alpha={info.alpha:.10g} "
                  f"mu={info.mu:.10g} ({time.time() - t0:.1f} s)", flush=True)
        out["numpy_version"] = np.array(np.__version__)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


if __name__ == "__main__":
    main()
