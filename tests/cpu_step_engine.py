"""CPU stand-in for ``engine.KfacEngine`` with the single-call step interface, used to
test the host-side state plumbing of ``paper_2405_15603_b200.optim`` and of the reference
plug-in (``paper_2405_15603_b200.plugin``) without a GPU.

It implements the calls ``optim.device_step`` makes (load/set state, set_batch,
launch_step / launch_star_step, finish_step, the read-backs) with the oracle's math, and
reports failures with the C ABI's status codes.  The interior residual is rebuilt from
the (r0, seeds, quad) split the device receives (pde.residual_terms).  Test
infrastructure only; installed through ``optim.ENGINE_FACTORY`` by the tests.
"""

from types import SimpleNamespace

import numpy as np

from oracle import kfac_oracle as orc


class CpuStepEngine:
    instances = 0
    force_code = None  # tests set a status code to exercise the error mapping

    def __init__(self, widths, n_interior, n_boundary, *, ema, damping, momentum,
                 ls_min_exp=-30, ls_max_exp=0, **_):
        CpuStepEngine.instances += 1
        self.widths = tuple(int(w) for w in widths)
        self.n_interior, self.n_boundary = int(n_interior), int(n_boundary)
        self.cfg = SimpleNamespace(ema=float(ema), damping=float(damping), momentum=float(momentum))
        self.grid = [2.0 ** e for e in range(ls_min_exp, ls_max_exp + 1)]
        self.w = self.b = self.kf = self.prev = None
        self._sc, self._code = np.zeros(4), 0

    # state ------------------------------------------------------------------
    def load_params(self, params):
        self.w = [np.array(w, dtype=np.float64) for w in params.weights]
        self.b = [np.array(b, dtype=np.float64) for b in params.biases]

    def set_factor_lists(self, a_int, b_int, a_bnd, b_bnd):
        cp = lambda lst: [np.array(m, dtype=np.float64) for m in lst]  # noqa: E731
        self.kf = orc.OracleKfac(cp(a_int), cp(b_int), cp(a_bnd), cp(b_bnd), 0.0, 0.0)

    def set_prev_mats(self, mats):
        self.prev = [np.array(m, dtype=np.float64) for m in mats]

    def set_batch(self, x_int, r0, seeds, x_bnd, targets, cdiag, quad=None):
        d = x_int.shape[1]
        r0, seeds = np.asarray(r0), np.asarray(seeds)
        qd = None if quad is None else np.asarray(quad)

        def residual(x, u, g, op):
            r = r0 + seeds[:, 0] * u + np.einsum("ni,ni->n", seeds[:, 1:d + 1], g) + seeds[:, d + 1] * op
            return r if qd is None else r + np.einsum("ni,ni->n", qd, g * g)

        def residual_grads(x, u, g, op):
            dg = seeds[:, 1:d + 1] if qd is None else seeds[:, 1:d + 1] + 2.0 * qd * g
            return seeds[:, 0], dg, seeds[:, d + 1]

        c = np.asarray(cdiag, dtype=np.float64)
        self.problem = SimpleNamespace(residual=residual, residual_grads=residual_grads,
                                       coeffs=SimpleNamespace(c=np.diag(c) if c.ndim == 1 else c))
        self.batch = SimpleNamespace(interior=np.array(x_int), boundary=np.array(x_bnd),
                                     boundary_targets=np.array(targets))

    # step -------------------------------------------------------------------
    def _run(self, fn):
        self.kf.ema, self.kf.damping = self.cfg.ema, self.cfg.damping
        st = orc.OracleState(self.w, self.b, self.kf, self.cfg.momentum, self.grid, self.prev,
                             model_damping=getattr(self.cfg, "model_damping", None))
        self._code = 0
        try:
            if self.force_code is not None:
                raise {3: orc.OracleLineSearchError, 2: orc.OracleNotPSD}[self.force_code]("forced")
            alpha, mu, li, lb = fn(st, self.batch, self.problem)
            self._sc = np.array([li, lb, alpha, mu])
        except orc.OracleLineSearchError:
            self._code = 3
        except orc.OracleNotPSD:
            self._code = 2
        except FloatingPointError:
            self._code = 4
            self._sc = np.array([np.nan, np.nan, np.nan, np.nan])
        self.w, self.b, self.prev = st.weights, st.biases, st.prev_update

    def launch_step(self):
        self._run(orc.kfac_step)

    def launch_star_step(self):
        self._run(orc.kfac_star_step)

    def finish_step(self):
        return self._sc.copy(), self._code

    # read-backs -------------------------------------------------------------
    def param_mats(self):
        return [np.hstack([w, b[:, None]]) for w, b in zip(self.w, self.b)]

    def prev_mats(self):
        return [m.copy() for m in self.prev]

    def factor_lists(self):
        cp = lambda lst: [m.copy() for m in lst]  # noqa: E731
        return cp(self.kf.a_int), cp(self.kf.b_int), cp(self.kf.a_bnd), cp(self.kf.b_bnd)
