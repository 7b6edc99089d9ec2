"""The reference-side plug-in (paper_2405_15603_b200.plugin) with the real device engine.

The reference package cannot travel to the GPU box, so the dispatch table it patches is a
stand-in module with the reference's shape (``_STEP_FNS``, ``StepInfo``,
``LineSearchError``; src/optim.py:37-38,217-226,387-402) and the state is a plain
reference-shaped ``TrainState`` (src/optim.py:81-92) holding plain factor lists.  The
steps must reproduce the reference's own golden vectors (tests/golden/c1_10.npz,
c1_star_10.npz).  The CPU twin on the real reference harness is tests/test_plugin.py.
"""

import types
from dataclasses import dataclass, field

import numpy as np
import pytest

from golden_util import compare, has, load, pack_factors

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200 import plugin  # noqa: E402
from paper_2405_15603_b200.network import mats_to_vec  # noqa: E402
from paper_2405_15603_b200.optim import LineSearchError, OptimizerConfig, StepInfo  # noqa: E402


@dataclass
class RefKfacState:  # src/curvature.py:43-59
    a_interior: list
    b_interior: list
    a_boundary: list
    b_boundary: list
    ema: float
    damping: float
    init_mode: str = "identity"


@dataclass
class RefTrainState:  # src/optim.py:81-92
    params: object
    config: object
    step: int = 0
    prev_update: list = field(default_factory=list)
    kfac: RefKfacState | None = None


def _ref_module():
    mod = types.ModuleType("refoptim_standin")
    mod.StepInfo, mod.LineSearchError = StepInfo, LineSearchError
    mod._STEP_FNS = {"kfac": None, "kfac_star": None}

    def optimizer_step(state, batch, problem):  # src/optim.py:396-402
        info = mod._STEP_FNS[state.config.kind](state, batch, problem)
        for w, b in zip(state.params.weights, state.params.biases):
            if not (np.all(np.isfinite(w)) and np.all(np.isfinite(b))):
                raise FloatingPointError("parameters became non-finite during the step")
        return info

    mod.optimizer_step = optimizer_step
    return mod


@pytest.mark.parametrize("name,kind", [("c1_10", "kfac"), ("c1_star_10", "kfac_star")])
def test_plugin_steps_match_reference_golden(name, kind):
    g = load(name)
    wl = cfgs.WORKLOADS["c1"]
    prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
    mod = _ref_module()
    plugin.install(mod)
    cfg = OptimizerConfig(kind=kind, damping=float(g["damping"]), ema=float(g["ema"]),
                          momentum=float(g["momentum"]))
    ws = params.weights
    eye = lambda k: np.eye(k)  # noqa: E731
    kf = RefKfacState([eye(w.shape[1] + 1) for w in ws], [eye(w.shape[0]) for w in ws],
                      [eye(w.shape[1] + 1) for w in ws], [eye(w.shape[0]) for w in ws],
                      cfg.ema, cfg.damping)
    st = RefTrainState(params, cfg, 0, [np.zeros((w.shape[0], w.shape[1] + 1)) for w in ws], kf)
    a_list = kf.a_interior
    t = 1
    while f"s{t}/alpha" in g:
        info = mod.optimizer_step(st, batch, prob)
        p, tol = f"s{t}/", (1e-10 if t == 1 else 1e-8)
        assert st.step == t
        if kind == "kfac":
            assert info.alpha == float(g[p + "alpha"])
        else:
            assert abs(info.alpha - float(g[p + "alpha"])) <= tol * abs(float(g[p + "alpha"]))
        assert abs(info.loss_interior - float(g[p + "loss_interior"])) <= tol * abs(float(g[p + "loss_interior"]))
        if has(g, p + "theta"):
            theta = np.concatenate([np.hstack([w, b[:, None]]).ravel(order="F")
                                    for w, b in zip(st.params.weights, st.params.biases)])
            assert compare(g, p + "theta", theta, tol) <= tol
            assert compare(g, p + "prev_update", mats_to_vec(st.prev_update), tol) <= tol
            assert st.kfac is kf and st.kfac.a_interior is a_list
            for key in ("a_interior", "b_interior", "a_boundary", "b_boundary"):
                assert compare(g, p + key, pack_factors(getattr(st.kfac, key)), tol) <= tol, key
        t += 1
    assert t == 11
