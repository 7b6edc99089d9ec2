"""Drop-in KFAC optimizer interface (mirror of src/optim.py) backed by the B200 path.

Same names, arguments, defaults, validation and error behaviour as the
reference (/root/reference/pkg/src/pinnopt/optim.py):

* ``OptimizerConfig``  ↔ optim.py:41-78 (all five kinds validate as in the
  reference; only ``kind="kfac"`` steps on the device);
* ``TrainState``       ↔ optim.py:81-92 (``params`` is a host ``Parameters`` of
  float64 arrays after every step; ``kfac`` / ``prev_update`` are device-backed
  and materialised on access);
* ``StepInfo``, ``LineSearchError`` ↔ optim.py:217-226, 37-38;
* ``init_train_state`` ↔ optim.py:102-117;
* ``optimizer_step``   ↔ optim.py:396-402 — one KFAC step (optim.py:251-263) as
  one C-ABI call (``kp_kfac_step``) on the GPU; it mutates ``state`` in place.
  ``kind="kfac_star"`` (optim.py:266-320) runs ``kp_kfac_star_step``: the same
  factors and direction plus exact Gramian-vector products and the 2 x 2 model.

The reference's objects (its ``Parameters``, ``Batch``, ``PdeProblem``) are
accepted as they are (duck typing), so the reference harness's
``run_training`` loop can call this ``optimizer_step`` unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import network
from .curvature import KfacState
from .engine import KfacEngine, LineSearchError, pack_mats
from .pde import residual_terms
from .taylor import coeff_matrix

__all__ = [
    "OptimizerConfig",
    "TrainState",
    "StepInfo",
    "LineSearchError",
    "init_train_state",
    "optimizer_step",
    "OPTIMIZER_KINDS",
]

OPTIMIZER_KINDS = ("kfac", "kfac_star", "engd", "sgd", "adam")

# The device engine class.  The only substitute is the CPU stand-in of the plug-in tests
# (tests/cpu_step_engine.py), which checks the host-side state plumbing without a GPU.
ENGINE_FACTORY = KfacEngine


@dataclass
class OptimizerConfig:
    kind: str
    lr: float = 1e-3
    momentum: float = 0.0
    ema: float = 0.9
    damping: float = 1e-2
    init_mode: str = "identity"
    rcond: float = 1e-10
    line_search_min_exp: int = -30
    line_search_max_exp: int = 0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8

    def __post_init__(self):
        self.validate()

    def validate(self):
        """Reference validation rules, same messages (optim.py:61-75)."""
        if self.kind not in OPTIMIZER_KINDS:
            raise ValueError(f"unknown optimizer {self.kind!r}; known: {OPTIMIZER_KINDS}")
        if not 0.0 <= self.ema < 1.0:
            raise ValueError(f"ema must lie in [0, 1), got {self.ema}")
        if self.momentum < 0.0:
            raise ValueError(f"momentum must be >= 0, got {self.momentum}")
        if self.kind in ("kfac", "kfac_star") and self.damping <= 0.0:
            raise ValueError(f"{self.kind} requires damping > 0")
        if self.kind in ("sgd", "adam") and self.lr <= 0.0:
            raise ValueError(f"{self.kind} requires lr > 0")
        if self.kind == "engd" and self.damping < 0.0:
            raise ValueError("engd damping must be >= 0")
        if self.line_search_min_exp > self.line_search_max_exp:
            raise ValueError("line search exponent range is empty")

    def line_search_grid(self):
        return [2.0 ** e for e in range(self.line_search_min_exp, self.line_search_max_exp + 1)]


@dataclass
class StepInfo:
    alpha: float
    mu: float
    loss_interior: float
    loss_boundary: float

    @property
    def loss_total(self) -> float:
        return self.loss_interior + self.loss_boundary


@dataclass
class TrainState:
    """Optimizer state; device-resident for kind="kfac" (see module docstring)."""

    params: object
    config: OptimizerConfig
    step: int = 0
    _prev_host: list = field(default_factory=list, repr=False)
    _kfac_host: KfacState | None = field(default=None, repr=False)
    _engine: KfacEngine | None = field(default=None, repr=False)
    _params_seen: object = field(default=None, repr=False)
    _prev_snapshot: list | None = field(default=None, repr=False)
    adam_m: list = field(default_factory=list)
    adam_v: list = field(default_factory=list)
    gramian_ema: object = None

    # -- reference-visible fields backed by the device --------------------
    @property
    def prev_update(self) -> list:
        if self._engine is None:
            return self._prev_host
        if self._prev_snapshot is None:
            mats = self._engine.prev_mats()
            self._prev_snapshot = [m.copy() for m in mats]
            self._prev_host = mats
        return self._prev_host

    @prev_update.setter
    def prev_update(self, mats):
        self._prev_host = list(mats)
        if self._engine is not None:
            self._engine.set_prev_mats(self._prev_host)
            self._prev_snapshot = [np.asarray(m).copy() for m in self._prev_host]

    @property
    def kfac(self) -> KfacState | None:
        if self._kfac_host is not None and self._engine is not None and self._kfac_host._stale:
            self._kfac_host._refresh(*self._engine.factor_lists())
        return self._kfac_host

    @kfac.setter
    def kfac(self, value):
        self._kfac_host = value
        if value is not None and self._engine is not None:
            self._engine.set_factor_lists(value.a_interior, value.b_interior, value.a_boundary,
                                          value.b_boundary)
            value._mark_synced()


def init_train_state(params, config: OptimizerConfig) -> TrainState:
    """Fresh state (optim.py:102-117): zero previous update, identity/zero factors."""
    config.validate()
    zero = [np.zeros((w.shape[0], w.shape[1] + 1)) for w in params.weights]
    state = TrainState(params=params, config=config, _prev_host=zero)
    if config.kind in ("kfac", "kfac_star"):
        if config.init_mode not in ("zero", "identity"):
            raise ValueError(f"init_mode must be 'zero' or 'identity', got {config.init_mode!r}")
        mk = np.eye if config.init_mode == "identity" else (lambda k: np.zeros((k, k)))
        state._kfac_host = KfacState(
            [mk(w.shape[1] + 1) for w in params.weights], [mk(w.shape[0]) for w in params.weights],
            [mk(w.shape[1] + 1) for w in params.weights], [mk(w.shape[0]) for w in params.weights],
            config.ema, config.damping, config.init_mode)
    return state


def _engine_for(state: TrainState, batch, widths) -> KfacEngine:
    cfg = state.config
    ni, nb = batch.interior.shape[0], batch.boundary.shape[0]
    eng = state._engine
    if eng is not None and eng.widths == tuple(widths) and eng.n_interior == ni and eng.n_boundary == nb:
        return eng
    # (re)build: carry the current host-visible optimizer state onto the device
    kf = state.kfac
    prev = state.prev_update
    eng = ENGINE_FACTORY(widths, ni, nb, ema=cfg.ema, damping=cfg.damping, momentum=cfg.momentum,
                     ls_min_exp=cfg.line_search_min_exp, ls_max_exp=cfg.line_search_max_exp)
    eng.set_factor_lists(kf.a_interior, kf.b_interior, kf.a_boundary, kf.b_boundary)
    eng.set_prev_mats(prev)
    eng.load_params(state.params)
    state._engine = eng
    state._params_seen = state.params
    kf._mark_synced()
    state._prev_snapshot = [np.asarray(m).copy() for m in prev]
    return eng


def _sync_host_edits(state: TrainState, eng: KfacEngine):
    """Push host-side edits of params / factors / prev_update back to the device."""
    if state.params is not state._params_seen:
        eng.load_params(state.params)
        state._params_seen = state.params
    kf = state._kfac_host
    if kf is not None and kf._dirty():
        eng.set_factor_lists(kf.a_interior, kf.b_interior, kf.a_boundary, kf.b_boundary)
        kf._mark_synced()
    if state._prev_snapshot is not None:
        if any(not np.array_equal(a, b) for a, b in zip(state._prev_host, state._prev_snapshot)):
            eng.set_prev_mats(state._prev_host)


def device_step(state: TrainState, batch, problem) -> tuple:
    """One step on the device; returns (StepInfo, status code) without raising.

    On success and on non-finite parameters (status 4) the state is updated the way the
    reference's step mutates it before ``optimizer_step`` raises (src/optim.py:259-262,
    396-402): new params, previous update and ``step += 1``.  The factors always carry the
    step's EMA update (the reference updates them before the line search can fail,
    src/optim.py:237-248)."""
    params = state.params
    widths = (params.weights[0].shape[1],) + tuple(w.shape[0] for w in params.weights)
    cdiag = coeff_matrix(problem.coeffs)
    x = np.asarray(batch.interior, dtype=np.float64)
    r0, seeds, quad = residual_terms(problem, x)
    eng = _engine_for(state, batch, widths)
    _sync_host_edits(state, eng)
    if state._kfac_host is not None:
        eng.cfg.ema = float(state._kfac_host.ema)
        eng.cfg.damping = float(state._kfac_host.damping)
        eng.cfg.model_damping = float(state.config.damping)  # KFAC* model (optim.py:303)
        if eng.cfg.damping <= 0:
            raise ValueError("damping must be positive for Kronecker preconditioning")
    eng.set_batch(x, r0, seeds, np.asarray(batch.boundary, dtype=np.float64),
                  np.asarray(batch.boundary_targets, dtype=np.float64), cdiag, quad)
    if state.config.kind == "kfac_star":
        eng.launch_star_step()
    else:
        eng.launch_step()
    sc, code = eng.finish_step()
    if state._kfac_host is not None:
        state._kfac_host._stale = True
    state._prev_snapshot = None
    if code == 0 or code == 4:  # ok, or non-finite params (params were replaced first)
        # mirror the device state back to the reference-visible fields
        mats = eng.param_mats()
        cls = type(params) if hasattr(type(params), "__dataclass_fields__") else network.Parameters
        new_params = cls([m[:, :-1].copy() for m in mats], [m[:, -1].copy() for m in mats],
                         getattr(params, "activation", "tanh"))
        state.params = new_params
        state._params_seen = new_params
        state.step += 1
    return StepInfo(float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])), code


def _kfac_device_step(state: TrainState, batch, problem) -> StepInfo:
    from .engine import raise_for_status

    info, code = device_step(state, batch, problem)
    raise_for_status(code, "optimizer_step")
    return info


def optimizer_step(state: TrainState, batch, problem) -> StepInfo:
    """One optimisation step (optim.py:396-402); kinds "kfac" and "kfac_star" run on the B200."""
    if state.config.kind not in ("kfac", "kfac_star"):
        raise NotImplementedError(
            f"optimizer kind {state.config.kind!r} is outside the accelerated KFAC path")
    return _kfac_device_step(state, batch, problem)
