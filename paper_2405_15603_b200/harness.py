"""Training-loop integration: the reference harness on the device.

Mirror of `pkg/src/pinnopt/harness.py` for the KFAC optimizers:

* ``RunConfig``        ↔ harness.py:69-128 (same fields, defaults, validation, JSON I/O);
* ``run_training``     ↔ harness.py:236-323 — same seeding (``SeedSequence`` sub-streams,
  harness.py:54-66), same resampling schedule, divergence handling and wall-clock stop;
  every step is ``optimizer_step`` on the B200 and the evaluation forward of
  ``eval_l2`` runs on the device (``kp_mlp_forward``);
* the CSV log (harness.py:42-51, 169-196) and the JSON checkpoint (harness.py:199-233)
  are written in the reference's formats, so its tooling reads them unchanged.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .configs import stream_seed
from .engine import LineSearchError, _ptr, raise_for_status
from .network import Architecture, Parameters, init_params
from .optim import OPTIMIZER_KINDS, OptimizerConfig, init_train_state, optimizer_step
from .pde import make_problem, sample_batch

__all__ = ["RunConfig", "TrainLog", "CSV_COLUMNS", "eval_l2", "run_training",
           "save_checkpoint", "load_checkpoint"]

CSV_COLUMNS = ("step", "wall_time_s", "loss_interior", "loss_boundary", "loss_total",
               "l2_rel_error", "alpha", "mu")
STREAM_INIT, STREAM_BATCH, STREAM_EVAL = 0, 1, 2
OUTPUT_DIR_ENV = "PINNOPT_OUTPUT_DIR"
DEFAULT_RESAMPLE_EVERY = {"sgd": 1, "adam": 1, "engd": 1, "kfac": 100, "kfac_star": 100}


@dataclass
class RunConfig:
    problem: str
    widths: list
    optimizer: str
    problem_params: dict = field(default_factory=dict)
    lr: float = 1e-3
    momentum: float = 0.0
    ema: float = 0.9
    damping: float = 1e-2
    init_mode: str = "identity"
    rcond: float = 1e-10
    n_interior: int = 900
    n_boundary: int = 120
    resample_every: int | None = None
    max_steps: int = 1000
    max_wall_seconds: float = 0.0
    eval_every: int = 100
    n_eval_points: int = 2000
    seed: int = 0
    output_dir: str = "runs/out"

    def __post_init__(self):
        if self.n_interior < 1 or self.n_boundary < 1:
            raise ValueError("batch sizes must be positive")
        if self.max_steps < 0 or self.eval_every < 1 or self.n_eval_points < 1:
            raise ValueError("step and evaluation counts must be positive")
        if self.optimizer not in OPTIMIZER_KINDS:
            raise ValueError(f"unknown optimizer {self.optimizer!r}; known: {OPTIMIZER_KINDS}")
        if self.resample_every is None:
            self.resample_every = DEFAULT_RESAMPLE_EVERY[self.optimizer]
        if self.resample_every < 0:
            raise ValueError("resample_every must be >= 0 (0 keeps the batch fixed)")

    @classmethod
    def from_dict(cls, d: dict) -> "RunConfig":
        unknown = set(d) - {f.name for f in dataclasses.fields(cls)}
        if unknown:
            raise ValueError(f"unknown config keys: {sorted(unknown)}")
        return cls(**d)

    @classmethod
    def from_json(cls, path: str) -> "RunConfig":
        with open(path, "r", encoding="utf-8") as fh:
            return cls.from_dict(json.load(fh))

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)

    def optimizer_config(self) -> OptimizerConfig:
        return OptimizerConfig(kind=self.optimizer, lr=self.lr, momentum=self.momentum,
                               ema=self.ema, damping=self.damping, init_mode=self.init_mode,
                               rcond=self.rcond)


@dataclass
class TrainLog:
    rows: list = field(default_factory=list)
    diverged: bool = False

    def column(self, name: str) -> list:
        i = CSV_COLUMNS.index(name)
        return [r[i] for r in self.rows]

    @property
    def final(self):
        return self.rows[-1]


class DeviceEvaluator:
    """u(x) on the device for a fixed point set (the eval_l2 forward pass)."""

    def __init__(self, widths, n_points: int):
        import torch

        self.torch = torch
        self.lib = _capi.load()
        self.widths = tuple(widths)
        self.n = int(n_points)
        ctx = C.c_void_p()
        raise_for_status(self.lib.kp_context_create(torch.cuda.current_device(), C.byref(ctx)))
        self.ctx = ctx
        self.prob = _capi.kp_problem()
        self.prob.net = _capi.make_net(self.widths)
        self.prob.n_interior, self.prob.n_boundary, self.prob.n_candidates = 1, self.n, 1
        nb = C.c_size_t()
        raise_for_status(self.lib.kp_workspace_bytes(self.ctx, C.byref(self.prob), C.byref(nb)))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ws_bytes = int(nb.value)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.x = torch.empty(self.n * self.widths[0], dtype=torch.float64, device=dev)
        self.u = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.theta = torch.empty(int(self.lib.kp_param_count(C.byref(self.prob.net))),
                                 dtype=torch.float64, device=dev)
        self._x_id = None

    def __call__(self, params, pts) -> np.ndarray:
        from .engine import pack_params

        t = self.torch
        if self._x_id is not id(pts):
            self.x.copy_(t.from_numpy(np.ascontiguousarray(pts, np.float64).ravel()))
            self._x_id = id(pts)
        self.theta.copy_(t.from_numpy(pack_params(params)))
        s = t.cuda.current_stream()
        raise_for_status(self.lib.kp_mlp_forward(
            self.ctx, C.byref(self.prob), C.c_void_p(_ptr(self.theta)), C.c_void_p(_ptr(self.x)),
            C.c_void_p(_ptr(self.u)), C.c_void_p(_ptr(self.ws)), C.c_size_t(self.ws_bytes),
            C.c_void_p(s.cuda_stream)))
        return self.u.cpu().numpy()

    def __del__(self):
        try:
            self.lib.kp_context_destroy(self.ctx)
        except Exception:
            pass


_EVALUATORS: dict = {}


def eval_l2(params, problem, n_points: int, seed: int) -> float:
    """Relative L2 error on a seeded uniform point set (harness.py:155-166); the network
    forward runs on the device."""
    if n_points < 1:
        raise ValueError("need at least one evaluation point")
    gen = np.random.default_rng(seed)
    pts = gen.uniform(problem.lower, problem.upper, size=(n_points, problem.dim))
    widths = (params.weights[0].shape[1],) + tuple(w.shape[0] for w in params.weights)
    key = (widths, n_points)
    ev = _EVALUATORS.get(key)
    if ev is None:
        ev = _EVALUATORS[key] = DeviceEvaluator(widths, n_points)
    u = ev(params, pts)
    u_true = problem.true_solution(pts)
    denom = float(u_true @ u_true)
    if denom <= 0.0:
        raise ValueError("true solution is identically zero on the evaluation set")
    return float(np.sqrt(float((u - u_true) @ (u - u_true)) / denom))


def _fmt(x) -> str:
    return format(float(x), ".17g")


class _CsvWriter:
    def __init__(self, path, meta: str):
        self.fh = open(path, "w", encoding="utf-8", newline="\n") if path else None
        if self.fh:
            self.fh.write(f"# {meta}\n" + ",".join(CSV_COLUMNS) + "\n")
            self.fh.flush()

    def row(self, values):
        if self.fh:
            self.fh.write(",".join([str(int(values[0]))] + [_fmt(v) for v in values[1:]]) + "\n")
            self.fh.flush()

    def comment(self, text):
        if self.fh:
            self.fh.write(f"# {text}\n")
            self.fh.flush()

    def close(self):
        if self.fh:
            self.fh.close()
            self.fh = None


def save_checkpoint(path, params, config: RunConfig | None = None):
    """Reference JSON checkpoint (harness.py:199-220): widths, activation, row-major layers."""
    widths = (params.weights[0].shape[1],) + tuple(w.shape[0] for w in params.weights)
    payload = {"widths": list(widths), "activation": getattr(params, "activation", "tanh"),
               "layers": [{"shape": list(w.shape), "weight": [float(v) for v in w.ravel()],
                           "bias": [float(v) for v in b.ravel()]}
                          for w, b in zip(params.weights, params.biases)]}
    if config is not None:
        payload["config"] = config.to_dict()
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh)


def load_checkpoint(path):
    with open(path, "r", encoding="utf-8") as fh:
        payload = json.load(fh)
    ws = [np.array(l["weight"], dtype=np.float64).reshape(tuple(l["shape"])) for l in payload["layers"]]
    bs = [np.array(l["bias"], dtype=np.float64) for l in payload["layers"]]
    return Parameters(ws, bs, payload.get("activation", "tanh")), payload.get("config")


def run_training(config: RunConfig) -> TrainLog:
    """The reference training loop (harness.py:236-323) with every step on the B200."""
    problem = make_problem(config.problem, **config.problem_params)
    arch = Architecture(tuple(config.widths), "tanh")
    if arch.input_dim != problem.dim:
        raise ValueError(f"network input width {arch.input_dim} does not match problem dim {problem.dim}")
    params = init_params(arch, stream_seed(config.seed, STREAM_INIT))
    state = init_train_state(params, config.optimizer_config())
    out_dir = os.environ.get(OUTPUT_DIR_ENV) or config.output_dir
    os.makedirs(out_dir, exist_ok=True)
    meta = json.dumps({"format": "pinnopt-log-v1",
                       "rng": "numpy PCG64; SeedSequence(entropy=seed, spawn_key=(tag, k)); "
                              "tags init=0 batch=1 eval=2",
                       "config": config.to_dict()}, sort_keys=True)
    writer = _CsvWriter(os.path.join(out_dir, "log.csv"), meta)
    eval_seed = stream_seed(config.seed, STREAM_EVAL)
    log = TrainLog()
    start = time.perf_counter()

    def record(step, l_int, l_bnd, alpha, mu):
        err = eval_l2(state.params, problem, config.n_eval_points, eval_seed)
        row = (step, time.perf_counter() - start, l_int, l_bnd, l_int + l_bnd, err, alpha, mu)
        log.rows.append(row)
        writer.row(row)

    batch = sample_batch(problem, config.n_interior, config.n_boundary,
                         stream_seed(config.seed, STREAM_BATCH, 0))
    l_int, l_bnd = _initial_losses(state, batch, problem)
    record(0, l_int, l_bnd, 0.0, 0.0)
    resamples = 0
    try:
        for t in range(1, config.max_steps + 1):
            if config.resample_every > 0 and t > 1 and (t - 1) % config.resample_every == 0:
                resamples += 1
                batch = sample_batch(problem, config.n_interior, config.n_boundary,
                                     stream_seed(config.seed, STREAM_BATCH, resamples))
            info = optimizer_step(state, batch, problem)
            if not np.isfinite(info.loss_total):
                log.diverged = True
                record(t, info.loss_interior, info.loss_boundary, info.alpha, info.mu)
                writer.comment(f"diverged step={t}")
                break
            if t % config.eval_every == 0 or t == config.max_steps:
                record(t, info.loss_interior, info.loss_boundary, info.alpha, info.mu)
            if config.max_wall_seconds > 0 and time.perf_counter() - start > config.max_wall_seconds:
                if t % config.eval_every != 0 and t != config.max_steps:
                    record(t, info.loss_interior, info.loss_boundary, info.alpha, info.mu)
                break
    except (LineSearchError, FloatingPointError) as exc:
        log.diverged = True
        writer.comment(f"diverged: {exc}")
    finally:
        writer.close()
        save_checkpoint(os.path.join(out_dir, "checkpoint.json"), state.params, config)
    return log


def _initial_losses(state, batch, problem):
    """evaluate_losses at the initial parameters (harness.py:326-329), on the device (this also
    builds the engine the first optimizer_step reuses)."""
    from .optim import _engine_for
    from .pde import residual_terms
    from .taylor import coeff_matrix

    params = state.params
    widths = (params.weights[0].shape[1],) + tuple(w.shape[0] for w in params.weights)
    x = np.asarray(batch.interior, dtype=np.float64)
    r0, seeds, quad = residual_terms(problem, x)
    eng = _engine_for(state, batch, widths)
    eng.set_batch(x, r0, seeds, np.asarray(batch.boundary, np.float64),
                  np.asarray(batch.boundary_targets, np.float64), coeff_matrix(problem.coeffs), quad)
    return eng.evaluate_losses()
