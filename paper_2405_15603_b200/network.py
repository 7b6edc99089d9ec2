"""Host-side MLP parameter containers (mirror of the reference interface).

Mirrors `pkg/src/pinnopt/network.py` so that a caller of the reference can hand
its objects to this package unchanged:

* ``Architecture`` / ``Parameters``  ↔ network.py:105-146 (same fields, same
  validation, ``[W | b]`` per linear layer, W of shape ``h_out x h_in``);
* ``init_params``                    ↔ network.py:149-161 (same numpy PCG64
  draw order: per layer the weight block row-major, then the bias), so seeded
  parameters are bit-identical to the reference's;
* ``add_scaled`` / flattening        ↔ network.py:259-305 (column-stacked
  ``[W | b]`` vectorisation).

Nothing here computes on the hot path; the device keeps its own packed copy of
the parameters (see ``engine.py``) and this module only describes them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Architecture",
    "Parameters",
    "init_params",
    "add_scaled",
    "mats_to_vec",
    "vec_to_mats",
    "params_to_vec",
    "vec_to_params",
    "params_to_mats",
]

ACTIVATIONS = ("tanh",)


@dataclass(frozen=True)
class Architecture:
    """Layer widths ``(d, h_1, ..., 1)`` plus the activation name (network.py:72-96)."""

    widths: tuple
    activation: str = "tanh"

    def __post_init__(self):
        widths = tuple(int(w) for w in self.widths)
        object.__setattr__(self, "widths", widths)
        if len(widths) < 2:
            raise ValueError("need at least input and output widths")
        if min(widths) < 1:
            raise ValueError(f"all widths must be >= 1, got {widths}")
        if widths[-1] != 1:
            raise ValueError(f"output width must be 1, got {widths[-1]}")
        if self.activation not in ACTIVATIONS:
            raise ValueError(f"unknown activation {self.activation!r}")

    @property
    def input_dim(self) -> int:
        return self.widths[0]

    @property
    def n_linear(self) -> int:
        return len(self.widths) - 1


@dataclass
class Parameters:
    """Per-linear-layer weights ``(h_out, h_in)`` and biases ``(h_out,)`` (network.py:105-146)."""

    weights: list
    biases: list
    activation: str = "tanh"

    def __post_init__(self):
        if len(self.weights) != len(self.biases):
            raise ValueError("weights and biases must pair up")
        prev_out = None
        for i, (w, b) in enumerate(zip(self.weights, self.biases)):
            if w.ndim != 2 or b.shape != (w.shape[0],):
                raise ValueError(f"layer {i}: weight {w.shape} / bias {b.shape} mismatch")
            if prev_out is not None and w.shape[1] != prev_out:
                raise ValueError(f"layer {i}: input width does not match previous layer")
            prev_out = w.shape[0]

    @property
    def widths(self) -> tuple:
        return (self.weights[0].shape[1],) + tuple(w.shape[0] for w in self.weights)

    @property
    def n_linear(self) -> int:
        return len(self.weights)

    @property
    def input_dim(self) -> int:
        return self.weights[0].shape[1]

    @property
    def n_params(self) -> int:
        return int(sum(w.size + b.size for w, b in zip(self.weights, self.biases)))

    def architecture(self) -> Architecture:
        return Architecture(self.widths, self.activation)

    def copy(self) -> "Parameters":
        return Parameters([w.copy() for w in self.weights], [b.copy() for b in self.biases],
                          self.activation)


def init_params(arch: Architecture, seed: int) -> Parameters:
    """U(-1/sqrt(fan_in), 1/sqrt(fan_in)) init, reference draw order (network.py:149-161)."""
    gen = np.random.default_rng(seed)
    ws, bs = [], []
    for fan_in, fan_out in zip(arch.widths[:-1], arch.widths[1:]):
        lim = 1.0 / np.sqrt(fan_in)
        ws.append(gen.uniform(-lim, lim, size=(fan_out, fan_in)))
        bs.append(gen.uniform(-lim, lim, size=fan_out))
    return Parameters(ws, bs, arch.activation)


def params_to_mats(params) -> list:
    """Per-layer augmented ``[W | b]`` matrices (``q x p`` with ``p = h_in + 1``)."""
    return [np.hstack([np.asarray(w, np.float64), np.asarray(b, np.float64)[:, None]])
            for w, b in zip(params.weights, params.biases)]


def add_scaled(params, mats: list, alpha: float) -> Parameters:
    """``params + alpha * mats`` with ``[dW | db]`` blocks (network.py:299-305)."""
    ws = [w + alpha * m[:, :-1] for w, m in zip(params.weights, mats)]
    bs = [b + alpha * m[:, -1] for b, m in zip(params.biases, mats)]
    return Parameters(ws, bs, getattr(params, "activation", "tanh"))


def mats_to_vec(mats: list) -> np.ndarray:
    """Column-stacked flattening of ``[W | b]`` blocks, layers concatenated (network.py:266-268)."""
    return np.concatenate([np.asarray(m, np.float64).ravel(order="F") for m in mats])


def vec_to_mats(vec, params) -> list:
    """Inverse of :func:`mats_to_vec` for the layer shapes of ``params`` (network.py:271-282)."""
    vec = np.asarray(vec, dtype=np.float64)
    out, off = [], 0
    for w in params.weights:
        q, p = w.shape[0], w.shape[1] + 1
        out.append(vec[off:off + p * q].reshape((q, p), order="F"))
        off += p * q
    if off != vec.size:
        raise ValueError(f"vector of length {vec.size} does not match parameter count {off}")
    return out


def params_to_vec(params) -> np.ndarray:
    return mats_to_vec(params_to_mats(params))


def vec_to_params(vec, template) -> Parameters:
    mats = vec_to_mats(vec, template)
    return Parameters([m[:, :-1].copy() for m in mats], [m[:, -1].copy() for m in mats],
                      getattr(template, "activation", "tanh"))
