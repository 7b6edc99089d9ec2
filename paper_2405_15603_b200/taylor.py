"""Operator coefficients of the forward-Laplacian (Taylor-mode) engine.

Mirror of ``OperatorCoeffs`` in `pkg/src/pinnopt/taylor.py:43-87`: a symmetric
``d x d`` matrix ``c`` of the operator ``sum_ij c_ij d^2/dx_i dx_j``.  The
device kernels take the diagonal only (every catalog operator and every
BASELINE configuration is diagonal: the Laplacian, or the partial Laplacian of
the heat problem, pde.py:199); a non-diagonal ``c`` is rejected by the device
path with ``NotImplementedError`` rather than silently mishandled.

Per-sample state layout on the device follows the reference
(taylor.py:3-16): ``S = d + 2`` rows per collocation point — value, the ``d``
directional first derivatives, and the operator row — stored row-major as an
``(N * S, h)`` matrix.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["OperatorCoeffs"]


@dataclass(frozen=True, eq=False)
class OperatorCoeffs:
    c: np.ndarray

    def __post_init__(self):
        c = np.asarray(self.c, dtype=np.float64)
        if c.ndim != 2 or c.shape[0] != c.shape[1]:
            raise ValueError(f"coefficients must be square, got shape {c.shape}")
        if c.size and float(np.max(np.abs(c - c.T))) > 1e-12:
            raise ValueError("coefficient matrix must be symmetric")
        object.__setattr__(self, "c", c)
        diag = np.diagonal(c).copy()
        is_diag = bool(np.array_equal(c, np.diag(diag)))
        object.__setattr__(self, "_diag", diag if is_diag else None)

    @property
    def dim(self) -> int:
        return self.c.shape[0]

    @property
    def is_diagonal(self) -> bool:
        return self._diag is not None

    @property
    def diagonal(self) -> np.ndarray:
        return np.diagonal(self.c).copy()

    def apply(self, g) -> np.ndarray:
        """Contract ``c`` over the derivative axis of an ``(N, d, h)`` stack (taylor.py:63-75)."""
        if self._diag is not None:
            return g * self._diag[None, :, None]
        return np.einsum("ij,njh->nih", self.c, g)

    @classmethod
    def laplacian(cls, dim: int) -> "OperatorCoeffs":
        return cls(np.eye(dim))

    @classmethod
    def partial_laplacian(cls, dim: int, active) -> "OperatorCoeffs":
        c = np.zeros((dim, dim))
        for i in active:
            c[i, i] = 1.0
        return cls(c)


def coeff_matrix(coeffs) -> np.ndarray:
    """The symmetric d x d coefficient matrix of any coefficient object with a ``c``."""
    return np.asarray(coeffs.c, dtype=np.float64)


def coeff_spectrum(c):
    """``(lam, rot)`` with c = rot diag(lam) rot^T for the device engine.

    Diagonal c (every catalog operator, reference pde.py:84-268; the test at
    taylor.py:56-57) gives ``(diag(c), None)`` and the coordinate derivative rows of
    the reference.  A dense c (taylor.py:72-75) gives its eigendecomposition: the
    engine then propagates derivatives along the eigenvectors, where the operator's
    quadratic form is diagonal.  A 1-D ``c`` is taken as the diagonal.
    """
    c = np.asarray(c, dtype=np.float64)
    if c.ndim == 1:
        return c.copy(), None
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise ValueError(f"coefficients must be square, got shape {c.shape}")
    diag = np.diagonal(c).copy()
    if np.array_equal(c, np.diag(diag)):
        return diag, None
    lam, rot = np.linalg.eigh(0.5 * (c + c.T))
    return lam, np.ascontiguousarray(rot)


def coeff_diagonal(coeffs) -> np.ndarray:
    """Diagonal of any coefficient object with a ``c`` matrix; raises if not diagonal."""
    c = coeff_matrix(coeffs)
    diag = np.diagonal(c).copy()
    if not np.array_equal(c, np.diag(diag)):
        raise NotImplementedError("coefficients are not diagonal; use coeff_spectrum")
    return diag
