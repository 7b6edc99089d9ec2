"""Kronecker-factor state (mirror of ``KfacState``, src/curvature.py:43-76).

The authoritative factors live on the GPU (``engine.KfacEngine``); this host
object exposes them with the reference's field names.  Lists are refreshed from
the device lazily after each step and edits made through the lists (as the
reference's tests do, e.g. pkg/tests/test_curvature.py:148-169) are detected and
pushed back before the next step.
"""

from __future__ import annotations

import numpy as np

__all__ = ["KfacState", "init_kfac_state"]


class KfacState:
    def __init__(self, a_interior, b_interior, a_boundary, b_boundary, ema, damping,
                 init_mode="identity"):
        self.a_interior = list(a_interior)
        self.b_interior = list(b_interior)
        self.a_boundary = list(a_boundary)
        self.b_boundary = list(b_boundary)
        self.ema = ema
        self.damping = damping
        self.init_mode = init_mode
        self._stale = False
        self._snap = None

    def _lists(self):
        return (self.a_interior, self.b_interior, self.a_boundary, self.b_boundary)

    def _refresh(self, a_int, b_int, a_bnd, b_bnd):
        self.a_interior[:] = a_int
        self.b_interior[:] = b_int
        self.a_boundary[:] = a_bnd
        self.b_boundary[:] = b_bnd
        self._stale = False
        self._mark_synced()

    def _mark_synced(self):
        self._snap = [[np.asarray(m).copy() for m in lst] for lst in self._lists()]

    def _dirty(self) -> bool:
        if self._stale or self._snap is None:
            return False
        for lst, snap in zip(self._lists(), self._snap):
            if len(lst) != len(snap):
                return True
            for m, s in zip(lst, snap):
                if m is not s and not np.array_equal(m, s):
                    return True
        return False

    def __repr__(self):
        return (f"KfacState(layers={len(self.a_interior)}, ema={self.ema}, damping={self.damping}, "
                f"init_mode={self.init_mode!r})")


def init_kfac_state(params, ema: float, damping: float, init_mode: str = "identity") -> KfacState:
    """Identity or zero factors per linear layer (src/curvature.py:62-76)."""
    if init_mode not in ("zero", "identity"):
        raise ValueError(f"init_mode must be 'zero' or 'identity', got {init_mode!r}")
    mk = np.eye if init_mode == "identity" else (lambda k: np.zeros((k, k)))
    ws = params.weights
    return KfacState([mk(w.shape[1] + 1) for w in ws], [mk(w.shape[0]) for w in ws],
                     [mk(w.shape[1] + 1) for w in ws], [mk(w.shape[0]) for w in ws],
                     ema, damping, init_mode)
