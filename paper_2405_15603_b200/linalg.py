"""Error types of the dense linear-algebra layer (mirror of src/linalg.py:39-44).

The device Kronecker-sum solve (csrc/kp_step.cu ``kron_solve``) reports its
failures as C-ABI status codes; the Python mirror raises these classes, which
subclass ``ValueError`` exactly like the reference's.
"""

from __future__ import annotations

__all__ = ["NotSymmetricError", "NotPositiveSemidefiniteError", "PSD_TOL", "SYMMETRY_TOL"]

SYMMETRY_TOL = 1e-10   # src/linalg.py:33
PSD_TOL = 1e-6         # src/linalg.py:36


class NotSymmetricError(ValueError):
    """A matrix is not square or not symmetric within tolerance."""


class NotPositiveSemidefiniteError(ValueError):
    """A matrix has eigenvalues below the negative tolerance (or is not PD)."""
