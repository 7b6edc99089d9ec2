"""Data-parallel KFAC step over several GPUs (one process per GPU, NCCL over NVLink).

Every N-dependent quantity of the step is a sum over collocation points
(factors src/curvature.py:113-115,133-134; gradient src/optim.py:173-176;
losses src/pde.py:351,359), so points are sharded contiguously across ranks
and the parameters / optimizer state are replicated.  A step
has exactly two exchange points, both sum all-reduces of one contiguous
device buffer:

1. after the local forward/backward: the UNNORMALISED factor sums, the
   residual-weighted gradient and sum r^2 (``kp_reduce_buffer``);
2. after the local line search: the 2 x 31 per-candidate sums of r^2
   (``kp_linesearch_buffer``).

Normalisation by the global point counts, the EMA and the argmin are then
computed redundantly — and bit-identically, since the all-reduced inputs are
identical — on every rank.  The per-layer Kronecker-sum solves
(src/curvature.py:150-163) are distributed by layer when any factor is too
large for the on-device solver: each layer is owned by
one rank (``layer_owners``), the owner writes its Delta rows and every other
rank zeros, and a third sum all-reduce of ``kp_direction_buffer`` (Delta plus
status slots) hands every rank the owners' Delta bit for bit.  Networks whose
factors all fit the on-device solver (one launch for every layer) solve
redundantly: an exchange would cost more than it saves.
"""

from __future__ import annotations

import numpy as np

from .engine import KfacEngine, raise_for_status
from .pde import residual_terms
from .taylor import coeff_matrix


def shard_bounds(n: int, rank: int, world: int):
    """Contiguous, balanced shard [lo, hi) of n points for `rank` of `world`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


SMALL_EIG_MAX_N = 96  # factor pairs up to this size use the one-launch device solver (kp_step.cu)


def layer_owners(widths, world: int):
    """Owner rank of each layer's Kronecker solve, or None to solve redundantly.

    Greedy longest-processing-time assignment on the solve cost p^3 + q^3 of the layer's
    two generalised eigenproblems (p = h_l + 1, q = h_{l+1}); deterministic, so every
    rank computes the same table.
    """
    widths = [int(w) for w in widths]
    sizes = [(widths[l] + 1, widths[l + 1]) for l in range(len(widths) - 1)]
    if world <= 1 or all(max(p, q) <= SMALL_EIG_MAX_N for p, q in sizes):
        return None
    cost = [float(p) ** 3 + float(q) ** 3 for p, q in sizes]
    load = [0.0] * world
    owners = [0] * len(sizes)
    for l in sorted(range(len(sizes)), key=lambda i: (-cost[i], i)):
        r = min(range(world), key=lambda k: (load[k], k))
        owners[l] = r
        load[r] += cost[l]
    return owners


class ShardedKfacStep:
    """Drives one rank's engine through the phased step with all-reduces in between.

    ``engine`` is anything with ``phase(name)``, ``reduce_buffer()``,
    ``linesearch_buffer()`` and ``finish_step()`` (the ``KfacEngine`` on GPUs;
    tests inject a CPU stand-in to check this orchestration under gloo).
    """

    def __init__(self, engine, all_reduce, owners=None, rank: int = 0):
        self.engine = engine
        self.all_reduce = all_reduce
        # owners: per-layer owner rank (layer_owners) or None for redundant solves
        self.owned = None if owners is None else [o == rank for o in owners]

    def _precondition(self):
        e = self.engine
        if self.owned is None:
            e.phase("precondition")
            return
        e.phase("precondition_owned", owned=self.owned)
        self.all_reduce(e.direction_buffer())
        e.phase("direction")

    def step(self):
        e = self.engine
        e.phase("accumulate")
        self.all_reduce(e.reduce_buffer())
        self._precondition()
        e.phase("linesearch")
        self.all_reduce(e.linesearch_buffer())
        e.phase("update")
        sc, code = e.finish_step()
        raise_for_status(code, "sharded kfac step")
        return float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])


class ShardedKfacStarStep(ShardedKfacStep):
    """KFAC* over P ranks: the factor/gradient all-reduce, then one all-reduce of the
    partial Gramian-vector products (kp_gvp_buffer) before the 2 x 2 model solve."""

    def step(self):
        e = self.engine
        e.phase("accumulate")
        self.all_reduce(e.reduce_buffer())
        self._precondition()
        e.phase("star_gvp")
        self.all_reduce(e.gvp_buffer())
        e.phase("star_update")
        sc, code = e.finish_step()
        raise_for_status(code, "sharded kfac_star step")
        return float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])


def make_rank_engine(widths, batch, problem, rank: int, world: int, *, ema, damping, momentum,
                     ls_min_exp=-30, ls_max_exp=0, chunk=None):
    """Engine for this rank's shard of ``batch`` with global normalisers."""
    n_int, n_bnd = batch.interior.shape[0], batch.boundary.shape[0]
    if n_int < world or n_bnd < world:
        raise ValueError("every rank needs at least one interior and one boundary point")
    i0, i1 = shard_bounds(n_int, rank, world)
    b0, b1 = shard_bounds(n_bnd, rank, world)
    eng = KfacEngine(widths, i1 - i0, b1 - b0, ema=ema, damping=damping, momentum=momentum,
                     ls_min_exp=ls_min_exp, ls_max_exp=ls_max_exp, chunk=chunk,
                     n_interior_global=n_int, n_boundary_global=n_bnd)
    upload_shard(eng, batch, problem, rank, world)
    return eng


def upload_shard(eng, batch, problem, rank: int, world: int):
    n_int, n_bnd = batch.interior.shape[0], batch.boundary.shape[0]
    i0, i1 = shard_bounds(n_int, rank, world)
    b0, b1 = shard_bounds(n_bnd, rank, world)
    x = np.asarray(batch.interior, dtype=np.float64)[i0:i1]
    r0, seeds, quad = residual_terms(problem, x)
    eng.set_batch(x, r0, seeds, np.asarray(batch.boundary, dtype=np.float64)[b0:b1],
                  np.asarray(batch.boundary_targets, dtype=np.float64)[b0:b1],
                  coeff_matrix(problem.coeffs), quad)


def torch_all_reduce(group=None):
    import torch.distributed as dist

    def _ar(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return _ar
