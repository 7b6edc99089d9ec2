"""The five BASELINE.json workloads as (problem, widths, batch sizes, optimizer config).

Inputs are built exactly as the reference harness builds them:
parameters from ``init_params(Architecture(widths), stream_seed(seed, 0))`` and
the batch from ``sample_batch(problem, N, Nb, stream_seed(seed, 1, 0))``
(reference src/harness.py:54-66, 249, 284-286), KFAC with damping 1e-3,
EMA 0.95, momentum 0 and identity init.  All data are synthetic.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

from .network import Architecture, init_params
from .pde import make_problem, sample_batch
from .taylor import OperatorCoeffs

STREAM_INIT, STREAM_BATCH = 0, 1


def stream_seed(seed: int, tag: int, index: int = 0) -> int:
    """``SeedSequence(entropy=seed, spawn_key=(tag, index))`` word (reference harness.py:64-66)."""
    return int(np.random.SeedSequence(entropy=seed, spawn_key=(tag, index)).generate_state(1)[0])


@dataclass(frozen=True)
class Workload:
    name: str
    problem: str
    problem_params: tuple
    widths: tuple
    n_interior: int
    n_boundary: int
    damping: float = 1e-3
    ema: float = 0.95
    momentum: float = 0.0
    steps: int = 10
    dense_coeffs_seed: int | None = None  # replace c by a random dense symmetric matrix

    def make_problem(self):
        prob = make_problem(self.problem, **dict(self.problem_params))
        if self.dense_coeffs_seed is not None:
            # the reference's own dense-coefficient test matrices (pkg/tests/test_taylor.py:22-24,
            # test_acceptance.py:34-35): c = (R + R^T) / 2, R standard normal
            r = np.random.default_rng(self.dense_coeffs_seed).standard_normal((prob.dim, prob.dim))
            prob = dataclasses.replace(prob, coeffs=OperatorCoeffs(0.5 * (r + r.T)))
        return prob

    def build(self, seed: int = 0, n_interior: int | None = None, n_boundary: int | None = None):
        """(problem, params, batch) with the reference seeding recipe."""
        prob = self.make_problem()
        params = init_params(Architecture(self.widths), stream_seed(seed, STREAM_INIT))
        ni = self.n_interior if n_interior is None else n_interior
        nb = self.n_boundary if n_boundary is None else n_boundary
        batch = sample_batch(prob, ni, nb, stream_seed(seed, STREAM_BATCH, 0))
        return prob, params, batch


WORKLOADS = {
    # c1: 2d Poisson, u* = prod sin(pi x_i) (reference poisson2d_sin)
    "c1": Workload("c1_poisson2d", "poisson2d_sin", (), (2, 64, 64, 48, 48, 1), 3000, 500),
    # c2: 5d Poisson, u* = sum cos(pi x_i) (reference poisson_cos_sum)
    "c2": Workload("c2_poisson5d", "poisson_cos_sum", (("dim", 5),), (5, 64, 64, 48, 48, 1), 3000, 500),
    # c3: 4+1d heat, u* = exp(-pi^2 t) prod sin(pi x_i); 500 initial + 500 spatial-boundary pts
    "c3": Workload("c3_heat4p1d", "heat", (("spatial_dim", 4), ("solution", "sine_product")),
                   (5, 64, 64, 48, 48, 1), 3000, 1000),
    # c4: 10d Poisson, u* = sum cos(pi x_i)
    "c4": Workload("c4_poisson10d", "poisson_cos_sum", (("dim", 10),),
                   (10, 256, 256, 128, 128, 1), 3000, 1000),
    # c5: 100d Poisson, u* = ||x||^2 / 100 (f = -2); N swept 3000 / 16384 / 65536, Nb = N // 3
    "c5": Workload("c5_poisson100d", "poisson_norm2", (("dim", 100), ("divisor", 100.0)),
                   (100, 768, 768, 512, 512, 1), 3000, 1000),
}

# Not a BASELINE config: the reference catalog's log-Fokker-Planck problem (pde.py:234-276),
# whose residual is quadratic in grad u — exercises the non-affine seed path.
WORKLOADS["lfp"] = Workload("lfp_logfokkerplanck9p1d", "log_fokker_planck", (),
                            (10, 48, 48, 32, 1), 500, 200)

# Not a BASELINE config: c2's network and residual with a dense, indefinite operator
# coefficient matrix (reference taylor.py:72-75, the non-diagonal branch of OperatorCoeffs.apply).
WORKLOADS["dense"] = Workload("dense_poisson5d", "poisson_cos_sum", (("dim", 5),),
                              (5, 64, 64, 48, 48, 1), 400, 100, dense_coeffs_seed=5)

C5_SWEEP = (3000, 16384, 65536)


def flops_per_step(widths, n_int: int, n_bnd: int, n_candidates: int = 31,
                   optimizer: str = "kfac") -> float:
    """Algorithmic FP64 flops of one KFAC step (SURVEY.md §8d formula).

    Forward: layer 0 on value rows only (its derivative rows are e_i, operator
    row 0); every later layer on all S = d + 2 rows; boundary plain forward.
    Backward: Gbar W_l for l >= 1.  Gradient/A/B contractions over all rows.
    The N-independent Kronecker-sum solve is excluded (reported separately).
    """
    d = widths[0]
    S = d + 2
    M = n_int * S
    L = len(widths) - 1
    h = widths
    f_fwd = 2.0 * n_int * h[0] * h[1] + sum(2.0 * M * h[l] * h[l + 1] for l in range(1, L))
    f_fwd += sum(2.0 * n_bnd * h[l] * h[l + 1] for l in range(L))
    f_bwd = sum(2.0 * (M + n_bnd) * h[l + 1] * h[l] for l in range(1, L))
    f_grad = 2.0 * n_int * h[1] * (h[0] + 1) + 2.0 * n_int * h[1] * h[0]
    f_grad += sum(2.0 * M * h[l + 1] * (h[l] + 1) for l in range(1, L))
    f_grad += sum(2.0 * n_bnd * h[l + 1] * (h[l] + 1) for l in range(L))
    f_a = n_int * (h[0] + 1) * (h[0] + 2) + sum(M * (h[l] + 1) * (h[l] + 2) for l in range(1, L))
    f_a += sum(n_bnd * (h[l] + 1) * (h[l] + 2) for l in range(L))
    f_b = sum(M * h[l + 1] * (h[l + 1] + 1) for l in range(L))
    f_b += sum(n_bnd * h[l + 1] * (h[l + 1] + 1) for l in range(L))
    if optimizer == "kfac_star":
        # no line search; two exact Gramian-vector products G.delta, G.prev (optim.py:266-320),
        # each a Jacobian-vector product (the forward GEMM shapes) plus a weighted gradient
        # contraction
        return f_fwd + f_bwd + f_grad + f_a + f_b + 2 * (f_fwd + f_grad)
    return (1 + n_candidates) * f_fwd + f_bwd + f_grad + f_a + f_b


def forward_gemm_flops(widths, n_int: int) -> float:
    """Flops of the interior hidden-layer forward GEMMs of ONE forward pass (l = 1..L-2)."""
    d = widths[0]
    M = n_int * (d + 2)
    L = len(widths) - 1
    return sum(2.0 * M * widths[l] * widths[l + 1] for l in range(1, L - 1))
