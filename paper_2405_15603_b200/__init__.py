"""B200-native KFAC step for PINN losses (arXiv 2405.15603), drop-in for the reference's
``OptimizerConfig`` / ``init_train_state`` / ``optimizer_step`` (kind="kfac").

Host-side mirror of the reference interface in Python; all compute in
``libkfac_pinn_b200.so`` (hand-written FP64 sm_100a kernels, C ABI in
``include/kfac_pinn_b200.h``).
"""

from .network import Architecture, Parameters, add_scaled, init_params
from .pde import Batch, PdeProblem, PROBLEM_NAMES, make_problem, sample_batch
from .taylor import OperatorCoeffs
from .linalg import NotPositiveSemidefiniteError, NotSymmetricError
from .curvature import KfacState, init_kfac_state
from .optim import (
    LineSearchError,
    OptimizerConfig,
    StepInfo,
    TrainState,
    init_train_state,
    optimizer_step,
)

__version__ = "0.1.0"

__all__ = [
    "Architecture", "Parameters", "add_scaled", "init_params",
    "Batch", "PdeProblem", "PROBLEM_NAMES", "make_problem", "sample_batch",
    "OperatorCoeffs", "NotPositiveSemidefiniteError", "NotSymmetricError",
    "KfacState", "init_kfac_state",
    "LineSearchError", "OptimizerConfig", "StepInfo", "TrainState",
    "init_train_state", "optimizer_step",
]
