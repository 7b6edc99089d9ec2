"""ctypes binding of the C ABI in include/kfac_pinn_b200.h.

The shared library ``libkfac_pinn_b200.so`` is built in-tree by
``paper_2405_15603_b200/csrc/Makefile`` (``__graft_entry__.build()``).  There is
no fallback: if the library is missing, importing the device path raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkfac_pinn_b200.so")
MAX_LAYERS = 16
ABI_VERSION = 5

KP_OK = 0
KP_ERR_INVALID = 1
KP_ERR_NOT_PSD = 2
KP_ERR_LINE_SEARCH = 3
KP_ERR_NONFINITE = 4
KP_ERR_CUDA = 5
KP_ERR_EIG = 6
KP_ERR_WORKSPACE = 7


class kp_net(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("widths", C.c_int32 * (MAX_LAYERS + 1))]


class kp_problem(C.Structure):
    _fields_ = [("net", kp_net), ("n_interior", C.c_int64), ("n_boundary", C.c_int64),
                ("chunk", C.c_int64), ("n_candidates", C.c_int32), ("pad_", C.c_int32)]


class kp_kfac_config(C.Structure):
    _fields_ = [("ema", C.c_double), ("damping", C.c_double), ("momentum", C.c_double),
                ("ls_min_exp", C.c_int32), ("ls_max_exp", C.c_int32),
                ("n_interior_global", C.c_double), ("n_boundary_global", C.c_double),
                ("model_damping", C.c_double)]


class kp_state(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("theta", "prev_update", "a_int", "b_int", "a_bnd", "b_bnd")]


class kp_batch(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("x_int", "r0", "seeds", "x_bnd", "targets", "coeff_diag",
                                          "quad", "coeff_rot")]


class kp_step_out(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("scalars", "status", "ls_losses", "grad", "delta")]


P = C.POINTER
_SIGS = {
    "kp_abi_version": (C.c_int32, []),
    "kp_status_string": (C.c_char_p, [C.c_int32]),
    "kp_context_create": (C.c_int32, [C.c_int32, P(C.c_void_p)]),
    "kp_context_destroy": (C.c_int32, [C.c_void_p]),
    "kp_profile_enable": (C.c_int32, [C.c_void_p, C.c_int32]),
    "kp_profile_read": (C.c_int32, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_int64),
                                    P(C.c_int64)]),
    "kp_solver_sweeps": (C.c_int32, [P(C.c_int32), P(C.c_int32), P(C.c_int32), C.c_int32]),
    "kp_profile_read_hbm": (C.c_int32, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_int64)]),
    "kp_profile_read_cat": (C.c_int32, [C.c_void_p, C.c_int32, P(C.c_double), P(C.c_double),
                                        P(C.c_int64)]),
    "kp_param_count": (C.c_int64, [P(kp_net)]),
    "kp_factor_count": (C.c_int64, [P(kp_net), C.c_int32]),
    "kp_workspace_bytes": (C.c_int32, [C.c_void_p, P(kp_problem), P(C.c_size_t)]),
    "kp_bytes_per_interior_point": (C.c_int32, [P(kp_net), P(C.c_size_t)]),
    "kp_init_state": (C.c_int32, [C.c_void_p, P(kp_net), P(kp_state), C.c_int32, C.c_void_p]),
    "kp_kfac_step": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config), P(kp_state),
                                 P(kp_batch), P(kp_step_out), C.c_void_p, C.c_size_t, C.c_void_p]),
    "kp_reduce_buffer": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(C.c_void_p),
                                     P(C.c_int64)]),
    "kp_linesearch_buffer": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(C.c_void_p),
                                         P(C.c_int64)]),
    "kp_kfac_phase_accumulate": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                             P(kp_state), P(kp_batch), P(kp_step_out), C.c_void_p,
                                             C.c_size_t, C.c_void_p]),
    "kp_kfac_phase_precondition": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                               P(kp_state), P(kp_step_out), C.c_void_p,
                                               C.c_size_t, C.c_void_p]),
    "kp_direction_buffer": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(C.c_void_p),
                                        P(C.c_int64)]),
    "kp_kfac_phase_precondition_owned": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                                     P(kp_state), P(kp_step_out), P(C.c_int32),
                                                     C.c_void_p, C.c_size_t, C.c_void_p]),
    "kp_kfac_phase_direction": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                            P(kp_state), P(kp_step_out), C.c_void_p, C.c_size_t,
                                            C.c_void_p]),
    "kp_kfac_phase_linesearch": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                             P(kp_state), P(kp_batch), P(kp_step_out), C.c_void_p,
                                             C.c_size_t, C.c_void_p]),
    "kp_kfac_phase_update": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                         P(kp_state), P(kp_step_out), C.c_void_p, C.c_size_t,
                                         C.c_void_p]),
    "kp_kfac_star_step": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config), P(kp_state),
                                      P(kp_batch), P(kp_step_out), C.c_void_p, C.c_size_t,
                                      C.c_void_p]),
    "kp_kfac_step_graphed": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config), P(kp_state),
                                         P(kp_batch), P(kp_step_out), C.c_void_p, C.c_size_t,
                                         C.c_void_p, C.c_int32]),
    "kp_gvp_buffer": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(C.c_void_p),
                                  P(C.c_int64)]),
    "kp_kfac_star_phase_gvp": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                           P(kp_state), P(kp_batch), P(kp_step_out), C.c_void_p,
                                           C.c_size_t, C.c_void_p]),
    "kp_kfac_star_phase_update": (C.c_int32, [C.c_void_p, P(kp_problem), P(kp_kfac_config),
                                              P(kp_state), P(kp_step_out), C.c_void_p,
                                              C.c_size_t, C.c_void_p]),
    "kp_taylor_forward": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(kp_batch),
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                      C.c_void_p]),
    "kp_mlp_forward": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.c_void_p]),
    "kp_evaluate_losses": (C.c_int32, [C.c_void_p, P(kp_problem), C.c_void_p, P(kp_batch),
                                       C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "kp_kron_solve_workspace_bytes": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32,
                                                  P(C.c_size_t)]),
    "kp_kron_sum_solve": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_size_t, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library and attach prototypes; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the KFAC device path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kp_abi_version() != ABI_VERSION:
        raise ImportError(f"ABI version mismatch: library {lib.kp_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def make_net(widths) -> kp_net:
    widths = [int(w) for w in widths]
    if len(widths) - 1 > MAX_LAYERS:
        raise ValueError(f"at most {MAX_LAYERS} linear layers are supported")
    net = kp_net()
    net.n_layers = len(widths) - 1
    for i, w in enumerate(widths):
        net.widths[i] = w
    return net
