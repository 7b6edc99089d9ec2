"""Device-resident KFAC state and the calls into the C ABI.

``KfacEngine`` owns, on one GPU, everything the reference keeps in
``TrainState`` / ``KfacState`` (src/optim.py:81-92, src/curvature.py:43-59):
the packed parameters theta, the previous update, the four factor lists, plus
the batch buffers and one scratch workspace.  PyTorch is used only as the
device allocator and for the current CUDA stream; all arithmetic happens in
``libkfac_pinn_b200.so`` (hand-written sm_100a kernels).  There is no CPU
fallback: without a CUDA device or without the library this raises.

Packed layouts (see include/kfac_pinn_b200.h): per layer the augmented matrix
``[W | b]`` (``q x p``) row-major, layers concatenated; factors ``p x p`` /
``q x q`` row-major, concatenated.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from .linalg import NotPositiveSemidefiniteError
from .taylor import coeff_spectrum


class LineSearchError(RuntimeError):
    """Raised when the loss is non-finite at every grid step size (src/optim.py:37-38)."""


def raise_for_status(code: int, where: str = ""):
    if code == _capi.KP_OK:
        return
    msg = _capi.load().kp_status_string(code).decode()
    if where:
        msg = f"{where}: {msg}"
    if code == _capi.KP_ERR_NOT_PSD:
        raise NotPositiveSemidefiniteError(msg)
    if code == _capi.KP_ERR_LINE_SEARCH:
        raise LineSearchError(msg)
    if code == _capi.KP_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if code == _capi.KP_ERR_EIG:
        raise np.linalg.LinAlgError(msg)
    if code == _capi.KP_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


def pack_params(params) -> np.ndarray:
    """Row-major ``[W | b]`` per layer, concatenated (device layout)."""
    return np.concatenate([np.hstack([np.asarray(w, np.float64), np.asarray(b, np.float64)[:, None]]).ravel()
                           for w, b in zip(params.weights, params.biases)])


def unpack_mats(vec: np.ndarray, widths) -> list:
    out, off = [], 0
    for h_in, h_out in zip(widths[:-1], widths[1:]):
        p, q = h_in + 1, h_out
        out.append(vec[off:off + p * q].reshape(q, p).copy())
        off += p * q
    return out


def pack_mats(mats) -> np.ndarray:
    return np.concatenate([np.asarray(m, np.float64).ravel() for m in mats])


def unpack_factors(vec: np.ndarray, sizes) -> list:
    out, off = [], 0
    for k in sizes:
        out.append(vec[off:off + k * k].reshape(k, k).copy())
        off += k * k
    return out


class KfacEngine:
    """One rank's device state for the KFAC step of one network shape and batch size."""

    def __init__(self, widths, n_interior: int, n_boundary: int, *, ema: float, damping: float,
                 momentum: float, ls_min_exp: int = -30, ls_max_exp: int = 0, device=None,
                 chunk: int | None = None, n_interior_global: int | None = None,
                 n_boundary_global: int | None = None, mem_fraction: float = 0.8):
        import torch

        self.torch = torch
        self.lib = _capi.load()
        if not torch.cuda.is_available():
            raise RuntimeError("the KFAC device path needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.widths = tuple(int(w) for w in widths)
        self.net = _capi.make_net(self.widths)
        self.D = int(self.lib.kp_param_count(C.byref(self.net)))
        if self.D <= 0:
            raise ValueError(f"invalid network widths {self.widths}")
        self.FA = int(self.lib.kp_factor_count(C.byref(self.net), 0))
        self.FB = int(self.lib.kp_factor_count(C.byref(self.net), 1))
        self.d = self.widths[0]
        self.S = self.d + 2
        self.n_interior, self.n_boundary = int(n_interior), int(n_boundary)
        self.ncand = ls_max_exp - ls_min_exp + 1
        ctx = C.c_void_p()
        raise_for_status(self.lib.kp_context_create(self.device.index, C.byref(ctx)), "context")
        self.ctx = ctx

        self.cfg = _capi.kp_kfac_config()
        self.cfg.ema, self.cfg.damping, self.cfg.momentum = float(ema), float(damping), float(momentum)
        self.cfg.ls_min_exp, self.cfg.ls_max_exp = int(ls_min_exp), int(ls_max_exp)
        self.cfg.n_interior_global = float(n_interior_global or n_interior)
        self.cfg.n_boundary_global = float(n_boundary_global or n_boundary)

        dev, f64 = self.device, torch.float64
        z = lambda n: torch.zeros(max(int(n), 1), dtype=f64, device=dev)  # noqa: E731
        self.theta, self.prev = z(self.D), z(self.D)
        self.a_int, self.b_int, self.a_bnd, self.b_bnd = z(self.FA), z(self.FB), z(self.FA), z(self.FB)
        self.st = _capi.kp_state(_ptr(self.theta), _ptr(self.prev), _ptr(self.a_int),
                                 _ptr(self.b_int), _ptr(self.a_bnd), _ptr(self.b_bnd))
        self.scalars = z(4)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ls_losses = z(2 * self.ncand)
        self.grad, self.delta = z(self.D), z(self.D)
        self.out = _capi.kp_step_out(_ptr(self.scalars), _ptr(self.status), _ptr(self.ls_losses),
                                     _ptr(self.grad), _ptr(self.delta))
        self.x_int = z(self.n_interior * self.d)
        self.r0 = z(self.n_interior)
        self.seeds = z(self.n_interior * self.S)
        self.x_bnd = z(self.n_boundary * self.d)
        self.targets = z(self.n_boundary)
        self.cdiag = z(self.d)
        self.quad = None  # allocated on first non-affine batch
        self.rot = None   # eigenvectors of a dense coefficient matrix (first use)
        self._coeff_key = self._lam = self._rot_host = None
        self.batch = _capi.kp_batch(_ptr(self.x_int), _ptr(self.r0), _ptr(self.seeds),
                                    _ptr(self.x_bnd), _ptr(self.targets), _ptr(self.cdiag), 0)
        self.prob = _capi.kp_problem()
        self.prob.net = self.net
        self.prob.n_interior, self.prob.n_boundary = self.n_interior, self.n_boundary
        self.prob.n_candidates = self.ncand
        self.prob.chunk = int(chunk) if chunk else self._auto_chunk(mem_fraction)
        nbytes = C.c_size_t()
        raise_for_status(self.lib.kp_workspace_bytes(self.ctx, C.byref(self.prob), C.byref(nbytes)),
                         "workspace")
        self.ws_bytes = int(nbytes.value)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self._pin = {}

    # ------------------------------------------------------------------ setup
    def _auto_chunk(self, mem_fraction: float) -> int:
        """Largest interior chunk whose workspace fits in ``mem_fraction`` of free HBM."""
        free, _ = self.torch.cuda.mem_get_info(self.device)
        budget = int(free * mem_fraction)
        per = C.c_size_t()
        raise_for_status(self.lib.kp_bytes_per_interior_point(C.byref(self.net), C.byref(per)))
        nb = C.c_size_t()
        self.prob.chunk = 1
        raise_for_status(self.lib.kp_workspace_bytes(self.ctx, C.byref(self.prob), C.byref(nb)))
        fixed = int(nb.value) - int(per.value)
        chunk = max(1, (budget - fixed) // max(int(per.value), 1))
        return int(min(chunk, self.n_interior))

    @property
    def stream(self):
        return self.torch.cuda.current_stream(self.device)

    def _h2d(self, dst, arr):
        """Host -> device copy through a pinned staging buffer (non-blocking)."""
        arr = np.ascontiguousarray(arr, dtype=np.float64).ravel()
        key = (id(dst), arr.size)
        buf = self._pin.get(key)
        if buf is None:
            buf = self.torch.empty(arr.size, dtype=self.torch.float64, pin_memory=True)
            self._pin[key] = buf
        buf.numpy()[:] = arr
        dst[: arr.size].copy_(buf, non_blocking=True)

    def _d2h(self, src, n) -> np.ndarray:
        return src[:n].cpu().numpy().copy()

    def load_params(self, params):
        self._h2d(self.theta, pack_params(params))

    def init_factors(self, identity: bool = True):
        raise_for_status(self.lib.kp_init_state(self.ctx, C.byref(self.net), C.byref(self.st),
                                                int(bool(identity)), C.c_void_p(self.stream.cuda_stream)))

    def set_batch(self, x_int, r0, seeds, x_bnd, targets, cdiag, quad=None):
        """Upload one batch; ``quad`` (N x d) makes the residual quadratic in grad u
        (pde.residual_terms), None keeps it affine.  ``cdiag`` is the operator's
        coefficient diagonal (d,) or its full symmetric matrix (d, d); a non-diagonal
        matrix switches the engine to its eigenbasis (taylor.coeff_spectrum)."""
        if x_int.shape != (self.n_interior, self.d) or x_bnd.shape != (self.n_boundary, self.d):
            raise ValueError("batch shape does not match the engine")
        cmat = np.asarray(cdiag, dtype=np.float64)
        key = (cmat.shape, cmat.tobytes())
        if key != self._coeff_key:
            lam, rot = coeff_spectrum(cmat)
            if lam.shape != (self.d,):
                raise ValueError(f"operator dim {lam.size} does not match input dim {self.d}")
            self._coeff_key, self._lam, self._rot_host = key, lam, rot
            if rot is not None:
                if self.rot is None:
                    self.rot = self.torch.zeros(self.d * self.d, dtype=self.torch.float64,
                                                device=self.device)
                self._h2d(self.rot, rot)
        cdiag = self._lam
        if self._rot_host is not None:
            if quad is not None:
                raise NotImplementedError(
                    "a residual quadratic in grad u with non-diagonal operator coefficients")
            self.batch.coeff_rot = _ptr(self.rot)
        else:
            self.batch.coeff_rot = 0
        if quad is None:
            self.batch.quad = 0
        else:
            if self.quad is None:
                self.quad = self.torch.zeros(self.n_interior * self.d, dtype=self.torch.float64,
                                             device=self.device)
            self._h2d(self.quad, quad)
            self.batch.quad = _ptr(self.quad)
        self._h2d(self.x_int, x_int)
        self._h2d(self.r0, r0)
        self._h2d(self.seeds, seeds)
        self._h2d(self.x_bnd, x_bnd)
        self._h2d(self.targets, targets)
        self._h2d(self.cdiag, cdiag)

    # ------------------------------------------------------------------ reads
    def theta_numpy(self) -> np.ndarray:
        return self._d2h(self.theta, self.D)

    def param_mats(self) -> list:
        return unpack_mats(self.theta_numpy(), self.widths)

    def prev_mats(self) -> list:
        return unpack_mats(self._d2h(self.prev, self.D), self.widths)

    def set_prev_mats(self, mats):
        self._h2d(self.prev, pack_mats(mats))

    def factor_lists(self):
        ps = [w + 1 for w in self.widths[:-1]]
        qs = list(self.widths[1:])
        return (unpack_factors(self._d2h(self.a_int, self.FA), ps),
                unpack_factors(self._d2h(self.b_int, self.FB), qs),
                unpack_factors(self._d2h(self.a_bnd, self.FA), ps),
                unpack_factors(self._d2h(self.b_bnd, self.FB), qs))

    def set_factor_lists(self, a_int, b_int, a_bnd, b_bnd):
        self._h2d(self.a_int, pack_mats(a_int))
        self._h2d(self.b_int, pack_mats(b_int))
        self._h2d(self.a_bnd, pack_mats(a_bnd))
        self._h2d(self.b_bnd, pack_mats(b_bnd))

    # ------------------------------------------------------------------ step
    def _args(self):
        return (self.ctx, C.byref(self.prob), C.byref(self.cfg), C.byref(self.st),
                C.byref(self.batch), C.byref(self.out), C.c_void_p(_ptr(self.ws)),
                C.c_size_t(self.ws_bytes), C.c_void_p(self.stream.cuda_stream))

    use_graph = True  # replay small (device-solver-only) steps from a captured CUDA graph

    def launch_step(self):
        """Enqueue one whole KFAC step on the current stream (no host sync)."""
        if self.use_graph:
            raise_for_status(self.lib.kp_kfac_step_graphed(*self._args(), 0), "kp_kfac_step")
        else:
            raise_for_status(self.lib.kp_kfac_step(*self._args()), "kp_kfac_step")

    def finish_step(self):
        """Synchronise, read StepInfo scalars and raise on a device-side failure."""
        self.stream.synchronize()
        sc = self.scalars.cpu().numpy()
        code = int(self.status.cpu().item())
        return sc, code

    def step(self):
        self.launch_step()
        sc, code = self.finish_step()
        raise_for_status(code, "kfac step")
        return float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])

    def launch_star_step(self):
        """Enqueue one KFAC* step (src/optim.py:266-320) on the current stream."""
        if self.use_graph:
            raise_for_status(self.lib.kp_kfac_step_graphed(*self._args(), 1), "kp_kfac_star_step")
        else:
            raise_for_status(self.lib.kp_kfac_star_step(*self._args()), "kp_kfac_star_step")

    def star_step(self):
        self.launch_star_step()
        sc, code = self.finish_step()
        raise_for_status(code, "kfac_star step")
        return float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])

    # phased step for sharded multi-GPU runs
    def reduce_buffer(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        raise_for_status(self.lib.kp_reduce_buffer(self.ctx, C.byref(self.prob),
                                                   C.c_void_p(_ptr(self.ws)), C.byref(ptr), C.byref(cnt)))
        return self._view(ptr.value, cnt.value)

    def linesearch_buffer(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        raise_for_status(self.lib.kp_linesearch_buffer(self.ctx, C.byref(self.prob),
                                                       C.c_void_p(_ptr(self.ws)), C.byref(ptr), C.byref(cnt)))
        return self._view(ptr.value, cnt.value)

    def direction_buffer(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        raise_for_status(self.lib.kp_direction_buffer(self.ctx, C.byref(self.prob),
                                                      C.c_void_p(_ptr(self.ws)), C.byref(ptr),
                                                      C.byref(cnt)))
        return self._view(ptr.value, cnt.value)

    def gvp_buffer(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        raise_for_status(self.lib.kp_gvp_buffer(self.ctx, C.byref(self.prob), C.c_void_p(_ptr(self.ws)),
                                                C.byref(ptr), C.byref(cnt)))
        return self._view(ptr.value, cnt.value)

    def _view(self, ptr: int, count: int):
        base = _ptr(self.ws)
        off = ptr - base
        assert off % 8 == 0 and off >= 0
        return self.ws[off: off + 8 * count].view(self.torch.float64)

    def phase(self, name: str, owned=None):
        """Run one phase; ``precondition_owned`` solves only the layers flagged in ``owned``."""
        a = self._args()
        if name == "precondition_owned":
            flags = (C.c_int32 * (len(self.widths) - 1))(*[1 if o else 0 for o in owned])
            rc = self.lib.kp_kfac_phase_precondition_owned(*a[:4], *a[5:6], flags, *a[6:])
        elif name == "direction":
            rc = self.lib.kp_kfac_phase_direction(*a[:4], *a[5:])
        elif name == "accumulate":
            rc = self.lib.kp_kfac_phase_accumulate(*a)
        elif name == "linesearch":
            rc = self.lib.kp_kfac_phase_linesearch(*a)
        elif name == "precondition":
            rc = self.lib.kp_kfac_phase_precondition(*a[:4], *a[5:])
        elif name == "update":
            rc = self.lib.kp_kfac_phase_update(*a[:4], *a[5:])
        elif name == "star_gvp":
            rc = self.lib.kp_kfac_star_phase_gvp(*a)
        elif name == "star_update":
            rc = self.lib.kp_kfac_star_phase_update(*a[:4], *a[5:])
        else:
            raise ValueError(name)
        raise_for_status(rc, f"phase {name}")

    # ------------------------------------------------------------------ other entry points
    def taylor_forward(self, theta=None):
        t = self.torch
        val = t.empty(self.n_interior, dtype=t.float64, device=self.device)
        grad = t.empty(self.n_interior * self.d, dtype=t.float64, device=self.device)
        op = t.empty(self.n_interior, dtype=t.float64, device=self.device)
        th = self.theta if theta is None else theta
        raise_for_status(self.lib.kp_taylor_forward(
            self.ctx, C.byref(self.prob), C.c_void_p(_ptr(th)), C.byref(self.batch),
            C.c_void_p(_ptr(val)), C.c_void_p(_ptr(grad)), C.c_void_p(_ptr(op)),
            C.c_void_p(_ptr(self.ws)), C.c_size_t(self.ws_bytes), C.c_void_p(self.stream.cuda_stream)))
        self.stream.synchronize()
        return val.cpu().numpy(), grad.cpu().numpy().reshape(self.n_interior, self.d), op.cpu().numpy()

    def evaluate_losses(self, theta=None):
        t = self.torch
        out = t.zeros(2, dtype=t.float64, device=self.device)
        th = self.theta if theta is None else theta
        raise_for_status(self.lib.kp_evaluate_losses(
            self.ctx, C.byref(self.prob), C.c_void_p(_ptr(th)), C.byref(self.batch),
            C.c_void_p(_ptr(out)), C.c_void_p(_ptr(self.ws)), C.c_size_t(self.ws_bytes),
            C.c_void_p(self.stream.cuda_stream)))
        self.stream.synchronize()
        o = out.cpu().numpy()
        return float(o[0]), float(o[1])

    def profile(self, enable: bool):
        self.lib.kp_profile_enable(self.ctx, int(bool(enable)))

    def profile_read(self):
        ms, fl, n, k = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        raise_for_status(self.lib.kp_profile_read(self.ctx, C.byref(ms), C.byref(fl), C.byref(n),
                                                  C.byref(k)))
        return ms.value, fl.value, n.value, k.value

    def profile_read_hbm(self):
        """(ms, algorithmic bytes, launches) of the activation-adjoint kernel since enable."""
        ms, by, n = C.c_double(), C.c_double(), C.c_int64()
        raise_for_status(self.lib.kp_profile_read_hbm(self.ctx, C.byref(ms), C.byref(by), C.byref(n)))
        return ms.value, by.value, n.value

    def profile_read_cat(self, cat: int):
        """(ms, work, launches) of category ``cat`` since enable: 0 = the line search's INT8
        tensor-core (CRT) layers (work: FP64-equivalent flops), 1 = their residue slicing
        (work: algorithmic DRAM bytes)."""
        ms, wk, n = C.c_double(), C.c_double(), C.c_int64()
        raise_for_status(self.lib.kp_profile_read_cat(self.ctx, int(cat), C.byref(ms), C.byref(wk),
                                                      C.byref(n)))
        return ms.value, wk.value, n.value

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.stream.synchronize()
            self.lib.kp_context_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kron_sum_solve_device(a1, b1, a2, b2, g, device=None):
    """kron_sum_solve (src/linalg.py:136-174) through the C ABI; returns X (q x p) with
    B1 X A1 + B2 X A2 = G.  ``g`` is the q x p matrix (reference passes vec_F(g))."""
    import torch

    lib = _capi.load()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = C.c_void_p()
    raise_for_status(lib.kp_context_create(dev.index, C.byref(ctx)))
    try:
        p, q = a1.shape[0], b1.shape[0]
        T = lambda m: torch.as_tensor(np.ascontiguousarray(m, np.float64), device=dev)  # noqa: E731
        ta1, tb1, ta2, tb2, tg = T(a1), T(b1), T(a2), T(b2), T(g)
        x = torch.empty(q * p, dtype=torch.float64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        nb = C.c_size_t()
        raise_for_status(lib.kp_kron_solve_workspace_bytes(ctx, p, q, C.byref(nb)))
        ws = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
        s = torch.cuda.current_stream(dev)
        raise_for_status(lib.kp_kron_sum_solve(ctx, p, q, _ptr(ta1), _ptr(tb1), _ptr(ta2), _ptr(tb2),
                                               _ptr(tg), _ptr(x), _ptr(status), _ptr(ws),
                                               C.c_size_t(int(nb.value)), C.c_void_p(s.cuda_stream)))
        s.synchronize()
        raise_for_status(int(status.cpu().item()), "kron_sum_solve")
        return x.cpu().numpy().reshape(q, p)
    finally:
        lib.kp_context_destroy(ctx)
