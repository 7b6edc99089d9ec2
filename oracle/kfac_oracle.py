"""CPU oracle: a NumPy restatement of the reference KFAC step for PINN losses.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
module, and only as the checker / the CPU baseline.  The product path
(``paper_2405_15603_b200``) never imports it and has no CPU fallback.

What it restates (reference = ``/root/reference/pkg/src/pinnopt``, "src/"):

====================================  ======================================
oracle function                       reference it follows
====================================  ======================================
``tanh_derivs``                       src/network.py:54-62
``taylor_forward``                    src/taylor.py:124-203 (initial_state,
                                      linear layer :134-148, activation
                                      :151-169)
``taylor_backward``                   src/taylor.py:206-276 (layer adjoints
                                      only; the unused ``weight_grads`` GEMM
                                      at :269 is not needed by KFAC)
``plain_forward`` / ``plain_backward``  src/network.py:200-232
``evaluate_batch``                    src/optim.py:155-189 with the losses of
                                      src/pde.py:344-360
``interior_factors`` / ``boundary_factors``  src/curvature.py:88-137
``kron_sum_solve``                    src/linalg.py:124-174 (same
                                      simultaneous-diagonalisation route: 4 eigh)
``precondition``                      src/curvature.py:140-163
``line_search``                       src/optim.py:195-211
``kfac_step`` / ``optimizer_step``     src/optim.py:237-263, 396-402
``kfac_star_step``                    src/optim.py:266-320 (exact Gramian-vector
                                      products from the per-sample residual
                                      Jacobian rows, src/curvature.py:169-194,253-260)
====================================  ======================================

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src``), plus the reference's own known-answer tests
restated in ``tests/test_oracle_kat.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PSD_TOL = 1e-6          # src/linalg.py:36
SYMMETRY_TOL = 1e-10    # src/linalg.py:33


class OracleLineSearchError(RuntimeError):
    pass


class OracleNotPSD(ValueError):
    pass


# ---------------------------------------------------------------------------
# activation


def tanh_derivs(z, order=3):
    """s0 = tanh z, s1 = 1 - s0^2, s2 = -2 s0 s1, s3 = -2 s1^2 - 2 s0 s2 (network.py:54-62)."""
    s0 = np.tanh(z)
    s1 = 1.0 - s0 * s0
    s2 = -2.0 * s0 * s1
    s3 = (-2.0 * s1 * s1 - 2.0 * s0 * s2) if order >= 3 else None
    return s0, s1, s2, s3


# ---------------------------------------------------------------------------
# forward-Laplacian engine


def _apply_c(cdiag, g):
    """Contract the coefficients over the derivative axis of an (N, d, h) stack
    (taylor.py:66-75): ``cdiag`` is the diagonal (d,) or the dense matrix (d, d)."""
    if cdiag.ndim == 1:
        return g * cdiag[None, :, None]
    return np.einsum("ij,njh->nih", cdiag, g)


def coeffs_of(problem):
    """Diagonal of the problem's c when it is diagonal (taylor.py:56-57), else c itself."""
    c = np.asarray(problem.coeffs.c, dtype=np.float64)
    diag = np.diagonal(c).copy()
    return diag if np.array_equal(c, np.diag(diag)) else c


def taylor_forward(weights, biases, x, cdiag):
    """Propagate [value | d/dx_1..d | Lz] rows through the MLP (taylor.py:172-203).

    Returns ``(lin_in, pre, out)``: ``lin_in[l]`` is the (N, S, h_l) input of
    linear layer l (states[2l] in the reference), ``pre[l]`` its (N, S, h_{l+1})
    output (states[2l+1]); ``out`` = (value, gradient, operator) of the scalar
    network output.
    """
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    z = np.zeros((n, d + 2, d))          # initial_state, taylor.py:124-131
    z[:, 0, :] = x
    z[:, 1:d + 1, :] = np.eye(d)
    lin_in, pre = [], []
    n_lin = len(weights)
    for l, (w, b) in enumerate(zip(weights, biases)):
        lin_in.append(z)
        y = (z.reshape(n * (d + 2), -1) @ w.T).reshape(n, d + 2, w.shape[0])
        y[:, 0, :] += b                   # bias on the value row only, taylor.py:147
        pre.append(y)
        if l == n_lin - 1:
            break
        s0, s1, s2, _ = tanh_derivs(y[:, 0, :], order=2)
        g = y[:, 1:d + 1, :]
        quad = np.sum(_apply_c(cdiag, g) * g, axis=1)
        z = np.empty_like(y)              # taylor_forward_activation, taylor.py:151-169
        z[:, 0, :] = s0
        z[:, 1:d + 1, :] = s1[:, None, :] * g
        z[:, d + 1, :] = s1 * y[:, d + 1, :] + s2 * quad
    last = pre[-1]
    out = (last[:, 0, 0].copy(), last[:, 1:d + 1, 0].copy(), last[:, d + 1, 0].copy())
    return lin_in, pre, out


def activation_backward(y, gout, cdiag):
    """Adjoint of the Taylor activation (taylor.py:206-239); ``y`` is the pre-activation state."""
    d = cdiag.shape[0]
    s0, s1, s2, s3 = tanh_derivs(y[:, 0, :], order=3)
    g = y[:, 1:d + 1, :]
    ell = y[:, d + 1, :]
    vb, gb, lb = gout[:, 0, :], gout[:, 1:d + 1, :], gout[:, d + 1, :]
    cg = _apply_c(cdiag, g)
    quad = np.sum(cg * g, axis=1)
    gin = np.empty_like(gout)
    gin[:, d + 1, :] = s1 * lb
    gin[:, 1:d + 1, :] = s1[:, None, :] * gb + 2.0 * s2[:, None, :] * cg * lb[:, None, :]
    gin[:, 0, :] = s1 * vb + s2 * np.sum(g * gb, axis=1) + s2 * ell * lb + s3 * quad * lb
    return gin


def taylor_backward(weights, pre, seeds, cdiag):
    """Per-layer output adjoints ``Gbar_l`` (N, S, h_{l+1}) (taylor.py:242-276)."""
    n_lin = len(weights)
    out = [None] * n_lin
    g = np.asarray(seeds, dtype=np.float64)[:, :, None]
    for l in range(n_lin - 1, -1, -1):
        out[l] = g
        if l == 0:
            break
        g = np.matmul(g, weights[l])                     # taylor.py:271
        g = activation_backward(pre[l - 1], g, cdiag)    # taylor.py:274
    return out


def plain_forward(weights, biases, x):
    """Plain batched MLP forward (network.py:200-213): (u, linear inputs, pre-activations)."""
    z = np.asarray(x, dtype=np.float64)
    lin_in, pre = [], []
    for l, (w, b) in enumerate(zip(weights, biases)):
        lin_in.append(z)
        z = z @ w.T + b
        pre.append(z)
        if l < len(weights) - 1:
            z = np.tanh(z)
    return pre[-1][:, 0], lin_in, pre


def plain_backward(weights, pre, seed):
    """Per-layer output gradients of seed_n u_n (network.py:216-232)."""
    n_lin = len(weights)
    grads = [None] * n_lin
    g = np.asarray(seed, dtype=np.float64)[:, None]
    for l in range(n_lin - 1, -1, -1):
        grads[l] = g
        if l > 0:
            g = g @ weights[l]
            g = g * tanh_derivs(pre[l - 1], order=2)[1]
    return grads


def _augment_rows(z):
    """Bias entry appended to an (N, S, h) state: 1 on the value row, 0 elsewhere (curvature.py:88-93)."""
    n, s, h = z.shape
    out = np.zeros((n, s, h + 1))
    out[:, :, :h] = z
    out[:, 0, h] = 1.0
    return out


# ---------------------------------------------------------------------------
# batch evaluation, factors, preconditioner


@dataclass
class Eval:
    loss_interior: float
    loss_boundary: float
    r_int: np.ndarray
    r_bnd: np.ndarray
    lin_in: list
    gbar: list
    bnd_lin_in: list
    bnd_grads: list
    grad_mats: list


def evaluate_batch(weights, biases, batch, problem, cdiag):
    """Losses, reverse pass and residual-weighted gradient (optim.py:155-189, pde.py:344-360)."""
    x = np.asarray(batch.interior, dtype=np.float64)
    lin_in, pre, (u, gu, lu) = taylor_forward(weights, biases, x, cdiag)
    r = np.asarray(problem.residual(x, u, gu, lu), dtype=np.float64)
    loss_int = float(r @ r) / (2.0 * r.size) if r.size else 0.0
    du, dg, dop = problem.residual_grads(x, u, gu, lu)
    seeds = np.concatenate([np.broadcast_to(du, (x.shape[0],))[:, None],
                            np.broadcast_to(dg, x.shape),
                            np.broadcast_to(dop, (x.shape[0],))[:, None]], axis=1)
    gbar = taylor_backward(weights, pre, seeds, cdiag)

    ub, bnd_in, bnd_pre = plain_forward(weights, biases, batch.boundary)
    res = ub - np.asarray(batch.boundary_targets, dtype=np.float64)
    loss_bnd = float(res @ res) / (2.0 * res.size) if res.size else 0.0
    bgr = plain_backward(weights, bnd_pre, np.ones(res.size))

    w_int = r / max(r.size, 1)
    w_bnd = res / max(res.size, 1)
    grads = []
    for l in range(len(weights)):
        g = gbar[l]
        n, s, q = g.shape
        zh = _augment_rows(lin_in[l]).reshape(n * s, -1)
        m = (g * w_int[:, None, None]).reshape(n * s, q).T @ zh
        zb = np.hstack([bnd_in[l], np.ones((bnd_in[l].shape[0], 1))])
        m = m + (bgr[l] * w_bnd[:, None]).T @ zb
        grads.append(m)
    return Eval(loss_int, loss_bnd, r, res, lin_in, gbar, bnd_in, bgr, grads)


def _sym(m):
    return 0.5 * (m + m.T)


def interior_factors(lin_in, gbar):
    """Batch factors A = sum zhat zhat^T/(N S), B = sum g g^T / N (curvature.py:96-118)."""
    a_new, b_new = [], []
    for z, g in zip(lin_in, gbar):
        n, s, _ = z.shape
        zh = _augment_rows(z).reshape(n * s, -1)
        gf = g.reshape(n * s, -1)
        a_new.append(_sym(zh.T @ zh / (n * s)))
        b_new.append(_sym(gf.T @ gf / n))
    return a_new, b_new


def boundary_factors(lin_in, grads):
    """Condition-term factors over bias-augmented plain inputs (curvature.py:121-137)."""
    a_new, b_new = [], []
    for z, g in zip(lin_in, grads):
        n = z.shape[0]
        zh = np.hstack([z, np.ones((n, 1))])
        a_new.append(_sym(zh.T @ zh / n))
        b_new.append(_sym(g.T @ g / n))
    return a_new, b_new


def _eigh_checked(m):
    if m.size and float(np.max(np.abs(m - m.T))) > SYMMETRY_TOL:
        raise ValueError("matrix is not symmetric to 1e-10")       # linalg.py:65-76
    return np.linalg.eigh(m)


def _pd_inv_sqrt(m):
    lam, q = _eigh_checked(m)                                        # linalg.py:124-133
    top = float(np.max(np.abs(lam))) if lam.size else 0.0
    if lam.size == 0 or float(lam[0]) <= 1e-14 * max(top, 1e-300):
        raise OracleNotPSD("matrix must be positive definite")
    return (q * lam ** -0.5) @ q.T


def _psd_check(lam):
    top = float(np.max(np.abs(lam))) if lam.size else 0.0            # linalg.py:79-83
    if lam.size and float(lam[0]) < -PSD_TOL * max(top, 1e-300):
        raise OracleNotPSD("smallest eigenvalue below -PSD_TOL * norm")


def kron_sum_solve(a1, b1, a2, b2, gmat):
    """Solve B1 X A1 + B2 X A2 = G for the q x p matrix X (linalg.py:136-174)."""
    ia = _pd_inv_sqrt(a2)
    ib = _pd_inv_sqrt(b2)
    ta, tb = ia @ a1 @ ia, ib @ b1 @ ib
    la, ea = _eigh_checked(_sym(ta))
    lb, eb = _eigh_checked(_sym(tb))
    _psd_check(la)
    _psd_check(lb)
    x = ib @ gmat @ ia
    y = (eb.T @ x @ ea) / (np.outer(lb, la) + 1.0)
    return ib @ (eb @ y @ ea.T) @ ia


def precondition(kf, grad_mats):
    """Damped two-term Kronecker-sum preconditioning, Delta = -(...)^-1 grad (curvature.py:140-163)."""
    lam = kf.damping
    if lam <= 0:
        raise ValueError("damping must be positive for Kronecker preconditioning")
    out = []
    for l, g in enumerate(grad_mats):
        q, p = g.shape
        ea, eb = lam * np.eye(p), lam * np.eye(q)
        v = kron_sum_solve(kf.a_int[l] + ea, kf.b_int[l] + eb, kf.a_bnd[l] + ea, kf.b_bnd[l] + eb, g)
        out.append(-v)
    return out


# ---------------------------------------------------------------------------
# state + step


@dataclass
class OracleKfac:
    a_int: list
    b_int: list
    a_bnd: list
    b_bnd: list
    ema: float
    damping: float


@dataclass
class OracleState:
    weights: list
    biases: list
    kfac: OracleKfac
    momentum: float
    grid: list
    prev_update: list = field(default_factory=list)
    step: int = 0
    # KFAC*'s quadratic-model damping is OptimizerConfig.damping (optim.py:303), the factor
    # damping KfacState.damping (curvature.py:150-152); None: the same value
    model_damping: float | None = None


def init_state(weights, biases, ema=0.9, damping=1e-2, momentum=0.0, init_mode="identity",
               ls_min_exp=-30, ls_max_exp=0):
    """init_train_state for kind="kfac" (optim.py:102-117, curvature.py:62-76)."""
    mk = (lambda k: np.eye(k)) if init_mode == "identity" else (lambda k: np.zeros((k, k)))
    ws = [np.array(w, dtype=np.float64) for w in weights]
    bs = [np.array(b, dtype=np.float64) for b in biases]
    kf = OracleKfac([mk(w.shape[1] + 1) for w in ws], [mk(w.shape[0]) for w in ws],
                    [mk(w.shape[1] + 1) for w in ws], [mk(w.shape[0]) for w in ws], ema, damping)
    grid = [2.0 ** e for e in range(ls_min_exp, ls_max_exp + 1)]    # optim.py:77-78
    prev = [np.zeros((w.shape[0], w.shape[1] + 1)) for w in ws]
    return OracleState(ws, bs, kf, momentum, grid, prev)


def losses_at(weights, biases, batch, problem, cdiag):
    """evaluate_losses (optim.py:148-152): forward-only interior + boundary losses."""
    x = np.asarray(batch.interior, dtype=np.float64)
    _, _, (u, gu, lu) = taylor_forward(weights, biases, x, cdiag)
    r = np.asarray(problem.residual(x, u, gu, lu), dtype=np.float64)
    li = float(r @ r) / (2.0 * r.size) if r.size else 0.0
    ub, _, _ = plain_forward(weights, biases, batch.boundary)
    res = ub - np.asarray(batch.boundary_targets, dtype=np.float64)
    lb = float(res @ res) / (2.0 * res.size) if res.size else 0.0
    return li, lb


def line_search(loss_fn, weights, biases, direction, grid):
    """Grid argmin, ascending, strict '<', finite only (optim.py:195-211)."""
    best_a, best_l, all_losses = None, np.inf, []
    for a in grid:
        ws = [w + a * m[:, :-1] for w, m in zip(weights, direction)]
        bs = [b + a * m[:, -1] for b, m in zip(biases, direction)]
        li, lb = loss_fn(ws, bs)
        loss = li + lb
        all_losses.append((li, lb))
        if np.isfinite(loss) and loss < best_l:
            best_a, best_l = a, loss
    if best_a is None:
        raise OracleLineSearchError("loss is non-finite at every line-search step size")
    return best_a, best_l, all_losses


def kfac_step(st: OracleState, batch, problem, record=None):
    """One KFAC step (optim.py:237-263) + non-finite check (optim.py:396-402).

    ``record`` (a dict, optional) receives the intermediates the parity tests
    compare: grad_mats, delta, direction, line-search losses.
    """
    cdiag = coeffs_of(problem)
    ev = evaluate_batch(st.weights, st.biases, batch, problem, cdiag)
    kf = st.kfac
    a_new, b_new = interior_factors(ev.lin_in, ev.gbar)
    beta = kf.ema
    kf.a_int = [beta * o + (1.0 - beta) * n for o, n in zip(kf.a_int, a_new)]   # curvature.py:79-85
    kf.b_int = [beta * o + (1.0 - beta) * n for o, n in zip(kf.b_int, b_new)]
    a_new, b_new = boundary_factors(ev.bnd_lin_in, ev.bnd_grads)
    kf.a_bnd = [beta * o + (1.0 - beta) * n for o, n in zip(kf.a_bnd, a_new)]
    kf.b_bnd = [beta * o + (1.0 - beta) * n for o, n in zip(kf.b_bnd, b_new)]
    delta = precondition(kf, ev.grad_mats)
    direction = [dl + st.momentum * pu for dl, pu in zip(delta, st.prev_update)]  # optim.py:254

    def loss_fn(ws, bs):
        return losses_at(ws, bs, batch, problem, cdiag)

    alpha, _, ls = line_search(loss_fn, st.weights, st.biases, direction, st.grid)
    st.weights = [w + alpha * m[:, :-1] for w, m in zip(st.weights, direction)]
    st.biases = [b + alpha * m[:, -1] for b, m in zip(st.biases, direction)]
    st.prev_update = [alpha * m for m in direction]
    st.step += 1
    for w, b in zip(st.weights, st.biases):
        if not (np.all(np.isfinite(w)) and np.all(np.isfinite(b))):
            raise FloatingPointError("parameters became non-finite during the step")
    if record is not None:
        record.update(grad_mats=ev.grad_mats, delta=delta, direction=direction,
                      ls_losses=np.array(ls), r_int=ev.r_int, r_bnd=ev.r_bnd)
    return alpha, st.momentum, ev.loss_interior, ev.loss_boundary


# ---------------------------------------------------------------------------
# KFAC* (optim.py:266-320)


def jacobian_rows(ev):
    """Per-sample residual Jacobian rows, interior and boundary (curvature.py:169-194).

    Row layout: per layer the (q x p) matrix sum_s g_{n,s} zhat_{n,s}^T flattened
    column-stacked, layers concatenated (the package-wide convention)."""
    segs_i, segs_b = [], []
    for l in range(len(ev.gbar)):
        zh = _augment_rows(ev.lin_in[l])                  # (N, S, p)
        blk = np.matmul(zh.transpose(0, 2, 1), ev.gbar[l])  # (N, p, q)
        segs_i.append(blk.reshape(blk.shape[0], -1))
        zb = np.hstack([ev.bnd_lin_in[l], np.ones((ev.bnd_lin_in[l].shape[0], 1))])
        bb = zb[:, :, None] * ev.bnd_grads[l][:, None, :]
        segs_b.append(bb.reshape(bb.shape[0], -1))
    return np.concatenate(segs_i, axis=1), np.concatenate(segs_b, axis=1)


def _vec(mats):
    return np.concatenate([np.asarray(m).ravel(order="F") for m in mats])


def solve_quadratic_model(have_prev, m11, m12, m22, rhs1, rhs2):
    """Minimise the (alpha, mu) quadratic model (optim.py:266-286)."""
    tiny = 1e-300
    det = m11 * m22 - m12 * m12
    scale = max(abs(m11 * m22), m12 * m12, tiny)
    if have_prev and det > 1e-12 * scale:
        return (-rhs1 * m22 + rhs2 * m12) / det, (rhs1 * m12 - rhs2 * m11) / det
    if m11 <= tiny:
        return 0.0, 0.0
    return -rhs1 / m11, 0.0


def kfac_star_step(st: OracleState, batch, problem, record=None):
    """One KFAC* step (optim.py:296-320) + non-finite check (optim.py:398-401)."""
    cdiag = coeffs_of(problem)
    ev = evaluate_batch(st.weights, st.biases, batch, problem, cdiag)
    kf = st.kfac
    beta = kf.ema
    a_new, b_new = interior_factors(ev.lin_in, ev.gbar)
    kf.a_int = [beta * o + (1.0 - beta) * n for o, n in zip(kf.a_int, a_new)]
    kf.b_int = [beta * o + (1.0 - beta) * n for o, n in zip(kf.b_int, b_new)]
    a_new, b_new = boundary_factors(ev.bnd_lin_in, ev.bnd_grads)
    kf.a_bnd = [beta * o + (1.0 - beta) * n for o, n in zip(kf.a_bnd, a_new)]
    kf.b_bnd = [beta * o + (1.0 - beta) * n for o, n in zip(kf.b_bnd, b_new)]
    delta = precondition(kf, ev.grad_mats)
    ri, rb = jacobian_rows(ev)

    def gvp(v):
        out = ri.T @ (ri @ v) / ri.shape[0]
        return out + rb.T @ (rb @ v) / rb.shape[0]

    dv, pv, gv = _vec(delta), _vec(st.prev_update), _vec(ev.grad_mats)
    lam = kf.damping if st.model_damping is None else st.model_damping
    g_dv = gvp(dv)
    m11 = float(dv @ g_dv + lam * dv @ dv)
    rhs1 = float(dv @ gv)
    have_prev = bool(pv @ pv > 0.0)
    if have_prev:
        g_pv = gvp(pv)
        m12 = float(dv @ g_pv + lam * dv @ pv)
        m22 = float(pv @ g_pv + lam * pv @ pv)
        rhs2 = float(pv @ gv)
    else:
        m12 = m22 = rhs2 = 0.0
    alpha, mu = solve_quadratic_model(have_prev, m11, m12, m22, rhs1, rhs2)
    update = [alpha * dl + mu * pu for dl, pu in zip(delta, st.prev_update)]
    st.weights = [w + 1.0 * m[:, :-1] for w, m in zip(st.weights, update)]
    st.biases = [b + 1.0 * m[:, -1] for b, m in zip(st.biases, update)]
    st.prev_update = update
    st.step += 1
    for w, b in zip(st.weights, st.biases):
        if not (np.all(np.isfinite(w)) and np.all(np.isfinite(b))):
            raise FloatingPointError("parameters became non-finite during the step")
    if record is not None:
        record.update(grad_mats=ev.grad_mats, delta=delta, m=(m11, m12, m22, rhs1, rhs2))
    return alpha, mu, ev.loss_interior, ev.loss_boundary
