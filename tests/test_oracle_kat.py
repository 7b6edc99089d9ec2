"""The reference's own known-answer tests for this path, restated against the oracle.

Each test cites the reference test it restates (pkg/tests/...).  Together with
tests/test_oracle_golden.py (reference-generated vectors) these pin the oracle.
"""

import numpy as np
import pytest

from oracle import kfac_oracle as orc
from paper_2405_15603_b200.network import Architecture, init_params
from paper_2405_15603_b200.pde import make_problem, sample_batch


def test_initial_state_and_bias_only_on_value_row():
    # test_taylor.py:44-66: Z0 = [x; I; 0]; bias on the value row only
    w = np.array([[1.0, 2.0]])
    b = np.array([5.0])
    lin_in, pre, out = orc.taylor_forward([w], [b], np.array([[3.0, 4.0]]), np.ones(2))
    z0 = lin_in[0]
    assert np.array_equal(z0[0, 0], [3.0, 4.0]) and np.array_equal(z0[0, 1:3], np.eye(2))
    assert np.array_equal(z0[0, 3], [0.0, 0.0])
    assert out[0][0] == 16.0 and np.array_equal(out[1][0], [1.0, 2.0]) and out[2][0] == 0.0


def test_one_hidden_layer_closed_form_laplacian():
    # test_taylor.py:159-173: Lap u = sum_j a_j s''(w_j.x+b_j) ||w_j||^2, grad = W^T (a s')
    p = init_params(Architecture((2, 7, 1)), 8)
    pts = np.random.default_rng(9).uniform(-1, 1, size=(6, 2))
    _, _, (u, g, lap) = orc.taylor_forward(p.weights, p.biases, pts, np.ones(2))
    w1, b1, a = p.weights[0], p.biases[0], p.weights[1][0]
    for i, x in enumerate(pts):
        s0, s1, s2, _ = orc.tanh_derivs(w1 @ x + b1)
        assert abs(lap[i] - np.sum(a * s2 * np.sum(w1 ** 2, axis=1))) <= 1e-10
        assert np.max(np.abs(g[i] - w1.T @ (a * s1))) <= 1e-10


def test_value_row_equals_plain_forward():
    # test_taylor.py:147-157
    p = init_params(Architecture((3, 8, 8, 1)), 6)
    pts = np.random.default_rng(7).standard_normal((4, 3))
    lin_in, pre, out = orc.taylor_forward(p.weights, p.biases, pts, np.ones(3))
    u, plin, ppre = orc.plain_forward(p.weights, p.biases, pts)
    assert np.max(np.abs(out[0] - u)) <= 1e-12
    for l in range(3):
        assert np.max(np.abs(pre[l][:, 0, :] - ppre[l])) <= 1e-12


def test_partial_laplacian_ignores_inactive_direction():
    # test_taylor.py:175-194: junk in a c_ii = 0 derivative row must not reach L u
    p = init_params(Architecture((3, 6, 1)), 10)
    x = np.random.default_rng(11).standard_normal((2, 3))
    cd = np.array([0.0, 1.0, 1.0])
    _, _, out_a = orc.taylor_forward(p.weights, p.biases, x, cd)
    # perturb the time-direction weights: changes grad[:, 0] but not the operator
    w = [m.copy() for m in p.weights]
    w[0][:, 0] += 123.456
    _, _, out_b = orc.taylor_forward(w, p.biases, x, cd)
    assert not np.array_equal(out_a[1][:, 0], out_b[1][:, 0])


def test_value_seed_backward_matches_plain_backprop():
    # test_taylor.py:206-219
    p = init_params(Architecture((2, 8, 8, 1)), 12)
    pts = np.random.default_rng(13).uniform(-1, 1, size=(5, 2))
    lin_in, pre, _ = orc.taylor_forward(p.weights, p.biases, pts, np.ones(2))
    seeds = np.zeros((5, 4))
    seeds[:, 0] = 1.0
    gbar = orc.taylor_backward(p.weights, pre, seeds, np.ones(2))
    _, plin, ppre = orc.plain_forward(p.weights, p.biases, pts)
    pg = orc.plain_backward(p.weights, ppre, np.ones(5))
    for l in range(3):
        assert np.max(np.abs(gbar[l][:, 0, :] - pg[l])) <= 1e-12


def test_factors_match_literal_loops_and_rank_one():
    # test_curvature.py:64-92: factors == literal per-column loops; rank-1 exactness
    prob = make_problem("poisson2d_sin")
    p = init_params(Architecture((2, 4, 1)), 9)
    batch = sample_batch(prob, 3, 3, 13)
    ev = orc.evaluate_batch(p.weights, p.biases, batch, prob, np.ones(2))
    a_new, b_new = orc.interior_factors(ev.lin_in, ev.gbar)
    for l in range(2):
        zh = orc._augment_rows(ev.lin_in[l])
        n, s, _ = zh.shape
        a_ref = sum(np.outer(zh[i, j], zh[i, j]) for i in range(n) for j in range(s)) / (n * s)
        g = ev.gbar[l]
        b_ref = sum(np.outer(g[i, j], g[i, j]) for i in range(n) for j in range(s)) / n
        assert np.max(np.abs(a_new[l] - a_ref)) <= 1e-12
        assert np.max(np.abs(b_new[l] - b_ref)) <= 1e-12
    rng = np.random.default_rng(0)
    z = rng.standard_normal((1, 1, 3))
    g = rng.standard_normal((1, 1, 2))
    a1, b1 = orc.interior_factors([z], [g])
    zh = np.append(z[0, 0], 1.0)
    jac = np.kron(zh[:, None], g[0, 0][:, None])
    assert np.max(np.abs(np.kron(a1[0], b1[0]) - jac @ jac.T)) <= 1e-12


def test_boundary_factor_hand_checked():
    # test_curvature.py:94-103
    a, b = orc.boundary_factors([np.array([[3.0, 4.0]])], [np.array([[1.0]])])
    assert np.allclose(a[0], [[9.0, 12.0, 3.0], [12.0, 16.0, 4.0], [3.0, 4.0, 1.0]])
    assert np.allclose(b[0], [[1.0]])


def test_damping_only_preconditioner_is_half_gradient():
    # test_curvature.py:140-146
    kf = orc.OracleKfac([np.zeros((3, 3)), np.zeros((4, 4))], [np.zeros((3, 3)), np.zeros((1, 1))],
                        [np.zeros((3, 3)), np.zeros((4, 4))], [np.zeros((3, 3)), np.zeros((1, 1))],
                        0.0, 1.0)
    grads = [np.ones((3, 3)), np.ones((1, 4))]
    for g, dl in zip(grads, orc.precondition(kf, grads)):
        assert np.allclose(dl, -g / 2.0, atol=1e-12)


def test_kron_sum_solve_matches_dense():
    # test_linalg.py:117-146 and test_curvature.py:148-169
    rng = np.random.default_rng(3)
    for p, q in ((3, 3), (1, 5), (6, 2), (8, 8)):
        mk = lambda k: (lambda a: a @ a.T + k * np.eye(k))(rng.standard_normal((k, k)))  # noqa: E731
        a1, a2, b1, b2 = mk(p), mk(p), mk(q), mk(q)
        g = rng.standard_normal((q, p))
        x = orc.kron_sum_solve(a1, b1, a2, b2, g)
        dense = np.linalg.solve(np.kron(a1, b1) + np.kron(a2, b2), g.ravel(order="F"))
        assert np.linalg.norm(x.ravel(order="F") - dense) <= 1e-8 * np.linalg.norm(dense)
    assert np.allclose(orc.kron_sum_solve(np.eye(2), np.eye(2), np.eye(2), np.eye(2),
                                          np.arange(4.0).reshape(2, 2, order="F")),
                       np.arange(4.0).reshape(2, 2, order="F") / 2)
    with pytest.raises(orc.OracleNotPSD):
        orc.kron_sum_solve(np.eye(2), np.eye(2), np.diag([1.0, 0.0]), np.eye(2), np.zeros((2, 2)))


def test_line_search_grid_and_rules():
    # test_optim.py:40-97: 31 points 2^-30..2^0; ties keep the smaller step; all-NaN raises
    st = orc.init_state([np.zeros((1, 1))], [np.zeros(1)])
    assert len(st.grid) == 31 and st.grid[0] == 2.0 ** -30 and st.grid[-1] == 1.0

    def quad(ws, bs):
        return 0.5 * (ws[0][0, 0] - 1.0) ** 2, 0.0

    a, loss, _ = orc.line_search(quad, [np.zeros((1, 1))], [np.zeros(1)], [np.array([[1.0, 0.0]])], st.grid)
    assert a == 1.0 and loss == 0.0

    def flat(ws, bs):
        return float(ws[0][0, 0] ** 2), 0.0

    a, _, _ = orc.line_search(flat, [np.array([[0.5]])], [np.zeros(1)], [np.zeros((1, 2))], st.grid)
    assert a == 2.0 ** -30
    with pytest.raises(orc.OracleLineSearchError):
        orc.line_search(lambda ws, bs: (float("nan"), 0.0), [np.zeros((1, 1))], [np.zeros(1)],
                        [np.ones((1, 2))], st.grid)


def test_momentum_recurrence():
    # test_optim.py:101-123: second update = alpha * (Delta_2 + first update) exactly
    prob = make_problem("poisson2d_sin")
    p = init_params(Architecture((2, 6, 1)), 0)
    batch = sample_batch(prob, 10, 6, 0)
    st = orc.init_state(p.weights, p.biases, ema=0.5, damping=1e-2, momentum=1.0)
    orc.kfac_step(st, batch, prob)
    first = [m.copy() for m in st.prev_update]
    before = [w.copy() for w in st.weights]
    rec = {}
    alpha, _, _, _ = orc.kfac_step(st, batch, prob, record=rec)
    for l in range(2):
        expect = alpha * (rec["delta"][l] + first[l])
        assert np.max(np.abs((st.weights[l] - before[l]) - expect[:, :-1])) <= 1e-12


def test_kfac_star_quadratic_model_rules():
    # pkg/tests/test_optim.py:184-207: identity-Gramian Rayleigh solution; parallel
    # directions fall back to the alpha-only solve
    rng = np.random.default_rng(5)
    dv, gv = rng.standard_normal(4), rng.standard_normal(4)
    a, m = orc.solve_quadratic_model(False, float(dv @ dv), 0.0, 0.0, float(dv @ gv), 0.0)
    assert abs(a + float(dv @ gv) / float(dv @ dv)) <= 1e-14 and m == 0.0
    d = np.array([1.0, 2.0])
    m11 = float(d @ d)
    k = 2.5
    a, m = orc.solve_quadratic_model(True, m11, k * m11, k * k * m11, 3.0, 3.0 * k)
    assert m == 0.0 and abs(a + 3.0 / m11) <= 1e-14


def test_kfac_star_first_step_is_alpha_only_and_stationary():
    # pkg/tests/test_optim.py:159-183, 209-237: mu = 0 without a previous update, and the
    # solved (alpha, mu) zero the gradient of the quadratic model on the next step
    prob = make_problem("poisson2d_sin")
    p = init_params(Architecture((2, 6, 1)), 3)
    batch = sample_batch(prob, 12, 6, 6)
    st = orc.init_state(p.weights, p.biases, ema=0.5, damping=1e-3)
    _, mu, _, _ = orc.kfac_star_step(st, batch, prob)
    assert mu == 0.0
    rec = {}
    alpha, mu, _, _ = orc.kfac_star_step(st, batch, prob, record=rec)
    m11, m12, m22, rhs1, rhs2 = rec["m"]
    res = np.array([m11 * alpha + m12 * mu + rhs1, m12 * alpha + m22 * mu + rhs2])
    gnorm = np.linalg.norm(np.concatenate([g.ravel() for g in rec["grad_mats"]]))
    assert np.linalg.norm(res) <= 1e-8 * gnorm
