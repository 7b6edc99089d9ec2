"""GPU parity: the B200 path (through the C ABI) vs the reference's golden vectors and the oracle.

Bars (BASELINE.json north star): 1e-10 relative after one step, 1e-8 after more;
the line-search alpha must be identical.  "Relative" = max|x - ref| / max|ref|
per array.
"""

import numpy as np
import pytest

from golden_util import (FULL_WL, NAMES, NAMES10, NAMES_FULL, STAR10, STAR_FULL, STAR_NAMES, compare, has, line_search_rel, load,
                         pack_factors)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import kfac_oracle as orc  # noqa: E402
from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200.network import Architecture, Parameters, init_params, mats_to_vec  # noqa: E402
from paper_2405_15603_b200.optim import OptimizerConfig, init_train_state, optimizer_step  # noqa: E402
from paper_2405_15603_b200.pde import make_problem, sample_batch  # noqa: E402

WL_OF = {"c1": "c1", "c2": "c2", "c3": "c3", "c4": "c4", "c5": "c5", "c1_momentum": "c1",
         "c1_star": "c1", "c3_star": "c3", "c5_star": "c5", "lfp": "lfp", "lfp_star": "lfp",
         "dense": "dense", "dense_star": "dense",
         "c1_10": "c1", "c2_10": "c2", "c3_10": "c3", "c4_10": "c4", "c5_10": "c5",
         "lfp_10": "lfp", "dense_10": "dense", "c1_star_10": "c1", "lfp_star_10": "lfp",
         "c3_star_10": "c3", "c5_star_10": "c5", "c1_momentum_10": "c1", "c4_zero_10": "c4",
         **FULL_WL}


def _theta_colstack(params):
    return np.concatenate([np.hstack([w, b[:, None]]).ravel(order="F")
                           for w, b in zip(params.weights, params.biases)])


def _device_mats_to_vec(vec, widths):
    """Device row-major [W|b] packing -> reference column-stacked vector."""
    out, off = [], 0
    for h_in, h_out in zip(widths[:-1], widths[1:]):
        p, q = h_in + 1, h_out
        out.append(vec[off:off + p * q].reshape(q, p).ravel(order="F"))
        off += p * q
    return np.concatenate(out)


@pytest.mark.parametrize("name", NAMES + NAMES10 + NAMES_FULL)
def test_kfac_steps_match_reference_golden(name):
    g = load(name)
    wl = cfgs.WORKLOADS[WL_OF[name]]
    prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
    cfg = OptimizerConfig(kind="kfac", damping=float(g["damping"]), ema=float(g["ema"]),
                          momentum=float(g["momentum"]),
                          init_mode="zero" if int(g.get("init_zero", 0)) else "identity")
    state = init_train_state(params, cfg)
    t = 1
    while f"s{t}/alpha" in g:
        info = optimizer_step(state, batch, prob)
        p = f"s{t}/"
        tol = 1e-10 if t == 1 else 1e-8
        assert info.alpha == float(g[p + "alpha"]), (t, info.alpha, float(g[p + "alpha"]))
        for key, val in (("loss_interior", info.loss_interior), ("loss_boundary", info.loss_boundary)):
            ref = float(g[p + key])
            assert abs(val - ref) <= tol * abs(ref), (key, val, ref)
        eng = state._engine
        rel = line_search_rel(eng.ls_losses.cpu().numpy(), g[p + "ls_losses"])
        assert rel <= tol, rel
        if not has(g, p + "theta"):  # ten-step runs record arrays at steps 1 and 10 only
            t += 1
            continue
        widths = eng.widths
        assert compare(g, p + "grad", _device_mats_to_vec(eng.grad.cpu().numpy(), widths), tol) <= tol
        assert compare(g, p + "delta", _device_mats_to_vec(eng.delta.cpu().numpy(), widths), tol) <= tol
        assert compare(g, p + "theta", _theta_colstack(state.params), tol) <= tol
        assert compare(g, p + "prev_update", mats_to_vec(state.prev_update), tol) <= tol
        kf = state.kfac
        for key, mats in (("a_interior", kf.a_interior), ("b_interior", kf.b_interior),
                          ("a_boundary", kf.a_boundary), ("b_boundary", kf.b_boundary)):
            assert compare(g, p + key, pack_factors(mats), tol) <= tol, key
        t += 1
    assert t > (10 if name in NAMES10 or name.endswith("full10") else 3 if name in NAMES_FULL else 1)


def _oracle_vs_device(widths, problem, n_int, n_bnd, steps, momentum=0.0, ema=0.95, damping=1e-3,
                      seed=3, chunk=None):
    arch = Architecture(widths)
    params = init_params(arch, seed)
    batch = sample_batch(problem, n_int, n_bnd, seed + 100)
    st = orc.init_state(params.weights, params.biases, ema=ema, damping=damping, momentum=momentum)
    cfg = OptimizerConfig(kind="kfac", damping=damping, ema=ema, momentum=momentum)
    state = init_train_state(params, cfg)
    if chunk is not None:
        from paper_2405_15603_b200.optim import _engine_for
        _engine_for(state, batch, tuple(widths))
        eng = state._engine
        from paper_2405_15603_b200.engine import KfacEngine
        new = KfacEngine(widths, n_int, n_bnd, ema=ema, damping=damping, momentum=momentum,
                         chunk=chunk)
        kf = state.kfac
        new.set_factor_lists(kf.a_interior, kf.b_interior, kf.a_boundary, kf.b_boundary)
        new.set_prev_mats(state.prev_update)
        new.load_params(state.params)
        state._engine = new
        del eng
    worst = 0.0
    for t in range(steps):
        a_ref, _, li_ref, lb_ref = orc.kfac_step(st, batch, problem)
        info = optimizer_step(state, batch, problem)
        assert info.alpha == a_ref
        th_ref = np.concatenate([np.hstack([w, b[:, None]]).ravel() for w, b in zip(st.weights, st.biases)])
        th = np.concatenate([np.hstack([w, b[:, None]]).ravel()
                             for w, b in zip(state.params.weights, state.params.biases)])
        err = max(abs(info.loss_interior - li_ref) / abs(li_ref),
                  abs(info.loss_boundary - lb_ref) / abs(lb_ref),
                  np.max(np.abs(th - th_ref)) / np.max(np.abs(th_ref)))
        worst = max(worst, err)
        assert err <= (1e-10 if t == 0 else 1e-8), (t, err)
    return worst


@pytest.mark.parametrize("widths,problem", [
    ((2, 1), "poisson2d_sin"),                      # single linear layer
    ((2, 7, 1), "poisson2d_sin"),                   # one hidden layer (first act only)
    ((3, 5, 9, 1), "poisson_norm2"),                # odd widths, K/N tails
    ((5, 33, 17, 65, 1), "heat4"),                  # partial Laplacian, ragged tiles
    ((10, 130, 70, 1), "poisson_harmonic_mixed"),   # > 128 wide, 10d
    ((3, 600, 1), "poisson_norm2"),                 # split-record cluster Jacobi (n = 601, 600)
    ((3, 1100, 1), "poisson_norm2"),                # > 1087: the streaming Jacobi
])
def test_device_matches_oracle_various_shapes(widths, problem):
    if problem == "heat4":
        prob = make_problem("heat", spatial_dim=4)
    elif problem == "poisson_norm2":
        prob = make_problem("poisson_norm2", dim=3)
    else:
        prob = make_problem(problem)
    _oracle_vs_device(widths, prob, 37, 11, 3, momentum=0.5)


def _with_dense_coeffs(prob, seed):
    """The problem with c replaced by a random dense symmetric matrix (the reference's
    own dense-coefficient tests: pkg/tests/test_taylor.py:22-24)."""
    import dataclasses
    from paper_2405_15603_b200.taylor import OperatorCoeffs
    r = np.random.default_rng(seed).standard_normal((prob.dim, prob.dim))
    return dataclasses.replace(prob, coeffs=OperatorCoeffs(0.5 * (r + r.T)))


@pytest.mark.parametrize("widths,problem,chunk", [
    ((2, 1), "poisson2d_sin", None),
    ((2, 7, 1), "poisson2d_sin", None),
    ((5, 33, 17, 65, 1), "heat4", None),             # u_t seed: the rotated seed path
    ((10, 130, 70, 1), "poisson_harmonic_mixed", None),
    ((5, 40, 24, 1), "heat4", 13),                  # chunked interior
])
def test_dense_coefficients_match_oracle(widths, problem, chunk):
    """Non-diagonal operator coefficients (reference taylor.py:72-75): the device works in
    the eigenbasis of c; results must match the oracle's dense contraction."""
    prob = make_problem("heat", spatial_dim=4) if problem == "heat4" else make_problem(problem)
    _oracle_vs_device(widths, _with_dense_coeffs(prob, 7), 37, 11, 3, momentum=0.5, chunk=chunk)


def test_dense_coefficients_taylor_forward_matches_reference():
    from paper_2405_15603_b200.engine import KfacEngine
    from paper_2405_15603_b200.pde import residual_terms
    g = load("dense")
    wl = cfgs.WORKLOADS["dense"]
    prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
    eng = KfacEngine(wl.widths, batch.interior.shape[0], batch.boundary.shape[0], ema=0.95,
                     damping=1e-3, momentum=0.0)
    eng.load_params(params)
    r0, seeds, _ = residual_terms(prob, batch.interior)
    eng.set_batch(batch.interior, r0, seeds, batch.boundary, batch.boundary_targets, prob.coeffs.c)
    u, gu, lu = eng.taylor_forward()
    for key, arr in (("value", u), ("gradient", gu), ("operator", lu)):
        assert compare(g, "taylor/" + key, arr, 1e-12) <= 1e-12, key
    eng.close()


def test_dense_coefficients_with_quadratic_residual_rejected():
    prob = _with_dense_coeffs(make_problem("log_fokker_planck"), 1)
    params = init_params(Architecture((10, 8, 1)), 0)
    batch = sample_batch(prob, 10, 5, 0)
    state = init_train_state(params, OptimizerConfig(kind="kfac", damping=1e-3))
    with pytest.raises(NotImplementedError):
        optimizer_step(state, batch, prob)


def test_chunked_interior_matches_unchunked():
    prob = make_problem("poisson_cos_sum")
    _oracle_vs_device((5, 64, 48, 1), prob, 300, 50, 2, chunk=70)


def test_chunked_mid_size_pairs_match_oracle():
    """Chunked interior with factor pairs on the cluster solver (n = 131, 130) and early
    preconditioning: the per-layer events come from the last chunk's contractions."""
    prob = make_problem("poisson_harmonic_mixed")
    _oracle_vs_device((10, 130, 70, 1), prob, 240, 60, 3, chunk=70)


def test_taylor_forward_matches_oracle():
    from paper_2405_15603_b200.engine import KfacEngine, pack_params
    prob = make_problem("heat", spatial_dim=4)
    params = init_params(Architecture((5, 40, 24, 1)), 11)
    batch = sample_batch(prob, 53, 7, 12)
    eng = KfacEngine((5, 40, 24, 1), 53, 7, ema=0.9, damping=1e-2, momentum=0.0)
    eng.load_params(params)
    from paper_2405_15603_b200.pde import affine_residual_terms
    r0, seeds = affine_residual_terms(prob, batch.interior)
    eng.set_batch(batch.interior, r0, seeds, batch.boundary, batch.boundary_targets,
                  np.diagonal(prob.coeffs.c))
    u, gu, lu = eng.taylor_forward()
    cd = np.diagonal(prob.coeffs.c).copy()
    _, _, (u_r, g_r, l_r) = orc.taylor_forward(params.weights, params.biases, batch.interior, cd)
    assert np.max(np.abs(u - u_r)) <= 1e-13 * max(1, np.max(np.abs(u_r)))
    assert np.max(np.abs(gu - g_r)) <= 1e-13 * max(1, np.max(np.abs(g_r)))
    assert np.max(np.abs(lu - l_r)) <= 1e-12 * max(1, np.max(np.abs(l_r)))
    li, lb = eng.evaluate_losses()
    li_r, lb_r = orc.losses_at(params.weights, params.biases, batch, prob, cd)
    assert abs(li - li_r) <= 1e-12 * abs(li_r) and abs(lb - lb_r) <= 1e-12 * abs(lb_r)


def test_kron_sum_solve_matches_dense():
    from paper_2405_15603_b200.engine import kron_sum_solve_device
    rng = np.random.default_rng(4)
    # small (one-CTA), mid (cluster shared memory) and large (L2-resident cluster Jacobi)
    # routes, and mixed small/large pairs
    for p, q in ((5, 3), (65, 64), (101, 1), (257, 256), (513, 512), (769, 768), (300, 40),
                 (1201, 1100)):
        mk = lambda k: (lambda a: a @ a.T / k + 0.3 * np.eye(k))(rng.standard_normal((k, k)))  # noqa: E731
        a1, a2, b1, b2 = mk(p), mk(p), mk(q), mk(q)
        g = rng.standard_normal((q, p))
        x = kron_sum_solve_device(a1, b1, a2, b2, g)
        if p * q <= 4000:
            dense = np.kron(a1, b1) + np.kron(a2, b2)
            want = np.linalg.solve(dense, g.ravel(order="F")).reshape((q, p), order="F")
        else:
            want = orc.kron_sum_solve(a1, b1, a2, b2, g)
        assert np.max(np.abs(x - want)) <= 1e-10 * np.max(np.abs(want)), (p, q)
        # residual check of B1 X A1 + B2 X A2 = G
        res = b1 @ x @ a1 + b2 @ x @ a2 - g
        assert np.max(np.abs(res)) <= 1e-10 * np.max(np.abs(g))


def test_kron_sum_solve_rejects_indefinite():
    from paper_2405_15603_b200.engine import kron_sum_solve_device
    from paper_2405_15603_b200.linalg import NotPositiveSemidefiniteError
    a = np.eye(3)
    bad = -np.eye(3)
    with pytest.raises(NotPositiveSemidefiniteError):
        kron_sum_solve_device(a, np.eye(2), bad, np.eye(2), np.ones((2, 3)))


def test_damping_only_gives_half_negative_gradient():
    # zero factors, damping 1: Delta = -g / 2 (pkg/tests/test_curvature.py:140-146)
    from paper_2405_15603_b200.engine import kron_sum_solve_device
    g = np.ones((3, 3))
    x = kron_sum_solve_device(np.eye(3), np.eye(3), np.eye(3), np.eye(3), g)
    assert np.allclose(-x, -g / 2.0, atol=1e-12)


@pytest.mark.parametrize("wkey,steps", [("c2", 2), ("c4", 4)])
def test_step_is_bit_deterministic(wkey, steps):
    """Two fresh runs give bitwise-identical parameters (c4: the cluster eigensolver, cold
    and warm-started, and its DSMEM exchange)."""
    wl = cfgs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, 500, 100)
    out = []
    for _ in range(2):
        state = init_train_state(params.copy(), OptimizerConfig(kind="kfac", damping=1e-3, ema=0.95))
        for _ in range(steps):
            optimizer_step(state, batch, prob)
        out.append(np.concatenate([w.ravel() for w in state.params.weights]))
    assert np.array_equal(out[0], out[1])


def test_line_search_error_on_nonfinite_params():
    from paper_2405_15603_b200.optim import LineSearchError
    wl = cfgs.WORKLOADS["c1"]
    prob, params, batch = wl.build(0, 50, 20)
    params.weights[1][0, 0] = np.nan
    state = init_train_state(params, OptimizerConfig(kind="kfac", damping=1e-3, ema=0.95))
    with pytest.raises((LineSearchError, FloatingPointError, ValueError)):
        optimizer_step(state, batch, prob)


def test_unsupported_residual_rejected():
    # a residual quadratic in u (seed dr/du depends on u) is outside the device family
    from paper_2405_15603_b200.pde import PdeProblem
    base = make_problem("poisson2d_sin")
    prob = PdeProblem(**{**base.__dict__,
                         "residual": lambda x, u, g, op: u * u - op,
                         "residual_grads": lambda x, u, g, op: (2 * u, np.zeros_like(g), -np.ones_like(u))})
    params = init_params(Architecture((2, 8, 1)), 0)
    batch = sample_batch(prob, 10, 5, 0)
    state = init_train_state(params, OptimizerConfig(kind="kfac", damping=1e-3))
    with pytest.raises(NotImplementedError):
        optimizer_step(state, batch, prob)


@pytest.mark.parametrize("name", STAR_NAMES + STAR10 + STAR_FULL)
def test_kfac_star_steps_match_reference_golden(name):
    """KFAC* on the device (kp_kfac_star_step): exact Gramian-vector products via JVP +
    weighted reverse contraction vs the reference's Jacobian-row route."""
    g = load(name)
    wl = cfgs.WORKLOADS[WL_OF[name]]
    prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
    cfg = OptimizerConfig(kind="kfac_star", damping=float(g["damping"]), ema=float(g["ema"]),
                          momentum=float(g["momentum"]))
    state = init_train_state(params, cfg)
    t = 1
    while f"s{t}/alpha" in g:
        info = optimizer_step(state, batch, prob)
        p = f"s{t}/"
        tol = 1e-10 if t == 1 else 1e-8
        a_ref, m_ref = float(g[p + "alpha"]), float(g[p + "mu"])
        assert abs(info.alpha - a_ref) <= tol * abs(a_ref), (info.alpha, a_ref)
        assert abs(info.mu - m_ref) <= tol * max(abs(m_ref), 1.0), (info.mu, m_ref)
        for key, val in (("loss_interior", info.loss_interior), ("loss_boundary", info.loss_boundary)):
            ref = float(g[p + key])
            assert abs(val - ref) <= tol * abs(ref), (key, val, ref)
        if not has(g, p + "theta"):  # ten-step runs record arrays at steps 1 and 10 only
            t += 1
            continue
        eng = state._engine
        widths = eng.widths
        assert compare(g, p + "delta", _device_mats_to_vec(eng.delta.cpu().numpy(), widths), tol) <= tol
        assert compare(g, p + "theta", _theta_colstack(state.params), tol) <= tol
        assert compare(g, p + "prev_update", mats_to_vec(state.prev_update), tol) <= tol
        t += 1
    assert t > (10 if name in STAR10 else 1)


def test_kfac_star_chunked_matches_single_chunk():
    """Multi-chunk KFAC* recomputes the interior states for the Gramian products."""
    from paper_2405_15603_b200.engine import KfacEngine
    from paper_2405_15603_b200.pde import affine_residual_terms
    wl = cfgs.WORKLOADS["c2"]
    prob, params, batch = wl.build(0, 240, 60)
    r0, seeds = affine_residual_terms(prob, batch.interior)
    out = []
    for chunk in (None, 70):
        eng = KfacEngine(wl.widths, 240, 60, ema=0.95, damping=1e-3, momentum=0.0, chunk=chunk)
        eng.set_batch(batch.interior, r0, seeds, batch.boundary, batch.boundary_targets,
                      np.diagonal(prob.coeffs.c))
        eng.load_params(params)
        eng.init_factors(True)
        res = [eng.star_step() for _ in range(2)]
        out.append((res, eng.theta_numpy()))
    (r1, t1), (r2, t2) = out
    for a, b in zip(r1, r2):
        assert abs(a[0] - b[0]) <= 1e-10 * abs(b[0]) and abs(a[1] - b[1]) <= 1e-10 * max(abs(b[1]), 1)
    assert np.max(np.abs(t1 - t2)) <= 1e-10 * np.max(np.abs(t2))


@pytest.mark.parametrize("star", [False, True], ids=["kfac", "kfac_star"])
def test_graph_replay_is_bit_identical(star):
    """kp_kfac_step_graphed (whole step replayed from a captured CUDA graph) == the plain
    call, bit for bit, over several steps (the graph is captured on the second step)."""
    from paper_2405_15603_b200.dist import make_rank_engine
    wl = cfgs.WORKLOADS["c3"]
    prob, params, batch = wl.build(0, 300, 80)
    runs = []
    for graph in (False, True):
        eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                               momentum=0.3)
        eng.use_graph = graph
        eng.load_params(params)
        eng.init_factors(True)
        fn = eng.star_step if star else eng.step
        infos = [fn() for _ in range(4)]
        runs.append((infos, eng.theta_numpy(), eng.factor_lists()))
        eng.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    for fa, fb in zip(runs[0][2], runs[1][2]):
        for a, b in zip(fa, fb):
            assert np.array_equal(a, b)


def test_ten_steps_match_oracle_warm_started_eigensolver():
    """Ten steps (step 10 within 1e-8): from step 2 on, the on-device
    eigensolver starts from the previous step's generalised eigenvectors."""
    prob = make_problem("poisson2d_sin")
    worst = _oracle_vs_device((2, 24, 24, 16, 1), prob, 120, 40, 10, momentum=0.3)
    assert worst <= 1e-8


def test_line_search_phase_is_bit_reproducible():
    """The line-search phase re-run on one state gives bitwise-identical candidate sums.
    (Regression: the fused layer's C staging used to overwrite its live mbarriers, which
    produced sporadic NaN rows at c5 scale.)"""
    from paper_2405_15603_b200.dist import make_rank_engine
    wl = cfgs.WORKLOADS["c5"]
    prob, params, batch = wl.build(0, 4096, 1365)
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                           momentum=wl.momentum)
    eng.load_params(params)
    eng.init_factors(True)
    eng.phase("accumulate")
    eng.phase("precondition")
    ref = None
    for _ in range(6):
        eng.phase("linesearch")
        torch.cuda.synchronize()
        ls = eng.linesearch_buffer().clone()
        assert torch.isfinite(ls).all()
        if ref is None:
            ref = ls
        assert torch.equal(ls, ref)
    eng.close()


@pytest.mark.parametrize("n_int,n_bnd", [(1, 1), (2, 1), (5, 3)])
def test_tiny_batches_match_oracle(n_int, n_bnd):
    """Ragged edge: one or a few collocation points (single-sample tiles, partial splits)."""
    _oracle_vs_device((2, 16, 8, 1), make_problem("poisson2d_sin"), n_int, n_bnd, 2)
    _oracle_vs_device((5, 64, 64, 48, 48, 1), make_problem("heat", spatial_dim=4), n_int, n_bnd, 2)


@pytest.mark.parametrize("cluster", ["8", "0"], ids=["cluster8", "cusolver"])
def test_mid_size_pairs_other_routes_match_reference(cluster):
    """c4's mid-size factor pairs through the 8-CTA-cluster solver and (KP_MID_CLUSTER=0)
    through the L2-resident large-pair solver match the reference goldens too
    (KP_MID_CLUSTER is read once per process, hence the subprocess)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, KP_MID_CLUSTER=cluster)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "test_kfac_steps_match_reference_golden and c4"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-500:]


@pytest.mark.parametrize("env", [{"KP_LARGE_SPLIT": "0"}, {"KP_LARGE_ACCV": "1", "KP_MID_ACCV": "1"},
                                 {"KP_OZAKI": "1"}])
def test_c5_alternative_solver_routes_match_reference(env):
    """c5 at the BASELINE size through the other routes — the all-L2 Jacobi for the 768 / 769
    pairs instead of the split-record one, both cluster Jacobis accumulating V (T^T = V^T L^-1)
    instead of T' = K^-T U, and the line-search layers on the INT8 tensor cores (Ozaki
    emulation of FP64) — against the reference's goldens (the switches are read once per
    process, hence the subprocess)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "test_kfac_steps_match_reference_golden and c5_full3"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-500:]
