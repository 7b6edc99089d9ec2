"""Host-side logic that runs without a GPU: the C-ABI library's exports, config
validation, the affine-residual split, parameter packing and shard bounds."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2405_15603_b200 import _capi
from paper_2405_15603_b200.dist import shard_bounds
from paper_2405_15603_b200.engine import pack_mats, pack_params, unpack_factors, unpack_mats
from paper_2405_15603_b200.network import Architecture, init_params
from paper_2405_15603_b200.optim import OptimizerConfig, init_train_state
from paper_2405_15603_b200.pde import affine_residual_terms, make_problem, sample_batch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "kfac_pinn_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(kp_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(syms) == sorted(_capi.EXPORTED)


def test_size_queries_without_gpu():
    lib = _capi.load()
    net = _capi.make_net((100, 768, 768, 512, 512, 1))
    assert lib.kp_param_count(C.byref(net)) == 1325057  # PAPER.md D for the 100d net
    assert lib.kp_factor_count(C.byref(net), 0) == 101 ** 2 + 2 * 769 ** 2 + 2 * 513 ** 2
    assert lib.kp_factor_count(C.byref(net), 1) == 2 * 768 ** 2 + 2 * 512 ** 2 + 1
    bad = _capi.make_net((3, 4, 2))
    assert lib.kp_param_count(C.byref(bad)) == -1
    assert lib.kp_status_string(2).decode().startswith("matrix not positive")


def test_ctypes_struct_layout_matches_header():
    assert C.sizeof(_capi.kp_net) == 4 * 18
    assert _capi.kp_problem.n_interior.offset == 72
    assert C.sizeof(_capi.kp_problem) == 104
    assert C.sizeof(_capi.kp_kfac_config) == 56
    assert C.sizeof(_capi.kp_step_out) == 5 * 8


def test_config_validation_mirrors_reference():
    # pkg/tests/test_optim.py:30-44
    for kw in ({"kind": "newton"}, {"kind": "kfac", "damping": 0.0}, {"kind": "sgd", "lr": 0.0},
               {"kind": "kfac", "ema": -0.1}, {"kind": "kfac", "ema": 1.0},
               {"kind": "sgd", "lr": 0.1, "momentum": -1.0},
               {"kind": "kfac", "line_search_min_exp": 1, "line_search_max_exp": 0}):
        with pytest.raises(ValueError):
            OptimizerConfig(**kw)
    grid = OptimizerConfig(kind="kfac").line_search_grid()
    assert len(grid) == 31 and grid[0] == 2.0 ** -30 and grid[-1] == 1.0


def test_init_train_state_shapes():
    p = init_params(Architecture((2, 5, 3, 1)), 0)
    st = init_train_state(p, OptimizerConfig(kind="kfac", init_mode="zero"))
    assert [m.shape for m in st.prev_update] == [(5, 3), (3, 6), (1, 4)]
    assert [a.shape for a in st.kfac.a_interior] == [(3, 3), (6, 6), (4, 4)]
    assert not np.any(st.kfac.b_boundary[1])
    st = init_train_state(p, OptimizerConfig(kind="kfac"))
    assert np.array_equal(st.kfac.a_boundary[0], np.eye(3))


@pytest.mark.parametrize("name,kw", [("poisson2d_sin", {}), ("poisson_cos_sum", {"dim": 10}),
                                     ("heat", {"spatial_dim": 4, "solution": "sine_product"}),
                                     ("poisson_norm2", {"dim": 100, "divisor": 100.0}),
                                     ("poisson_harmonic_mixed", {})])
def test_affine_residual_split_reproduces_residual(name, kw):
    prob = make_problem(name, **kw)
    b = sample_batch(prob, 64, 8, 1)
    r0, seeds = affine_residual_terms(prob, b.interior)
    rng = np.random.default_rng(0)
    n, d = b.interior.shape
    u, g, op = rng.standard_normal(n), rng.standard_normal((n, d)), rng.standard_normal(n)
    want = prob.residual(b.interior, u, g, op)
    got = r0 + seeds[:, 0] * u + np.einsum("ni,ni->n", seeds[:, 1:d + 1], g) + seeds[:, d + 1] * op
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def test_nonaffine_residual_is_rejected():
    prob = make_problem("log_fokker_planck")
    b = sample_batch(prob, 16, 4, 0)
    with pytest.raises(NotImplementedError):
        affine_residual_terms(prob, b.interior)


def test_log_fokker_planck_is_quadratic_in_grad():
    # pde.py:253-263: r = u_t - s/2 - x.grad_x u / 2 - |grad_x u|^2 - Lu
    from paper_2405_15603_b200.pde import residual_terms
    prob = make_problem("log_fokker_planck")
    b = sample_batch(prob, 32, 8, 2)
    r0, seeds, quad = residual_terms(prob, b.interior)
    assert np.allclose(r0, -4.5)
    assert np.allclose(quad[:, 0], 0.0) and np.allclose(quad[:, 1:], -1.0)
    assert np.allclose(seeds[:, 1], 1.0) and np.allclose(seeds[:, 2:11], -0.5 * b.interior[:, 1:])
    assert np.allclose(seeds[:, 11], -1.0)
    # affine problems keep quad = None
    assert residual_terms(make_problem("poisson2d_sin"), b.interior[:, :2])[2] is None


def test_heat_sine_product_solution_solves_pde():
    # u = exp(-pi^2 t) prod sin(pi x_i): u_t = -pi^2 u, 1/4 Lap_x u = 1/4 * (-4 pi^2) u
    prob = make_problem("heat", spatial_dim=4, solution="sine_product")
    x = np.random.default_rng(0).uniform(size=(5, 5))
    u = prob.true_solution(x)
    ut = -np.pi ** 2 * u
    lap = -4 * np.pi ** 2 * u
    assert np.allclose(prob.residual(x, u, np.column_stack([ut, np.zeros((5, 4))]), lap), 0.0)


def test_packing_roundtrip():
    p = init_params(Architecture((3, 4, 2, 1)), 0)
    v = pack_params(p)
    mats = unpack_mats(v, (3, 4, 2, 1))
    for m, w, b in zip(mats, p.weights, p.biases):
        assert np.array_equal(m[:, :-1], w) and np.array_equal(m[:, -1], b)
    assert np.array_equal(pack_mats(mats), v)
    f = unpack_factors(np.arange(4 + 9, dtype=float), [2, 3])
    assert f[1].shape == (3, 3) and f[1][0, 0] == 4.0


@pytest.mark.parametrize("n,world", [(3000, 8), (7, 2), (65536, 3), (5, 5)])
def test_shard_bounds_cover_exactly(n, world):
    spans = [shard_bounds(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, _) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_run_config_mirrors_reference_validation():
    from paper_2405_15603_b200.harness import RunConfig
    cfg = RunConfig(problem="heat", widths=[2, 8, 1], optimizer="kfac")
    assert cfg.resample_every == 100 and cfg.to_dict()["optimizer"] == "kfac"
    for bad in ({"n_interior": 0}, {"eval_every": 0}, {"resample_every": -1}, {"optimizer": "lbfgs"}):
        with pytest.raises(ValueError):
            RunConfig(**{**dict(problem="heat", widths=[2, 8, 1], optimizer="kfac"), **bad})
    with pytest.raises(ValueError):
        RunConfig.from_dict({"problem": "heat", "widths": [2, 1], "optimizer": "kfac", "bogus": 1})


def test_checkpoint_roundtrip(tmp_path):
    from paper_2405_15603_b200.harness import load_checkpoint, save_checkpoint
    p = init_params(Architecture((3, 4, 1)), 2)
    save_checkpoint(str(tmp_path / "c.json"), p)
    q, conf = load_checkpoint(str(tmp_path / "c.json"))
    assert conf is None
    for a, b in zip(p.weights + p.biases, q.weights + q.biases):
        assert np.array_equal(a, b)


def test_coeff_spectrum_diagonal_and_dense():
    from paper_2405_15603_b200.taylor import coeff_spectrum
    lam, rot = coeff_spectrum(np.diag([0.0, 1.0, 2.0]))
    assert rot is None and np.array_equal(lam, [0.0, 1.0, 2.0])
    lam, rot = coeff_spectrum(np.array([1.0, 3.0]))  # 1-D = the diagonal
    assert rot is None and np.array_equal(lam, [1.0, 3.0])
    r = np.random.default_rng(0).standard_normal((5, 5))
    c = 0.5 * (r + r.T)
    lam, rot = coeff_spectrum(c)
    assert np.allclose(rot @ np.diag(lam) @ rot.T, c, atol=1e-13)
    assert np.allclose(rot.T @ rot, np.eye(5), atol=1e-13)
    # the rotated diagonal quadratic form equals the dense one (the device identity)
    g = np.random.default_rng(1).standard_normal((7, 5))
    gp = g @ rot
    assert np.allclose(np.einsum("ni,ij,nj->n", g, c, g), (gp * gp) @ lam, atol=1e-12)
    with pytest.raises(ValueError):
        coeff_spectrum(np.zeros((2, 3)))


def test_residual_terms_cache_tracks_batch_contents():
    from paper_2405_15603_b200.pde import residual_terms
    prob = make_problem("poisson_cos_sum")
    x = sample_batch(prob, 40, 8, 3).interior.copy()
    r0a, sa, _ = residual_terms(prob, x)
    r0b, sb, _ = residual_terms(prob, x.copy())        # same contents: cached
    assert r0b is r0a and sb is sa and not r0a.flags.writeable
    x[0, 0] += 0.25                                     # in-place edit: recomputed
    r0c, _, _ = residual_terms(prob, x)
    assert r0c is not r0a and r0c[0] != r0a[0] and np.array_equal(r0c[1:], r0a[1:])
    other = make_problem("poisson_cos_sum")             # another problem object: recomputed
    assert residual_terms(other, x)[0] is not r0c
