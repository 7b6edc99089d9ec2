"""The reference-side plug-in (option B) on the reference's own harness.

``paper_2405_15603_b200.plugin.install()`` replaces ``_STEP_FNS["kfac"]`` /
``["kfac_star"]`` of the reference (src/optim.py:387-393).  These CPU tests run the
UNMODIFIED reference ``run_training`` (src/harness.py:236-323, which binds
``init_train_state`` / ``optimizer_step`` at import, :22-28) once stock and once through
the plug-in, with the device engine replaced by the oracle-backed CPU stand-in
(tests/cpu_step_engine.py), and require the same log and checkpoint; and they check the
in-place ``TrainState`` mutations and the error classes the reference's callers see.
The same adapter on the GPU (real engine) is tests/test_gpu_plugin.py.

Needs the reference sources (``/root/reference``, build container only); skipped elsewhere.
"""

import json
import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"
if not os.path.isdir(os.path.join(REF_SRC, "pinnopt")):
    pytest.skip("reference sources not present", allow_module_level=True)
if REF_SRC not in sys.path:
    sys.path.append(REF_SRC)

from cpu_step_engine import CpuStepEngine  # noqa: E402
from pinnopt import network as ref_network  # noqa: E402  (the reference)
from pinnopt import optim as ref_optim  # noqa: E402
from pinnopt import pde as ref_pde  # noqa: E402
from pinnopt.harness import RunConfig, _stream_seed, load_checkpoint, run_training  # noqa: E402

from paper_2405_15603_b200 import optim as b200_optim  # noqa: E402
from paper_2405_15603_b200 import plugin  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = json.load(open(os.path.join(HERE, "golden", "training_logs.json")))


@pytest.fixture
def patched(monkeypatch):
    monkeypatch.setattr(b200_optim, "ENGINE_FACTORY", CpuStepEngine)
    CpuStepEngine.force_code = None
    saved = plugin.install(ref_optim)
    yield
    plugin.uninstall(saved, ref_optim)
    CpuStepEngine.force_code = None


def _run(kw, out_dir):
    log = run_training(RunConfig(output_dir=str(out_dir), **kw))
    rows = np.array([[r[0]] + list(r[2:]) for r in log.rows], dtype=np.float64)
    params, _ = load_checkpoint(str(out_dir / "checkpoint.json"))
    return rows, log.diverged, params


@pytest.mark.parametrize("name", ["train_kfac_poisson2d", "train_kfac_star_heat"])
def test_reference_run_training_through_plugin_matches_stock(name, tmp_path, monkeypatch):
    kw = CONFIGS[name]["config"]
    stock_rows, stock_div, stock_params = _run(kw, tmp_path / "stock")
    monkeypatch.setattr(b200_optim, "ENGINE_FACTORY", CpuStepEngine)
    saved = plugin.install(ref_optim)
    try:
        n0 = CpuStepEngine.instances
        rows, div, params = _run(kw, tmp_path / "plugin")
        assert CpuStepEngine.instances == n0 + 1  # one engine for the whole run (resampling reuses it)
    finally:
        plugin.uninstall(saved, ref_optim)
    assert ref_optim._STEP_FNS["kfac"] is ref_optim.kfac_step
    assert div == stock_div and rows.shape == stock_rows.shape
    assert np.array_equal(rows[:, 0], stock_rows[:, 0])
    if kw["optimizer"] == "kfac":
        assert np.array_equal(rows[:, 5], stock_rows[:, 5])  # line-search alpha, exact
    np.testing.assert_allclose(rows[:, 1:], stock_rows[:, 1:], rtol=1e-10, atol=1e-14)
    for w, w_ref in zip(params.weights + params.biases, stock_params.weights + stock_params.biases):
        np.testing.assert_allclose(w, w_ref, rtol=0, atol=1e-10 * np.max(np.abs(w_ref)))


def _inputs(kind, momentum=0.5, n=120, nb=40):
    prob = ref_pde.make_problem("poisson2d_sin")
    params = ref_network.init_params(ref_network.Architecture((2, 12, 10, 1)), _stream_seed(0, 0))
    batch = ref_pde.sample_batch(prob, n, nb, _stream_seed(0, 1, 0))
    cfg = ref_optim.OptimizerConfig(kind=kind, damping=1e-3, ema=0.9, momentum=momentum)
    return prob, params, batch, cfg


def _assert_states_equal(a, b, tol=1e-11):
    assert a.step == b.step
    for x, y in zip(a.params.weights + a.params.biases, b.params.weights + b.params.biases):
        np.testing.assert_allclose(x, y, rtol=tol, atol=1e-14)
    for x, y in zip(a.prev_update, b.prev_update):
        np.testing.assert_allclose(x, y, rtol=tol, atol=1e-14)
    for f in ("a_interior", "b_interior", "a_boundary", "b_boundary"):
        for x, y in zip(getattr(a.kfac, f), getattr(b.kfac, f)):
            np.testing.assert_allclose(x, y, rtol=tol, atol=1e-14)


@pytest.mark.parametrize("kind", ["kfac", "kfac_star"])
def test_plugin_mutates_reference_train_state_like_stock(kind, patched):
    prob, params, batch, cfg = _inputs(kind)
    # stock run on a copy of the same inputs
    stock_fns = {"kfac": ref_optim.kfac_step, "kfac_star": ref_optim.kfac_star_step}
    stock = ref_optim.init_train_state(params, cfg)
    mine = ref_optim.init_train_state(params, cfg)
    kf_obj, a_list = mine.kfac, mine.kfac.a_interior

    def both(fn):
        for st, use_stock in ((stock, True), (mine, False)):
            cur = ref_optim._STEP_FNS[kind]
            if use_stock:
                ref_optim._STEP_FNS[kind] = stock_fns[kind]
            try:
                fn(st)
            finally:
                ref_optim._STEP_FNS[kind] = cur

    for _ in range(3):
        both(lambda st: ref_optim.optimizer_step(st, batch, prob))
    assert type(mine.params) is ref_network.Parameters
    assert mine.kfac is kf_obj and mine.kfac.a_interior is a_list  # entries replaced in place
    _assert_states_equal(mine, stock)

    # host-side edits between steps are honoured: new params object, an edited factor,
    # a replaced prev_update list, a changed damping
    def edit(st):
        st.params = ref_network.add_scaled(st.params, st.prev_update, 0.5)
        st.kfac.b_interior[1] = st.kfac.b_interior[1] * 1.5
        st.kfac.a_boundary[0][0, 0] += 0.25  # in-place edit of an entry
        st.prev_update = [0.5 * m for m in st.prev_update]
        st.kfac.damping = 2e-3

    both(edit)
    for _ in range(2):
        both(lambda st: ref_optim.optimizer_step(st, batch, prob))
    _assert_states_equal(mine, stock, tol=1e-10)

    # a whole new KfacState object (what init_train_state builds) is adopted too
    def reset(st):
        st.kfac = ref_optim.curvature.init_kfac_state(st.params, 0.8, 1e-3, "zero")

    both(reset)
    both(lambda st: ref_optim.optimizer_step(st, batch, prob))
    _assert_states_equal(mine, stock, tol=1e-10)


def test_plugin_raises_reference_error_classes(patched, tmp_path):
    prob, params, batch, cfg = _inputs("kfac")
    st = ref_optim.init_train_state(params, cfg)
    CpuStepEngine.force_code = 3
    with pytest.raises(ref_optim.LineSearchError):
        ref_optim.optimizer_step(st, batch, prob)
    assert st.step == 0
    CpuStepEngine.force_code = 2
    from pinnopt.linalg import NotPositiveSemidefiniteError

    with pytest.raises(NotPositiveSemidefiniteError):
        ref_optim.optimizer_step(st, batch, prob)
    # the reference harness catches the reference class and marks the run diverged
    CpuStepEngine.force_code = 3
    kw = dict(CONFIGS["train_kfac_poisson2d"]["config"], max_steps=3)
    log = run_training(RunConfig(output_dir=str(tmp_path), **kw))
    assert log.diverged and len(log.rows) == 1


def test_plugin_nonfinite_params_raise_what_stock_raises(patched):
    prob, params, batch, cfg = _inputs("kfac")
    raised = []
    for stock in (True, False):
        st = ref_optim.init_train_state(params, cfg)
        bad = ref_network.Parameters([w.copy() for w in params.weights],
                                     [b.copy() for b in params.biases], params.activation)
        bad.weights[-1][0, 0] = 1e308  # the output weight: the candidates overflow
        st.params = bad
        cur = ref_optim._STEP_FNS["kfac"]
        if stock:
            ref_optim._STEP_FNS["kfac"] = ref_optim.kfac_step
        try:
            ref_optim.optimizer_step(st, batch, prob)
            raised.append(None)
        except Exception as exc:  # noqa: BLE001 - the class is what is compared
            raised.append(type(exc))
        finally:
            ref_optim._STEP_FNS["kfac"] = cur
    assert raised[0] is not None and raised[0] is raised[1], raised
