"""Bit-reproducibility across runs and graph replay with the cluster eigensolver's side streams
busy next to main-stream work: KFAC* issues G·prev before the preconditioner, so the mid-size
eigenproblems (warm-started, on side streams) overlap long GEMMs.  A missing ordering of the
warm-start flags' reset against those streams once showed up here as runs that differed from
step 2 on (tools/star_repeat_check.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wkey,n", [("c4", 3000), ("c5", 2048)])  # sizes where it showed
def test_star_steps_reproducible_plain_and_graphed(wkey, n):
    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import make_rank_engine
    wl = configs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, n, max(1, n // 3))
    runs = []
    for graph in (False, False, True):
        eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                               momentum=wl.momentum)
        eng.use_graph = graph
        eng.load_params(params)
        eng.init_factors(True)
        outs = [tuple(eng.star_step()) for _ in range(6)]
        runs.append((outs, eng.theta_numpy()))
        eng.close()
    for outs, theta in runs[1:]:
        assert outs == runs[0][0]
        assert np.array_equal(theta, runs[0][1])
