"""Training-loop integration: run_training on the B200 vs the
reference harness's own logs (tests/golden/training_logs.json, made by running the
reference run_training, tests/golden/make_golden_training.py)."""

import csv
import json
import os

import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("name", ["train_kfac_poisson2d", "train_kfac_star_heat"])
def test_run_training_matches_reference_log(name, tmp_path):
    from paper_2405_15603_b200.harness import RunConfig, load_checkpoint, run_training

    gold = json.load(open(os.path.join(HERE, "golden", "training_logs.json")))[name]
    cfg = RunConfig(output_dir=str(tmp_path), **gold["config"])
    log = run_training(cfg)
    ref = np.array(gold["rows"])
    got = np.array([[r[0]] + list(r[2:]) for r in log.rows])
    assert got.shape == ref.shape and log.diverged == gold["diverged"]
    assert np.array_equal(got[:, 0], ref[:, 0])                      # recorded steps
    if cfg.optimizer == "kfac":
        assert np.array_equal(got[:, 5], ref[:, 5])                  # line-search alpha (exact)
    else:
        assert np.allclose(got[:, 5:7], ref[:, 5:7], rtol=1e-8, atol=1e-12)
    assert np.allclose(got[:, 1:5], ref[:, 1:5], rtol=1e-8, atol=0)  # losses, total, L2 error
    # the reference's file formats
    rows = list(csv.reader(l for l in open(tmp_path / "log.csv") if not l.startswith("#")))
    assert rows[0] == ["step", "wall_time_s", "loss_interior", "loss_boundary", "loss_total",
                       "l2_rel_error", "alpha", "mu"]
    assert len(rows) - 1 == len(ref)
    params, conf = load_checkpoint(str(tmp_path / "checkpoint.json"))
    assert conf["optimizer"] == cfg.optimizer and params.n_linear == len(cfg.widths) - 1
