"""Golden training logs from the REFERENCE harness (build container only).

    python tests/golden/make_golden_training.py

Runs the reference ``run_training`` (src/harness.py:236-323) on small configs and stores
the log rows (minus the wall-time column) for tests/test_gpu_training.py.
"""
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from pinnopt.harness import RunConfig, run_training  # noqa: E402  (the reference)

CONFIGS = {
    "train_kfac_poisson2d": dict(problem="poisson2d_sin", widths=[2, 16, 16, 1], optimizer="kfac",
                                 damping=1e-3, ema=0.95, momentum=0.5, n_interior=200,
                                 n_boundary=50, max_steps=12, eval_every=3, n_eval_points=500,
                                 resample_every=5, seed=0),
    "train_kfac_star_heat": dict(problem="heat", problem_params={"spatial_dim": 1},
                                 widths=[2, 16, 16, 1], optimizer="kfac_star", damping=1e-3,
                                 ema=0.95, n_interior=200, n_boundary=60, max_steps=8,
                                 eval_every=2, n_eval_points=400, resample_every=4, seed=1),
}


def main():
    out = {}
    for name, kw in CONFIGS.items():
        with tempfile.TemporaryDirectory() as d:
            cfg = RunConfig(output_dir=d, **kw)
            log = run_training(cfg)
            rows = np.array([[r[0]] + list(r[2:]) for r in log.rows], dtype=np.float64)
            out[name] = {"config": kw, "rows": rows.tolist(), "diverged": log.diverged}
            print(name, rows[-1])
    with open(os.path.join(HERE, "training_logs.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
