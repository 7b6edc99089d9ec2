"""The c5 line search with its hidden layers on the INT8 tensor cores (CRT construction,
csrc/kp_crt.cu, the default) against the same steps with every layer on the FP64 DMMA kernel
(KP_CRT=0): every candidate loss within 1e-12 relative, identical step sizes, and not
bit-identical (so the emulated path did run).  Every CTA organisation of the kernel is
covered: independent CTAs (the default), CTA pairs sharing one cta_group::2 MMA, and 2 x 2
multicast clusters (KP_CRT_CLUSTER = 1 / 2 / 4)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _run(tmp_path, crt, n, steps, cluster=1):
    out = tmp_path / f"crt{crt}_{n}_{cluster}.json"
    env = dict(os.environ, KP_CRT=str(crt), KP_CRT_CLUSTER=str(cluster))
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "crt_check.py"), "--workload", "c5",
                    "--n-interior", str(n), "--steps", str(steps), "--out", str(out)],
                   env=env, check=True, cwd=ROOT, timeout=900)
    return json.load(open(out))


@pytest.mark.parametrize("n,cluster", [(1000, 1), (3001, 1), (1000, 2), (1001, 4)])
def test_c5_linesearch_crt_matches_fp64_layers(tmp_path, n, cluster):
    a = _run(tmp_path, 0, n, 3)
    b = _run(tmp_path, 1, n, 3, cluster)
    worst = 0.0
    for sa, sb in zip(a["steps"], b["steps"]):
        assert sa["code"] == sb["code"] == 0
        assert sa["alpha"] == sb["alpha"]
        la, lb = np.asarray(sa["ls"]), np.asarray(sb["ls"])
        fin = np.isfinite(la)
        assert np.array_equal(fin, np.isfinite(lb))
        worst = max(worst, float(np.max(np.abs(la[fin] - lb[fin]) / np.abs(la[fin]))))
    assert 0.0 < worst < 1e-12, worst
