"""bench.py's reference arm (``--impl reference``) on CPU: the JSON line the driver parses.

The reference arm times the oracle (the CPU restatement of the reference step) on the host
cores; these tests run it on a tiny sample so the keys, the optimizer switch and the
one-line-from-rank-0 rule under torchrun are checked without a GPU.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = ["--workload", "c1", "--steps", "1", "--warmup", "0", "--cpu-points", "8"]


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("optimizer", ["kfac", "kfac_star"])
def test_reference_arm_line(optimizer):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--optimizer", optimizer,
                        *TINY], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    ln = lines[0]
    assert ln["impl"] == "reference"
    assert ln["metric"] == "collocation_pts_per_s" and ln["higher_is_better"] is True
    assert ln["value"] > 0 and ln["steps"] == 1 and ln["warmup"] == 0
    assert ln["config"]["optimizer"] == optimizer
    cb = ln["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == ln["value"]
    assert ("kfac_star_step" in cb["sample"]) == (optimizer == "kfac_star")
    assert ln["e2e"] == {"value": ln["value"], "unit": ln["unit"], "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}


def test_reference_arm_under_torchrun_prints_once():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "0", "bench.py", "--gpus", "2",
           "--impl", "reference", *TINY]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    # torchrun exports OMP_NUM_THREADS=1; the reference arm still uses every host core
    assert lines[0]["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_reference_arm_describes_the_gpu_arms_batch():
    """The reference arm times bounded samples and reports the fitted step time at the GPU
    arm's own N (BASELINE c5: 16384 on one GPU, 65536 global under strong scaling)."""
    for extra, n in (([], 16384), (["--gpus", "4"], 65536), (["--gpus", "2", "--scaling", "weak"], 32768)):
        r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", *TINY, *extra],
                           cwd=ROOT, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        ln = _json_lines(r.stdout)[0]
        cb = ln["cpu_baseline"]
        assert ln["extrapolated"] and cb["extrapolated"] and cb["same_config"]
        assert ln["config"]["n_interior_total"] == n == cb["n_interior"]
        assert [s["n_interior"] for s in cb["samples"]] == [4, 12]
        assert abs(ln["value"] - n / (cb["fit"]["fixed_s"] + cb["fit"]["per_point_s"] * n)) <= 1e-9 * ln["value"]


def test_fixed_plus_per_point_fit():
    sys.path.insert(0, ROOT)
    import bench

    a, b = bench.fit_fixed_per_point([(64, 1.0 + 64 * 0.01), (192, 1.0 + 192 * 0.01),
                                      (64, 1.0 + 64 * 0.01)])
    assert abs(a - 1.0) < 1e-12 and abs(b - 0.01) < 1e-14
    a, b = bench.fit_fixed_per_point([(64, 2.0), (192, 1.0)])  # noisy: pure per-point rate
    assert a == 0.0 and abs(b - 3.0 / 256) < 1e-15
