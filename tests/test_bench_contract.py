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
