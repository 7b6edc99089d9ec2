"""bench.py's N > 1 path end to end under torchrun (dist init, sharded stepper with distributed
solves, barriers, max-over-ranks timing, the sharded e2e leg), on the one GPU of a test box:
every rank runs on that GPU and the collectives go over gloo (KP_BENCH_DIST_BACKEND=gloo;
host-side, no kernel waits on another rank).  The losses after the timed steps must equal the
N = 1 run on the same global batch to summation-order roundoff."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _line(cmd, env):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return lines[0]


@pytest.mark.parametrize("workload,world,optimizer,scaling", [("c4", 2, "kfac", "weak"),
                                                               ("c3", 4, "kfac_star", "strong")])
def test_bench_sharded_matches_single_gpu(workload, world, optimizer, scaling):
    """weak: launched under torchrun, --n-interior per rank.  strong: plain ``bench.py --gpus
    N`` (bench.py re-executes itself under torch.distributed.run), --n-total split across
    the ranks."""
    n_loc, nb_loc = 256, 80
    common = ["--workload", workload, "--optimizer", optimizer, "--steps", "2", "--warmup", "3",
              "--no-cpu"]
    env = dict(os.environ, KP_BENCH_DIST_BACKEND="gloo")
    if scaling == "weak":
        multi = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                       "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                       "--master-port", str(_port()), "bench.py", "--gpus", str(world),
                       "--scaling", "weak", "--n-interior", str(n_loc), "--n-boundary",
                       str(nb_loc), *common], env)
    else:
        multi = _line([sys.executable, "bench.py", "--gpus", str(world), "--n-total",
                       str(n_loc * world), *common], env)
    env.pop("KP_BENCH_DIST_BACKEND")
    single = _line([sys.executable, "bench.py", "--n-interior", str(n_loc * world),
                    "--n-boundary", str(nb_loc * world if scaling == "weak" else n_loc * world // 3),
                    *common], env)
    assert multi["n_gpus"] == world and single["n_gpus"] == 1 and multi["scaling"] == scaling
    assert multi["config"]["n_interior_total"] == single["config"]["n_interior_total"]
    assert multi["e2e"] is not None and multi["gpu_launches"] > 0
    for a, b in zip(multi["losses_last_step"], single["losses_last_step"]):
        assert abs(a - b) <= 1e-10 * abs(b), (multi["losses_last_step"], single["losses_last_step"])
