"""The multi-GPU step's device glue under a real NCCL communicator (world size 1 on the one
GPU this build has): the sharded step (phases + NCCL all-reduces of the reduce and
line-search / Gramian buffers, dist.ShardedKfacStep) must reproduce the single-call step
bit for bit.  The rank-count-dependent orchestration is covered under gloo
(tests/test_dist_gloo.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("star", [False, True], ids=["kfac", "kfac_star"])
def test_nccl_sharded_step_matches_single_call(nccl_group, star):
    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import (ShardedKfacStarStep, ShardedKfacStep, make_rank_engine,
                                            torch_all_reduce)
    wl = configs.WORKLOADS["c3"]
    prob, params, batch = wl.build(0, 600, 200)
    runs = []
    for sharded in (False, True):
        eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                               momentum=0.4)
        eng.use_graph = False
        eng.load_params(params)
        eng.init_factors(True)
        if sharded:
            stepper = (ShardedKfacStarStep if star else ShardedKfacStep)(eng, torch_all_reduce())
            infos = [stepper.step() for _ in range(3)]
        else:
            fn = eng.star_step if star else eng.step
            infos = [fn() for _ in range(3)]
        runs.append((infos, eng.theta_numpy()))
        eng.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
