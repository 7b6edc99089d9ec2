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


@pytest.mark.parametrize("star", [False, True], ids=["kfac", "kfac_star"])
def test_nccl_owned_solves_match_single_call(nccl_group, star):
    """The distributed-solve phases (precondition_owned -> NCCL all-reduce of the direction
    buffer -> direction) at world size 1, every layer owned by rank 0, on c4's widths (factor
    pairs of 128-257: the cuSOLVER route)."""
    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import (ShardedKfacStarStep, ShardedKfacStep, make_rank_engine,
                                            torch_all_reduce)
    wl = configs.WORKLOADS["c4"]
    prob, params, batch = wl.build(0, 300, 100)
    runs = []
    for sharded in (False, True):
        eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                               momentum=0.4)
        eng.use_graph = False
        eng.load_params(params)
        eng.init_factors(True)
        if sharded:
            cls = ShardedKfacStarStep if star else ShardedKfacStep
            stepper = cls(eng, torch_all_reduce(), owners=[0] * (len(wl.widths) - 1), rank=0)
            infos = [stepper.step() for _ in range(3)]
        else:
            fn = eng.star_step if star else eng.step
            infos = [fn() for _ in range(3)]
        runs.append((infos, eng.theta_numpy()))
        eng.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("wkey", ["c4", "c1"])
def test_two_rank_distributed_solves_bit_identical(wkey):
    """Two engines in one process play two ranks that each own part of the layers: each
    solves only its layers, the direction buffers are summed (what the NCCL all-reduce does)
    and both ranks continue — parameters, losses and step sizes must equal the single-call
    step bit for bit.  No kernel waits on the other engine (sequential host calls)."""
    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import make_rank_engine
    wl = configs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, 300, 100)
    L = len(wl.widths) - 1
    owners = [l % 2 for l in range(L)]

    def fresh():
        e = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                             momentum=0.4)
        e.use_graph = False
        e.load_params(params)
        e.init_factors(True)
        return e

    ref = fresh()
    ref_infos = [ref.step() for _ in range(3)]
    ref_theta = ref.theta_numpy()
    ref.close()
    ranks = [fresh(), fresh()]
    infos = []
    for _ in range(3):
        for e in ranks:
            e.phase("accumulate")
        for r, e in enumerate(ranks):
            e.phase("precondition_owned", owned=[o == r for o in owners])
        b0, b1 = ranks[0].direction_buffer(), ranks[1].direction_buffer()
        total = b0 + b1
        b0.copy_(total)
        b1.copy_(total)
        out = []
        for e in ranks:
            e.phase("direction")
            e.phase("linesearch")
            e.phase("update")
            sc, code = e.finish_step()
            assert code == 0
            out.append((float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])))
        assert out[0] == out[1]
        infos.append(out[0])
    assert infos == ref_infos
    for e in ranks:
        assert np.array_equal(e.theta_numpy(), ref_theta)
        e.close()


@pytest.mark.parametrize("wkey", ["c4", "c1"])
def test_distributed_solve_failure_reaches_every_rank(wkey):
    """A not-positive-definite factor pair detected by the owner of its layer must fail the
    step on every rank (status slots of the direction buffer): both ranks end with
    NotPositiveSemidefiniteError's code."""
    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import make_rank_engine
    wl = configs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, 200, 60)
    L = len(wl.widths) - 1
    owners = [l % 2 for l in range(L)]  # layer 1 belongs to rank 1
    ranks = []
    for _ in range(2):
        e = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                             momentum=0.0)
        e.use_graph = False
        e.load_params(params)
        e.init_factors(True)
        a_int, b_int, a_bnd, b_bnd = e.factor_lists()
        a_bnd[1] = -100.0 * np.eye(a_bnd[1].shape[0])  # EMA keeps it indefinite
        e.set_factor_lists(a_int, b_int, a_bnd, b_bnd)
        ranks.append(e)
    for e in ranks:
        e.phase("accumulate")
    for r, e in enumerate(ranks):
        e.phase("precondition_owned", owned=[o == r for o in owners])
    b0, b1 = ranks[0].direction_buffer(), ranks[1].direction_buffer()
    total = b0 + b1
    b0.copy_(total)
    b1.copy_(total)
    codes = []
    for e in ranks:
        e.phase("direction")
        e.phase("linesearch")
        e.phase("update")
        codes.append(e.finish_step()[1])
        e.close()
    assert codes == [2, 2], codes  # KP_ERR_NOT_PSD on both ranks
