"""World-size-2 gloo test of the sharded KFAC step orchestration (dist.py) on CPU.

Each rank owns a contiguous shard of the interior and boundary points
(``shard_bounds``), runs the phased step through ``ShardedKfacStep`` with
gloo all-reduces at the two exchange points, and must reproduce the
single-process reference algorithm (oracle) on the whole batch.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, star=False, wkey="c3", owners=None):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_shard_engine import CpuShardEngine
        from paper_2405_15603_b200 import configs
        from paper_2405_15603_b200.dist import (ShardedKfacStarStep, ShardedKfacStep, shard_bounds,
                                                torch_all_reduce)

        wl = configs.WORKLOADS[wkey]
        prob, params, batch = wl.build(0, 90, 31)
        i0, i1 = shard_bounds(90, rank, world)
        b0, b1 = shard_bounds(31, rank, world)
        eng = CpuShardEngine(params.weights, params.biases, batch.interior[i0:i1],
                             batch.boundary[b0:b1], batch.boundary_targets[b0:b1], prob, 90, 31,
                             ema=wl.ema, damping=wl.damping, momentum=0.3)
        stepper = (ShardedKfacStarStep if star else ShardedKfacStep)(eng, torch_all_reduce(),
                                                                      owners=owners, rank=rank)
        infos = [stepper.step() for _ in range(3)]
        q.put((rank, infos, [w.copy() for w in eng.w]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("star,wkey,owners", [(False, "c3", None), (True, "c3", None),
                                               (False, "dense", None), (False, "c3", [0, 1, 1, 0, 1]),
                                               (True, "c3", [1, 0, 0, 1, 0])],
                         ids=["kfac", "kfac_star", "kfac_dense_coeffs", "kfac_distributed_solves",
                              "kfac_star_distributed_solves"])
def test_sharded_step_matches_single_process_oracle(star, wkey, owners):
    from oracle import kfac_oracle as orc
    from paper_2405_15603_b200 import configs

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, star, wkey, owners)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])

    wl = configs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, 90, 31)
    st = orc.init_state(params.weights, params.biases, ema=wl.ema, damping=wl.damping, momentum=0.3)
    step = orc.kfac_star_step if star else orc.kfac_step
    ref = [step(st, batch, prob) for _ in range(3)]
    for rank, infos, ws in res:
        for t, ((a, mu, li, lb), (ar, mur, lir, lbr)) in enumerate(zip(infos, ref)):
            if star:
                assert abs(a - ar) <= 1e-9 * abs(ar) and abs(mu - mur) <= 1e-9 * max(abs(mur), 1.0)
            else:
                assert a == ar
            tol = 1e-10 if t == 0 else 1e-8
            assert abs(li - lir) <= tol * abs(lir) and abs(lb - lbr) <= tol * abs(lbr)
        for w, wr in zip(ws, st.weights):
            assert np.max(np.abs(w - wr)) <= 1e-8 * np.max(np.abs(wr))
    # every rank ends with identical parameters (replicated state)
    for w0, w1 in zip(res[0][2], res[1][2]):
        assert np.array_equal(w0, w1)


def test_layer_owners():
    from paper_2405_15603_b200.dist import layer_owners

    # all factors fit the one-launch device solver: redundant solves, no exchange
    assert layer_owners([2, 64, 64, 48, 48, 1], 4) is None
    c5 = [100, 768, 768, 512, 512, 1]
    assert layer_owners(c5, 1) is None
    # one owner per layer, the two largest layers on different ranks, deterministic
    o2 = layer_owners(c5, 2)
    assert o2 == layer_owners(c5, 2) and set(o2) == {0, 1} and o2[1] != o2[2]
    assert sorted(layer_owners(c5, 8)) == [0, 1, 2, 3, 4]
    c4 = [10, 256, 256, 128, 128, 1]
    o4 = layer_owners(c4, 4)
    assert len(o4) == 5 and set(o4) == {0, 1, 2, 3}
