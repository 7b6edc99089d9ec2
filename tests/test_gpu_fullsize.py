"""The benched c5 size itself (N_Omega = 16384, N_b = 5461), where no CPU reference finishes
in test time (the reference needs ~57 min and ~214 GB per step).

Size-independent property: every N-dependent quantity of the step is a sum over points
(src/curvature.py:113-115,133-134, src/optim.py:173-176, src/pde.py:351,359), so streaming
the interior batch through the Taylor engine in four chunks must give the same step as one
chunk, up to the summation order.  Checked over two KFAC steps and one KFAC* step: losses,
line-search losses and the step-1 factor sums agree to 1e-12 relative, parameters, previous
update and later factors (which pass through the Kronecker solves) to 1e-10; the
line-search alpha is identical.  The parity of the same code path
against the reference itself is c5_full3 (N_Omega = 3000) in test_gpu_parity.py.
"""

import gc

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_util import max_rel  # noqa: E402
from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200.dist import make_rank_engine  # noqa: E402

N, NB = 16384, 5461


def _run(chunk, kind, steps, n=N, nb=NB):
    wl = cfgs.WORKLOADS["c5"]
    prob, params, batch = wl.build(0, n, nb)
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                           momentum=wl.momentum, chunk=chunk)
    eng.use_graph = False
    eng.load_params(params)
    eng.init_factors(True)
    out = []
    for _ in range(steps):
        alpha, mu, li, lb = eng.star_step() if kind == "kfac_star" else eng.step()
        rec = {"scalars": np.array([li, lb, alpha, mu]), "theta": eng.theta_numpy(),
               "prev": eng._d2h(eng.prev, eng.D),
               "ls": eng.ls_losses.cpu().numpy().copy()}
        for name, t, n in (("a_int", eng.a_int, eng.FA), ("b_int", eng.b_int, eng.FB),
                           ("a_bnd", eng.a_bnd, eng.FA), ("b_bnd", eng.b_bnd, eng.FB)):
            rec[name] = eng._d2h(t, n)
        out.append(rec)
    eng.close()
    del eng
    gc.collect()
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("kind,steps", [("kfac", 2), ("kfac_star", 1)])
def test_c5_n16384_four_chunks_equal_one_chunk(kind, steps):
    one = _run(N, kind, steps)
    four = _run(N // 4, kind, steps)
    for t, (a, b) in enumerate(zip(one, four)):
        tol1 = 1e-12 if t == 0 else 1e-10
        if kind == "kfac":
            assert a["scalars"][2] == b["scalars"][2], (t, a["scalars"], b["scalars"])  # alpha
            tot = a["ls"].reshape(-1, 2).sum(axis=1)
            keep = np.isfinite(tot) & (tot <= 1e3 * np.nanmin(tot))
            assert max_rel(b["ls"].reshape(-1, 2)[keep], a["ls"].reshape(-1, 2)[keep]) <= tol1
        else:
            assert max_rel(b["scalars"][2:], a["scalars"][2:]) <= 1e-10  # alpha, mu
        assert max_rel(b["scalars"][:2], a["scalars"][:2]) <= tol1
        for key in ("theta", "prev", "a_int", "b_int", "a_bnd", "b_bnd"):
            # step-1 factors are plain sums over points; the rest passes through the solves
            tol = 1e-12 if (t == 0 and key not in ("theta", "prev")) else 1e-10
            assert max_rel(b[key], a[key]) <= tol, (t, key, max_rel(b[key], a[key]))


def test_c5_n65536_eight_point_shards_match_one_gpu():
    """SURVEY.md §8(e) at BASELINE c5's largest sweep point (N_Omega = 65536, N_b = 21845):
    eight point shards (one engine per emulated rank, exchange buffers summed on the host in
    rank order, per-layer solves distributed by dist.layer_owners) take the same two KFAC
    steps as one GPU with the whole batch: identical line-search alpha, losses and line-search
    losses to 1e-12 / 1e-10, parameters to 1e-10 on every rank."""
    from paper_2405_15603_b200.dist import layer_owners

    n, nb, world = 65536, 21845, 8
    one = _run(0, "kfac", 2, n, nb)
    wl = cfgs.WORKLOADS["c5"]
    prob, params, batch = wl.build(0, n, nb)
    owners = layer_owners(wl.widths, world)
    ranks = []
    for r in range(world):
        e = make_rank_engine(wl.widths, batch, prob, r, world, ema=wl.ema, damping=wl.damping,
                             momentum=wl.momentum, chunk=1024)
        e.use_graph = False
        e.load_params(params)
        e.init_factors(True)
        ranks.append(e)

    def all_reduce(bufs):
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)

    try:
        for t in range(2):
            for e in ranks:
                e.phase("accumulate")
            all_reduce([e.reduce_buffer() for e in ranks])
            for r, e in enumerate(ranks):
                e.phase("precondition_owned", owned=[o == r for o in owners])
            all_reduce([e.direction_buffer() for e in ranks])
            for e in ranks:
                e.phase("direction")
                e.phase("linesearch")
            all_reduce([e.linesearch_buffer() for e in ranks])
            for e in ranks:
                e.phase("update")
            outs = []
            for e in ranks:
                sc, code = e.finish_step()
                assert code == 0, (t, code)
                outs.append(np.array([sc[0], sc[1], sc[2], sc[3]]))
            assert all(np.array_equal(o, outs[0]) for o in outs)
            ref = one[t]
            tol = 1e-12 if t == 0 else 1e-10
            assert outs[0][2] == ref["scalars"][2], (t, outs[0], ref["scalars"])  # alpha
            assert max_rel(outs[0][:2], ref["scalars"][:2]) <= tol
            thetas = [e.theta_numpy() for e in ranks]
            assert all(np.array_equal(th, thetas[0]) for th in thetas[1:])
            assert max_rel(thetas[0], ref["theta"]) <= 1e-10, (t, max_rel(thetas[0], ref["theta"]))
            ls, lref = ranks[0].ls_losses.cpu().numpy(), ref["ls"]
            tot = lref.reshape(-1, 2).sum(axis=1)
            keep = np.isfinite(tot) & (tot <= 1e3 * np.nanmin(tot))
            assert max_rel(ls.reshape(-1, 2)[keep], lref.reshape(-1, 2)[keep]) <= tol
    finally:
        for e in ranks:
            e.close()
