"""the sharded step must match the reference for P in {1, 2, 4, 8} on the same
global batch.  The build has one GPU, so P ranks are P engines in one process, each holding
its contiguous shard of the reference-golden batch with the global normalisers; between
phases the host sums their exchange buffers (reduce, direction, line-search / Gramian) in a
fixed order and writes the sum back to every rank — what the NCCL all-reduces of
dist.ShardedKfacStep do.  No kernel waits on another engine (sequential host calls).

The per-rank partial sums are added in a different order than the single-GPU step adds them,
so parity is at the §8(c) tolerance against the reference goldens (1e-10 after one step,
1e-8 after ten), not bit-exact; every rank must end with identical parameters.
"""

import numpy as np
import pytest

from golden_util import compare, has, line_search_rel, load

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200.dist import layer_owners, make_rank_engine  # noqa: E402

WL_OF = {"c1_10": "c1", "c3_10": "c3", "c4_10": "c4", "c4_zero_10": "c4", "lfp_10": "lfp",
         "dense_10": "dense", "c1_star_10": "c1", "c3_star_10": "c3", "c1_momentum_10": "c1", "c2_10": "c2", "c5_10": "c5",
         "c5_star_10": "c5", "c4_full10": "c4", "c5_full3": "c5"}


def _device_mats_to_vec(vec, widths):
    """Device row-major [W|b] packing -> reference column-stacked vector."""
    out, off = [], 0
    for h_in, h_out in zip(widths[:-1], widths[1:]):
        p, q = h_in + 1, h_out
        out.append(vec[off:off + p * q].reshape(q, p).ravel(order="F"))
        off += p * q
    return np.concatenate(out)


def _all_reduce(bufs):
    total = bufs[0].clone()
    for b in bufs[1:]:
        total += b
    for b in bufs:
        b.copy_(total)


def _emulated_steps(name, world, owners_mode):
    g = load(name)
    wl = cfgs.WORKLOADS[WL_OF[name]]
    star = "_star" in name
    prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
    L = len(wl.widths) - 1
    if owners_mode == "lpt":
        owners = layer_owners(wl.widths, world)
    elif owners_mode == "round_robin":
        owners = [l % world for l in range(L)]
    else:
        owners = None
    ranks = []
    for r in range(world):
        e = make_rank_engine(wl.widths, batch, prob, r, world, ema=float(g["ema"]),
                             damping=float(g["damping"]), momentum=float(g["momentum"]))
        e.use_graph = False
        e.load_params(params)
        e.init_factors(not int(g.get("init_zero", 0)))
        ranks.append(e)
    t = 1
    try:
        while f"s{t}/alpha" in g:
            for e in ranks:
                e.phase("accumulate")
            _all_reduce([e.reduce_buffer() for e in ranks])
            if owners is None:
                for e in ranks:
                    e.phase("precondition")
            else:
                for r, e in enumerate(ranks):
                    e.phase("precondition_owned", owned=[o == r for o in owners])
                _all_reduce([e.direction_buffer() for e in ranks])
                for e in ranks:
                    e.phase("direction")
            if star:
                for e in ranks:
                    e.phase("star_gvp")
                _all_reduce([e.gvp_buffer() for e in ranks])
                for e in ranks:
                    e.phase("star_update")
            else:
                for e in ranks:
                    e.phase("linesearch")
                _all_reduce([e.linesearch_buffer() for e in ranks])
                for e in ranks:
                    e.phase("update")
            outs = []
            for e in ranks:
                sc, code = e.finish_step()
                assert code == 0, (t, code)
                outs.append((float(sc[2]), float(sc[3]), float(sc[0]), float(sc[1])))
            assert all(o == outs[0] for o in outs), outs  # every rank took the same step
            alpha, mu, li, lb = outs[0]
            p = f"s{t}/"
            tol = 1e-10 if t == 1 else 1e-8
            if star:
                a_ref, m_ref = float(g[p + "alpha"]), float(g[p + "mu"])
                assert abs(alpha - a_ref) <= tol * abs(a_ref), (t, alpha, a_ref)
                assert abs(mu - m_ref) <= tol * max(abs(m_ref), 1.0), (t, mu, m_ref)
            else:
                assert alpha == float(g[p + "alpha"]), (t, alpha, float(g[p + "alpha"]))
                assert line_search_rel(ranks[0].ls_losses.cpu().numpy(), g[p + "ls_losses"]) <= tol
            for key, val in (("loss_interior", li), ("loss_boundary", lb)):
                ref = float(g[p + key])
                assert abs(val - ref) <= tol * abs(ref), (t, key, val, ref)
            thetas = [e.theta_numpy() for e in ranks]
            assert all(np.array_equal(th, thetas[0]) for th in thetas[1:])
            if has(g, p + "theta"):
                th = _device_mats_to_vec(thetas[0], wl.widths)
                assert compare(g, p + "theta", th, tol) <= tol, t
                d = _device_mats_to_vec(ranks[0].delta.cpu().numpy(), wl.widths)
                assert compare(g, p + "delta", d, tol) <= tol, t
            t += 1
    finally:
        for e in ranks:
            e.close()
    assert t > (3 if name.endswith("full3") else 10)


@pytest.mark.parametrize("name,world,owners_mode", [
    ("c1_10", 2, "replicated"), ("c1_10", 8, "round_robin"), ("c1_momentum_10", 4, "round_robin"),
    ("c3_10", 4, "replicated"), ("c4_10", 2, "lpt"), ("c4_10", 8, "lpt"),
    ("c4_zero_10", 4, "lpt"), ("lfp_10", 4, "round_robin"), ("dense_10", 2, "round_robin"),
    ("c1_star_10", 4, "round_robin"), ("c3_star_10", 8, "replicated"), ("c2_10", 4, "replicated"),
    ("c5_10", 8, "lpt"), ("c5_10", 2, "lpt"), ("c5_star_10", 4, "lpt"),
    # the BASELINE sizes: c4 at N = 3000 (ten steps) and c5 at N = 3000 (three steps)
    ("c4_full10", 4, "lpt"), ("c5_full3", 8, "lpt"),
])
def test_point_sharded_steps_match_reference_golden(name, world, owners_mode):
    _emulated_steps(name, world, owners_mode)
