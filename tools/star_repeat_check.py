"""Bit-reproducibility of KFAC* steps: plain / plain / graph-replayed runs of the same steps.

    python tools/star_repeat_check.py --workload c4 --steps 25
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--steps", type=int, default=25)
ap.add_argument("--n-interior", type=int, default=None)
a = ap.parse_args()
from paper_2405_15603_b200 import configs
from paper_2405_15603_b200.dist import make_rank_engine
wl = configs.WORKLOADS[a.workload]
prob, params, batch = wl.build(0, a.n_interior, None)
runs = {}
for name, graph in (("plain_a", False), ("plain_b", False), ("graph", True)):
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping, momentum=wl.momentum)
    eng.use_graph = graph
    eng.load_params(params); eng.init_factors(True)
    first_diff = None
    outs = [tuple(eng.star_step()) for _ in range(a.steps)]
    runs[name] = (outs, eng.theta_numpy())
    eng.close()
res = {"workload": wl.name}
for name in ("plain_b", "graph"):
    o, th = runs[name]
    ref, rth = runs["plain_a"]
    diff = [i for i in range(a.steps) if o[i] != ref[i]]
    res[name] = {"first_differing_step": diff[0] + 1 if diff else None,
                 "theta_identical": bool((th == rth).all())}
print(json.dumps(res))
