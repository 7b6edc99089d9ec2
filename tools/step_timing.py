"""Wall-clock per KFAC step (engine.step, incl. host sync + scalar read), graph vs no graph."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1")
ap.add_argument("--n-interior", type=int, default=None)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--star", action="store_true")
a = ap.parse_args()
import torch
from paper_2405_15603_b200 import configs
from paper_2405_15603_b200.dist import make_rank_engine
wl = configs.WORKLOADS[a.workload]
prob, params, batch = wl.build(0, a.n_interior, None)
res = {"workload": wl.name, "star": a.star}
for graph in (False, True):
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping, momentum=wl.momentum)
    eng.use_graph = graph
    eng.load_params(params); eng.init_factors(True)
    fn = eng.star_step if a.star else eng.step
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        out = fn()
    res[f"ms_per_step_graph={graph}"] = round((time.perf_counter() - t0) / a.steps * 1e3, 3)
    res[f"out_graph={graph}"] = [float(x) for x in out]
    eng.close()
print(json.dumps(res))
