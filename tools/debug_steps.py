"""Run several consecutive device KFAC steps and report the status of each (diagnostic)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5")
ap.add_argument("--n-interior", type=int, default=16384)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
from paper_2405_15603_b200 import configs
from paper_2405_15603_b200.dist import make_rank_engine
wl = configs.WORKLOADS[a.workload]
prob, params, batch = wl.build(0, a.n_interior, max(1, a.n_interior // 3))
eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping, momentum=wl.momentum)
eng.load_params(params)
eng.init_factors(True)
for t in range(a.steps):
    eng.launch_step()
    sc, code = eng.finish_step()
    print(f"step {t}: status={code} alpha={sc[2]} losses={sc[0]:.6e},{sc[1]:.6e}", flush=True)
