"""Line-search agreement of the CRT (INT8 tensor-core) layers with the FP64 DMMA layers.

    KP_CRT=0 python tools/crt_check.py --workload c5 --n-interior 3000 --steps 5 --out a.json
    KP_CRT=1 python tools/crt_check.py --workload c5 --n-interior 3000 --steps 5 --out b.json
    python tools/crt_check.py --compare a.json b.json

Runs `steps` KFAC steps phase by phase and records every step's line-search losses (all grid
candidates, interior and boundary) and the chosen step size.  --compare prints the largest
relative difference of the candidate losses, whether every argmin agrees, and the smallest
relative gap between the best and the runner-up candidate (the margin an argmin flip needs).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    import numpy as np
    import torch

    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import make_rank_engine

    wl = configs.WORKLOADS[a.workload]
    nb = wl.n_boundary if a.n_interior == wl.n_interior else a.n_interior // 3
    prob, params, batch = wl.build(0, a.n_interior, nb)
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                           momentum=wl.momentum)
    eng.load_params(params)
    eng.init_factors(True)
    out = {"workload": wl.name, "n_interior": a.n_interior, "n_boundary": nb,
           "crt": os.environ.get("KP_CRT", ""),
           "steps": []}
    for _ in range(a.steps):
        eng.phase("accumulate")
        eng.phase("precondition")
        eng.phase("linesearch")
        ls = eng.linesearch_buffer().cpu().numpy().copy()
        eng.phase("update")
        sc, code = eng.finish_step()
        torch.cuda.synchronize()
        out["steps"].append({"ls": ls.tolist(), "alpha": float(sc[2]), "code": int(code)})
    with open(a.out, "w") as f:
        json.dump(out, f)
    print(json.dumps({"alphas": [s["alpha"] for s in out["steps"]]}))


def compare(pa, pb):
    import numpy as np

    A = json.load(open(pa))
    B = json.load(open(pb))
    worst, agree, gap = 0.0, True, float("inf")
    for sa, sb in zip(A["steps"], B["steps"]):
        # ls[2k] / ls[2k+1]: interior / boundary sums of squares of candidate k
        la, lb = np.asarray(sa["ls"]).reshape(-1, 2), np.asarray(sb["ls"]).reshape(-1, 2)
        w = np.array([1.0 / A["n_interior"], 1.0 / A["n_boundary"]])
        tot_a, tot_b = la @ w, lb @ w
        fin = np.isfinite(tot_a) & np.isfinite(tot_b)
        worst = max(worst, float(np.max(np.abs(la[fin] - lb[fin]) / np.abs(la[fin]))))
        agree = agree and sa["alpha"] == sb["alpha"]
        s = np.sort(tot_a[fin])
        if s.size > 1:
            gap = min(gap, float((s[1] - s[0]) / abs(s[0])))
    print(json.dumps({"a": pa, "b": pb, "max_rel_diff_candidate_losses": worst,
                      "argmin_agree": agree, "min_rel_gap_best_vs_runner_up": gap,
                      "alphas_a": [s["alpha"] for s in A["steps"]],
                      "alphas_b": [s["alpha"] for s in B["steps"]]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--n-interior", type=int, default=3000)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default="crt_check.json")
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a)


if __name__ == "__main__":
    main()
