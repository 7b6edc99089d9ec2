"""Parity margins of the device step against the reference goldens (diagnostic).

    python tools/parity_report.py c5_full3 c4_full10 c5_star_n1000 ...

For each golden (tests/golden/<name>.npz, made by running the reference itself) runs the
same steps through the public optimizer_step and prints, per step, the worst relative
discrepancy of the losses, alpha / mu and (where recorded) the gradient, the direction,
the parameters, the previous update and the four factor lists, plus the per-step Jacobi
sweep counts of the device eigensolvers and the step time.  The bars are 1e-10 after one
step and 1e-8 after more (BASELINE.json north star); the tests assert them, this prints the
margins.
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden_util import FULL_WL, compare, has, line_search_rel, load, pack_factors  # noqa: E402
from paper_2405_15603_b200 import configs as cfgs  # noqa: E402
from paper_2405_15603_b200.network import mats_to_vec  # noqa: E402
from paper_2405_15603_b200.optim import OptimizerConfig, init_train_state, optimizer_step  # noqa: E402


def wl_of(name):
    return FULL_WL.get(name) or name.split("_")[0]


def dev_to_ref(vec, widths):
    out, off = [], 0
    for h_in, h_out in zip(widths[:-1], widths[1:]):
        p, q = h_in + 1, h_out
        out.append(vec[off:off + p * q].reshape(q, p).ravel(order="F"))
        off += p * q
    return np.concatenate(out)


def main():
    import torch

    for name in sys.argv[1:]:
        g = load(name)
        wl = cfgs.WORKLOADS[wl_of(name)]
        prob, params, batch = wl.build(0, int(g["n_interior"]), int(g["n_boundary"]))
        kind = "kfac_star" if "star" in name else "kfac"
        cfg = OptimizerConfig(kind=kind, damping=float(g["damping"]), ema=float(g["ema"]),
                              momentum=float(g["momentum"]))
        state = init_train_state(params, cfg)
        t = 1
        while f"s{t}/alpha" in g:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            info = optimizer_step(state, batch, prob)
            dt = time.perf_counter() - t0
            eng = state._engine
            sw = [C.c_int32() for _ in range(3)]
            eng.lib.kp_solver_sweeps(*[C.byref(v) for v in sw], 1)
            p = f"s{t}/"
            rel = lambda a, b: abs(a - b) / max(abs(b), 1e-300)  # noqa: E731
            rec = {"golden": name, "step": t, "ms": round(dt * 1e3, 2),
                   "sweeps": {"small": sw[0].value, "mid": sw[1].value, "large": sw[2].value},
                   "loss_interior": rel(info.loss_interior, float(g[p + "loss_interior"])),
                   "loss_boundary": rel(info.loss_boundary, float(g[p + "loss_boundary"])),
                   "alpha": rel(info.alpha, float(g[p + "alpha"])),
                   "mu": abs(info.mu - float(g[p + "mu"])) / max(abs(float(g[p + "mu"])), 1.0)}
            if p + "ls_losses" in g:
                rec["ls_losses"] = line_search_rel(eng.ls_losses.cpu().numpy(), g[p + "ls_losses"])
            if has(g, p + "theta"):
                w = eng.widths
                theta = np.concatenate([np.hstack([a, b[:, None]]).ravel(order="F")
                                        for a, b in zip(state.params.weights, state.params.biases)])
                rec["theta"] = compare(g, p + "theta", theta, 0)
                rec["prev_update"] = compare(g, p + "prev_update", mats_to_vec(state.prev_update), 0)
                rec["delta"] = compare(g, p + "delta", dev_to_ref(eng.delta.cpu().numpy(), w), 0)
                if has(g, p + "grad"):
                    rec["grad"] = compare(g, p + "grad", dev_to_ref(eng.grad.cpu().numpy(), w), 0)
                kf = state.kfac
                for key, mats in (("a_interior", kf.a_interior), ("b_interior", kf.b_interior),
                                  ("a_boundary", kf.a_boundary), ("b_boundary", kf.b_boundary)):
                    rec[key] = compare(g, p + key, pack_factors(mats), 0)
            worst = max(v for k, v in rec.items() if isinstance(v, float) and k != "ms")
            rec["worst"] = worst
            rec["bar"] = 1e-10 if t == 1 else 1e-8
            print(json.dumps(rec), flush=True)
            t += 1


if __name__ == "__main__":
    main()
