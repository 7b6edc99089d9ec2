"""Per-layer timing of the device Kronecker-sum solve on real factors (diagnostic).

    python tools/solve_timing.py --workload c5 --n-interior 3000 --steps 2 [--reps 3]

Runs ``--steps`` KFAC steps of the workload, takes the EMA factors of every layer, and times
kp_kron_sum_solve (src/linalg.py:136-174 through curvature.py:150-161: the damped interior and
boundary pairs, cold, no warm start) per layer with CUDA events, printing the factor sizes,
milliseconds and the Jacobi sweeps each route used.  The solve is the same device route the
step uses for each pair size (one-CTA / cluster shared memory / split records / L2).
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--n-interior", type=int, default=3000)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import make_rank_engine
    from paper_2405_15603_b200.engine import kron_sum_solve_device

    wl = configs.WORKLOADS[a.workload]
    prob, params, batch = wl.build(0, a.n_interior, a.n_interior // 3)
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                           momentum=wl.momentum)
    eng.use_graph = False
    eng.load_params(params)
    eng.init_factors(True)
    for _ in range(a.steps):
        eng.step()
    ai, bi, ab, bb = eng.factor_lists()
    grad = eng.grad.cpu().numpy()
    lam = wl.damping
    lib = eng.lib
    off = 0
    for l, (A1, B1, A2, B2) in enumerate(zip(ai, bi, ab, bb)):
        p, q = A1.shape[0], B1.shape[0]
        g = grad[off:off + p * q].reshape(q, p)
        off += p * q
        I = lambda k: np.eye(k) * lam  # noqa: E731, E741
        args = (A1 + I(p), B1 + I(q), A2 + I(p), B2 + I(q), g)
        ts = []
        for _ in range(a.reps):
            sw = [C.c_int32() for _ in range(3)]
            lib.kp_solver_sweeps(*[C.byref(v) for v in sw], 1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kron_sum_solve_device(*args)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        lib.kp_solver_sweeps(*[C.byref(v) for v in sw], 1)
        print(json.dumps({"layer": l, "p": p, "q": q, "ms_min": min(ts), "ms": ts,
                          "sweeps": {"small": sw[0].value, "mid": sw[1].value,
                                     "large": sw[2].value}}), flush=True)


if __name__ == "__main__":
    main()
