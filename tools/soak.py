"""Soak test: K consecutive KFAC steps of a workload, printed as (alpha, loss) pairs, so that
two runs can be compared for bitwise run-to-run reproducibility (diagnostic).
    NI=16384 STEPS=30 python tools/soak.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_15603_b200 import configs  # noqa: E402
from paper_2405_15603_b200.dist import make_rank_engine  # noqa: E402

wl = configs.WORKLOADS[os.environ.get("WL", "c5")]
N = int(os.environ.get("NI", 16384))
prob, params, batch = wl.build(0, N, N // 3)
eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping, momentum=wl.momentum)
eng.load_params(params)
eng.init_factors(True)
for t in range(int(os.environ.get("STEPS", 30))):
    a, mu, li, lb = eng.step()
    print(t, repr(a), repr(li), repr(lb), flush=True)
