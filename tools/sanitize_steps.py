"""Small KFAC / KFAC* steps for compute-sanitizer (racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_steps.py

Covers every kernel family of the step at sizes the sanitizer finishes in minutes:
c1 (one-launch small eigensolver, grouped TN contractions, candidate-batched line search),
c4 at reduced N (mid-size cluster eigensolver ``k_eig_mid`` with DSMEM + cluster barriers,
TMA-fed ``k_gemm_act`` / ``k_gemm_nt_tma`` / ``k_gemm_tn_tma``) and c5 at N = 24 (the
768-wide layers, the large factor pairs), KFAC and KFAC*, with the KFAC* G.prev-ahead
ordering (KP_STAR_AHEAD, default on).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2405_15603_b200 import configs  # noqa: E402
from paper_2405_15603_b200.optim import OptimizerConfig, init_train_state, optimizer_step  # noqa: E402

CASES = [("c1", 3000, 500, "kfac", 2), ("c4", 400, 130, "kfac", 2), ("c4", 400, 130, "kfac_star", 2),
         ("c5", 24, 8, "kfac", 2), ("c5", 24, 8, "kfac_star", 2)]
only = set(sys.argv[1:])
for wkey, n, nb, kind, steps in CASES:
    if only and wkey not in only:
        continue
    wl = configs.WORKLOADS[wkey]
    prob, params, batch = wl.build(0, n, nb)
    state = init_train_state(params, OptimizerConfig(kind=kind, damping=wl.damping, ema=wl.ema))
    for _ in range(steps):
        info = optimizer_step(state, batch, prob)
    print(f"{wkey} {kind} N={n}: alpha={info.alpha} mu={info.mu} loss={info.loss_total:.12e}",
          flush=True)
