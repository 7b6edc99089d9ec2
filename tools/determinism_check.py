"""Bitwise reproducibility of the accumulate and line-search phases (diagnostic).

Runs each phase REPS times on the same state and compares the reduce / line-search
buffers bit for bit.  FILL=zero|nan pre-fills the workspace (uninitialised-read probe).
    NI=16384 REPS=6 python tools/determinism_check.py
"""
import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2405_15603_b200 import configs
from paper_2405_15603_b200.dist import make_rank_engine
wl = configs.WORKLOADS[os.environ.get("WL", "c5")]
N = int(os.environ.get("NI", 16384))
prob, params, batch = wl.build(0, N, N // 3)
eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping, momentum=wl.momentum)
eng.load_params(params); eng.init_factors(True)
fill = os.environ.get("FILL")
if fill == "zero":
    eng.ws.zero_()
elif fill == "nan":
    eng.ws.view(torch.float64)[:].fill_(float("nan")) if eng.ws.numel() % 8 == 0 else None
torch.cuda.synchronize()
K = int(os.environ.get("REPS", 5))
ref = None
bad = 0
for r in range(K):
    eng.phase("accumulate"); torch.cuda.synchronize()
    red = eng.reduce_buffer().clone()
    if ref is None: ref = red
    else:
        d = (red != ref) | torch.isnan(red)
        if d.any():
            bad += 1
            idx = torch.nonzero(d).flatten()
            print("accumulate rep", r, "differs at", idx.numel(), "entries; first", idx[:5].tolist(), "nan", int(torch.isnan(red).sum()))
print("accumulate reps", K, "bad", bad, "nan_in_ref", int(torch.isnan(ref).sum()))
eng.phase("precondition"); torch.cuda.synchronize()
d0 = eng.delta.clone()
print("delta nan", int(torch.isnan(d0).sum()), "status", int(eng.status.item()))
lref = None; bad = 0
for r in range(K):
    eng.phase("linesearch"); torch.cuda.synchronize()
    ls = eng.linesearch_buffer().clone()
    if lref is None: lref = ls
    elif not torch.equal(ls, lref):
        bad += 1
        print("linesearch rep", r, "differs:", int((ls != lref).sum()), "nan", int(torch.isnan(ls).sum()), int(torch.isnan(lref).sum()), "idx", torch.nonzero(ls != lref).flatten().tolist(), "vals", [ (float(ls[i]), float(lref[i])) for i in torch.nonzero(ls != lref).flatten().tolist()][:4])
print("linesearch reps", K, "bad", bad)
