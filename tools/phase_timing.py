"""Per-phase CUDA-event timing of one KFAC step (diagnostic, not the bench).

    python tools/phase_timing.py --workload c5 --n-interior 3000 [--chunk 0] [--reps 3]
                                 [--owned-world W]

--owned-world W: also time the precondition phase as each rank r < W of a W-GPU run does it
with distributed Kronecker solves (dist.layer_owners; the direction all-reduce excluded) and
report the slowest rank's time as "precondition_owned_max_ms".
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--n-interior", type=int, default=3000)
    ap.add_argument("--n-boundary", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--owned-world", type=int, default=0)
    ap.add_argument("--star", action="store_true", help="KFAC* phases (star_gvp, star_update)")
    a = ap.parse_args()
    import torch

    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import layer_owners, make_rank_engine

    wl = configs.WORKLOADS[a.workload]
    nb = a.n_boundary if a.n_boundary is not None else (wl.n_boundary if a.n_interior == wl.n_interior else a.n_interior // 3)
    prob, params, batch = wl.build(0, a.n_interior, nb)
    eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                           momentum=wl.momentum, chunk=a.chunk or None)
    eng.load_params(params)
    eng.init_factors(True)
    res = {}
    for rep in range(a.reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        evs[0].record()
        eng.phase("accumulate")
        evs[1].record()
        eng.phase("precondition")
        evs[2].record()
        eng.phase("star_gvp" if a.star else "linesearch")
        evs[3].record()
        eng.phase("star_update" if a.star else "update")
        evs[4].record()
        sc, code = eng.finish_step()
        names = (["accumulate", "precondition", "star_gvp", "star_update"] if a.star
                 else ["accumulate", "precondition", "linesearch", "update"])
        res = {n: evs[i].elapsed_time(evs[i + 1]) for i, n in enumerate(names)}
        res["total_ms"] = evs[0].elapsed_time(evs[4])
        res["status"] = code
        res["alpha"] = float(sc[2])
    owners = layer_owners(wl.widths, a.owned_world) if a.owned_world > 1 else None
    if owners is not None:
        worst = 0.0
        for r in range(a.owned_world):
            t = []
            for rep in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                eng.phase("accumulate")
                e0.record()
                eng.phase("precondition_owned", owned=[o == r for o in owners])
                e1.record()
                torch.cuda.synchronize()
                t.append(e0.elapsed_time(e1))
            worst = max(worst, min(t))
        res["owners"] = owners
        res["precondition_owned_max_ms"] = worst
    # the single-call step (early preconditioning overlaps the accumulate) for comparison
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn = eng.star_step if a.star else eng.step
    eng.use_graph = False
    fn()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    res["single_call_ms"] = e0.elapsed_time(e1)
    f = configs.flops_per_step(wl.widths, a.n_interior, nb,
                               optimizer="kfac_star" if a.star else "kfac")
    res["alg_tflops_per_s"] = f / (res["total_ms"] / 1e3) / 1e12
    res["workload"] = wl.name
    res["n_interior"] = a.n_interior
    res["chunk"] = int(eng.prob.chunk)
    import ctypes as C
    sw = [C.c_int32() for _ in range(3)]
    eng.lib.kp_solver_sweeps(*[C.byref(v) for v in sw], 0)
    res["max_sweeps"] = {"small": sw[0].value, "mid": sw[1].value, "large": sw[2].value}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
