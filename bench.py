"""Benchmark: KFAC steps of the 100d Poisson PINN (BASELINE.json config c5) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n-interior N_per_gpu]
    python bench.py --impl reference ...      # the reference algorithm on the host CPU

One "step" = one full KFAC optimizer step (reference src/optim.py:251-263): the
forward-Laplacian forward + reverse pass over the batch, factor/gradient
accumulation, the damped Kronecker-sum preconditioner, momentum, the 31-point
grid line search (31 more forward passes) and the update.  Metric: interior
collocation points processed per second (N_Omega x KFAC steps/s), whole job.

Multi-GPU (torchrun, one process per GPU, NCCL): weak scaling — every rank owns
``--n-interior`` interior and ``--n-interior // 3`` boundary points of one global
batch; factor sums / gradient and line-search losses are all-reduced.

Printed JSON also carries: ``roofline`` for the dominant kernel (the FP64 DMMA
forward GEMM, k_gemm_nt) measured with CUDA events inside the timed region;
``cpu_baseline`` (the CPU oracle restating the reference, bounded sample on
this host); ``e2e`` (the public optimizer_step API with host numpy buffers,
H2D of the batch and D2H of parameters + StepInfo inside the timed region);
``clocks`` sampled by nvidia-smi during the timed region; ``gpu_launches``.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1  # measured, profiles/r01_fp64_peaks.txt (register-only DMMA, 1965 MHz)
CPU_SAMPLE_POINTS = 128       # interior points per CPU-oracle step (bounded sample, ~10 s on the box;
                              # the per-point rate is within 1% of a 192-point step)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--optimizer", choices=("kfac", "kfac_star"), default="kfac",
                    help="kfac (the BASELINE metric) or kfac_star (src/optim.py:266-320)")
    ap.add_argument("--n-interior", type=int, default=16384, help="interior points per GPU")
    ap.add_argument("--n-boundary", type=int, default=None, help="boundary points per GPU")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-points", type=int, default=CPU_SAMPLE_POINTS,
                    help="interior points per CPU-oracle step (reference arm and cpu_baseline)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the sharded NCCL step even at world size 1 (plumbing check)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out = self.proc.communicate(timeout=10)[0]
        sm, smax, reasons = [], None, set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_step_fn(optimizer):
    """The oracle's step for --optimizer (reference src/optim.py:251-263 / :266-320)."""
    from oracle import kfac_oracle as orc

    return orc.kfac_star_step if optimizer == "kfac_star" else orc.kfac_step


def all_host_blas_threads():
    """Context giving the oracle's BLAS every host core: torchrun exports OMP_NUM_THREADS=1,
    which OpenBLAS reads when NumPy loads."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=host_cores(), user_api="blas")


def blas_threads():
    from threadpoolctl import threadpool_info

    return max([d["num_threads"] for d in threadpool_info() if d["user_api"] == "blas"] or [1])


def cpu_reference_step_time(wl, n_points, n_bnd, optimizer="kfac"):
    """Time one oracle KFAC step (the reference algorithm, NumPy/OpenBLAS) on this host with
    every host core; returns (seconds, BLAS threads used)."""
    with all_host_blas_threads():
        return _cpu_reference_step_time(wl, n_points, n_bnd, optimizer), blas_threads()


def _cpu_reference_step_time(wl, n_points, n_bnd, optimizer):
    from oracle import kfac_oracle as orc

    step = oracle_step_fn(optimizer)

    prob, params, batch = wl.build(0, n_points, n_bnd)
    # warm the BLAS/LAPACK paths on a tiny batch first
    _, _, small = wl.build(0, 4, 2)
    st0 = orc.init_state(params.weights, params.biases, ema=wl.ema, damping=wl.damping,
                         momentum=wl.momentum)
    step(st0, small, prob)
    st = orc.init_state(params.weights, params.biases, ema=wl.ema, damping=wl.damping,
                        momentum=wl.momentum)
    t0 = time.perf_counter()
    step(st, batch, prob)
    return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    """--impl reference: the reference KFAC step (restated CPU oracle) on host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2405_15603_b200 import configs

    wl = configs.WORKLOADS[args.workload]
    n_s = args.cpu_points
    nb_s = max(1, n_s // 3)
    prob, params, batch = wl.build(0, n_s, nb_s)
    from oracle import kfac_oracle as orc

    step = oracle_step_fn(args.optimizer)
    ref_lines = "266-320" if args.optimizer == "kfac_star" else "251-263"

    st = orc.init_state(params.weights, params.biases, ema=wl.ema, damping=wl.damping,
                        momentum=wl.momentum)
    with all_host_blas_threads():
        cores = blas_threads()
        for _ in range(args.warmup):
            step(st, batch, prob)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step(st, batch, prob)
        dt = (time.perf_counter() - t0) / max(args.steps, 1)
    value = n_s / dt
    n_int_full = args.n_interior * args.gpus
    line = {
        "impl": "reference", "metric": "collocation_pts_per_s", "value": value,
        "unit": "interior collocation points/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference seeding recipe, SURVEY.md §8d)",
        "config": {"workload": wl.name, "optimizer": args.optimizer, "widths": list(wl.widths),
                   "n_interior_per_step": n_s, "n_boundary_per_step": nb_s,
                   "arm_n_interior_total": n_int_full},
        "cpu_baseline": {"value": value, "unit": "interior collocation points/s", "cores": cores,
                         "kind": "port",
                         "sample": f"oracle/kfac_oracle.py {step.__name__} (NumPy/OpenBLAS restatement of "
                                   f"the reference src/optim.py:{ref_lines}) on {n_s} interior + {nb_s} boundary "
                                   f"points of {wl.name}; per-point work is N-linear except the "
                                   f"N-independent Kronecker solve"},
        "e2e": {"value": value, "unit": "interior collocation points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2405_15603_b200 import configs
    from paper_2405_15603_b200.dist import (ShardedKfacStarStep, ShardedKfacStep, layer_owners,
                                            make_rank_engine, torch_all_reduce)
    from paper_2405_15603_b200.engine import KfacEngine

    rank, world, local = dist_env()
    # KP_BENCH_DIST_BACKEND=gloo: plumbing check of the N > 1 path with every rank on the one
    # GPU of a test box (host-side collectives; no kernel waits on another rank).  Never a
    # bench number.
    backend = os.environ.get("KP_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.force_dist
    if sharded:
        if "RANK" not in os.environ:  # --force-dist outside torchrun: a world of one
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0",
                               "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    wl = configs.WORKLOADS[args.workload]
    n_loc = args.n_interior
    nb_loc = args.n_boundary if args.n_boundary is not None else max(1, n_loc // 3)
    n_glob, nb_glob = n_loc * world, nb_loc * world
    prob, params, batch = wl.build(0, n_glob, nb_glob)

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()

    if sharded:
        eng = make_rank_engine(wl.widths, batch, prob, rank, world, ema=wl.ema, damping=wl.damping,
                               momentum=wl.momentum, chunk=args.chunk or None)
        cls = ShardedKfacStarStep if args.optimizer == "kfac_star" else ShardedKfacStep
        stepper = cls(eng, torch_all_reduce(), owners=layer_owners(wl.widths, world), rank=rank)
        do_step = stepper.step
    else:
        eng = make_rank_engine(wl.widths, batch, prob, 0, 1, ema=wl.ema, damping=wl.damping,
                               momentum=wl.momentum, chunk=args.chunk or None)
        do_step = eng.star_step if args.optimizer == "kfac_star" else eng.step

    def reset_state():
        eng.load_params(params)
        eng.init_factors(identity=True)

    reset_state()
    for _ in range(args.warmup):
        do_step()
    reset_state()
    barrier()
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    clocks.start()
    eng.profile(True)
    _, _, _, k0 = eng.profile_read()
    eng.profile(True)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    infos = []
    for _ in range(args.steps):
        infos.append(do_step())
    e1.record()
    barrier()
    ms_total = e0.elapsed_time(e1)
    gemm_ms, gemm_flops, gemm_launches, k1 = eng.profile_read()
    eng.profile(False)
    clk = clocks.stop()
    launches = (k1 - k0) // max(args.steps, 1)
    chunk = int(eng.prob.chunk)

    t = torch.tensor([ms_total, gemm_ms], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, gemm_ms_max = float(t[0]), float(t[1])
    ms_step = ms_total / args.steps
    steps_per_s = 1e3 / ms_step
    value = n_glob * steps_per_s
    f_step = configs.flops_per_step(wl.widths, n_loc, nb_loc, optimizer=args.optimizer) * world
    achieved_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None

    # end to end through the public API (host numpy in, host numpy out), 1 GPU
    e2e = None
    if not args.no_e2e and not sharded:
        eng.close()  # release the device-timed engine's workspace first
        del eng, do_step
        torch.cuda.empty_cache()
        e2e = run_e2e(args, wl, prob, params, batch)
        eng = None
    elif not args.no_e2e and sharded:
        e2e = run_e2e_sharded(args, wl, prob, params, batch, rank, world, eng, stepper)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_s = args.cpu_points
        dt, cores = cpu_reference_step_time(wl, n_s, max(1, n_s // 3), args.optimizer)
        cpu = {"value": n_s / dt, "unit": "interior collocation points/s", "cores": cores,
               "kind": "port",
               "sample": f"one oracle {args.optimizer}_step (NumPy/OpenBLAS restatement of "
                         f"reference src/optim.py:"
                         f"{'266-320' if args.optimizer == 'kfac_star' else '251-263'}) on {n_s} interior + {n_s // 3} boundary points of "
                         f"{wl.name}, {dt:.2f} s"}

    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "gemm_act_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            # only valid for the workload it was captured on (bytes scale with N)
            if tj.get("n_interior") == args.n_interior and tj.get("workload") == wl.name:
                traffic = tj.get("dram_bytes_per_launch")
                traffic_note = {"launch": tj.get("kernel"),
                                "algorithmic_bytes_per_launch": tj.get("algorithmic_bytes_per_launch")}
        except (OSError, ValueError):
            traffic = None

    if rank == 0:
        line = {
            "metric": "collocation_pts_per_s", "value": value,
            "unit": "interior collocation points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference seeding recipe, SURVEY.md §8d)",
            "config": {"workload": wl.name, "optimizer": args.optimizer,
                       "widths": list(wl.widths), "n_interior_per_gpu": n_loc,
                       "n_boundary_per_gpu": nb_loc, "n_interior_total": n_glob,
                       "n_boundary_total": nb_glob, "chunk": chunk,
                       "parallelism": f"dp{world}",
                       "l2": "working set (Taylor states, GBs) far larger than the 126 MB L2"},
            "kfac_steps_per_s": steps_per_s,
            "alg_tflops_per_s": f_step * steps_per_s / 1e12,
            "alg_frac_fp64_peak": f_step * steps_per_s / 1e12 / (FP64_DMMA_PEAK_TFLOPS * world),
            "roofline": {"bound": "tensor", "kernel": "k_gemm_act (TMA-fed FP64 DMMA forward GEMM fused with the Taylor activation; hidden-layer forwards)",
                         "achieved": achieved_tflops, "peak": FP64_DMMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s",
                         "frac": (achieved_tflops / FP64_DMMA_PEAK_TFLOPS) if achieved_tflops else None,
                         "traffic": traffic, "traffic_of": traffic_note, "launches_per_step": gemm_launches // max(args.steps, 1),
                         "share_of_step": gemm_ms / ms_total if ms_total else None,
                         "peak_source": "measured DMMA issue peak, profiles/r01_fp64_peaks.txt "
                                        "(MEASURED_PEAKS.json has no FP64 entry; cuBLAS DGEMM 35.4)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "losses_last_step": infos[-1][2:] if infos else None,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, wl, prob, params, batch):
    """optimizer_step (public API) per step: H2D batch + D2H params/StepInfo inside the timer."""
    import torch

    from paper_2405_15603_b200.optim import OptimizerConfig, init_train_state, optimizer_step

    cfg = OptimizerConfig(kind=args.optimizer, damping=wl.damping, ema=wl.ema, momentum=wl.momentum)
    state = init_train_state(params.copy(), cfg)
    # warm-up on the same state, as a training loop runs: the first call builds the device
    # engine (workspace, context, plans, solver handles) outside the timer
    for _ in range(max(1, args.warmup)):
        optimizer_step(state, batch, prob)
    state_engine = None
    steps = args.e2e_steps or args.steps
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        optimizer_step(state, batch, prob)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    n, nb, d = batch.interior.shape[0], batch.boundary.shape[0], batch.interior.shape[1]
    h2d = 8 * (n * d + n + n * (d + 2) + nb * d + nb + d)
    D = sum(w.size + b.size for w, b in zip(params.weights, params.biases))
    d2h = 8 * (D + 4) + 4
    del state_engine
    return {"value": n / dt, "unit": "interior collocation points/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
            "api": "paper_2405_15603_b200.optimizer_step (host numpy batch/params)"}


def run_e2e_sharded(args, wl, prob, params, batch, rank, world, eng, stepper):
    import torch
    import torch.distributed as dist

    from paper_2405_15603_b200.dist import upload_shard

    steps = args.e2e_steps or args.steps
    eng.load_params(params)
    eng.init_factors(True)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        upload_shard(eng, batch, prob, rank, world)
        stepper.step()
        eng.param_mats()
    torch.cuda.synchronize()
    dt = torch.tensor([(time.perf_counter() - t0) / steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    n = batch.interior.shape[0]
    d = batch.interior.shape[1]
    nloc = eng.n_interior
    h2d = 8 * (nloc * d + nloc + nloc * (d + 2) + eng.n_boundary * (d + 1) + d)
    return {"value": n / float(dt[0]), "unit": "interior collocation points/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * eng.D + 36,
            "ms_per_step": float(dt[0]) * 1e3, "api": "dist.ShardedKfacStep + host shard upload"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
