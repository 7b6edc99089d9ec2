"""Benchmark: KFAC steps of the 100d Poisson PINN (BASELINE.json config c5) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n-interior N_per_gpu]
    python bench.py --impl reference ...      # the reference algorithm on the host CPU

One "step" = one full KFAC optimizer step (reference src/optim.py:251-263): the
forward-Laplacian forward + reverse pass over the batch, factor/gradient
accumulation, the damped Kronecker-sum preconditioner, momentum, the 31-point
grid line search (31 more forward passes) and the update.  Metric: interior
collocation points processed per second (N_Omega x KFAC steps/s), whole job.

Multi-GPU (one process per GPU, NCCL): ``--gpus N`` outside torchrun re-executes itself
under ``torch.distributed.run --nproc-per-node N``.  N > 1 defaults to strong scaling:
one global batch of ``--n-total`` (default 65536, the top of the BASELINE c5 sweep)
interior and ``--n-total // 3`` boundary points split contiguously across the ranks;
``--scaling weak`` gives every rank ``--n-interior`` points instead.  Factor sums /
gradient and line-search losses are all-reduced; the per-layer Kronecker solves are
distributed across ranks.

Printed JSON also carries: ``roofline`` for the dominant kernel -- with KFAC the line
search's fused layer on the INT8 tensor cores (k_crt_act, the FP64 product emulated exactly
by the CRT; int8 tensor operations against the measured tcgen05 int8 peak, the
FP64-equivalent rate alongside), otherwise the FP64 DMMA forward GEMM (k_gemm_act), which
is ``roofline_dmma`` when it is not the dominant one -- measured with CUDA events inside
the timed region; ``roofline_hbm`` for the HBM-bound activation adjoint (k_act_bwd) and
``roofline_hbm_slice`` for the residue slicing, also timed with CUDA events in the timed
region; ``cpu_baseline`` (the CPU oracle restating the
reference, timed on this host at two bounded sample sizes and extrapolated to the
arm's N with a fixed + per-point cost fit); ``e2e`` (the public optimizer_step API with host numpy buffers,
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
INT8_UMMA_PEAK_TOPS = 4570.0   # measured tcgen05 kind::i8 issue peak, profiles/r02_umma_i8_peak.txt
CRT_MODULI = 13               # csrc/kp_crt.cu NMOD
HBM_COPY_PEAK_GBS = 6552.6    # measured copy bandwidth (profiles/r01_fp64_peaks.txt) when
                              # MEASURED_PEAKS.json is absent
CPU_SAMPLE_POINTS = 128       # mean interior points per CPU-oracle step: the steps alternate
                              # between 64 and 192 points (bounded samples, ~5 / ~15 s on the box)
STRONG_N_TOTAL = 65536        # BASELINE c5's largest sweep point (global batch for N > 1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--optimizer", choices=("kfac", "kfac_star"), default="kfac",
                    help="kfac (the BASELINE metric) or kfac_star (src/optim.py:266-320)")
    ap.add_argument("--n-interior", type=int, default=16384,
                    help="interior points per GPU (N = 1, and every N under --scaling weak)")
    ap.add_argument("--n-total", type=int, default=STRONG_N_TOTAL,
                    help="global interior points under --scaling strong (N > 1)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default=None,
                    help="N > 1: strong (default, fixed --n-total) or weak (--n-interior per GPU)")
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
        sm, smax, reasons, pw = [], None, set(), []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "sm_min_mhz": float(np.min(sm)) if sm else None,
                "power_w_median": float(np.median(pw)) if pw else None,
                "power_w_max": float(np.max(pw)) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def crt_smem_roof(int8_tops, clk):
    """Shared-memory traffic of k_crt_act against the 128 B/clk/SM port: every M 128 x N 112 x
    K 32 MMA reads 4096 + 3584 B of operands and TMA writes 4096 + 3328 B (104 of the 112 rows)
    for a later one, for 2 * 128 * 102 * 32 algorithmic int8 operations."""
    bytes_per_op = (4096 + 3584 + 4096 + 3328) / (2.0 * 128 * 102 * 32)
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
    per_clk = int8_tops * 1e12 * bytes_per_op / 148.0 / (mhz * 1e6)
    return {"bytes_per_clk_per_sm": per_clk, "peak": 128.0, "frac": per_clk / 128.0,
            "at_sm_mhz": mhz, "bytes_per_int8_op": bytes_per_op}


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


def cpu_sizes(args):
    """The two bounded CPU sample sizes (interior points): mean = --cpu-points."""
    n1 = max(2, args.cpu_points // 2)
    return n1, max(n1 + 1, (3 * args.cpu_points) // 2)


def fit_fixed_per_point(samples):
    """Least-squares t(n) = fixed + per_point * n over (n, seconds) samples.  The step is
    linear in N except for the N-independent Kronecker solves."""
    n = np.array([s[0] for s in samples], dtype=np.float64)
    t = np.array([s[1] for s in samples], dtype=np.float64)
    if np.ptp(n) == 0:
        return 0.0, float(t.mean() / n.mean())
    b = float(np.sum((n - n.mean()) * (t - t.mean())) / np.sum((n - n.mean()) ** 2))
    a = float(t.mean() - b * n.mean())
    if a < 0 or b <= 0:  # noisy samples: fall back to a pure per-point rate
        return 0.0, float(t.sum() / n.sum())
    return a, b


def cpu_reference_fit(wl, sizes, optimizer="kfac"):
    """One oracle step (the reference algorithm, NumPy/OpenBLAS, every host core) at each
    sample size; returns ([(n, seconds)], BLAS threads used)."""
    with all_host_blas_threads():
        return [(n, _cpu_reference_step_time(wl, n, max(1, n // 3), optimizer)) for n in sizes], \
            blas_threads()


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


def cpu_line(samples, cores, n_arm, nb_arm, wl, optimizer, what):
    """cpu_baseline object: the fit extrapolated to the GPU arm's interior batch."""
    a, b = fit_fixed_per_point(samples)
    t_arm = a + b * n_arm
    ref_lines = "266-320" if optimizer == "kfac_star" else "251-263"
    desc = ", ".join(f"{n} pts: {t:.2f} s" for n, t in samples)
    return {"value": n_arm / t_arm, "unit": "interior collocation points/s", "cores": cores,
            "kind": "port", "extrapolated": True, "same_config": True,
            "n_interior": n_arm, "n_boundary": nb_arm,
            "fit": {"fixed_s": a, "per_point_s": b, "step_s_at_n": t_arm},
            "samples": [{"n_interior": n, "n_boundary": max(1, n // 3), "s_per_step": t}
                        for n, t in samples],
            "sample": f"{what} oracle {optimizer}_step (NumPy/OpenBLAS restatement of reference "
                      f"src/optim.py:{ref_lines}) on {wl.name} at bounded sample sizes ({desc}); "
                      f"t(N) = fixed + per_point * N fitted over the samples and evaluated at "
                      f"the GPU arm's N = {n_arm} interior / {nb_arm} boundary points "
                      f"(extrapolated: the reference step is linear in N apart from the "
                      f"N-independent Kronecker solves)"}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def resolve_scaling(args, world):
    return args.scaling or ("strong" if world > 1 else "weak")


def job_points(args, world):
    """(interior, boundary) points of the whole job and the scaling mode."""
    scaling = resolve_scaling(args, world)
    n = args.n_total if scaling == "strong" else args.n_interior * world
    if args.n_boundary is not None:
        nb = args.n_boundary * (world if scaling == "weak" else 1)
    else:
        nb = max(1, n // 3)
    return n, nb, scaling


def run_reference(args):
    """--impl reference: the reference KFAC step (restated CPU oracle) on host cores.

    Steps alternate between two bounded sample sizes of the arm's workload; the per-step
    times are fitted as fixed + per-point cost and evaluated at the GPU arm's N (value =
    that N / the fitted step time).  Under torchrun only rank 0 runs and prints."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2405_15603_b200 import configs
    from oracle import kfac_oracle as orc

    wl = configs.WORKLOADS[args.workload]
    step = oracle_step_fn(args.optimizer)
    n_arm, nb_arm, scaling = job_points(args, max(world, args.gpus))
    runs = []
    for n_s in cpu_sizes(args):
        prob, params, batch = wl.build(0, n_s, max(1, n_s // 3))
        st = orc.init_state(params.weights, params.biases, ema=wl.ema, damping=wl.damping,
                            momentum=wl.momentum)
        runs.append((n_s, st, batch, prob))
    samples = []
    with all_host_blas_threads():
        cores = blas_threads()
        for k in range(max(args.warmup, 0)):
            n_s, st, batch, prob = runs[k % 2]
            step(st, batch, prob)
        for k in range(max(args.steps, 2)):  # at least one step per sample size
            n_s, st, batch, prob = runs[k % 2]
            t0 = time.perf_counter()
            step(st, batch, prob)
            samples.append((n_s, time.perf_counter() - t0))
    per_size = [(n, float(np.median([t for m, t in samples if m == n]))) for n in cpu_sizes(args)]
    cpu = cpu_line(samples, cores, n_arm, nb_arm, wl, args.optimizer,
                   f"{len(samples)} timed steps (alternating sizes) of the")
    cpu["samples"] = [{"n_interior": n, "n_boundary": max(1, n // 3), "s_per_step": t}
                      for n, t in per_size]
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": "collocation_pts_per_s", "value": value,
        "unit": "interior collocation points/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": cpu["fit"]["step_s_at_n"] * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference seeding recipe, SURVEY.md §8d)",
        "config": {"workload": wl.name, "optimizer": args.optimizer, "widths": list(wl.widths),
                   "n_interior_total": n_arm, "n_boundary_total": nb_arm,
                   "parallelism": f"dp{args.gpus}"},
        "extrapolated": True,
        "cpu_baseline": cpu,
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
    n_glob, nb_glob, scaling = job_points(args, world)
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
    # the timed steps continue the warm-up run: steps W+1 .. W+K of one optimisation from
    # identity factors (the Kronecker solves warm-start from the previous step's eigenbasis,
    # as in a training run; the first steps after an identity start need more Jacobi sweeps)
    for _ in range(args.warmup):
        do_step()
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
    hbm_ms, hbm_bytes, hbm_launches = eng.profile_read_hbm()
    crt_ms, crt_flops, crt_launches = eng.profile_read_cat(0)
    slice_ms, slice_bytes, slice_launches = eng.profile_read_cat(1)
    eng.profile(False)
    n_loc, nb_loc = eng.n_interior, eng.n_boundary
    clk = clocks.stop()
    launches = (k1 - k0) // max(args.steps, 1)
    chunk = int(eng.prob.chunk)

    t = torch.tensor([ms_total, gemm_ms, hbm_ms], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, gemm_ms_max = float(t[0]), float(t[1])
    ms_step = ms_total / args.steps
    steps_per_s = 1e3 / ms_step
    value = n_glob * steps_per_s
    f_step = configs.flops_per_step(wl.widths, n_glob, nb_glob, optimizer=args.optimizer)
    achieved_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    hbm_peak, hbm_peak_src = HBM_COPY_PEAK_GBS, "measured copy bandwidth, profiles/r01_fp64_peaks.txt"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            hbm_peak = float(json.load(open(mp))["hbm_gbs"])
            hbm_peak_src = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
        except (OSError, ValueError, KeyError):
            pass
    hbm_gbs = hbm_bytes / (hbm_ms / 1e3) / 1e9 if hbm_ms > 0 else None

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
        samples, cores = cpu_reference_fit(wl, cpu_sizes(args), args.optimizer)
        cpu = cpu_line(samples, cores, n_glob, nb_glob, wl, args.optimizer, "one")

    def stored_traffic(fname):
        """DRAM bytes per launch from a stored ncu --set full capture (profiles/<fname>): only
        valid for the workload it was captured on (bytes scale with N)."""
        tp = os.path.join(ROOT, "profiles", fname)
        if not os.path.exists(tp):
            return None, None
        try:
            tj = json.load(open(tp))
            if tj.get("n_interior") == args.n_interior and tj.get("workload") == wl.name:
                return tj.get("dram_bytes_per_launch"), {
                    "launch": tj.get("kernel"),
                    "algorithmic_bytes_per_launch": tj.get("algorithmic_bytes_per_launch"),
                    "source": f"stored ncu --set full capture of the same launch (profiles/{fname}), "
                              "not measured in this run"}
        except (OSError, ValueError):
            pass
        return None, None

    traffic, traffic_note = stored_traffic("gemm_act_traffic.json")
    per_step = max(args.steps, 1)
    dmma_roof = {"bound": "tensor", "kernel": "k_gemm_act (TMA-fed FP64 DMMA forward GEMM fused with the Taylor "
                                              "activation: the stored forward pass, and every line-search layer "
                                              "with KP_CRT=0)",
                 "achieved": achieved_tflops, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                 "frac": (achieved_tflops / FP64_DMMA_PEAK_TFLOPS) if achieved_tflops else None,
                 "traffic": traffic, "traffic_of": traffic_note,
                 "launches_per_step": gemm_launches // per_step,
                 "share_of_step": gemm_ms / ms_total if ms_total else None,
                 "peak_source": "measured DMMA issue peak, profiles/r01_fp64_peaks.txt "
                                "(MEASURED_PEAKS.json has no FP64 entry; cuBLAS DGEMM 35.4)"}
    crt_roof = None
    if crt_ms > 0:
        # every FP64-equivalent multiply-add is one int8 multiply-add per modulus (13)
        crt_tops = CRT_MODULI * crt_flops / (crt_ms / 1e3) / 1e12
        ctraffic, ctraffic_note = stored_traffic("crt_act_traffic.json")
        crt_roof = {"bound": "tensor",
                    "kernel": "k_crt_act (line-search hidden layers: FP64 product emulated exactly on the INT8 "
                              "tensor cores by the CRT over 13 moduli, tcgen05.mma kind::i8 fed by TMA, fold + "
                              "Taylor activation in the epilogue; src/taylor.py:134-169 in src/optim.py:195-211)",
                    "achieved": crt_tops, "peak": INT8_UMMA_PEAK_TOPS, "unit": "TFLOP/s",
                    "unit_note": "int8 tensor operations (2 per multiply-add), 13 per FP64 multiply-add",
                    "frac": crt_tops / INT8_UMMA_PEAK_TOPS,
                    "fp64_equivalent_tflops": crt_tops / CRT_MODULI,
                    "fp64_equivalent_vs_dmma_peak": crt_tops / CRT_MODULI / FP64_DMMA_PEAK_TFLOPS,
                    "traffic": ctraffic, "traffic_of": ctraffic_note,
                    "launches_per_step": crt_launches // per_step,
                    "share_of_step": crt_ms / ms_total if ms_total else None,
                    "smem": crt_smem_roof(crt_tops, clk),
                    "limit": "shared-memory bandwidth: a 128-unit x 112-row x 32-byte MMA reads 7.5 KB of operands "
                             "while TMA writes 7.5 KB for a later one, 15 KB per 56 tensor clocks against 128 B/clk "
                             "(measured 121 clk per MMA, DESIGN.md section 5); the fold state (12 B per output) "
                             "fills the register file, so the tile cannot grow",
                    "peak_source": "measured tcgen05 kind::i8 issue peak, tools/umma_i8_peak.cu "
                                   "(profiles/r02_umma_i8_peak.txt: 4570 TOPS at N = 128/256, 4257 at N = 112); "
                                   "MEASURED_PEAKS.json has no int8 entry (its bf16 burst figure x 2 = 3308)"}
    slice_roof = None
    if slice_ms > 0:
        sl_gbs = slice_bytes / (slice_ms / 1e3) / 1e9
        slice_roof = {"bound": "hbm", "kernel": "k_crt_slice_h (FP64 states -> 13 int8 residue planes + row exponents)",
                      "achieved": sl_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": sl_gbs / hbm_peak,
                      "traffic": None, "launches_per_step": slice_launches // per_step,
                      "share_of_step": slice_ms / ms_total if ms_total else None,
                      "peak_source": hbm_peak_src,
                      "bytes": "algorithmic: 8 B read + 13 B written per state element"}
    main_roof = crt_roof if (crt_roof and crt_ms > gemm_ms) else dmma_roof

    if rank == 0:
        line = {
            "metric": "collocation_pts_per_s", "value": value,
            "unit": "interior collocation points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference seeding recipe, SURVEY.md §8d)",
            "config": {"workload": wl.name, "optimizer": args.optimizer,
                       "widths": list(wl.widths), "n_interior_per_gpu": n_loc,
                       "n_boundary_per_gpu": nb_loc, "n_interior_total": n_glob,
                       "n_boundary_total": nb_glob, "chunk": chunk,
                       "parallelism": f"dp{world}",
                       "timed_steps": f"steps {args.warmup + 1}..{args.warmup + args.steps} of one run "
                                      "from identity factors (the warm-up steps come first)",
                       "l2": "working set (Taylor states, GBs) far larger than the 126 MB L2",
                       "line_search_layers": ("INT8 tensor cores, FP64 products emulated by the CRT "
                                              "(13 moduli, 45-bit operands: within 2e-14 of sum|h w|)"
                                              if crt_launches > 0 else "FP64 DMMA")},
            "kfac_steps_per_s": steps_per_s,
            "alg_tflops_per_s": f_step * steps_per_s / 1e12,
            "alg_frac_fp64_peak": f_step * steps_per_s / 1e12 / (FP64_DMMA_PEAK_TFLOPS * world),
            "alg_frac_note": "algorithmic FP64 flops of the step / measured FP64 DMMA peak; above 1 when the line "
                             "search runs its products on the INT8 tensor cores (roofline)",
            "roofline": main_roof,
            "roofline_dmma": dmma_roof if main_roof is not dmma_roof else None,
            "roofline_hbm_slice": slice_roof,
            "roofline_hbm": {"bound": "hbm", "kernel": "k_act_bwd (activation adjoint, src/taylor.py:206-239)",
                             "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": (hbm_gbs / hbm_peak) if hbm_gbs else None,
                             "frac_of_8tbs": (hbm_gbs / 8000.0) if hbm_gbs else None,
                             "traffic": None, "launches_per_step": hbm_launches // max(args.steps, 1),
                             "share_of_step": hbm_ms / ms_total if ms_total else None,
                             "peak_source": hbm_peak_src,
                             "bytes": "algorithmic: stored pre-activation state + incoming "
                                      "adjoint + outgoing adjoint, 8 B each per (point, row, unit)"},
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

    # continues the device-timed run (no reset: warm-started solves, as in the timed steps);
    # at most 5 steps unless --e2e-steps says otherwise (strong scaling at 65536 points makes
    # an N = 2 step ~9 s)
    steps = args.e2e_steps or min(args.steps, 5)
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


def reexec_under_torchrun(n):
    """``--gpus N`` (N > 1) outside torchrun: one process per GPU through torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    under_torchrun = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not under_torchrun:
        reexec_under_torchrun(args.gpus)
    if under_torchrun and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    run_ours(args)


if __name__ == "__main__":
    main()
