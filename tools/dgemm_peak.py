"""Measure cuBLAS FP64 DGEMM throughput on the box (burst + 4 s sustained).

Used once to fix the FP64 roofline denominator; the
result is recorded in profiles/ and DESIGN.md.
"""
import json
import subprocess
import time

import torch


def main():
    dev = torch.device("cuda:0")
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            a @ b
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / best / 1e9
    # sustained 4 s
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    torch.cuda.synchronize()
    t0 = time.time()
    cnt = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            a @ b
        cnt += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    lines = smi.communicate()[0].strip().splitlines()
    out["dgemm_8192_sustained_tflops"] = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
    out["clock_samples"] = lines[-8:]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
