"""Measure the FP64 roofline denominator on the box: cuBLAS DGEMM (torch.matmul float64).

Burst = best of 10 single 8192^3 launches; sustained = back-to-back for ~4 s.
Writes one JSON line (to stdout and, if given, to argv[1]).
"""
import json
import subprocess
import sys
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    flops = 2.0 * n ** 3
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "200"],
        stdout=subprocess.PIPE, text=True)
    reps = max(4, int(4.0 / best))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    sustained_s = e0.elapsed_time(e1) * 1e-3 / reps
    time.sleep(0.3)
    smi.terminate()
    lines = smi.communicate()[0].strip().splitlines()
    clocks = []
    for ln in lines:
        parts = [x.strip() for x in ln.split(",")]
        try:
            clocks.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3]))
        except (ValueError, IndexError):
            pass
    sm = sorted(x[0] for x in clocks) or [0.0]
    out = {
        "what": "cuBLAS DGEMM via torch.matmul float64, 8192^3",
        "fp64_tflops_burst": flops / best / 1e12,
        "fp64_tflops_sustained": flops / sustained_s / 1e12,
        "sustained_reps": reps,
        "sm_mhz_median": sm[len(sm) // 2],
        "sm_max_mhz": max((x[1] for x in clocks), default=0.0),
        "power_w_max": max((x[2] for x in clocks), default=0.0),
        "reasons": sorted({x[3] for x in clocks}),
        "gpu": torch.cuda.get_device_name(0),
    }
    s = json.dumps(out)
    print(s)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
