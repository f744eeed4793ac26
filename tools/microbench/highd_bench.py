"""Config 5 shapes: complex128 propagate at 6D n=29 (Q10 x 3 cells, L=5) and 9D n=9 (Q5 x 2 cells,
L=3); reports ms per propagate, per-pass GB/s (HBM-bound regime) and steps/s of a Strang step."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A
from paper_2605_20491_b200 import potentials as P

ctx = A.Context(0)
res = {}
for name, (L, cells, k, d, kind) in {"6d_n29": (5.0, 3, 10, 6, "coulomb-3d2"),
                                     "9d_n9": (3.0, 2, 5, 9, "coulomb-3d3")}.items():
    g = A.Grid.sem(L, cells, k, d)
    lap = g.laplacian(ctx)
    N = g.node_count()
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
    out = torch.empty_like(psi)
    for _ in range(2):
        lap.propagate(psi, 0.01, out=out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(ctx.stream)
    for _ in range(reps):
        lap.propagate(psi, 0.01, out=out)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    passes = 2 * d
    bytes_per_pass = 2 * 16 * N
    res[name] = {"n": g.shape[0], "dof": N, "ms_per_propagate": t * 1e3,
                 "gbs_per_pass": passes * bytes_per_pass / t / 1e9,
                 "tflops": 8.0 * g.shape[0] * d * N / t / 1e12}
    del psi, out, lap
    torch.cuda.empty_cache()
print(json.dumps(res))
