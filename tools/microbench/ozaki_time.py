"""Time the Ozaki (INT8 tcgen05) FP64-emulated solve against the DMMA FP64 solve at n^3."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 205
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["ozaki", "ozaki6", "ozaki5"]
ctx = A.Context(0)
g = A.Grid.sem(8.0, cells, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3)
b = A.splitmix_uniform(ctx, 1, g.node_count())
x = torch.empty_like(b)
ref = op.solve(b)
out = {"n": g.shape[0]}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for m in ["fp64"] + modes:
    f = (lambda: op.solve(b, out=x)) if m == "fp64" else (lambda: op.solve_lowp(b, m, out=x))
    f()
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
    e0.record(ctx.stream)
    for _ in range(3):
        f()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    out[m] = {"ms": e0.elapsed_time(e1) / 3, "rel": err}
print(json.dumps(out))
