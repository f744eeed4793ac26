"""Time the Ozaki complex propagate against the DMMA propagate at n^3."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 205
ctx = A.Context(0)
g = A.Grid.sem(8.0, cells, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3)
N = g.node_count()
psi = torch.view_as_complex(A.splitmix_uniform(ctx, 7, 2 * N).view(-1, 2))
ref = op.propagate(psi, 0.01)
x = torch.empty_like(psi)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"n": g.shape[0]}
for m in ["fp64", "ozaki"]:
    f = (lambda: op.propagate(psi, 0.01, out=x)) if m == "fp64" else (
        lambda: op.propagate_lowp(psi, 0.01, m, out=x))
    f()
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
    e0.record(ctx.stream)
    for _ in range(2):
        f()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    out[m] = {"ms": e0.elapsed_time(e1) / 2, "rel": err}
print(json.dumps(out))
