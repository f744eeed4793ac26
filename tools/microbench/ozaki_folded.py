"""1024^3 solve: dense DMMA / folded DMMA / dense Ozaki / folded Ozaki (ms, rel. diff)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 205
ctx = A.Context(0)
g = A.Grid.sem(8.0, cells, 5, 3)
f = [lambda t: t * t] * 3
ops = {"dense": g.separable_operator(ctx, f),
       "folded": g.separable_operator(ctx, f, folded=True)}
b = A.splitmix_uniform(ctx, 1, g.node_count())
ref = ops["dense"].solve(b)
x = torch.empty_like(b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"n": g.shape[0]}
for prec in ("fp64", "ozaki"):
    for name, op in ops.items():
        op.set_precision(prec)
        op.solve(b, out=x)
        torch.cuda.synchronize()
        err = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
        e0.record(ctx.stream)
        for _ in range(3):
            op.solve(b, out=x)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        out[name + "_" + prec] = {"ms": e0.elapsed_time(e1) / 3, "rel": err}
print(json.dumps(out))
