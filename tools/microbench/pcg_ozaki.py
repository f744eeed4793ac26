"""512^3 stirrer PCG (bench secondary setup) with FP64 DMMA vs the INT8 execution precision."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402
from paper_2605_20491_b200 import potentials as P  # noqa: E402

ctx = A.Context(0)
g = A.Grid.sem(8.0, int(sys.argv[1]) if len(sys.argv) > 1 else 27, 19, 3)
pot = P.build_potential("stirrer", g)
op = g.separable_operator(ctx, pot.separable)
v2 = pot.v2_device("cuda:0")
b = A.splitmix_uniform(ctx, 1, g.node_count())
out = {"n": g.shape[0]}
xs = {}
for prec in ("fp64", "ozaki"):
    op.set_precision(prec)
    x = torch.zeros_like(b)
    A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8, max_iter=2))
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    rep = A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8))
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    out[prec] = {"s": e0.elapsed_time(e1) / 1e3, "iterations": rep.iterations,
                 "residual": rep.final_residual}
    xs[prec] = x
out["rel_diff"] = float(torch.linalg.norm(xs["ozaki"] - xs["fp64"]) / torch.linalg.norm(xs["fp64"]))
print(json.dumps(out))
