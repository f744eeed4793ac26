"""Config-5 small-extent transforms: one kinetic propagate on the 9D n = 9 and 6D n = 29 grids
(complex128) and one 9D solve (real), CUDA events on the context stream (variant libraries via
KRONOP_LIB)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A


def timed(ctx, fn, reps=3):
    fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(reps):
        fn()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ctx = A.Context(0)
res = {"lib": os.environ.get("KRONOP_LIB", "default")}
for name, (L, cells, k, d) in {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6)}.items():
    g = A.Grid.sem(L, cells, k, d)
    lap = g.laplacian(ctx)
    N = g.node_count()
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
    o = torch.empty_like(psi)
    res[name + "_propagate_ms"] = timed(ctx, lambda: lap.propagate(psi, 0.005, out=o))
    ref = o.clone()
    del psi
    if name == "9d":
        b = A.splitmix_uniform(ctx, 4, N)
        x = torch.empty_like(b)
        op = g.separable_operator(ctx, [lambda t: t * t] * d)
        res[name + "_solve_ms"] = timed(ctx, lambda: op.solve(b, out=x))
        res[name + "_solve_checksum"] = float(x.double().abs().sum())
        del b, x, op
    res[name + "_propagate_checksum"] = float(torch.view_as_real(ref).abs().sum())
    del o, ref, lap
    torch.cuda.empty_cache()
print(json.dumps(res))
