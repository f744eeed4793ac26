"""Real-field small-extent transforms at the config-5 sizes: solve and FullOperator apply on the
6D n = 29 and 9D n = 9 grids (the inverse-iteration inner PCG's two transforms), CUDA events."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A

ctx = A.Context(0)
res = {}
for name, (L, cells, k, d) in {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6)}.items():
    g = A.Grid.sem(L, cells, k, d)
    op = g.separable_operator(ctx, [lambda t: t * t] * d, shift=-0.5)
    N = g.node_count()
    b = A.splitmix_uniform(ctx, 4, N)
    v2 = A.splitmix_uniform(ctx, 5, N) + 2.0
    x = torch.empty_like(b)
    fo = A.FullOperator(op, v2)
    for key, fn in (("solve", lambda: op.solve(b, out=x)), ("apply_v2", lambda: fo.apply(b, sigma=0.3, out=x))):
        fn()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(5):
            fn()
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        res["%s_%s_ms" % (name, key)] = e0.elapsed_time(e1) / 5
    del b, v2, x, fo, op
    torch.cuda.empty_cache()
print(json.dumps(res))
