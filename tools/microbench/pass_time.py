"""Per-axis FP64 pass times and the solve time at 1024^3 (CUDA events on the context stream)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402

ctx = A.Context(0)
g = A.Grid.sem(8.0, int(sys.argv[1]) if len(sys.argv) > 1 else 205, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3)
b = A.splitmix_uniform(ctx, 1, g.node_count())
y = torch.empty_like(b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {}
for ax in range(3):
    op.transform_pass(b, ax, True, out=y)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(3):
        op.transform_pass(b, ax, True, out=y)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    out["axis%d_ms" % ax] = e0.elapsed_time(e1) / 3
op.solve(b, out=y)
torch.cuda.synchronize()
e0.record(ctx.stream)
for _ in range(3):
    op.solve(b, out=y)
e1.record(ctx.stream)
torch.cuda.synchronize()
out["solve_ms"] = e0.elapsed_time(e1) / 3
print(json.dumps(out))
