"""Time the C-ABI host entry point (pinned H2D + solve + D2H) at 1024^3, several repetitions."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402

ctx = A.Context(0)
g = A.Grid.sem(8.0, 205, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3)
N = g.node_count()
b = A.splitmix_uniform(ctx, 1, N)
bh = torch.empty(N, dtype=torch.float64, pin_memory=True)
xh = torch.empty(N, dtype=torch.float64, pin_memory=True)
bh.copy_(b.cpu())
bn, xn = bh.numpy(), xh.numpy()
op.solve_host(bn, xn)
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    op.solve_host(bn, xn)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"ms": [t * 1e3 for t in ts], "gdofs": [N / t / 1e9 for t in ts]}))
