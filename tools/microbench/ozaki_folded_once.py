import sys, torch
sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A
ctx = A.Context(0); g = A.Grid.sem(8.0, 205, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3, folded=True).set_precision("ozaki")
b = A.splitmix_uniform(ctx, 1, g.node_count()); x = torch.empty_like(b)
for _ in range(2): op.solve(b, out=x)
torch.cuda.synchronize()
