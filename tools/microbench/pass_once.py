import sys, torch
sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A
ctx = A.Context(0); g = A.Grid.sem(8.0, 205, 5, 3); op = g.separable_operator(ctx, [lambda t: t * t] * 3)
b = A.splitmix_uniform(ctx, 1, g.node_count()); y = torch.empty_like(b)
for ax in range(3): op.transform_pass(b, ax, True, out=y)
torch.cuda.synchronize()
