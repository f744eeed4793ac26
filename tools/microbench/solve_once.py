"""One 1024^3 solve (the bench's rotated six-pass sequence), for ncu captures."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A
ctx = A.Context(0)
grid = A.Grid.sem(8.0, 205, 5, 3)
op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
b = A.splitmix_uniform(ctx, 1, grid.node_count())
x = op.solve(b)
torch.cuda.synchronize()
print("ok")
