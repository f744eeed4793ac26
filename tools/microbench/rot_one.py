"""One kinetic propagate on the 9D n = 9 or 6D n = 29 grid (for ncu captures of fused_rot)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A
ctx = A.Context(0)
L, cells, k, d = {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6)}[sys.argv[1]]
g = A.Grid.sem(L, cells, k, d)
lap = g.laplacian(ctx)
psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * g.node_count()).view(-1, 2))
o = lap.propagate(psi, 0.005)
torch.cuda.synchronize()
print("ok")
