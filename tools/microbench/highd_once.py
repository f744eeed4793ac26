"""One complex propagate on the config-5 shapes (for ncu: -k regex:fused_small)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A

ctx = A.Context(0)
which = sys.argv[1] if len(sys.argv) > 1 else "9d"
L, cells, k, d = {"6d": (5.0, 3, 10, 6), "9d": (3.0, 2, 5, 9)}[which]
g = A.Grid.sem(L, cells, k, d)
lap = g.laplacian(ctx)
N = g.node_count()
psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
out = torch.empty_like(psi)
lap.propagate(psi, 0.01, out=out)
torch.cuda.synchronize()
print("ok", which, N)
