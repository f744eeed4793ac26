"""One 512^3 stirrer PCG solve (BASELINE config 3), for ncu captures of the device-resident PCG
vector kernels (-k regex:k_pcg|k_dot|k_copy)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A  # noqa: E402
from paper_2605_20491_b200 import potentials as P  # noqa: E402

ctx = A.Context(0)
g = A.Grid.sem(8.0, 27, 19, 3)
pot = P.build_potential("stirrer", g)
op = g.separable_operator(ctx, pot.separable)
b = A.splitmix_uniform(ctx, 1, g.node_count())
x = torch.zeros_like(b)
rep = A.pcg(A.apply_map(op, pot.v2_device()), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8))
torch.cuda.synchronize()
print("pcg", rep.iterations, rep.final_residual)
