"""Strang (qHOP M = 1, merge) steps/s on the config-5 grids: the B phase applied by the next
Kronecker propagate's first group (default), as its own pass (KRONOP_BPHASE_PRE=0), or in the
last pass of the propagate before it (KRONOP_BPHASE_FUSED=1)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A, potentials as P

ctx = A.Context(0)
res = {"pre": os.environ.get("KRONOP_BPHASE_PRE", "1"),
       "post_fused": os.environ.get("KRONOP_BPHASE_FUSED", "0")}
for name, (L, cells, k, d) in {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6), "3d499": (8.0, 100, 5, 3)}.items():
    g = A.Grid.sem(L, cells, k, d)
    lap = g.laplacian(ctx)
    b = torch.from_numpy(np.ascontiguousarray(P.separable_sum(g, P.build_potential("harmonic", g)))).cuda()
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * g.node_count()).view(-1, 2))
    spec = A.SplitSpec(quad_points=1, dt=0.005, total_time=0.05, merge_across_steps=True)
    A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=0.01, merge_across_steps=True), lap, b, psi, stationary_eigenvalue=0.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, err, steps = A.evolve(spec, lap, b, psi, stationary_eigenvalue=0.0)
    torch.cuda.synchronize()
    res[name + "_steps_per_s"] = steps / (time.perf_counter() - t0)
    del lap, b, psi, st
    torch.cuda.empty_cache()
print(json.dumps(res))
