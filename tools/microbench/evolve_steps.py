"""Per-step cost of evolve (Strang, merged) on the config-5 9D grid vs the bare propagate, for
two run lengths (setup amortisation), CUDA events on the context stream."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A, potentials as P

ctx = A.Context(0)
name = sys.argv[1] if len(sys.argv) > 1 else "9d"
L, cells, k, d = {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6)}[name]
g = A.Grid.sem(L, cells, k, d)
lap = g.laplacian(ctx)
N = g.node_count()
b = torch.from_numpy(np.ascontiguousarray(P.separable_sum(g, P.build_potential("harmonic", g)))).cuda()
psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
o = torch.empty_like(psi)
lap.propagate(psi, 0.005, out=o)
torch.cuda.synchronize()
e0.record(ctx.stream)
for _ in range(5):
    lap.propagate(psi, 0.005, out=o)
e1.record(ctx.stream)
torch.cuda.synchronize()
res = {"propagate_ms": e0.elapsed_time(e1) / 5}
del o
for T in (0.05, 0.2):
    A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=0.01, merge_across_steps=True), lap, b, psi, stationary_eigenvalue=0.0)
    torch.cuda.synchronize()
    c0 = ctx.launch_count()
    e0.record(ctx.stream)
    st, err, steps = A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=T, merge_across_steps=True), lap, b, psi, stationary_eigenvalue=0.0)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    res["T=%g" % T] = {"steps": steps, "ms_per_step": e0.elapsed_time(e1) / steps, "launches": ctx.launch_count() - c0}
    del st
print(json.dumps(res))
