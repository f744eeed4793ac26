"""Strang split-step (bench secondary setup, 499^3) with the dense vs the even/odd folded kinetic
operator: steps/s and the final-state difference."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A  # noqa: E402
from paper_2605_20491_b200 import potentials as P  # noqa: E402

ctx = A.Context(0)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = A.Grid.sem(8.0, cells, 5, 3)
pot = P.build_potential("sep-osc", g, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
bdiag = torch.from_numpy(np.array(P.separable_sum(g, pot))).cuda()
box = g.sample(lambda c: np.sin(np.pi * (c[0] + 8.0) / 16.0) * np.sin(np.pi * (c[1] + 8.0) / 16.0)
               * np.sin(np.pi * (c[2] + 8.0) / 16.0))
psi0 = torch.from_numpy(box.astype(np.complex128)).cuda()
spec = A.SplitSpec(quad_points=1, composition="single", dt=5e-3, total_time=0.1,
                   merge_across_steps=True)
out = {"n": g.shape[0]}
states = {}
for name, folded in (("dense", False), ("folded", True), ("ozaki", False)):
    lap = g.laplacian(ctx, folded=folded)
    if name == "ozaki":
        lap.set_precision("ozaki")
    A.evolve(A.SplitSpec(quad_points=1, dt=5e-3, total_time=1e-2, merge_across_steps=True), lap,
             bdiag, psi0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    state, err, steps = A.evolve(spec, lap, bdiag, psi0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    out[name] = {"steps_per_s": steps / t, "steps": steps, "s": t}
    states[name] = state
    del lap
for k in ("folded", "ozaki"):
    d = states[k] - states["dense"]
    out["rel_diff_" + k] = float(torch.linalg.norm(d) / torch.linalg.norm(states["dense"]))
print(json.dumps(out))
