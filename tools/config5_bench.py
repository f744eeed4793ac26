"""BASELINE configs[4]: approximated qHOP and Magnus-2 (Yoshida) splitting for the multi-body
Coulomb Hamiltonians in 6D and 9D, complex128 on one B200 (one JSON line on stdout).

Workloads (potentials.cpp:40-54,116-127; splitting.cpp:107-146):
  6d: coulomb-3d2, delta = 0.01, c = 1, L = 5, SEM Q10 x 3 cells (n = 29, 29^6 = 5.9e8 DoF),
      A = -Delta (split=kinetic), B = V_trap + V_Coulomb;
  9d: coulomb-3d3, delta = 0.1, c = 1, L = 3, SEM Q5 x 2 cells (n = 9, 9^9 = 3.9e8 DoF),
      A = -Delta + V_trap (split=kinetic+v1), B = V_Coulomb.
Reference: the stationary solution e^{-i lambda_1 T} u_1 with (lambda_1, u_1) from PCG shifted
inverse iteration (ground_state.cpp:35-99, the reference's defaults: sigma = 0.9 lambda_min of the
separable part, eigen tol 1e-12, inner PCG tol 1e-12, stagnation window 100). T = 0.1, merge on.
For each (composition, M, dt): error, observed rate, device seconds of the march, steps/s and
propagations/s. The paper's runs are complex64 on GH200 (tables at); these are
complex128 (FP64) throughout.

  python tools/config5_bench.py [6d|9d|both] [--quick]
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_20491_b200 import api as A  # noqa: E402
from paper_2605_20491_b200 import potentials as P  # noqa: E402

SETUPS = {
    "6d": dict(kind="coulomb-3d2", delta=0.01, L=5.0, cells=3, k=10, d=6, split="kinetic"),
    "9d": dict(kind="coulomb-3d3", delta=0.1, L=3.0, cells=2, k=5, d=9, split="kinetic+v1"),
}
# (composition, M, dt grid): the paper's tables / figure
RUNS = {
    "single": {1: [0.1, 0.02, 0.005], 3: [0.1, 0.02, 0.005], 5: [0.1, 0.02, 0.005],
               7: [0.1, 0.02, 0.005]},
    "yoshida": {1: [0.1, 0.01, 0.005], 3: [0.1, 0.01, 0.005], 5: [0.1, 0.01], 7: [0.1, 0.01]},
}


def sync_time(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def run(name, quick=False):
    s = SETUPS[name]
    ctx = A.Context(0)
    g = A.Grid.sem(s["L"], s["cells"], s["k"], s["d"])
    pot = P.build_potential(s["kind"], g, coulomb_softening=s["delta"])
    sep = g.separable_operator(ctx, pot.separable)
    v2 = pot.v2_device()
    res = {"workload": "%s delta=%g L=%g Q%d x %d cells, n=%d, %dD, N=%d, split=%s, complex128"
                       % (s["kind"], s["delta"], s["L"], s["k"], s["cells"], g.shape[0], s["d"],
                          g.node_count(), s["split"])}
    ev, t = sync_time(lambda: A.inverse_iteration(A.FullOperator(sep, v2),
                                                  A.InverseIterationConfig(), sep.ground_state()))
    res["ground_state"] = {"eigenvalue": ev.eigenvalue, "outer_iterations": ev.outer_iterations,
                           "total_inner_iterations": ev.total_inner_iterations,
                           "seconds": t, "converged": ev.converged}
    if s["split"] == "kinetic":
        a_op = g.laplacian(ctx)
        bdiag = torch.from_numpy(np.ascontiguousarray(P.separable_sum(g, pot))).cuda() + v2
    else:
        a_op = sep
        bdiag = v2
    psi0 = ev.eigenvector.to(torch.complex128)
    del v2
    torch.cuda.empty_cache()
    # one A-propagation and one fused propagate + B phase (the unit of a split step)
    o = torch.empty_like(psi0)
    a_op.propagate(psi0, 0.005, out=o)
    _, t1 = sync_time(lambda: [a_op.propagate(psi0, 0.005, out=o) for _ in range(3)])
    res["propagate_ms"] = t1 / 3 * 1e3
    del o
    runs = {}
    for comp, ms in RUNS.items():
        for m, dts in ms.items():
            if quick and (m > 3 or comp == "yoshida" and m > 1):
                continue
            rows = []
            for dt in dts:
                spec = A.SplitSpec(quad_points=m, composition=comp, dt=dt, total_time=0.1,
                                   merge_across_steps=True)
                (st, err, steps), t = sync_time(lambda: A.evolve(
                    spec, a_op, bdiag, psi0, stationary_eigenvalue=ev.eigenvalue))
                del st
                props = steps * (3 if comp == "yoshida" else 1) * m  # merged A-propagations
                row = {"dt": dt, "steps": steps, "error": err, "seconds": t,
                       "steps_per_s": steps / t, "propagations_per_s": props / t}
                if rows:
                    row["rate"] = math.log(rows[-1]["error"] / err) / math.log(rows[-1]["dt"] / dt)
                rows.append(row)
            runs["%s_M%d" % (comp, m)] = rows
    res["splitting"] = runs
    return res


def main():
    which = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "both"
    quick = "--quick" in sys.argv
    out = {}
    for name in (["6d", "9d"] if which == "both" else [which]):
        out[name] = run(name, quick)
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
