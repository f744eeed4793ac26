"""BASELINE configs[3] diagnostics: where the a_u GPE flow's time goes at 1024^3.

Runs the product driver (kronop_gpe_gradient_flow, device-resident inner PCG) for K outer
iterations of the a_u flow (sep-osc V1 amp 100 quad 1, L = 8, SEM Q25 x 41 cells = 1024^3,
beta = 1600, tau = 1, constant init, the reference's inner PcgConfig: tol 1e-12, max 500,
stagnation window 100 -- harness.cpp:342-343, gpe.hpp:38), then replays the same K outer
iterations step by step through the public API (gpe.cpp:118-157 restated with api.pcg and
record_history=True) to record each inner solve's residual history: iterations, the best
residual reached, and whether the solve stopped on the tolerance or on the stagnation window.
The replay's energies must equal the driver's (same kernels, same order).

  python tools/config4_histories.py [K] [cells]     (defaults: 3 outer iterations, 41 cells)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_20491_b200 import api as A  # noqa: E402
from paper_2605_20491_b200 import potentials as P  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cells = int(sys.argv[2]) if len(sys.argv) > 2 else 41
    ctx = A.Context(0)
    g = A.Grid.sem(8.0, cells, 25, 3)
    pot = P.build_potential("sep-osc", g, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    sep = g.separable_operator(ctx, pot.separable)
    ham = A.FullOperator(sep)
    beta = 1600.0
    out = {"grid": "Q25 x %d cells, n = %d, N = %d" % (cells, g.shape[0], g.node_count()),
           "beta": beta, "outer_iterations": K}
    cfg = A.GpeFlowConfig(kind="au", step=1.0, energy_rel_tol=1e-30, max_iterations=K,
                          record_history=True, init="constant")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = A.gpe_gradient_flow(ham, g.laplacian(ctx), beta, cfg)
    torch.cuda.synchronize()
    out["driver"] = {"seconds": time.perf_counter() - t0,
                     "rows": [{"iteration": int(h[0]), "energy": h[1], "rel_change": h[2],
                               "linear_solves": int(h[3]), "seconds": h[4]} for h in r.history]}
    del r
    torch.cuda.empty_cache()
    # replay with inner residual histories (gpe.cpp:76-157)
    N = g.node_count()
    mass = g.mass
    u = torch.ones(N, dtype=torch.float64, device="cuda")
    u /= A.norm(ctx, u, g.shape, mass)
    w = torch.zeros_like(u)
    inner = []
    energies = []
    for it in range(K):
        dg = beta * (u * u)  # k_beta_square: beta (u u)
        t1 = time.perf_counter()
        rep = A.pcg(A.apply_map(sep, dg), A.solve_map(sep), u, w,
                    A.PcgConfig(rel_tol=1e-12, max_iter=500, stagnation_window=100,
                                record_history=True))
        torch.cuda.synchronize()
        hist = np.array(rep.history)
        inner.append({"outer": it + 1, "iterations": rep.iterations,
                      "converged": rep.converged, "final_residual": rep.final_residual,
                      "best_residual": float(hist.min()),
                      "iteration_of_best": int(hist.argmin()),
                      "stopped_by": "tolerance" if rep.converged else (
                          "stagnation window" if rep.iterations < 500 else "max_iter"),
                      "seconds": time.perf_counter() - t1,
                      "history_every_10": [float(x) for x in hist[::10]]})
        uu = A.inner(ctx, u, u, g.shape, mass)
        wu = A.inner(ctx, w, u, g.shape, mass)
        grad = u - (uu / wu) * w
        u = u - 1.0 * grad
        u /= A.norm(ctx, u, g.shape, mass)
        energies.append(A.gpe_energy(ham, beta, u))
        print(json.dumps(inner[-1])[:300], flush=True)
    out["replay"] = {"inner": inner, "energies": energies}
    out["replay_vs_driver_max_rel"] = max(
        abs(e - row["energy"]) / abs(row["energy"]) for e, row in zip(energies, out["driver"]["rows"]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
