"""Measurements for the BASELINE.json configs that are not the bench.py headline (one JSON line).

config 3: stirrer 512^3 (Q19 x 27 cells, L=8): PCG time-to-tol at 1e-8 and 1e-12 (seed-1 rhs,
          (-Delta+V1)^-1 preconditioner) and the shifted-inverse-iteration ground state
          (sigma = 0.9 lambda_min, eigen tol 1e-12, inner PCG tol 1e-12, stagnation 100).
config 4: GPE a_u flow at 1024^3 (sep-osc amp 100 quad 1, Q25 x 41 cells, L=8, beta = 1600,
          tau = 1, constant init): seconds and PCG iterations per outer iteration (2 iterations).
"3oz" / "4oz": configs 3 / 4 with kronop_op_set_precision("ozaki") (FP64 emulated on INT8).
config 5: 6D n=29 (coulomb-3d2, L=5, Q10 x 3) and 9D n=9 (coulomb-3d3, L=3, Q5 x 2) complex128:
          one A-propagation (split=kinetic) and Strang steps/s (qHOP M=1, merge, dt=0.005).
All times are device time (CUDA events / synchronised wall clock around device-resident calls).
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


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def config3(ctx, out, prec="fp64"):
    g = A.Grid.sem(8.0, 27, 19, 3)
    pot = P.build_potential("stirrer", g)
    op = g.separable_operator(ctx, pot.separable).set_precision(prec)
    v2 = pot.v2_device()
    b = A.splitmix_uniform(ctx, 1, g.node_count())
    res = {"n": g.shape[0], "dof": g.node_count()}
    for tol in (1e-8, 1e-12):
        x = torch.zeros_like(b)
        rep, t = timed(lambda: A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x,
                                     A.PcgConfig(rel_tol=tol)))
        res["pcg_tol_%g" % tol] = {"seconds": t, "iterations": rep.iterations,
                                   "final_residual": rep.final_residual,
                                   "converged": rep.converged}
    fo = A.FullOperator(op, v2)
    r, t = timed(lambda: A.inverse_iteration(fo, A.InverseIterationConfig(), op.ground_state()))
    res["inverse_iteration"] = {"seconds": t, "eigenvalue": r.eigenvalue,
                                "outer_iterations": r.outer_iterations,
                                "total_inner_iterations": r.total_inner_iterations,
                                "converged": r.converged}
    out["config3_stirrer_512" + ("" if prec == "fp64" else "_" + prec)] = res


def config4(ctx, out, iters=2, prec="fp64"):
    g = A.Grid.sem(8.0, 41, 25, 3)
    pot = P.build_potential("sep-osc", g, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    ham = A.FullOperator(g.separable_operator(ctx, pot.separable).set_precision(prec))
    lap = g.laplacian(ctx).set_precision(prec)
    cfg = A.GpeFlowConfig(kind="au", step=1.0, init="constant", energy_rel_tol=1e-30,
                          max_iterations=iters, record_history=True)
    r, t = timed(lambda: A.gpe_gradient_flow(ham, lap, 1600.0, cfg))
    out["config4_gpe_au_1024" + ("" if prec == "fp64" else "_" + prec)] = {
        "n": g.shape[0], "dof": g.node_count(), "beta": 1600.0, "outer_iterations": r.iterations,
        "seconds_total": t, "seconds_per_outer": t / max(1, r.iterations),
        "pcg_iterations_total": r.linear_solves,
        "pcg_per_outer": r.linear_solves / max(1, r.iterations),
        "energy_trace": [h[1] for h in r.history]}


def config5(ctx, out):
    for name, (L, cells, k, d, kind) in {"6d_n29": (5.0, 3, 10, 6, "coulomb-3d2"),
                                         "9d_n9": (3.0, 2, 5, 9, "coulomb-3d3")}.items():
        g = A.Grid.sem(L, cells, k, d)
        pot = P.build_potential(kind, g, coulomb_softening=0.01 if d == 6 else 0.1)
        lap = g.laplacian(ctx)
        bdiag = torch.from_numpy(P.separable_sum(g, pot) + pot.nonseparable).cuda()
        N = g.node_count()
        psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2)).contiguous()
        o = torch.empty_like(psi)
        lap.propagate(psi, 0.005, out=o)
        _, tp = timed(lambda: [lap.propagate(psi, 0.005, out=o) for _ in range(3)])
        spec = A.SplitSpec(quad_points=1, dt=0.005, total_time=0.05, merge_across_steps=True)
        A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=0.01, merge_across_steps=True),
                 lap, bdiag, psi, stationary_eigenvalue=0.0)
        (st, err, steps), ts = timed(lambda: A.evolve(spec, lap, bdiag, psi,
                                                      stationary_eigenvalue=0.0))
        out["config5_" + name] = {"n": g.shape[0], "d": d, "dof": N,
                                  "ms_per_propagate": tp / 3 * 1e3,
                                  "strang_steps_per_s": steps / ts, "steps": steps}
        del lap, bdiag, psi, o, st
        torch.cuda.empty_cache()


def main():
    ctx = A.Context(0)
    out = {"gpu": torch.cuda.get_device_name(0)}
    which = sys.argv[1:] or ["3", "4", "5"]
    if "3" in which:
        config3(ctx, out)
    if "5" in which:
        config5(ctx, out)
    if "4" in which:
        config4(ctx, out)
    # the same with every transform on the INT8 path (kronop_op_set_precision)
    if "3oz" in which:
        config3(ctx, out, "ozaki")
    if "4oz" in which:
        config4(ctx, out, prec="ozaki")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
