"""Pin the CPU oracle against the reference's own known answers (proj/tests/acceptance.cpp).

Test infrastructure only. Runs each acceptance criterion of the reference suite on the oracle and
writes the measured numbers next to the reference's golden values into
tests/golden/oracle_acceptance.json (committed). Usage:

    python oracle/pin_golden.py [criterion ...]      # default: all cheap + expensive ones

Where the reference's desk-scale grid is not converged enough to reach a golden value quoted from
the paper's 599^3-1099^3 runs, the script also runs a refinement study and records the converged
value next to the desk-grid value.
"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import kronop_oracle as K  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "oracle_acceptance.json")


def trap(dim):
    return dict(osc_amplitude=100.0, quad_coeffs=[1.0] * dim)


def solve_rel_error(cells, degree):
    """acceptance.cpp:85-103."""
    g = K.Grid.sem(1.0, cells, degree, 3)
    pot = K.build_potential("sep-osc", g, quad_coeffs=[1.0, 2.0, 3.0], osc_amplitude=1600.0)
    op = g.separable_operator(pot.separable)
    ustar = g.sample(lambda c: np.sin(np.pi * c[0]) * np.sin(2 * np.pi * c[1]) *
                     np.sin(3 * np.pi * c[2]))
    rhs = (14.0 * math.pi * math.pi + K.separable_sum_field(g, pot)) * ustar
    u = op.solve(rhs)
    return float(np.linalg.norm(u - ustar) / np.linalg.norm(ustar))


def c1():
    e16, e32, e64 = solve_rel_error(16, 2), solve_rel_error(32, 2), solve_rel_error(64, 2)
    e10 = solve_rel_error(8, 10)
    rate = math.log2(e16 / e32)
    return {
        "1a_rate_16_32": rate, "1a_need": ">= 3.7", "1a_pass": rate >= 3.7,
        "1a_errors": [e16, e32, e64], "1a_rate_32_64": math.log2(e32 / e64),
        "1a_note": "pre-asymptotic pair (acceptance.cpp:122-124 says so); rate -> 4 = k+2 on refinement,"
                   " and the 550-cell extrapolation (e32*(32/550)^4) matches PAPER.md:341 (1.93e-9)",
        "1b_err_q10_79": e10, "1b_pass": e10 <= 1e-8,
    }


def c2():
    """Dense-oracle equivalence (acceptance.cpp:131-200)."""
    trapf = lambda x: x * x
    worst = {"apply": 0.0, "solve": 0.0, "prop": 0.0}
    for bases, seed in (([K.assemble_sem(1.0, 13, 1), K.assemble_sem(1.0, 7, 2)], 101),
                        ([K.assemble_sem(1.0, 7, 1)] * 3, 102)):
        grid = K.Grid(list(bases))
        d = grid.dim
        op = K.FullOperator(grid.separable_operator([trapf] * d),
                            grid.sample(lambda c: 2.0 * np.exp(-sum((c[a] - 0.3) ** 2
                                                                    for a in range(d)))))
        ops = [K.dense_axis_operator(b, trapf) for b in bases]
        syms = [K.dense_sym_axis_operator(b, trapf) for b in bases]
        dense_full = K.dense_assemble(ops, op.diagonal)
        dense_sep = K.dense_assemble(ops)
        mw = K.mass_field(grid.shape, grid.mass)
        sq = np.sqrt(mw)
        t = 0.083
        uprop = (1.0 / sq)[:, None] * K.expm_hermitian(K.dense_assemble(syms), t) * sq[None, :]
        n = grid.node_count()
        vals = K.uniform_pm1(seed, 20 * 2 * n)
        pos = 0
        for _ in range(20):
            v = vals[pos:pos + n]
            pos += n
            hv = op.apply(v)
            ref = dense_full @ v
            worst["apply"] = max(worst["apply"], np.linalg.norm(hv - ref) / np.linalg.norm(ref))
            sol = op.sep.solve(v)
            sref = np.linalg.solve(dense_sep, v)
            worst["solve"] = max(worst["solve"], np.linalg.norm(sol - sref) / np.linalg.norm(sref))
            im = vals[pos:pos + n]
            pos += n
            psi = v + 1j * im
            pr = op.sep.propagate(psi, t)
            pref = uprop @ psi
            worst["prop"] = max(worst["prop"], np.linalg.norm(pr - pref) / np.linalg.norm(pref))
    return {"2_worst": worst, "2_pass": all(x <= 1e-10 for x in worst.values())}


def pcg_iterations(kind, half_width, cells, degree, laplacian_precond, seed):
    """acceptance.cpp:202-236."""
    g = K.Grid.sem(half_width, cells, degree, 3)
    pot = K.build_potential(kind, g)
    op = K.build_full_operator(g, pot)
    b = K.seeded_field(g.shape, seed)
    x = np.zeros_like(b)
    cfg = K.PcgConfig(rel_tol=1e-8)
    if laplacian_precond:
        lap = g.laplacian()
        v1 = K.separable_sum_field(g, pot)
        if pot.nonseparable is not None:
            v1 = v1 + pot.nonseparable
        kin = K.FullOperator(lap, v1)
        rep = K.pcg(kin.apply, lap.solve, b, x, cfg)
    else:
        rep = K.pcg(op.apply, op.sep.solve, b, x, cfg)
    return rep.iterations if rep.converged else -rep.iterations


def c3():
    st = [pcg_iterations("stirrer", l, c, 6, False, 1) for l in (8.0, 10.0) for c in (8, 16)]
    q47 = pcg_iterations("quartic", 8.0, 8, 6, False, 1)
    q95 = pcg_iterations("quartic", 8.0, 16, 6, False, 1)
    l47 = pcg_iterations("quartic", 8.0, 8, 6, True, 1)
    l95 = pcg_iterations("quartic", 8.0, 16, 6, True, 1)
    gain = min(abs(l47) / q47, abs(l95) / q95)
    return {"3_stirrer": st, "3a_pass": max(st) <= 10, "3b_pass": max(st) - min(st) <= 2,
            "3_quartic": [q47, q95], "3c_pass": abs(q47 - q95) <= 3,
            "3_laplacian": [l47, l95], "3d_gain": gain, "3d_pass": gain >= 5.0}


def c5():
    g = K.Grid.sem(8.0, 8, 10, 3)
    pot = K.build_potential("sep-osc", g, **trap(3))
    op = K.FullOperator(g.separable_operator(pot.separable))
    r = K.inverse_iteration(op, K.InverseIterationConfig(), np.ones(g.node_count()), g.mass)
    ref = 23.2878438176
    conv = {}
    for cells in (12, 16, 24):
        gg = K.Grid.sem(8.0, cells, 10, 3)
        pp = K.build_potential("sep-osc", gg, **trap(3))
        conv[gg.shape[0]] = 3.0 * float(gg.separable_operator(pp.separable).axes[0].eigenvalues[0])
    return {"5_lambda_79": r.eigenvalue, "5_rel": abs(r.eigenvalue - ref) / ref,
            "5a_pass": abs(r.eigenvalue - ref) / ref <= 1e-6,
            "5_outer": r.outer_iterations, "5b_pass": r.outer_iterations <= 15,
            "5c_pass": r.converged,
            "5_refinement_lambda": conv,
            "5_refined_rel_239": abs(conv[239] - ref) / ref,
            "5_note": "golden value is PAPER.md:946 at 599^3; at 79^3 the Q10 discretisation error is"
                      " 2.1e-5, on refinement the oracle reaches it (239^3: see 5_refined_rel_239)"}


def c4():
    """acceptance.cpp:262-289: preconditioned-spectrum clustering for the bump V2 over
    n in {49, 99} x L in {8, 16}: identical outlier counts, condition numbers within 5%."""
    trap_f = lambda x: x * x
    bump = lambda x: 8.0 * np.exp(-(x - 1.0) * (x - 1.0))
    counts, kappas = [], []
    for half in (8.0, 16.0):
        for cells in (2, 4):
            b = K.assemble_sem(half, cells, 25)
            v2 = np.array([bump(float(x)) for x in b.nodes])
            _, out, kappa = K.clustering_report([K.dense_sym_axis_operator(b, trap_f)], v2, 0.1)
            counts.append(out)
            kappas.append(kappa)
    kmin, kmax = min(kappas), max(kappas)
    return {"4_outliers": counts, "4a_pass": len(set(counts)) == 1, "4_kappa": kappas,
            "4b_pass": (kmax - kmin) <= 0.05 * kmin}


def c6():
    """acceptance.cpp:310-345: Hermite axes. 1-D oscillator levels {1,3,5,7}; 3-D lambda_1 = 3 by
    inverse iteration on Grid::hermite(40, 3); 99^3 solve residual with the accuracy potential."""
    b40 = K.hermite_basis(40)
    ax = K.build_hermite_axis(b40, lambda x: x * x)
    worst = float(np.max(np.abs(ax.eigenvalues[:4] - np.array([1.0, 3.0, 5.0, 7.0]))))
    g = K.Grid.hermite(40, 3)
    op = K.FullOperator(g.separable_operator([lambda x: x * x] * 3))
    r = K.inverse_iteration(op, K.InverseIterationConfig(), np.ones(g.node_count()), g.mass)
    g99 = K.Grid.hermite(99, 3)
    pot = K.build_potential("sep-osc", g99, osc_amplitude=1600.0, quad_coeffs=[1.0, 2.0, 3.0])
    h = g99.separable_operator(pot.separable)
    f = g99.sample(lambda c: np.sin(np.pi / 2 * (c[0] + 1.0)) * np.sin(np.pi * (c[1] + 1.0))
                   * np.sin(1.5 * np.pi * (c[2] + 1.0))
                   * np.exp(-(c[0] ** 2 + c[1] ** 2 + c[2] ** 2) / 4.0))
    u = h.solve(f)
    res = float(np.linalg.norm(h.apply(u) - f) / np.linalg.norm(f))
    return {"6_levels_err": worst, "6a_pass": worst <= 1e-9, "6_lambda": r.eigenvalue,
            "6b_pass": abs(r.eigenvalue - 3.0) <= 1e-9, "6_outer": r.outer_iterations,
            "6_residual_99": res, "6c_pass": res <= 1e-10}


def c7():
    cfg = K.InverseIterationConfig()
    grids = [K.Grid.sem(8.0, 2, 20, 3), K.Grid.sem(8.0, 4, 20, 3)]
    mk = lambda g: K.build_full_operator(g, K.build_potential("stirrer", g))
    pair, levels = K.multilevel_ground_state(grids, mk, cfg)
    ref = 5.286155366963
    fine = mk(grids[1])
    cold = K.inverse_iteration(fine, cfg, fine.sep.ground_state(), grids[1].mass)
    return {"7_lambda": pair.eigenvalue, "7_rel": abs(pair.eigenvalue - ref) / ref,
            "7a_pass": abs(pair.eigenvalue - ref) / ref <= 1e-6, "7_levels": levels,
            "7_cold_outer": cold.outer_iterations,
            "7b_pass": levels[1][1] < cold.outer_iterations}


def c8():
    g = K.Grid.sem(8.0, 5, 20, 3)
    pot = K.build_potential("sep-osc", g, **trap(3))
    prob = K.GpeProblem(K.FullOperator(g.separable_operator(pot.separable)), g.laplacian(), 0.0,
                        g.mass)

    def flow(beta, kind, init, tol):
        prob.beta = beta
        cfg = K.GpeFlowConfig(kind=kind, init=init, step=0.1 if kind == "h1" else 1.0,
                              energy_rel_tol=tol, max_iterations=40000)
        return K.gpe_gradient_flow(prob, cfg)
    out = {}
    h1 = flow(10.0, "h1", "eigenfunction", 1e-13)
    out.update({"8_b10_E": h1.energy, "8_b10_lambda": h1.eigenvalue, "8_b10_iters": h1.iterations,
                "8a_pass": abs(h1.energy - 14.1965761916) / 14.1965761916 <= 1e-6,
                "8b_pass": abs(h1.eigenvalue - 32.4916917439) / 32.4916917439 <= 1e-6})
    au = flow(10.0, "au", "eigenfunction", 1e-13)
    agree = abs(au.energy - h1.energy) / abs(h1.energy)
    out.update({"8_b10_au_E": au.energy, "8_b10_au_iters": au.iterations, "8c_agree": agree,
                "8c_pass": agree <= 1e-10})
    h1c = flow(10.0, "h1", "constant", 1e-13)
    out.update({"8_b10_const_iters": h1c.iterations, "8d_pass": h1.iterations < h1c.iterations})
    b100 = flow(100.0, "h1", "eigenfunction", 1e-13)
    out.update({"8_b100_E": b100.energy,
                "8e_pass": abs(b100.energy - 20.6824463703) / 20.6824463703 <= 1e-6})
    b1600 = flow(1600.0, "h1", "constant", 1e-13)
    out.update({"8_b1600_E": b1600.energy, "8_b1600_iters": b1600.iterations,
                "8f_pass": abs(b1600.energy - 33.80227900547) / 33.80227900547 <= 1e-5})
    return out


def lsq_slope(dts, errs):
    x, y = np.log(dts), np.log(errs)
    n = len(x)
    return float((n * np.sum(x * y) - x.sum() * y.sum()) / (n * np.sum(x * x) - x.sum() ** 2))


def c9():
    g = K.Grid.sem(8.0, 4, 8, 3)
    pot = K.build_potential("sep-osc", g, **trap(3))
    full = g.separable_operator(pot.separable)
    a = g.laplacian()
    b = K.separable_sum_field(g, pot)
    psi0 = K.box_state(g, 8.0).astype(np.complex128)

    def err(dt, total, m, comp):
        spec = K.SplitSpec(quad_points=m, composition=comp, dt=dt, total_time=total,
                           merge_across_steps=True)
        return K.evolve(spec, a, b, psi0, exact=full)[1]
    out = {}
    dts = [0.02, 0.01, 0.005]
    last = {}
    for m in (1, 3, 5):
        errs = [err(dt, 0.1, m, "single") for dt in dts]
        s = lsq_slope(dts, errs)
        out["9a_M%d_rate" % m] = s
        out["9a_M%d_errors" % m] = errs
        out["9a_M%d_pass" % m] = 1.8 <= s <= 2.2
        last[m] = errs[-1]
    out["9b_ratio"] = last[1] / last[3]
    out["9b_pass"] = out["9b_ratio"] >= 4.0
    for m in (1, 3):
        errs = [err(dt, 1.0, m, "yoshida") for dt in (0.2, 0.1, 0.05)]
        s = lsq_slope([0.2, 0.1, 0.05], errs)
        out["9c_M%d_rate" % m] = s
        out["9c_M%d_errors" % m] = errs
        out["9c_M%d_pass" % m] = 3.5 <= s <= 4.5
        errs2 = [err(dt, 1.0, m, "yoshida") for dt in (0.02, 0.01, 0.005)]
        out["9c_M%d_rate_small_dt" % m] = lsq_slope([0.02, 0.01, 0.005], errs2)
    return out


def c10():
    g = K.Grid.sem(8.0, 2, 20, 3)
    pot = K.build_potential("stirrer", g)
    op = K.build_full_operator(g, pot)
    pair = K.inverse_iteration(op, K.InverseIterationConfig(), op.sep.ground_state(), g.mass)
    psi0 = pair.eigenvector.astype(np.complex128)
    b_all = K.separable_sum_field(g, pot) + pot.nonseparable

    def err(a, b, dt):
        spec = K.SplitSpec(quad_points=1, dt=dt, total_time=0.1, merge_across_steps=True)
        return K.evolve(spec, a, b, psi0, stationary_eigenvalue=pair.eigenvalue)[1]
    v1_01, v1_005 = err(op.sep, pot.nonseparable, 0.01), err(op.sep, pot.nonseparable, 0.005)
    lap = g.laplacian()
    k01, k005 = err(lap, b_all, 0.01), err(lap, b_all, 0.005)
    rv, rk = math.log2(v1_01 / v1_005), math.log2(k01 / k005)
    return {"10_lambda": pair.eigenvalue, "10_errors": [v1_01, v1_005, k01, k005],
            "10a_pass": v1_01 <= k01 and v1_005 <= k005, "10_rates": [rv, rk],
            "10b_pass": 1.8 <= rv <= 2.2 and 1.8 <= rk <= 2.2}


def c11():
    g = K.Grid.sem(8.0, 7, 7, 1)
    basis = g.axes[0]
    n = basis.size
    a = g.laplacian()
    pot = K.build_potential("sep-osc", g, **trap(1))
    b = g.sample(lambda c: pot.separable_vec[0](c[0]))
    psi = K.seeded_complex_field((n,), 7)
    psi = psi / np.linalg.norm(psi)
    m = 3
    asym = K.dense_sym_axis_operator(basis, lambda x: 0.0)
    sq = np.sqrt(basis.mass)
    nodes, weights = K.gauss_legendre(m)

    def one(h):
        omega = np.zeros((n, n), dtype=complex)
        for k in range(m):
            sk = h * (1.0 + nodes[k]) / 2.0
            wk = weights[k] / 2.0
            ek = K.expm_hermitian(asym, -sk)
            omega += wk * (ek * b[None, :]) @ ek.conj().T
        uref = (1.0 / sq)[:, None] * (K.expm_hermitian(asym, h) @ K.expm_hermitian(omega, h)) \
            * sq[None, :]
        return float(np.linalg.norm(K.qhop_step(a, b, psi, h, m) - uref @ psi))
    ratio = one(0.01) / one(0.005)
    return {"11_ratio": ratio, "11a_pass": 6.0 <= ratio <= 10.0}


def c12():
    def ground(delta):
        cfg = K.InverseIterationConfig(shift_mode="offset")
        cfg.inner.rel_tol = 1e-9
        grids = [K.Grid.sem(8.0, 2, 10, 4), K.Grid.sem(8.0, 3, 10, 4)]
        mk = lambda g: K.build_full_operator(g, K.build_potential("coulomb-2d2", g,
                                                                  coulomb_softening=delta))
        return K.multilevel_ground_state(grids, mk, cfg)[0].eigenvalue
    l01 = ground(0.1)
    l001 = ground(0.01)
    ref = 5.060514417326
    return {"12_lambda_d01": l01, "12_rel": abs(l01 - ref) / ref, "12a_pass": abs(l01 - ref) / ref <= 1e-4,
            "12_lambda_d001": l001, "12b_pass": l001 > l01}


def c13():
    g = K.Grid.sem(8.0, 4, 8, 3)
    pot = K.build_potential("sep-osc", g, **trap(3))
    full = g.separable_operator(pot.separable)
    a = g.laplacian()
    b = K.separable_sum_field(g, pot)
    psi0 = K.box_state(g, 8.0).astype(np.complex128)
    spec = K.SplitSpec(quad_points=1, dt=1e-3, total_time=1.0, merge_across_steps=True)
    state, _, _ = K.evolve(spec, a, b, psi0, exact=full)
    mw = K.mass_field(g.shape, g.mass)
    nrm = psi0 / np.linalg.norm(psi0)
    n0 = K.norm(nrm, mw)
    drift = abs(K.norm(state, mw) - n0) / n0
    return {"13a_drift": drift, "13a_pass": drift <= 1e-8}


CRITERIA = {"1": c1, "2": c2, "3": c3, "4": c4, "5": c5, "6": c6, "7": c7, "8": c8, "9": c9, "10": c10, "11": c11,
            "12": c12, "13": c13}


def main():
    which = sys.argv[1:] or list(CRITERIA)
    results = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            results = json.load(f)
    for c in which:
        t0 = time.time()
        r = CRITERIA[c]()
        r["seconds"] = time.time() - t0
        results[c] = r
        print(c, json.dumps(r, default=float))
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        with open(OUT, "w") as f:
            json.dump(results, f, indent=1, default=float, sort_keys=True)


if __name__ == "__main__":
    main()
