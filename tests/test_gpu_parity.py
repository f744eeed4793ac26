"""GPU parity: libkronop.so (sm_100a) against the CPU oracle on identical inputs.

Two levels, as in the reference's own tests:
  * kernel parity — the oracle is handed the SAME per-axis factors (T, T^-1, lambda) the product
    built, so differences are pure transform arithmetic (bound 1e-13 relative, the reference's
    dense-Kronecker tolerance, proj/tests/test_tensor.cpp:64-84);
  * end-to-end parity — each side builds its own setup (C++ Householder+QL vs LAPACK), compared
    within the FP64 tolerances of SURVEY.md §8c (1e-12 for solutions / eigenvalues, equal PCG
    iteration counts, splitting errors to 1e-9 relative).
"""
import math

import numpy as np
import pytest
import torch

from oracle import kronop_oracle as K

pytestmark = pytest.mark.gpu


def api():
    from paper_2605_20491_b200 import api as a
    return a


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_op_from(prod_op, shift=0.0):
    """Oracle SeparableOperator built from the product's own axis factors (kernel parity)."""
    axes = [K.AxisEigens(a.eigenvalues.copy(), a.transform.copy(), a.inverse_transform.copy())
            for a in prod_op.axes]
    return K.SeparableOperator(axes, shift)


# ----------------------------------------------------------------------------- tensor --
@pytest.mark.parametrize("shape", [(3, 4, 5), (64, 64, 64), (13, 7, 33), (129, 3, 130), (32, 5, 6),
                                   (48, 3, 10), (6, 200, 2)])
@pytest.mark.parametrize("cplx", [False, True])
def test_mode_product_matches_dense(ctx, shape, cplx):
    A = api()
    n = int(np.prod(shape))
    x = K.uniform_pm1(17, 2 * n)
    x = x[0::2] + 1j * x[1::2] if cplx else x[:n]
    for axis in range(len(shape)):
        for m in (shape[axis], 7, 150):
            a = K.uniform_pm1(100 + axis + m, m * shape[axis]).reshape(m, shape[axis], order="F")
            y = host(A.mode_product(ctx, dev(x), shape, a, axis))
            ref = K.mode_product(x, shape, a, axis)
            assert rel(y, ref) < 1e-13, (axis, m)


def test_mode_product_rank_one_and_identity(ctx):
    # proj/tests/test_tensor.cpp:46-62
    A = api()
    x = K.uniform_pm1(5, 20)
    y = host(A.mode_product(ctx, dev(x), (4, 5), np.eye(4), 0))
    assert np.array_equal(y, x)
    e = np.zeros(6)
    e[1 + 3 * 1] = 1.0
    a = np.arange(1, 10, dtype=float).reshape(3, 3)
    r = host(A.mode_product(ctx, dev(e), (3, 2), a, 0))
    for i in range(3):
        for j in range(2):
            assert r[i + 3 * j] == (a[i, 1] if j == 1 else 0.0)


def test_mode_product_shape_errors(ctx):
    # proj/tests/test_tensor.cpp:86-91
    from paper_2605_20491_b200 import ParameterError
    A = api()
    x = dev(np.zeros(12))
    with pytest.raises(ParameterError):
        A.mode_product(ctx, x, (3, 4), np.zeros((3, 5)), 0)
    with pytest.raises(ParameterError):
        A.mode_product(ctx, x, (3, 4), np.zeros((3, 5)), 2)


def test_kron_apply_and_round_trip(ctx):
    # proj/tests/test_tensor.cpp:93-117
    A = api()
    a = np.array([[0.3, -1.2], [0.7, 2.0]])
    b = np.array([[1.5, 0.25], [-0.6, 0.1]])
    x = K.uniform_pm1(23, 4)
    y = host(A.kron_apply(ctx, dev(x), (2, 2), [a, b]))
    full = np.kron(b, a)
    assert np.abs(y - full @ x).max() < 1e-13
    basis = A.assemble_sem(1.0, 5, 8)
    ax = A.build_axis(basis, lambda t: t * t)
    u = K.uniform_pm1(29, ax.size * ax.size)
    shp = (ax.size, ax.size)
    v = A.kron_apply(ctx, A.kron_apply(ctx, dev(u), shp, [ax.transform, ax.transform]), shp,
                     [ax.inverse_transform, ax.inverse_transform])
    assert np.abs(host(v) - u).max() < 1e-9 * np.abs(u).max()
    # rectangular (multilevel prolongation shapes) + identity entries
    c = A.assemble_sem(8.0, 2, 6)
    f = A.assemble_sem(8.0, 4, 6)
    p = A.interp_matrix(c, f)
    g = K.uniform_pm1(3, c.size ** 3)
    out = host(A.kron_apply(ctx, dev(g), (c.size,) * 3, [p, None, p]))
    ref, _ = K.kron_apply(g, (c.size,) * 3, [p, None, p])
    assert rel(out, ref) < 1e-13


def test_inner_mass_direct_sum_splitmix(ctx):
    A = api()
    grid = A.Grid.sem(2.0, 3, 4, 3)
    shape = grid.shape
    u = K.uniform_pm1(3, grid.node_count())
    v = K.uniform_pm1(4, grid.node_count())
    mw = K.mass_field(shape, grid.mass)
    assert abs(A.inner(ctx, dev(u), dev(v), shape) - float(u @ v)) < 1e-12 * np.abs(u * v).sum()
    got = A.inner(ctx, dev(u), dev(v), shape, grid.mass)
    assert abs(got - float(np.sum(mw * u * v))) < 1e-12 * np.abs(mw * u * v).sum()
    uc = K.seeded_complex_field(shape, 9)
    vc = K.seeded_complex_field(shape, 10)
    gc = A.inner(ctx, dev(uc), dev(vc), shape)
    assert abs(gc - np.vdot(uc, vc)) < 1e-12 * np.abs(uc).sum()
    # mass_field / direct_sum_grid are bitwise: same operation order as tensor.cpp:183-209
    assert np.array_equal(host(A.mass_field(ctx, shape, grid.mass)), mw)
    vals = [K.uniform_pm1(7 + a, shape[a]) for a in range(3)]
    assert np.array_equal(host(A.direct_sum_grid(ctx, vals)), K.direct_sum_grid(vals))
    # SplitMix64 on the device is bit-identical to rng.hpp
    assert np.array_equal(host(A.splitmix_uniform(ctx, 1, 100000)), K.uniform_pm1(1, 100000))
    assert np.array_equal(host(A.splitmix_uniform(ctx, 7, 1000, start=123)),
                          K.uniform_pm1(7, 1000, start=123))


# -------------------------------------------------------------------------- operators --
def _trap_op(A, ctx, grid, shift=0.0):
    return grid.separable_operator(ctx, [lambda t: t * t] * grid.dim, shift)


@pytest.mark.parametrize("spec", [(1.0, 4, 3, 2), (2.0, 3, 4, 3), (8.0, 13, 5, 3), (8.0, 8, 10, 3),
                                  (1.5, 5, 6, 1)])
def test_separable_apply_solve_propagate_kernel_parity(ctx, spec):
    A = api()
    grid = A.Grid.sem(*spec)
    op = _trap_op(A, ctx, grid, 0.5)
    ko = oracle_op_from(op, 0.5)
    n = grid.node_count()
    u = K.uniform_pm1(11, n)
    psi = K.seeded_complex_field(grid.shape, 12)
    assert rel(host(op.apply(dev(u))), ko.apply(u)) < 1e-13
    assert rel(host(op.solve(dev(u))), ko.solve(u)) < 1e-13
    assert rel(host(op.apply(dev(psi))), ko.apply(psi)) < 1e-13
    assert rel(host(op.solve(dev(psi))), ko.solve(psi)) < 1e-13
    for dt in (0.083, -0.2, 1e-3):
        assert rel(host(op.propagate(dev(psi), dt)), ko.propagate(psi, dt)) < 1e-13
    assert np.array_equal(host(op.propagate(dev(psi), 0.0)), psi)
    assert np.array_equal(host(op.eigenvalue_grid()), ko.lam)
    assert np.array_equal(host(op.ground_state()), ko.ground_state())
    s, lo, hi = op.info()
    assert (s, lo, hi) == (0.5, ko.lambda_min, ko.lambda_max)


@pytest.mark.parametrize("spec", [(8.0, 13, 5, 3), (1.0, 4, 3, 2), (2.0, 3, 4, 4), (1.5, 5, 6, 1)])
def test_host_buffer_entry_points_pipelined(ctx, spec):
    """kronop_sep_{solve,apply,propagate}_host (slab-pipelined H2D/D2H) equal the device path."""
    A = api()
    grid = A.Grid.sem(*spec)
    op = _trap_op(A, ctx, grid, 0.25)
    ko = oracle_op_from(op, 0.25)
    n = grid.node_count()
    u = K.uniform_pm1(21, n)
    out = np.empty_like(u)
    assert rel(op.solve_host(u, out), ko.solve(u)) < 1e-13
    assert rel(op.apply_host(u, np.empty_like(u)), ko.apply(u)) < 1e-13
    psi = K.seeded_complex_field(grid.shape, 22)
    assert rel(op.propagate_host(psi, 0.07, np.empty_like(psi)), ko.propagate(psi, 0.07)) < 1e-13
    assert rel(op.solve_host(psi, np.empty_like(psi)), ko.solve(psi)) < 1e-13


@pytest.mark.parametrize("spec", [(8.0, 13, 5, 3), (3.0, 2, 5, 4)])
def test_host_batch_entry_points(ctx, spec):
    """kronop_sep_{solve,propagate}_host_batch: every item of a 5-item batch (distinct inputs,
    real and complex, one output aliasing its own input) equals the oracle; 1- and 0-item
    batches."""
    A = api()
    grid = A.Grid.sem(*spec)
    op = _trap_op(A, ctx, grid, 0.25)
    ko = oracle_op_from(op, 0.25)
    n = grid.node_count()
    bs = [K.uniform_pm1(90 + i, n) for i in range(5)]
    outs = [np.empty_like(b) for b in bs]
    outs[3] = bs[3]  # in place
    ref3 = ko.solve(bs[3].copy())
    refs = [ko.solve(b) for b in bs]
    refs[3] = ref3
    op.solve_host_batch(bs, outs)
    for o, r in zip(outs, refs):
        assert rel(o, r) < 1e-13
    cs = [K.seeded_complex_field(grid.shape, 95 + i) for i in range(3)]
    couts = [np.empty_like(c) for c in cs]
    op.propagate_host_batch(cs, 0.07, couts)
    for o, c in zip(couts, cs):
        assert rel(o, ko.propagate(c, 0.07)) < 1e-13
    op.solve_host_batch(cs[:2], couts[:2])
    for o, c in zip(couts[:2], cs[:2]):
        assert rel(o, ko.solve(c)) < 1e-13
    one = [np.empty_like(bs[0])]
    op.solve_host_batch(bs[:1], one)
    assert rel(one[0], ko.solve(bs[0])) < 1e-13
    op.solve_host_batch([], [])


def test_full_operator_apply_with_v2_and_sigma(ctx):
    A = api()
    grid = A.Grid.sem(1.0, 7, 1, 3)  # 6^3, acceptance.cpp:131-200 instance
    op = _trap_op(A, ctx, grid)
    v2 = grid.sample(lambda c: 2.0 * np.exp(-((c[0] - 0.3) ** 2 + (c[1] - 0.3) ** 2 + (c[2] - 0.3) ** 2)))
    ko = K.FullOperator(oracle_op_from(op), v2)
    u = K.uniform_pm1(101, grid.node_count())
    fo = A.FullOperator(op, dev(v2))
    assert rel(host(fo.apply(dev(u))), ko.apply(u)) < 1e-13
    assert rel(host(fo.apply(dev(u), sigma=1.7)), ko.apply(u) - 1.7 * u) < 1e-13
    # dense-oracle equivalence at the acceptance tolerance (acceptance.cpp:131-200)
    ops = [K.dense_axis_operator(K.assemble_sem(1.0, 7, 1), lambda t: t * t)] * 3
    dense = K.dense_assemble(ops, v2)
    assert rel(host(fo.apply(dev(u))), dense @ u) < 1e-10
    uc = K.seeded_complex_field(grid.shape, 5)
    assert rel(host(fo.apply(dev(uc))), ko.apply(uc)) < 1e-13


def test_singular_shift_refused(ctx):
    # proj/tests/test_operators.cpp:95-102
    from paper_2605_20491_b200 import NumericalError
    A = api()
    grid = A.Grid.sem(1.0, 4, 3, 2)
    op = _trap_op(A, ctx, grid)
    lam = op.axes[0].eigenvalues[1] + op.axes[1].eigenvalues[2]
    op.set_shift(lam)
    with pytest.raises(NumericalError):
        op.solve(dev(np.ones(grid.node_count())))
    op.set_shift(op.axes[0].eigenvalues[0] + op.axes[1].eigenvalues[0])  # = lambda_min
    with pytest.raises(NumericalError):
        op.solve(dev(np.ones(grid.node_count())))


def test_c1_manufactured_solve_64cubed(ctx):
    """BASELINE config 1: 64^3 (SEM k=5, 13 cells, L=8) harmonic, manufactured solution
    (harness.cpp:228-249): the GPU solution equals the oracle's own end-to-end solve."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 13, 5, 3)
    pot = P.build_potential("harmonic", grid)
    op = grid.separable_operator(ctx, pot.separable)
    kg = K.Grid.sem(8.0, 13, 5, 3)
    kp = K.build_potential("harmonic", kg)
    rhs, ustar = K.manufactured_rhs(kg, kp, 8.0)
    kop = kg.separable_operator(kp.separable)
    u_ref = kop.solve(rhs)
    u = host(op.solve(dev(rhs)))
    assert rel(u, u_ref) < 1e-12
    err_gpu, err_ref = rel(u, ustar), rel(u_ref, ustar)
    assert abs(err_gpu - err_ref) <= 1e-9 * err_ref
    # residual (harness.cpp:269-274)
    res = host(A.FullOperator(op).apply(dev(u))) - rhs
    assert np.linalg.norm(res) / np.linalg.norm(rhs) < 1e-12


# --------------------------------------------------------------------------------- pcg --
def test_pcg_identity_and_exact_preconditioner(ctx):
    # proj/tests/test_pcg.cpp:26-69: exact preconditioner converges in one iteration
    A = api()
    grid = A.Grid.sem(2.0, 3, 4, 3)
    op = _trap_op(A, ctx, grid)
    b = dev(K.uniform_pm1(3, grid.node_count()))
    x = torch.zeros_like(b)
    rep = A.pcg(A.apply_map(op), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-10))
    assert rep.converged and rep.iterations == 1
    r = host(A.FullOperator(op).apply(x)) - host(b)
    assert np.linalg.norm(r) / np.linalg.norm(host(b)) < 1e-10
    # warm start at the solution: zero iterations (test_pcg.cpp:129-142)
    rep2 = A.pcg(A.apply_map(op), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8))
    assert rep2.converged and rep2.iterations == 0


@pytest.mark.parametrize("kind,cells", [("stirrer", 8), ("quartic", 8)])
def test_pcg_iteration_parity_with_oracle(ctx, kind, cells):
    """acceptance.cpp:202-236 instances (Q6, L=8, seed 1, tol 1e-8): same iteration count and
    history as the oracle; solution within tolerance."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, cells, 6, 3)
    pot = P.build_potential(kind, grid)
    op = grid.separable_operator(ctx, pot.separable)
    v2 = pot.v2_device()
    b_np = K.seeded_field(grid.shape, 1)
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    assert np.array_equal(host(b), b_np)
    x = torch.zeros_like(b)
    cfg = A.PcgConfig(rel_tol=1e-8, record_history=True)
    rep = A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, cfg)
    kg = K.Grid.sem(8.0, cells, 6, 3)
    kop = K.build_full_operator(kg, K.build_potential(kind, kg))
    xr = np.zeros_like(b_np)
    krep = K.pcg(kop.apply, kop.sep.solve, b_np, xr, K.PcgConfig(rel_tol=1e-8, record_history=True))
    assert rep.converged == krep.converged
    assert rep.iterations == krep.iterations
    assert np.allclose(rep.history, krep.history, rtol=1e-8, atol=0)
    assert rel(host(x), xr) < 1e-10


def test_pcg_max_iter_returns_best_and_breakdown(ctx):
    from paper_2605_20491_b200 import NumericalError
    A = api()
    grid = A.Grid.sem(8.0, 4, 6, 3)
    from paper_2605_20491_b200 import potentials as P
    pot = P.build_potential("quartic", grid)
    op = grid.separable_operator(ctx, pot.separable)
    b = A.splitmix_uniform(ctx, 2, grid.node_count())
    x = torch.zeros_like(b)
    rep = A.pcg(A.apply_map(op, pot.v2_device()), A.solve_map(op), b, x,
                A.PcgConfig(rel_tol=1e-14, max_iter=3))
    assert not rep.converged and rep.iterations == 3
    # indefinite operator: A = sep.apply - sigma with sigma above lambda_max (test_pcg.cpp:144-154)
    s, lo, hi = op.info()
    x.zero_()
    with pytest.raises(NumericalError):
        A.pcg(A.apply_map(op, None, sigma=2 * hi), A.solve_map(op), b, x, A.PcgConfig())


# ------------------------------------------------------------------- inverse iteration --
def test_inverse_iteration_separable_criterion5(ctx):
    """acceptance.cpp:291-308 (79^3, sep-osc amp 100): eigenvalue equals the oracle's."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 8, 10, 3)
    pot = P.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    op = grid.separable_operator(ctx, pot.separable)
    init = torch.ones(grid.node_count(), dtype=torch.float64, device="cuda")
    r = A.inverse_iteration(A.FullOperator(op), A.InverseIterationConfig(), init)
    kg = K.Grid.sem(8.0, 8, 10, 3)
    kp = K.build_potential("sep-osc", kg, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    kr = K.inverse_iteration(K.FullOperator(kg.separable_operator(kp.separable)),
                             K.InverseIterationConfig(), np.ones(kg.node_count()), kg.mass)
    assert r.converged and r.outer_iterations == kr.outer_iterations
    assert abs(r.eigenvalue - kr.eigenvalue) <= 1e-12 * kr.eigenvalue
    assert rel(host(r.eigenvector), kr.eigenvector) < 1e-9


def test_inverse_iteration_stirrer_pcg_path(ctx):
    """Non-separable inverse iteration (stirrer, Q20 2 cells = 39^3; acceptance.cpp:347-368 level
    0 / criterion 10 setup): eigenvalue and inner iteration counts equal the oracle's."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 2, 20, 3)
    pot = P.build_potential("stirrer", grid)
    op = grid.separable_operator(ctx, pot.separable)
    fo = A.FullOperator(op, pot.v2_device())
    r = A.inverse_iteration(fo, A.InverseIterationConfig(), op.ground_state())
    kg = K.Grid.sem(8.0, 2, 20, 3)
    kop = K.build_full_operator(kg, K.build_potential("stirrer", kg))
    kr = K.inverse_iteration(kop, K.InverseIterationConfig(), kop.sep.ground_state(), kg.mass)
    assert r.outer_iterations == kr.outer_iterations
    assert r.inner_per_outer == kr.inner_per_outer
    assert abs(r.eigenvalue - kr.eigenvalue) <= 1e-12 * kr.eigenvalue


# --------------------------------------------------------------------------------- gpe --
@pytest.mark.parametrize("kind", ["h1", "au"])
def test_gpe_flow_trace_parity(ctx, kind):
    """GPE flows (gpe.cpp:55-165) on a 39^3 Q20 grid, beta = 10, 25 iterations: the energy
    trace equals the oracle's to 1e-11 relative."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 2, 20, 3)
    pot = P.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    ham = A.FullOperator(grid.separable_operator(ctx, pot.separable))
    lap = grid.laplacian(ctx)
    step = 0.1 if kind == "h1" else 1.0
    cfg = A.GpeFlowConfig(kind=kind, step=step, energy_rel_tol=1e-30, max_iterations=25,
                          record_history=True, init="constant")
    r = A.gpe_gradient_flow(ham, lap, 10.0, cfg)
    kg = K.Grid.sem(8.0, 2, 20, 3)
    kp = K.build_potential("sep-osc", kg, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    prob = K.GpeProblem(K.FullOperator(kg.separable_operator(kp.separable)), kg.laplacian(), 10.0,
                        kg.mass)
    kr = K.gpe_gradient_flow(prob, K.GpeFlowConfig(kind=kind, step=step, energy_rel_tol=1e-30,
                                                   max_iterations=25, record_history=True,
                                                   init="constant"))
    assert r.iterations == kr.iterations == 25
    e_gpu = np.array([h[1] for h in r.history])
    e_ref = np.array([h[1] for h in kr.history])
    assert np.max(np.abs(e_gpu - e_ref) / np.abs(e_ref)) < 1e-11
    assert [int(h[3]) for h in r.history] == [h[3] for h in kr.history]
    assert abs(r.energy - kr.energy) <= 1e-11 * abs(kr.energy)
    assert abs(A.gpe_energy(ham, 10.0, r.state) - r.energy) <= 1e-12 * abs(r.energy)


# --------------------------------------------------------------------------- splitting --
def test_yoshida_coeffs():
    # proj/tests/test_splitting.cpp:29-35
    g1, g2 = api().yoshida_coeffs()
    assert abs(2 * g1 + g2 - 1.0) < 1e-15
    assert abs(2 * g1 ** 3 + g2 ** 3) < 1e-14
    assert (g1, g2) == K.yoshida_coeffs()


def test_qhop_and_yoshida_step_kernel_parity(ctx):
    A = api()
    grid = A.Grid.sem(8.0, 4, 7, 2)
    a = grid.laplacian(ctx)
    ko = oracle_op_from(a)
    b = grid.sample(lambda c: c[0] ** 2 + 100 * np.sin(np.pi * c[0] / 4) ** 2 + c[1] ** 2)
    psi = K.seeded_complex_field(grid.shape, 2)
    for m in (1, 3, 5):
        out = host(A.qhop_step(a, dev(b), dev(psi), 0.013, m))
        assert rel(out, K.qhop_step(ko, b, psi, 0.013, m)) < 1e-12
        out = host(A.yoshida_step(a, dev(b), dev(psi), -0.02, m))
        assert rel(out, K.yoshida_step(ko, b, psi, -0.02, m)) < 1e-12
    # M = 1 is the explicit Strang half-kick form (test_splitting.cpp:37-54)
    ref = ko.propagate(psi, 0.013 / 2)
    ref = K.pointwise_phase(ref, b, 0.013)
    ref = ko.propagate(ref, 0.013 / 2)
    assert np.abs(host(A.qhop_step(a, dev(b), dev(psi), 0.013, 1)) - ref).max() < 1e-12


@pytest.mark.parametrize("m,comp,dt,total", [(1, "single", 0.01, 0.1), (3, "single", 0.005, 0.1),
                                             (1, "yoshida", 0.05, 1.0), (3, "yoshida", 0.1, 1.0)])
def test_evolve_criterion9_errors(ctx, m, comp, dt, total):
    """acceptance.cpp:424-489 setup (31^3 sep-osc, box psi0, exact reference, merge on): the
    split-step error equals the oracle's to 1e-9 relative."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 4, 8, 3)
    pot = P.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    full = grid.separable_operator(ctx, pot.separable)
    lap = grid.laplacian(ctx)
    b = P.separable_sum(grid, pot)
    kg = K.Grid.sem(8.0, 4, 8, 3)
    psi0 = K.box_state(kg, 8.0).astype(np.complex128)
    spec = A.SplitSpec(quad_points=m, composition=comp, dt=dt, total_time=total,
                       merge_across_steps=True)
    state, err, steps = A.evolve(spec, lap, dev(b), dev(psi0), exact=full)
    kp = K.build_potential("sep-osc", kg, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    kstate, kerr, ksteps = K.evolve(K.SplitSpec(quad_points=m, composition=comp, dt=dt,
                                                total_time=total, merge_across_steps=True),
                                    kg.laplacian(), K.separable_sum_field(kg, kp), psi0,
                                    exact=kg.separable_operator(kp.separable))
    assert steps == ksteps
    assert abs(err - kerr) <= 1e-9 * kerr
    assert rel(host(state), kstate) < 1e-10


def test_evolve_unitarity_and_stationary(ctx):
    """Mass-norm conservation (acceptance.cpp:611-645) over 200 steps and the stationary
    reference path (splitting.cpp:129-134)."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 4, 8, 3)
    pot = P.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    full = grid.separable_operator(ctx, pot.separable)
    lap = grid.laplacian(ctx)
    b = dev(P.separable_sum(grid, pot))
    psi0 = K.box_state(K.Grid.sem(8.0, 4, 8, 3), 8.0).astype(np.complex128)
    spec = A.SplitSpec(quad_points=1, dt=1e-3, total_time=0.2, merge_across_steps=True)
    state, err, steps = A.evolve(spec, lap, b, dev(psi0), exact=full)
    n0 = A.norm(ctx, dev(psi0 / np.linalg.norm(psi0)), grid.shape, grid.mass)
    drift = abs(A.norm(ctx, state, grid.shape, grid.mass) - n0) / n0
    assert drift <= 1e-8
    # stationary: psi0 = ground state of the separable full operator -> error ~ splitting error
    gs = full.ground_state().to(torch.complex128)
    st, e2, _ = A.evolve(A.SplitSpec(quad_points=1, dt=0.01, total_time=0.1,
                                     merge_across_steps=True), full, torch.zeros_like(b), gs,
                         stationary_eigenvalue=full.min_eigenvalue())
    assert e2 < 1e-10


def test_multilevel_ground_state_criterion7(ctx):
    """acceptance.cpp:347-368: stirrer, Q20, 2 -> 4 cells (39^3 -> 79^3). Same per-level outer
    and inner iteration counts as the oracle; eigenvalue equal to 1e-11 and to the reference's
    golden 5.286155366963 within its 1e-6."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grids = [A.Grid.sem(8.0, 2, 20, 3), A.Grid.sem(8.0, 4, 20, 3)]

    def mk(g):
        pot = P.build_potential("stirrer", g)
        return A.FullOperator(g.separable_operator(ctx, pot.separable), pot.v2_device())
    pair, levels = A.multilevel_ground_state(ctx, grids, mk, A.InverseIterationConfig())
    kgrids = [K.Grid.sem(8.0, 2, 20, 3), K.Grid.sem(8.0, 4, 20, 3)]
    kpair, klevels = K.multilevel_ground_state(
        kgrids, lambda g: K.build_full_operator(g, K.build_potential("stirrer", g)),
        K.InverseIterationConfig())
    assert [(lv.n, lv.outer_iterations, lv.total_inner_iterations) for lv in levels] == \
        [(l[0], l[1], l[2]) for l in klevels]
    assert abs(pair.eigenvalue - kpair.eigenvalue) <= 1e-11 * kpair.eigenvalue
    assert abs(pair.eigenvalue - 5.286155366963) <= 1e-6 * 5.286155366963


@pytest.mark.parametrize("spec", [(5.0, 2, 3, 6), (3.0, 2, 2, 9), (8.0, 2, 10, 4)])
def test_high_dimensional_operators(ctx, spec):
    """6D / 9D / 4D grids (config 5 families at parity-test size): apply / solve / propagate and
    a qHOP step with the soft-Coulomb B equal the oracle given the same factors."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(*spec)
    op = _trap_op(A, ctx, grid, 0.0)
    ko = oracle_op_from(op)
    u = K.uniform_pm1(31, grid.node_count())
    psi = K.seeded_complex_field(grid.shape, 32)
    assert rel(host(op.apply(dev(u))), ko.apply(u)) < 1e-13
    assert rel(host(op.solve(dev(u))), ko.solve(u)) < 1e-13
    assert rel(host(op.propagate(dev(psi), 0.01)), ko.propagate(psi, 0.01)) < 1e-13
    kind = {6: "coulomb-3d2", 9: "coulomb-3d3", 4: "coulomb-2d2"}[grid.dim]
    b = P.build_potential(kind, grid).nonseparable
    out = host(A.qhop_step(op, dev(b), dev(psi), 0.02, 3))
    assert rel(out, K.qhop_step(ko, b, psi, 0.02, 3)) < 1e-12


def test_slab_operator_single_rank_on_gpu(ctx):
    """slab.py with the libkronop pass backend (kronop_op_pass_ex) on one GPU (P = 1: the
    all-to-alls degenerate to copies) equals the single-device operators."""
    A = api()
    from paper_2605_20491_b200 import slab as S
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 13, 5, 3)
    pot = P.build_potential("stirrer", grid)
    op = grid.separable_operator(ctx, pot.separable, 0.0)
    v2 = pot.v2_device()
    sl = S.SlabOperator(op.axes, S.KronopPassBackend(ctx), shift=0.0, diag_slab=v2)
    u = dev(K.uniform_pm1(5, grid.node_count()))
    fo = A.FullOperator(op, v2)
    assert rel(host(sl.apply(u, sigma=0.3)), host(fo.apply(u, sigma=0.3))) < 1e-13
    assert rel(host(sl.solve(u)), host(op.solve(u))) < 1e-13
    psi = dev(K.seeded_complex_field(grid.shape, 6))
    assert rel(host(sl.propagate(psi, 0.02)), host(op.propagate(psi, 0.02))) < 1e-13
    x = torch.zeros_like(u)
    it, res, conv = S.slab_pcg(lambda v: sl.apply(v), sl.solve, u, x, sl.dot, rel_tol=1e-10)
    rep = A.pcg(A.apply_map(op, v2), A.solve_map(op), u, torch.zeros_like(u),
                A.PcgConfig(rel_tol=1e-10))
    assert conv and it == rep.iterations


# ------------------------------------------------------------------ even/odd folding --
@pytest.mark.parametrize("spec", [(8.0, 4, 7, 3), (8.0, 3, 5, 3), (2.0, 3, 4, 2), (1.5, 5, 6, 1),
                                  (8.0, 13, 5, 3), (8.0, 37, 7, 3), (1.0, 1, 3, 4), (8.0, 3, 3, 6)])
def test_folded_operator_matches_unfolded(ctx, spec):
    """The even/odd folded operator (kronop_op_create_folded) is the same operator as the dense
    one: apply / solve / propagate / FullOperator apply agree to 1e-12 on real and complex
    fields (odd and even extents, the n = 2 and 1-D edge cases, the fused-small regime)."""
    A = api()
    grid = A.Grid.sem(*spec)
    f = [lambda t: t * t] * grid.dim
    op = grid.separable_operator(ctx, f, 0.5)
    fo = grid.separable_operator(ctx, f, 0.5, folded=True)
    n = grid.node_count()
    u = dev(K.uniform_pm1(31, n))
    psi = dev(K.seeded_complex_field(grid.shape, 32))
    for a, b in ((fo.apply(u), op.apply(u)), (fo.solve(u), op.solve(u)),
                 (fo.apply(psi), op.apply(psi)), (fo.solve(psi), op.solve(psi))):
        assert rel(host(a), host(b)) < 1e-12
    # the two factorisations' eigenvalues differ by rounding (~eps lambda_max), which the phase
    # multiplies by dt: bound the propagate difference by that, not by a fixed 1e-12
    lmax = max(abs(fo.info()[2]), 1.0)
    for dt in (0.11, -1.3):
        bound = max(1e-12, 64 * 2.2e-16 * lmax * abs(dt))
        assert rel(host(fo.propagate(psi, dt)), host(op.propagate(psi, dt))) < bound
    v2 = grid.sample(lambda c: 2.0 * np.exp(-sum((ci - 0.3) ** 2 for ci in c)))
    fa, fb = A.FullOperator(fo, dev(v2)), A.FullOperator(op, dev(v2))
    assert rel(host(fa.apply(u, sigma=0.7)), host(fb.apply(u, sigma=0.7))) < 1e-12
    inplace = psi.clone()
    fo.propagate(inplace, 0.2, out=inplace)
    assert rel(host(inplace), host(op.propagate(psi, 0.2))) < max(1e-12, 64 * 2.2e-16 * lmax * 0.2)
    s0, lo0, hi0 = op.info()
    s1, lo1, hi1 = fo.info()
    assert s0 == s1 and abs(lo0 - lo1) <= 1e-12 * abs(hi0) and abs(hi0 - hi1) <= 1e-12 * abs(hi0)
    assert rel(host(fo.ground_state()), host(op.ground_state())) < 1e-10
    assert rel(fo.solve_host(host(u), np.empty(n)), host(op.solve(u))) < 1e-12


def test_folded_operator_pcg_and_inverse_iteration(ctx):
    """Folded preconditioner inside PCG (stirrer, acceptance.cpp:202-236 instance) and inside
    inverse iteration (criterion 5): the oracle's iteration counts and values."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, 8, 6, 3)
    pot = P.build_potential("stirrer", grid)
    op = grid.separable_operator(ctx, pot.separable, folded=True)
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    x = torch.zeros_like(b)
    cfg = A.PcgConfig(rel_tol=1e-8, record_history=True)
    rep = A.pcg(A.apply_map(op, pot.v2_device()), A.solve_map(op), b, x, cfg)
    kg = K.Grid.sem(8.0, 8, 6, 3)
    kop = K.build_full_operator(kg, K.build_potential("stirrer", kg))
    xr = np.zeros(kg.node_count())
    krep = K.pcg(kop.apply, kop.sep.solve, K.seeded_field(kg.shape, 1), xr,
                 K.PcgConfig(rel_tol=1e-8, record_history=True))
    assert rep.converged and rep.iterations == krep.iterations
    assert np.allclose(rep.history, krep.history, rtol=1e-7, atol=0)
    assert rel(host(x), xr) < 1e-10
    grid = A.Grid.sem(8.0, 8, 10, 3)
    pot = P.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    op = grid.separable_operator(ctx, pot.separable, folded=True)
    init = torch.ones(grid.node_count(), dtype=torch.float64, device="cuda")
    r = A.inverse_iteration(A.FullOperator(op), A.InverseIterationConfig(), init)
    assert r.converged
    kg = K.Grid.sem(8.0, 8, 10, 3)
    kp = K.build_potential("sep-osc", kg, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    kr = K.inverse_iteration(K.FullOperator(kg.separable_operator(kp.separable)),
                             K.InverseIterationConfig(), np.ones(kg.node_count()), kg.mass)
    assert abs(r.eigenvalue - kr.eigenvalue) <= 1e-12 * kr.eigenvalue


def test_folded_operator_refuses_per_pass_api(ctx):
    from paper_2605_20491_b200 import ParameterError
    A = api()
    grid = A.Grid.sem(2.0, 3, 4, 3)
    fo = grid.laplacian(ctx, folded=True)
    u = dev(K.uniform_pm1(3, grid.node_count()))
    with pytest.raises(ParameterError):
        fo.transform_pass(u, 0, True)


# ---------------------------------------------------------------------- Hermite axes --
def test_hermite_grid_criterion6(ctx):
    """acceptance.cpp:320-344 on the device: 3-D oscillator lambda_1 = 3 (Grid::hermite(40, 3),
    inverse iteration from the constant field) and the 99^3 solve residual with the accuracy
    potential; plus kernel parity of apply / solve / propagate on a Hermite grid."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    g = A.Grid.hermite(40, 3)
    op = g.separable_operator(ctx, [lambda x: x * x] * 3)
    init = torch.ones(g.node_count(), dtype=torch.float64, device="cuda")
    r = A.inverse_iteration(A.FullOperator(op), A.InverseIterationConfig(), init)
    assert r.converged and abs(r.eigenvalue - 3.0) <= 1e-9
    g99 = A.Grid.hermite(99, 3)
    pot = P.build_potential("sep-osc", g99, osc_amplitude=1600.0, quad_coeffs=[1.0, 2.0, 3.0])
    h = g99.separable_operator(ctx, pot.separable)
    f = g99.sample(lambda c: np.sin(np.pi / 2 * (c[0] + 1.0)) * np.sin(np.pi * (c[1] + 1.0))
                   * np.sin(1.5 * np.pi * (c[2] + 1.0))
                   * np.exp(-(c[0] ** 2 + c[1] ** 2 + c[2] ** 2) / 4.0))
    fd = dev(f)
    u = h.solve(fd)
    res = rel(host(h.apply(u)), f)
    assert res <= 1e-10
    ko = oracle_op_from(h)
    assert rel(host(u), ko.solve(f)) < 1e-13
    psi = K.seeded_complex_field(g99.shape, 7)
    assert rel(host(h.propagate(dev(psi), 0.01)), ko.propagate(psi, 0.01)) < 1e-13


def test_field_io_device_streaming(ctx, tmp_path):
    """Device dump/load (pinned double-buffered streaming) against the oracle's reader/writer,
    on a field larger than one 32 MiB staging chunk (real) and a complex field."""
    A = api()
    shape = (160, 160, 200)  # 5.1 M doubles = 41 MB: two chunks
    x = A.splitmix_uniform(ctx, 9, int(np.prod(shape)))
    p = str(tmp_path / "x.kf")
    A.dump_field(p, x, shape, ctx=ctx)
    got, shp = K.load_field(p)
    assert shp == shape and np.array_equal(got, host(x))
    y, shp2, cplx = A.load_field(p, ctx=ctx)
    assert shp2 == shape and not cplx and torch.equal(y, x)
    z = K.seeded_complex_field((31, 17, 9), 4)
    K.dump_field(p, z, (31, 17, 9))
    zt, _, cplx = A.load_field(p, ctx=ctx)
    assert cplx and np.array_equal(host(zt), z)


@pytest.mark.parametrize("axes", [[(2.0, 2, 3), (3.0, 2, 4), (1.5, 3, 4), (2.0, 2, 5), (1.0, 2, 2)],
                                  [(5.0, 3, 10), (2.0, 1, 5), (3.0, 2, 2)],
                                  [(2.0, 1, 7)] * 4,
                                  [(8.0, 3, 11), (8.0, 3, 11)]])
def test_small_extent_path_anisotropic(ctx, axes):
    """The rotating small-extent kernel on grids whose axes differ (extents and potentials): mixed
    group extents (DMMA path), equal extents with different matrices (DFMA, non-uniform), the
    phase / divide / multiply epilogues and the V2 + sigma AXPY, real and complex, against the
    oracle given the same factors."""
    A = api()
    grid = A.Grid([A.assemble_sem(*a) for a in axes])
    pots = [(lambda t, c=c: (1.0 + 0.3 * c) * t * t + 0.1 * c) for c in range(grid.dim)]
    op = grid.separable_operator(ctx, pots, 0.25)
    ko = oracle_op_from(op, 0.25)
    n = grid.node_count()
    u = K.uniform_pm1(41, n)
    psi = K.seeded_complex_field(grid.shape, 42)
    for x in (u, psi):
        assert rel(host(op.apply(dev(x))), ko.apply(x)) < 1e-13
        assert rel(host(op.solve(dev(x))), ko.solve(x)) < 1e-13
    assert rel(host(op.propagate(dev(psi), 0.07)), ko.propagate(psi, 0.07)) < 1e-13
    v2 = K.uniform_pm1(43, n) + 2.0
    fo = A.FullOperator(op, dev(v2))
    kf = K.FullOperator(ko, v2)
    assert rel(host(fo.apply(dev(u), sigma=0.3)), kf.apply(u) - 0.3 * u) < 1e-13
    assert rel(host(fo.apply(dev(psi))), kf.apply(psi)) < 1e-13


# ----------------------------------------------------- reduced precision (tcgen05 BF16) --
@pytest.mark.parametrize("axes", [[(8.0, 13, 5)] * 3, [(8.0, 5, 5), (8.0, 41, 1), (8.0, 17, 1)],
                                  [(8.0, 61, 5)] * 2 + [(8.0, 5, 5)]])
@pytest.mark.parametrize("prec", ["bf16", "tf32", "fp32"])
def test_lowp_tcgen05_solve(ctx, axes, prec):
    """The paper's BF16 / TF32 modes on the tcgen05 tensor cores (FP32 accumulation in TMEM):
    agree with the FP64 solve to the storage precision, and with a host emulation of the same
    rounding chain (rounded operands, FP32 accumulate, rounded intermediates) far more closely;
    edge tiles (R % 128, m % 256, K % BK != 0) included."""
    A = api()
    grid = A.Grid([A.assemble_sem(*a) for a in axes])
    op = grid.separable_operator(ctx, [lambda t: t * t] * grid.dim, 0.0)
    n = grid.node_count()
    b_np = K.uniform_pm1(5, n)
    b = dev(b_np)
    x64 = host(op.solve(b))
    x16 = host(op.solve_lowp(b, prec))
    assert rel(x16, x64) < {"bf16": 3e-2, "tf32": 5e-3, "fp32": 2e-5}[prec]
    if prec == "fp32":  # 3xTF32: FP32-level agreement is the whole check
        return

    def store(a):  # storage precision of the intermediate fields (TF32: FP32 rounded to TF32)
        t = torch.from_numpy(np.ascontiguousarray(a))
        if prec == "bf16":
            return t.to(torch.bfloat16).to(torch.float64).numpy()
        u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
        u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000  # round to nearest even, 10-bit mantissa
        return u.astype(np.uint32).view(np.float32).astype(np.float64)

    def operand(a):  # operands are stored pre-rounded: the tensor core multiplies them exactly
        return store(a)

    # emulation: contract the fastest axis, move it to the slow end, BF16 between passes
    d = grid.dim
    cur = store(b_np)
    shape = list(grid.shape)  # current layout, fastest first
    order = list(range(d))
    for direction in (0, 1):
        for a in range(d):
            ax = op.axes[a]
            mat = operand(store(ax.inverse_transform if direction == 0 else ax.transform))
            R = cur.size // shape[0]
            X = operand(cur).reshape(R, shape[0])
            Y = (X @ mat.T).astype(np.float32).astype(np.float64)  # [R][m]
            if direction == 0 and a == d - 1:
                lam = np.zeros(R)
                idx = np.arange(R)
                for j in range(d - 1):
                    lam = lam + op.axes[j].eigenvalues[idx % grid.shape[j]]
                    idx //= grid.shape[j]
                lam = lam[:, None] + ax.eigenvalues[None, :]
                Y = (Y.astype(np.float32) / lam.astype(np.float32)).astype(np.float64)
            cur = Y.T.reshape(-1)  # output [m][R]: the contracted axis is now the slowest
            shape = shape[1:] + [shape[0]]
            if not (direction == 1 and a == d - 1):
                cur = store(cur)
    # the emulation accumulates in FP64 then rounds to FP32; the tensor cores' FP32 accumulation
    # is not IEEE-sequential, which the solve's cancellation amplifies to ~3e-4 (TF32 storage);
    # a layout / descriptor error would be O(1)
    assert rel(x16, cur) < (2e-3 if prec == "bf16" else 1e-3)


# ------------------------------------------------------------------------- edge cases --
@pytest.mark.parametrize("axes", [[(1.0, 1, 2), (2.0, 3, 4), (1.0, 1, 2)],       # n = 1, 11, 1
                                  [(1.0, 1, 2)] * 9,                             # 9-D of n = 1
                                  [(2.0, 2, 2), (1.0, 1, 2), (3.0, 5, 7), (1.0, 2, 2)],
                                  [(8.0, 40, 5), (1.0, 1, 2)],                   # n = 199 (TMA) x 1
                                  [(1.0, 1, 2), (8.0, 13, 5), (8.0, 13, 5)]])
def test_degenerate_and_mixed_extents(ctx, axes):
    """Axes of extent 1, mixed small / large extents and d up to 9 (tensor.hpp:33-34): every
    operator path (small-extent kernel, TMA / cp.async passes) against the oracle, real and
    complex, in place and out of place."""
    A = api()
    grid = A.Grid([A.assemble_sem(*a) for a in axes])
    op = grid.separable_operator(ctx, [lambda t: t * t + 1.0] * grid.dim, 0.25)
    ko = oracle_op_from(op, 0.25)
    n = grid.node_count()
    u = K.uniform_pm1(61, n)
    psi = K.seeded_complex_field(grid.shape, 62)
    for x in (u, psi):
        assert rel(host(op.apply(dev(x))), ko.apply(x)) < 1e-13
        xs = dev(x)
        op.solve(xs, out=xs)  # in place
        assert rel(host(xs), ko.solve(x)) < 1e-13
    p = dev(psi)
    op.propagate(p, 0.3, out=p)
    assert rel(host(p), ko.propagate(psi, 0.3)) < 1e-13


# ------------------------------------------ FP64 emulation on INT8 tensor cores (Ozaki) --
@pytest.mark.parametrize("axes", [[(8.0, 13, 5)] * 3, [(8.0, 5, 5), (8.0, 41, 1), (8.0, 17, 1)],
                                  [(8.0, 4, 3), (6.0, 9, 5), (8.0, 3, 7)],
                                  [(8.0, 61, 5)] * 2 + [(8.0, 5, 5)],
                                  [(8.0, 3, 4)] * 4, [(8.0, 29, 5)]])
@pytest.mark.parametrize("prec,tol", [("ozaki", 1e-12), ("ozaki6", 2e-10), ("ozaki5", 3e-8)])
def test_ozaki_int8_solve(ctx, axes, prec, tol):
    """(-Delta+V1)^-1 with every transform as exact INT8 tcgen05 products of 7-bit slices
    (kind::i8, S32 accumulators in TMEM): equal to the FP64 (DMMA) solve to FP64 level with 7
    slices; fewer slices lose 8 bits each. Ragged extents (K % 32, m % 64, R % 128 != 0) and
    1-D / 4-D fields included."""
    A = api()
    grid = A.Grid([A.assemble_sem(*a) for a in axes])
    op = grid.separable_operator(ctx, [lambda t: t * t + 0.5 * t] * grid.dim, 0.0)
    n = grid.node_count()
    b = dev(K.uniform_pm1(11, n))
    x64 = host(op.solve(b))
    xoz = host(op.solve_lowp(b, prec))
    assert np.isfinite(x64).all()
    bad = np.flatnonzero(~np.isfinite(xoz))
    assert bad.size == 0, (bad.size, bad[:8], grid.shape)
    assert rel(xoz, x64) < tol
    # the low-order slices matter: a second right-hand side at a very different scale
    b2h = K.uniform_pm1(12, n) * 1e-200
    b2 = dev(b2h)
    z2 = host(op.solve(b2)) * 1e200  # (norms underflow)
    y2 = host(op.solve_lowp(b2, prec)) * 1e200
    assert np.array_equal(host(b2), b2h)  # the input is not touched
    zb = np.flatnonzero(~np.isfinite(z2))
    assert zb.size == 0, (zb.size, zb[:6], z2[zb[:3]], grid.shape, np.flatnonzero(~np.isfinite(y2)).size)
    assert rel(y2, z2) < tol
    assert np.array_equal(host(op.solve(b2)) * 1e200, z2)


@pytest.mark.parametrize("axes", [[(8.0, 13, 5)] * 3, [(8.0, 5, 5), (8.0, 41, 1), (8.0, 17, 1)],
                                  [(8.0, 4, 3), (6.0, 9, 5)], [(8.0, 29, 5)],
                                  [(8.0, 3, 4)] * 4])
def test_ozaki_int8_propagate(ctx, axes):
    """exp(-i dt (-Delta+V1)) on the INT8 path: re and im as separate real rows through the
    transforms, the phase in the epilogue of the last forward pass; equal to the FP64 (DMMA)
    propagate to FP64 level (the bound scales with dt * lambda_max like the folded test)."""
    A = api()
    grid = A.Grid([A.assemble_sem(*a) for a in axes])
    op = grid.separable_operator(ctx, [lambda t: t * t + 0.5 * t] * grid.dim, 0.25)
    psi = dev(K.seeded_complex_field(grid.shape, 21).reshape(-1))
    lmax = sum(float(np.max(a.eigenvalues)) for a in op.axes)
    for dt in (0.0, 1e-3, 0.05):
        ref = host(op.propagate(psi, dt))
        got = host(op.propagate_lowp(psi, dt, "ozaki"))
        assert np.isfinite(got).all()
        assert rel(got, ref) < max(1e-12, 64 * 2.2e-16 * lmax * dt), dt
    assert rel(host(op.propagate_lowp(psi, 0.05, "ozaki5")), host(op.propagate(psi, 0.05))) < 3e-8


@pytest.mark.parametrize("kind,cells", [("stirrer", 4), ("quartic", 5)])
def test_ozaki_execution_precision_drivers(ctx, kind, cells):
    """kronop_op_set_precision("ozaki"): every transform of the operator - and so the graph-
    captured device PCG built on it - runs on the INT8 path. Same iteration count and residual
    history as the oracle (acceptance.cpp:202-236 instances), apply / solve / FullOperator apply
    (V2, sigma) / complex solve equal to the FP64 operator's to 1e-12."""
    A = api()
    from paper_2605_20491_b200 import potentials as P
    grid = A.Grid.sem(8.0, cells, 6, 3)
    pot = P.build_potential(kind, grid)
    op64 = grid.separable_operator(ctx, pot.separable)
    op = grid.separable_operator(ctx, pot.separable).set_precision("ozaki")
    v2 = pot.v2_device()
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    for f in ("apply", "solve"):
        assert rel(host(getattr(op, f)(b)), host(getattr(op64, f)(b))) < 1e-12, f
    psi = dev(K.seeded_complex_field(grid.shape, 5).reshape(-1))
    assert rel(host(op.solve(psi)), host(op64.solve(psi))) < 1e-12
    fo, fo64 = A.FullOperator(op, v2), A.FullOperator(op64, v2)
    assert rel(host(fo.apply(b)), host(fo64.apply(b))) < 1e-12
    x = torch.zeros_like(b)
    cfg = A.PcgConfig(rel_tol=1e-8, record_history=True)
    rep = A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, cfg)
    b_np = host(b)
    kg = K.Grid.sem(8.0, cells, 6, 3)
    kop = K.build_full_operator(kg, K.build_potential(kind, kg))
    xr = np.zeros_like(b_np)
    krep = K.pcg(kop.apply, kop.sep.solve, b_np, xr, K.PcgConfig(rel_tol=1e-8, record_history=True))
    assert rep.converged and rep.iterations == krep.iterations
    assert np.allclose(rep.history, krep.history, rtol=1e-8, atol=0)
    assert rel(host(x), xr) < 1e-10
    op.set_precision("fp64")  # back to DMMA
    assert rel(host(op.solve(b)), host(op64.solve(b))) == 0.0


@pytest.mark.parametrize("spec", [(8.0, 4, 7, 3), (8.0, 3, 5, 3), (2.0, 3, 4, 2), (1.5, 5, 6, 1),
                                  (8.0, 13, 5, 3), (1.0, 1, 3, 4)])
def test_ozaki_folded_operator(ctx, spec):
    """The even/odd folded operator on the INT8 path (fold, two half-size INT8 passes per axis,
    unfold with the FullOperator AXPY): apply / solve / propagate / FullOperator apply equal to
    the dense FP64 operator's, real and complex, odd and even extents."""
    A = api()
    grid = A.Grid.sem(*spec)
    f = [lambda t: t * t] * grid.dim
    op = grid.separable_operator(ctx, f, 0.5)
    fo = grid.separable_operator(ctx, f, 0.5, folded=True).set_precision("ozaki")
    n = grid.node_count()
    u = dev(K.uniform_pm1(31, n))
    psi = dev(K.seeded_complex_field(grid.shape, 32).reshape(-1))
    for a, b in ((fo.apply(u), op.apply(u)), (fo.solve(u), op.solve(u)),
                 (fo.apply(psi), op.apply(psi)), (fo.solve(psi), op.solve(psi))):
        assert np.isfinite(host(a)).all() and rel(host(a), host(b)) < 1e-12
    lmax = max(abs(fo.info()[2]), 1.0)
    for dt in (0.11, -1.3):
        bound = max(1e-12, 64 * 2.2e-16 * lmax * abs(dt))
        assert rel(host(fo.propagate(psi, dt)), host(op.propagate(psi, dt))) < bound
    v2 = grid.sample(lambda c: 2.0 * np.exp(-sum((ci - 0.3) ** 2 for ci in c)))
    fa, fb = A.FullOperator(fo, dev(v2)), A.FullOperator(op, dev(v2))
    assert rel(host(fa.apply(u, sigma=0.7)), host(fb.apply(u, sigma=0.7))) < 1e-12
    x = torch.zeros_like(u)
    rep = A.pcg(A.apply_map(fo, dev(v2)), A.solve_map(fo), u, x, A.PcgConfig(rel_tol=1e-10))
    rep64 = A.pcg(A.apply_map(op, dev(v2)), A.solve_map(op), u, torch.zeros_like(u),
                  A.PcgConfig(rel_tol=1e-10))
    assert rep.converged and rep.iterations == rep64.iterations


_SPLIT_CHILD = r"""
import hashlib, sys
import torch
sys.path.insert(0, %r)
from paper_2605_20491_b200 import api as A
from oracle import kronop_oracle as K
ctx = A.Context(0)
h = hashlib.sha1()
for spec in [(3.0, 2, 2, 9), (5.0, 2, 3, 6), (2.0, 1, 7, 4), (8.0, 3, 11, 2)]:
    g = A.Grid.sem(*spec)
    op = g.separable_operator(ctx, [(lambda t: t * t)] * g.dim, 0.25)
    u = torch.from_numpy(K.uniform_pm1(7, g.node_count())).cuda()
    psi = torch.from_numpy(K.seeded_complex_field(g.shape, 8)).cuda()
    for t in (op.apply(u), op.solve(u), op.solve(psi), op.propagate(psi, 0.07)):
        h.update(torch.view_as_real(t).cpu().numpy().tobytes() if t.is_complex()
                 else t.cpu().numpy().tobytes())
print(h.hexdigest())
"""


@pytest.mark.parametrize("mode", ["1", "2"])
def test_small_extent_spectral_split_bitwise(mode):
    """The standalone spectral pass after an epilogue-free contraction (KRONOP_ROT_SPEC_SPLIT = 1,
    or 2, the default) gives bit-identical apply / solve / propagate results to the epilogue fused
    into the DMMA contraction (= 0) on 9D / 6D / 4D / 2D grids."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _SPLIT_CHILD % root
    dig = {}
    for m in ("0", mode):
        p = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                           env=dict(os.environ, KRONOP_ROT_SPEC_SPLIT=m), timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        dig[m] = p.stdout.strip().splitlines()[-1]
    assert dig["0"] == dig[mode]
