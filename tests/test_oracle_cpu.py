"""The C++ restatement of the reference CPU path (oracle/cpu/kronop_cpu.cpp, the timed CPU
reference arm of bench.py) against the numpy oracle, which is pinned against the reference's golden
values (tests/test_oracle_golden.py). Test infrastructure checking test infrastructure: no GPU."""
import numpy as np
import pytest

from oracle import kronop_oracle as K


@pytest.fixture(scope="module")
def C():
    from oracle import kronop_cpu
    kronop_cpu.lib()
    return kronop_cpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cells,degree,d", [(13, 5, 3), (3, 4, 2), (2, 3, 4), (5, 2, 1)])
def test_cpu_restatement_matches_oracle_operators(C, cells, degree, d):
    g = K.Grid.sem(8.0, cells, degree, d)
    pot = K.build_potential("harmonic", g)
    op = g.separable_operator(pot.separable, 0.3)
    co = C.CpuOperator(op.axes, 0.3)
    b = K.seeded_field(g.shape, 1)
    psi = K.seeded_complex_field(g.shape, 2)
    assert _rel(co.solve(b), op.solve(b)) < 1e-13
    assert _rel(co.apply(b), op.apply(b)) < 1e-13
    assert _rel(co.solve(psi), op.solve(psi)) < 1e-13
    assert _rel(co.apply(psi), op.apply(psi)) < 1e-13
    assert _rel(co.propagate(psi, 0.01), op.propagate(psi, 0.01)) < 1e-13
    assert np.array_equal(co.propagate(psi, 0.0), psi)


def test_cpu_restatement_singular_shift_and_full_apply(C):
    g = K.Grid.sem(8.0, 4, 5, 3)
    pot = K.build_potential("stirrer", g)
    op = g.separable_operator(pot.separable)
    co = C.CpuOperator(op.axes)
    u = K.seeded_field(g.shape, 5)
    full = K.FullOperator(op, pot.nonseparable)
    assert _rel(co.full_apply(pot.nonseparable, u), full.apply(u)) < 1e-13
    lam0 = float(op.axes[0].eigenvalues[1] + op.axes[1].eigenvalues[0] + op.axes[2].eigenvalues[0])
    co.set_shift(lam0)
    with pytest.raises(ArithmeticError, match="coincides"):
        co.solve(u)


@pytest.mark.parametrize("tol", [1e-8, 1e-12])
def test_cpu_restatement_pcg_matches_oracle(C, tol):
    """Stirrer pcg-bench pairing (harness.cpp:515-556): equal iteration counts and histories."""
    g = K.Grid.sem(8.0, 8, 6, 3)  # n = 47, acceptance criterion 3's coarse grid
    pot = K.build_potential("stirrer", g)
    op = g.separable_operator(pot.separable)
    full = K.FullOperator(op, pot.nonseparable)
    b = K.seeded_field(g.shape, 1)
    x = np.zeros_like(b)
    rep = K.pcg(full.apply, op.solve, b, x, K.PcgConfig(rel_tol=tol, record_history=True))
    co = C.CpuOperator(op.axes)
    xc = np.zeros_like(b)
    its, conv, fr, hist = C.pcg(co, pot.nonseparable, co, b, xc, rel_tol=tol, max_iter=500)
    assert its == rep.iterations and conv == rep.converged
    np.testing.assert_allclose(hist, rep.history, rtol=1e-8)
    assert _rel(xc, x) < 1e-11


def test_cpu_splitmix_stream_bitwise(C):
    for start, count in [(0, 1000), (12345, 777)]:
        assert np.array_equal(C.uniform_pm1(1, count, start), K.uniform_pm1(1, count, start))
