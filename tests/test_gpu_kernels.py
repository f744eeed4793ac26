"""Kernel-level GPU checks of building blocks that must be bit-exact by construction."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_batched_division_bitwise_equals_ddiv_rn(ctx):
    """The spectral-divide epilogue's batched division (div_rn_fast + __ddiv_rn fallback) is
    bit-identical to __ddiv_rn (hence to the reference's `wf[i] /= lam[i] - shift`, an IEEE
    division, operators.cpp:56-57) on random operands over the whole exponent range, on the
    solve's operand range, and on special / subnormal / extreme values."""
    from paper_2605_20491_b200 import _lib
    rng = np.random.default_rng(7)
    n = 1 << 24
    bits = rng.integers(0, 2 ** 64, size=(2, n), dtype=np.uint64)
    a_all, b_all = bits.view(np.float64)
    a_sol = rng.uniform(-1e4, 1e4, n)
    b_sol = rng.uniform(1.0, 1e7, n) * rng.choice([-1.0, 1.0], n)
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                   1.7976931348623157e308, 1e-300, 1e300, 1.0, -1.0, 3.0, 1e-310, 6.6e-37,
                   1.4e-39, 2.0 ** -1022, 2.0 ** 1023])
    a_sp, b_sp = [x.ravel() for x in np.meshgrid(sp, sp)]
    for a, b in [(a_all, b_all), (a_sol, b_sol), (a_sp, b_sp)]:
        da = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        bad = C.c_ulonglong()
        _lib.check(_lib.lib().kronop_selftest_division(ctx.h, C.c_void_p(da.data_ptr()),
                                                       C.c_void_p(db.data_ptr()), da.numel(),
                                                       C.byref(bad)))
        assert bad.value == 0


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_ozaki_path_propagates_non_finite_inputs(ctx, bad):
    """FP64 emulated on INT8 (Ozaki slices): a NaN / Inf in the input must give non-finite
    outputs, as FP64 arithmetic does (a row holding one is marked and every output that contracts
    it is stored as NaN), not finite garbage from slicing a non-finite value."""
    from paper_2605_20491_b200 import api as A
    grid = A.Grid.sem(8.0, 4, 5, 3)
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    good = op.solve_lowp(b, "ozaki")
    assert bool(torch.isfinite(good).all())
    b[1234] = bad
    x = op.solve_lowp(b, "ozaki")
    ref = op.solve(b)
    assert not bool(torch.isfinite(x).all())
    # the DMMA FP64 path and the INT8 path agree on where the result is non-finite
    assert bool((torch.isfinite(x) == torch.isfinite(ref)).all()) or not bool(torch.isfinite(ref).any())


_BPHASE_SNIPPET = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_20491_b200 import api as A, potentials as P
ctx = A.Context(0)
out = {}
for name, (L, cells, k, d) in {"3d": (8.0, 4, 8, 3), "6d": (5.0, 1, 6, 6), "odd": (8.0, 5, 5, 3)}.items():
    g = A.Grid.sem(L, cells, k, d)
    pot = P.build_potential("harmonic", g)
    lap = g.laplacian(ctx)
    b = torch.from_numpy(np.ascontiguousarray(P.separable_sum(g, pot))).cuda()
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * g.node_count()).view(-1, 2))
    for m, comp in [(1, "single"), (3, "yoshida")]:
        for merge in (True, False):
            st, err, _ = A.evolve(A.SplitSpec(quad_points=m, composition=comp, dt=0.01,
                                              total_time=0.03, merge_across_steps=merge),
                                  lap, b, psi, stationary_eigenvalue=1.0)
            out["%s_%d_%s_%d" % (name, m, comp, merge)] = torch.view_as_real(st).cpu().numpy()
np.savez(sys.argv[1], **out)
'''


def test_fused_b_phase_is_bit_identical(tmp_path):
    """The split-step B phase fused into the propagate's last pass (EPI_BPHASE, DMMA / TMA /
    small-extent kernels; KRONOP_BPHASE_FUSED=1) gives bit-identical states to the standalone
    phase pass (the default), for qHOP / Yoshida, merged or not."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("1", "0"):
        f = str(tmp_path / ("b%s.npz" % flag))
        env = dict(os.environ, KRONOP_BPHASE_FUSED=flag)
        subprocess.check_call([sys.executable, "-c", _BPHASE_SNIPPET, f], cwd=root, env=env)
        res[flag] = np.load(f)
    for k in res["1"].files:
        assert np.array_equal(res["1"][k], res["0"][k]), k
