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
