"""Every KRONOP_* A/B switch (environment variables read once per process) keeps
parity: each alternative path runs in a child process on the grid that exercises it and is checked
against the oracle (FP64 paths, 1e-13 with the product's own factors) or against the FP64 solve
at the alternative's storage precision (reduced-precision tcgen05 paths)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
from oracle import kronop_oracle as K
from paper_2605_20491_b200 import api as A
ctx = A.Context(0)
kind = sys.argv[1]

def oracle(op, shift=0.0):
    return K.SeparableOperator([K.AxisEigens(a.eigenvalues.copy(), a.transform.copy(),
                                             a.inverse_transform.copy()) for a in op.axes], shift)

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

L, cells, k, d = {"fp64_3d": (8.0, 13, 5, 3), "fp64_254": (8.0, 51, 5, 3),
                  "small_6d": (5.0, 2, 3, 6), "small_9d": (3.0, 1, 4, 7),
                  "lowp": (8.0, 13, 5, 3), "rot_9": (3.0, 2, 5, 6)}[kind]
g = A.Grid.sem(L, cells, k, d)
op = g.separable_operator(ctx, [lambda t: t * t] * d, shift=-0.25)
b = K.seeded_field(g.shape, 5)
psi = K.seeded_complex_field(g.shape, 6)
if kind == "lowp":
    bd = torch.from_numpy(b).cuda()
    x64 = op.solve(bd).cpu().numpy()
    worst = 0.0
    for prec, tol in (("bf16", 3e-2), ("tf32", 5e-3), ("fp32", 1e-4), ("ozaki", 1e-12)):
        e = rel(op.solve_lowp(bd, prec).cpu().numpy(), x64)
        assert e < tol, (prec, e)
    e = rel(op.propagate_lowp(torch.from_numpy(psi).cuda(), 0.01, "ozaki").cpu().numpy(),
            op.propagate(torch.from_numpy(psi).cuda(), 0.01).cpu().numpy())
    assert e < 1e-12, e
else:
    ko = oracle(op, -0.25)
    x = op.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    assert rel(x, ko.solve(b)) < 1e-13
    y = op.apply(torch.from_numpy(b).cuda()).cpu().numpy()
    assert rel(y, ko.apply(b)) < 1e-13
    z = op.propagate(torch.from_numpy(psi).cuda(), 0.02).cpu().numpy()
    assert rel(z, ko.propagate(psi, 0.02)) < 1e-13
print("ok", kind)
'''


@pytest.mark.parametrize("var,val,kind", [
    ("KRONOP_DISABLE_TMA", "1", "fp64_3d"),           # cp.async pass kernel for every geometry
    ("KRONOP_ROTATE_PASSES", "0", "fp64_3d"),         # axis-order passes (STRIDED TMA loader)
    ("KRONOP_ROTATE_PASSES", "0", "fp64_254"),
    ("KRONOP_TMA_CLUSTER", "2", "fp64_254"),          # X multicast across 2-CTA clusters
    ("KRONOP_TMA_CLUSTER", "4", "fp64_254"),          # ... 4-CTA clusters
    ("KRONOP_DISABLE_FUSED_SMALL", "1", "small_6d"),  # generic per-axis passes for n <= 32
    ("KRONOP_ROT_NO_DFMA", "1", "small_9d"),          # DMMA instead of DFMA for n <= 10
    ("KRONOP_ROT_CT", "0", "rot_9"),                  # runtime-geometry DFMA kernel, real n = 9
    ("KRONOP_ROT_SPEC_SPLIT", "0", "small_9d"),       # phase fused into the contraction
    ("KRONOP_KRON_PROP", "0", "small_9d"),            # transform / phase / transform propagate
    ("KRONOP_KRON_FOLD", "0", "rot_9"),               # dense E_a on parity-symmetric axes
    ("KRONOP_KRON_REAL", "0", "rot_9"),               # fused_rot DFMA for real small-extent fields
    ("KRONOP_ROT_SPEC_SPLIT", "1", "small_6d"),       # standalone spectral pass everywhere
    ("KRONOP_TC_CLUSTER", "2", "lowp"),               # B multicast in the tcgen05 pass
    ("KRONOP_TC_2SM", "0", "lowp"),                   # 1-SM tcgen05 kernels
    ("KRONOP_OZ_2SM", "0", "lowp"),                   # 1-SM INT8 (Ozaki) kernels
])
def test_switch_keeps_parity(var, val, kind):
    p = subprocess.run([sys.executable, "-c", _CHILD % ROOT, kind], cwd=ROOT, capture_output=True,
                       text=True, env=dict(os.environ, **{var: val}), timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert p.stdout.strip().endswith("ok " + kind)
