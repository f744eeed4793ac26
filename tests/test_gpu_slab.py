"""Slab decomposition through the C-ABI (kronop_slab_*, csrc/slab.cu) on one GPU.

Virtual slabs: P = 2, 3, 4 parts on the same device, each with its own stream, exchanging by the
same block copies (cudaMemcpy2D / 3DPeer) and all-gathers the multi-GPU path uses, so the
decomposition, the uneven splits, the global eigenvalue indexing of the fused epilogues, the
transposes and the device-resident drivers run on the hardware against the oracle. The NCCL
transport runs with a one-rank communicator (its own block and the all-gather go through NCCL's
code path; peer sends need a second GPU, which the round's runners do not provide).
"""
import numpy as np
import pytest
import torch

from oracle import kronop_oracle as K

pytestmark = pytest.mark.gpu


def api():
    from paper_2605_20491_b200 import api as a
    return a


def slabmod():
    from paper_2605_20491_b200 import slab as s
    return s


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_op(op, shift=0.0):
    return K.SeparableOperator([K.AxisEigens(a.eigenvalues.copy(), a.transform.copy(),
                                             a.inverse_transform.copy()) for a in op.axes], shift)


GRIDS = [  # (cells, degree, d) -> n = cells * degree - 1; uneven splits for P = 2, 3, 4
    (6, 4, 3),    # 23^3
    (5, 5, 3),    # 24^3 (STRIDED / CONTIG TMA geometries on the slabs)
    (3, 3, 4),    # 8^4
]


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("g", GRIDS)
def test_virtual_slab_operators_match_oracle(ctx, P, g):
    A, S = api(), slabmod()
    grid = A.Grid.sem(8.0, *g)
    op = grid.separable_operator(ctx, [lambda t: t * t] * grid.dim, shift=-0.3)
    so = S.DeviceSlabOperator(op.axes, shift=-0.3, mass=grid.mass, devices=[0] * P)
    ko = oracle_op(op, -0.3)
    N = grid.node_count()
    b = K.seeded_field(grid.shape, 11)
    v2 = K.seeded_field(grid.shape, 12) + 2.0
    bs = so.scatter(torch.from_numpy(b))
    v2s = so.scatter(torch.from_numpy(v2))
    assert [p["nz"] for p in so.parts] == S.plan(grid.shape[-1], P)[0]
    assert rel(host(so.gather(so.solve(bs))), ko.solve(b)) < 1e-13
    assert rel(host(so.gather(so.apply(bs))), ko.apply(b)) < 1e-13
    full = K.FullOperator(ko, v2)
    ref = full.apply(b) - 0.7 * b
    assert rel(host(so.gather(so.apply(bs, diag=v2s, sigma=0.7))), ref) < 1e-13
    psi = K.seeded_complex_field(grid.shape, 13)
    ps = so.scatter(torch.from_numpy(psi))
    assert rel(host(so.gather(so.propagate(ps, 0.02))), ko.propagate(psi, 0.02)) < 1e-13
    assert rel(host(so.gather(so.solve(ps))), ko.solve(psi)) < 1e-13
    assert abs(so.dot(bs, bs) - float(b @ b)) <= 1e-13 * float(b @ b)
    mw = K.mass_field(grid.shape, grid.mass)
    assert abs(so.dot(bs, bs, weighted=True) - float(np.sum(mw * b * b))) <= 1e-13 * float(b @ b)
    assert N == sum(p["elems"] for p in so.parts)
    so.close()


@pytest.mark.parametrize("P", [2, 3])
def test_virtual_slab_pcg_matches_oracle(ctx, P):
    """Stirrer pcg-bench instance (acceptance.cpp:202-236, Q6 8 cells = 47^3, seed 1,
    tol 1e-8) on P slabs: same iteration count and residual history as the oracle."""
    A, S = api(), slabmod()
    from paper_2605_20491_b200 import potentials as Pt
    grid = A.Grid.sem(8.0, 8, 6, 3)
    pot = Pt.build_potential("stirrer", grid)
    op = grid.separable_operator(ctx, pot.separable)
    so = S.DeviceSlabOperator(op.axes, mass=grid.mass, devices=[0] * P)
    b_np = K.seeded_field(grid.shape, 1)
    bs = so.scatter(torch.from_numpy(b_np))
    v2s = so.scatter(torch.from_numpy(pot.nonseparable))
    xs = [torch.zeros_like(t) for t in bs]
    rep = so.pcg(bs, xs, A.PcgConfig(rel_tol=1e-8, record_history=True), diag=v2s)
    kg = K.Grid.sem(8.0, 8, 6, 3)
    kop = K.build_full_operator(kg, K.build_potential("stirrer", kg))
    xr = np.zeros_like(b_np)
    krep = K.pcg(kop.apply, kop.sep.solve, b_np, xr, K.PcgConfig(rel_tol=1e-8, record_history=True))
    assert rep.converged and rep.iterations == krep.iterations
    np.testing.assert_allclose(rep.history, krep.history, rtol=1e-8, atol=0)
    assert rel(host(so.gather(xs)), xr) < 1e-10
    # warm start at the solution: zero iterations (test_pcg.cpp:129-142)
    rep2 = so.pcg(bs, xs, A.PcgConfig(rel_tol=1e-6), diag=v2s)
    assert rep2.converged and rep2.iterations == 0
    so.close()


def test_virtual_slab_gpe_au_matches_oracle(ctx):
    """a_u GPE flow (gpe.cpp:118-157; beta = 10, sep-osc, Q20 2 cells = 39^3, constant init,
    12 iterations) on 3 slabs: energy trace to 1e-11, same inner PCG counts as the oracle."""
    A, S = api(), slabmod()
    from paper_2605_20491_b200 import potentials as Pt
    grid = A.Grid.sem(8.0, 2, 20, 3)
    pot = Pt.build_potential("sep-osc", grid, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    op = grid.separable_operator(ctx, pot.separable)
    so = S.DeviceSlabOperator(op.axes, mass=grid.mass, devices=[0] * 3)
    cfg = A.GpeFlowConfig(kind="au", step=1.0, energy_rel_tol=1e-30, max_iterations=12,
                          record_history=True, init="constant")
    state, r = so.gpe_au(10.0, cfg)
    kg = K.Grid.sem(8.0, 2, 20, 3)
    kp = K.build_potential("sep-osc", kg, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    prob = K.GpeProblem(K.FullOperator(kg.separable_operator(kp.separable)), kg.laplacian(), 10.0,
                        kg.mass)
    kr = K.gpe_gradient_flow(prob, K.GpeFlowConfig(kind="au", step=1.0, energy_rel_tol=1e-30,
                                                   max_iterations=12, record_history=True,
                                                   init="constant"))
    assert r.iterations == kr.iterations == 12
    e_gpu = np.array([h[1] for h in r.history])
    e_ref = np.array([h[1] for h in kr.history])
    assert np.max(np.abs(e_gpu - e_ref) / np.abs(e_ref)) < 1e-11
    assert [int(h[3]) for h in r.history] == [h[3] for h in kr.history]
    assert abs(r.eigenvalue - kr.eigenvalue) <= 1e-10 * abs(kr.eigenvalue)
    assert rel(host(so.gather(state)), kr.state) < 1e-9
    so.close()


def test_slab_1024_two_virtual_parts_equal_single_device(ctx):
    """The headline workload (1024^3 solve, SEM Q5 x 205 cells, harmonic V1) on 2 virtual slabs
    equals the single-device solve (same kernels; only the order of the commuting backward
    passes differs) -- the decomposition at the production size."""
    A, S = api(), slabmod()
    grid = A.Grid.sem(8.0, 205, 5, 3)
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    x = op.solve(b)
    so = S.DeviceSlabOperator(op.axes, devices=[0, 0])
    xs = so.solve(so.scatter(b))
    del b
    torch.cuda.empty_cache()
    d = float(torch.linalg.norm(so.gather(xs) - x) / torch.linalg.norm(x))
    assert d < 1e-13
    so.close()


def test_nccl_slab_one_rank(ctx):
    """The NCCL transport (kronop_slab_create_nccl, libnccl dlopen'd) with a one-rank
    communicator: solve / propagate / PCG against the oracle."""
    A, S = api(), slabmod()
    import torch.cuda.nccl  # noqa: F401  (loads torch's libnccl.so.2 into the process)
    grid = A.Grid.sem(8.0, 5, 5, 3)
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3, shift=-0.3)
    uid = S.nccl_unique_id()
    so = S.DeviceSlabOperator(op.axes, shift=-0.3, mass=grid.mass, ctx=ctx, rank=0, nranks=1,
                              unique_id=uid)
    ko = oracle_op(op, -0.3)
    b = K.seeded_field(grid.shape, 3)
    bs = so.scatter(torch.from_numpy(b))
    assert rel(host(so.gather(so.solve(bs))), ko.solve(b)) < 1e-13
    psi = K.seeded_complex_field(grid.shape, 4)
    assert rel(host(so.gather(so.propagate(so.scatter(torch.from_numpy(psi)), 0.01))),
               ko.propagate(psi, 0.01)) < 1e-13
    xs = [torch.zeros_like(t) for t in bs]
    rep = so.pcg(bs, xs, A.PcgConfig(rel_tol=1e-10))
    assert rep.converged and rep.iterations == 1  # exact preconditioner
    so.close()


_FUSED_SNIPPET = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import kronop_oracle as K
from paper_2605_20491_b200 import api as A, slab as S
ctx = A.Context(0)
out = {}
for g, P in (((3, 11, 3), 3), ((3, 3, 4), 2), ((3, 11, 3), 4)):
    grid = A.Grid.sem(8.0, *g)
    op = grid.separable_operator(ctx, [lambda t: t * t] * grid.dim, shift=-0.3)
    so = S.DeviceSlabOperator(op.axes, shift=-0.3, mass=grid.mass, devices=[0] * P)
    b = K.seeded_field(grid.shape, 11)
    v2 = K.seeded_field(grid.shape, 12) + 2.0
    psi = K.seeded_complex_field(grid.shape, 13)
    bs, v2s = so.scatter(torch.from_numpy(b)), so.scatter(torch.from_numpy(v2))
    ps = so.scatter(torch.from_numpy(psi))
    key = "%d_%d_%d_%d" % (g + (P,))
    out["s" + key] = so.gather(so.solve(bs)).cpu().numpy()
    out["a" + key] = so.gather(so.apply(bs, diag=v2s, sigma=0.7)).cpu().numpy()
    out["p" + key] = so.gather(so.propagate(ps, 0.02)).cpu().numpy()
    out["n" + key] = np.array([so.fused_transforms()])
    so.close()
np.savez(sys.argv[1], **out)
'''


def test_virtual_slab_fused_exchange_bitwise(ctx, tmp_path):
    """The exchange-fused transposes (the pass before each transpose storing straight into the
    destination parts' slab buffers, SplitDst epilogue of the TMA pass kernel) give bit-identical
    solve / FullOperator apply / propagate to the copy exchange (KRONOP_SLAB_FUSED=0) on
    TMA-eligible virtual-slab grids (32^3 over 3 and 4 uneven parts, 8^4 over 2), ran fused for
    every application, and match the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for name, env_add in (("fused", {}), ("copy", {"KRONOP_SLAB_FUSED": "0"})):
        f = str(tmp_path / ("s%s.npz" % name))
        subprocess.check_call([sys.executable, "-c", _FUSED_SNIPPET, f], cwd=root,
                              env=dict(os.environ, **env_add))
        res[name] = np.load(f)
    for k in res["fused"].files:
        if k.startswith("n"):
            assert res["fused"][k][0] == 3, k  # solve, apply, propagate: all fused
            assert res["copy"][k][0] == 0, k
        else:
            assert np.array_equal(res["fused"][k], res["copy"][k]), k
    A = api()
    grid = A.Grid.sem(8.0, 3, 11, 3)
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3, shift=-0.3)
    ko = oracle_op(op, -0.3)
    b = K.seeded_field(grid.shape, 11)
    assert rel(res["fused"]["s3_11_3_3"], ko.solve(b)) < 1e-13
    psi = K.seeded_complex_field(grid.shape, 13)
    assert rel(res["fused"]["p3_11_3_3"], ko.propagate(psi, 0.02)) < 1e-13


def test_nccl_slab_one_rank_fused_exchange(ctx):
    """The NCCL transport's exchange-fused path at one rank: the CUDA IPC setup (receive buffers
    at complex size, handle all-gather over NCCL, the collective write-through probe and the
    agreement) runs, every application is fused, and solve / propagate match the single-device
    path (at P ranks the same code maps the peers' buffers and stores into them over NVLink)."""
    A, S = api(), slabmod()
    import torch.cuda.nccl  # noqa: F401
    grid = A.Grid.sem(8.0, 3, 11, 3)  # 32^3: both transposes TMA-eligible
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3, shift=-0.3)
    so = S.DeviceSlabOperator(op.axes, shift=-0.3, ctx=ctx, rank=0, nranks=1,
                              unique_id=S.nccl_unique_id())
    b = A.splitmix_uniform(ctx, 1, grid.node_count())
    x = op.solve(b)
    xs = so.gather(so.solve(so.scatter(b)))
    assert float(torch.linalg.norm(xs - x) / torch.linalg.norm(x)) < 1e-13
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 2, 2 * grid.node_count()).view(-1, 2))
    p = op.propagate(psi, 0.02)
    ps = so.gather(so.propagate(so.scatter(psi), 0.02))
    assert float(torch.linalg.norm(ps - p) / torch.linalg.norm(p)) < 1e-13
    assert so.fused_transforms() == 2
    so.close()
