"""CPU, world_size 2 (gloo): the slab-decomposed multi-GPU operators (paper_2605_20491_b200/slab.py)
against the single-process oracle on the full grid.

The local pass backend is injected: on the GPU it is libkronop.so (kronop_op_pass_ex); here it is a
numpy stand-in for the device kernel so the decomposition / all-to-all / global-index logic is
exercised with real collectives on CPU (the oracle stays the checker on the full grid).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kronop_oracle as K


class NumpyPassBackend:
    """Local passes restated on the CPU for the gloo test (same contract as KronopPassBackend)."""

    class Op:
        def __init__(self, mats_f, mats_b, lams, shift):
            self.f, self.b, self.lams, self.shift = mats_f, mats_b, lams, shift
            self.shape = tuple(len(l) for l in lams)

    def make_op(self, axes, lam_override, shift, mass=None):
        lams, mf, mb = [], [], []
        for a, ax in enumerate(axes):
            lam = lam_override.get(a)
            lams.append(np.asarray(ax.eigenvalues if lam is None else lam))
            mf.append(ax.inverse_transform)
            mb.append(ax.transform)
        return self.Op(mf, mb, lams, shift)

    def run(self, op, x, axis, forward, epi=0, dt=0.0, diag=None, sigma=0.0, u=None):
        xn = x.numpy()
        y = K.mode_product(xn, op.shape, (op.f if forward else op.b)[axis], axis)
        if epi in (1, 2, 3):
            ls = K.direct_sum_grid(op.lams) - op.shift
            if epi == 1:
                y = y * ls
            elif epi == 2:
                y = y / ls
            else:
                ph = -ls * dt
                y = y * (np.cos(ph) + 1j * np.sin(ph))
        elif epi == 4:
            un = u.numpy()
            if diag is not None:
                y = y + diag.numpy() * un
            y = y - sigma * un
        return torch.from_numpy(np.ascontiguousarray(y))

    def dot(self, a, b):
        return complex(torch.vdot(a, b)) if a.is_complex() else float(torch.dot(a, b))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_20491_b200 import slab as S
        grid = K.Grid([K.assemble_sem(1.0, 3, 2), K.assemble_sem(1.0, 4, 2), K.assemble_sem(1.0, 5, 2)])
        shape = grid.shape  # (5, 7, 9): uneven splits for P = 2
        f = lambda t: t * t + 0.5
        axes = [K.build_axis(b, f) for b in grid.axes]
        v2 = grid.sample(lambda c: np.exp(-(c[0] ** 2 + c[1] ** 2 + c[2] ** 2)))
        zs = S.split_extent(shape[2], world)
        z0 = S.offsets(zs)
        plane = shape[0] * shape[1]
        sl = slice(z0[rank] * plane, (z0[rank] + zs[rank]) * plane)
        be = NumpyPassBackend()
        op = S.SlabOperator(axes, be, shift=0.3, diag_slab=torch.from_numpy(v2[sl].copy()))
        u = K.uniform_pm1(3, grid.node_count())
        psi = K.seeded_complex_field(shape, 4)
        res = {}
        res["apply"] = op.apply(torch.from_numpy(u[sl].copy()), sigma=0.7).numpy()
        res["solve"] = op.solve(torch.from_numpy(u[sl].copy())).numpy()
        res["prop"] = op.propagate(torch.from_numpy(psi[sl].copy()), 0.05).numpy()
        res["dot"] = op.dot(torch.from_numpy(u[sl].copy()), torch.from_numpy(u[sl].copy()))
        b = torch.from_numpy(u[sl].copy())
        x = torch.zeros_like(b)
        it, rel, conv = S.slab_pcg(lambda v: op.apply(v), op.solve, b, x, op.dot, rel_tol=1e-10)
        res["pcg"] = (it, rel, conv, x.numpy())
        q.put((rank, res, (sl.start, sl.stop)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_slab_operators_match_full_grid_oracle(world):
    """World sizes 2, 3, 4 on a 5 x 7 x 9 grid: uneven z-slabs and y-slabs (4 ranks: 3,2,2,2 and
    2,2,2,1), every rank's piece of apply / solve / propagate / dot / PCG equal to the oracle."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda t: t[0])
    grid = K.Grid([K.assemble_sem(1.0, 3, 2), K.assemble_sem(1.0, 4, 2), K.assemble_sem(1.0, 5, 2)])
    f = lambda t: t * t + 0.5
    axes = [K.build_axis(b, f) for b in grid.axes]
    v2 = grid.sample(lambda c: np.exp(-(c[0] ** 2 + c[1] ** 2 + c[2] ** 2)))
    op = K.FullOperator(K.SeparableOperator(axes, 0.3), v2)
    u = K.uniform_pm1(3, grid.node_count())
    psi = K.seeded_complex_field(grid.shape, 4)
    full = {"apply": op.apply(u) - 0.7 * u, "solve": op.sep.solve(u), "prop": op.sep.propagate(psi, 0.05)}
    for key, ref in full.items():
        out = np.concatenate([r[1][key] for r in got])
        assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref), key
    assert abs(got[0][1]["dot"] - float(u @ u)) <= 1e-13 * float(u @ u)
    x = np.zeros_like(u)
    rep = K.pcg(op.apply, op.sep.solve, u, x, K.PcgConfig(rel_tol=1e-10))
    its = {r[1]["pcg"][0] for r in got}
    assert its == {rep.iterations}
    xs = np.concatenate([r[1]["pcg"][3] for r in got])
    assert np.linalg.norm(xs - x) <= 1e-10 * np.linalg.norm(x)
