"""Slab decomposition of the tensor-product operators across GPUs (north-star 4).

Rank p owns a contiguous slab of the slowest axis (axis d-1): planes [z0_p, z1_p), uneven splits
allowed when P does not divide n. Passes on axes 0..d-2 are local GEMMs on the slab. The last
axis is handled by an all-to-all transpose into slabs of axis d-2 (full axis d-1), where the
forward pass on axis d-1, the fused spectral divide / multiply / phase (with GLOBAL indices: each
rank's operator carries its lambda slice) and the backward pass on axis d-1 run locally; a second
all-to-all returns to z-slabs for the backward passes on axes 0..d-2 (the last one fuses the V2
term). Two all-to-alls per application, one scalar all-reduce per dot product; no other traffic.

Pass order differs from the single-device reference only in running backward axis d-1 before
axes 0..d-2 (the Kronecker factors commute exactly; results agree to rounding).

The transposes use torch.distributed all_to_all_single (NCCL on GPUs, grouped send/recv inside
NCCL); the packing is a strided copy on the z->y side only (the y->z receive side is contiguous per
peer). The same class runs on CPU under gloo with an injected local-pass backend, which is how the
multi-rank logic is tested without GPUs (tests/test_slab_gloo.py).
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def split_extent(n: int, parts: int) -> List[int]:
    """Contiguous, as-even-as-possible split of n planes into `parts` slabs (first n % parts get
    one extra)."""
    base, extra = divmod(n, parts)
    return [base + (1 if p < extra else 0) for p in range(parts)]


def offsets(sizes: Sequence[int]) -> List[int]:
    out, acc = [], 0
    for s in sizes:
        out.append(acc)
        acc += s
    return out


EPI_STORE, EPI_MUL, EPI_DIV, EPI_PHASE, EPI_AXPY = 0, 1, 2, 3, 4


class KronopPassBackend:
    """Local passes through libkronop.so (kronop_op_pass_ex) on this rank's GPU."""

    def __init__(self, ctx):
        self.ctx = ctx

    def make_op(self, axes, lam_override, shift, mass=None):
        from . import api
        eig = []
        for a, ax in enumerate(axes):
            if lam_override.get(a) is not None:
                lam = lam_override[a]
                eye = np.eye(len(lam))
                eig.append(api.AxisEigens(np.ascontiguousarray(lam), eye, eye))
            else:
                eig.append(ax)
        return api.SeparableOperator(self.ctx, eig, shift, mass=mass)

    def run(self, op, x, axis, forward, epi=EPI_STORE, dt=0.0, diag=None, sigma=0.0, u=None):
        import ctypes as C
        from . import _lib
        from .api import _Call, _ptr
        out = torch.empty_like(x)
        with _Call(self.ctx):
            _lib.check(_lib.lib().kronop_op_pass_ex(
                self.ctx.h, op.h, axis, int(forward), _ptr(x), int(x.is_complex()), _ptr(out), epi,
                dt, _ptr(diag), sigma, _ptr(u)))
        return out

    def dot(self, a, b):
        """Local dot product through kronop_inner (deterministic fixed-tree reduction)."""
        from . import api
        return api.inner(self.ctx, a, b, (a.numel(),))


class SlabOperator:
    """SeparableOperator / FullOperator distributed over the ranks of `group` by slabs of the
    slowest axis. Fields passed in and returned are this rank's z-slab (flat, axis 0 fastest)."""

    def __init__(self, axes, backend, shift: float = 0.0, diag_slab=None, group=None):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.r = dist.get_rank(group) if dist.is_initialized() else 0
        self.axes = list(axes)
        self.d = len(axes)
        assert self.d >= 2, "slab decomposition needs d >= 2"
        self.shape = tuple(a.size for a in axes)
        self.backend = backend
        self.shift = shift
        self.diag = diag_slab
        nz, ny = self.shape[-1], self.shape[-2]
        # the partition of the C-ABI slab operators (kronop_slab_plan, host code of libkronop.so)
        self.zs, self.z0 = plan(nz, self.P)
        self.ys, self.y0 = plan(ny, self.P)
        assert self.zs == split_extent(nz, self.P) and self.z0 == offsets(self.zs)
        r = self.r
        self.R = int(np.prod(self.shape[:-2]))  # extent of the axes below d-2
        lamz = axes[-1].eigenvalues[self.z0[r]:self.z0[r] + self.zs[r]]
        lamy = axes[-2].eigenvalues[self.y0[r]:self.y0[r] + self.ys[r]]
        # z-slab operator: axes 0..d-2 full, axis d-1 = this rank's planes (lambda only)
        self.op_z = backend.make_op(axes, {self.d - 1: lamz}, shift)
        # y-slab operator: axis d-2 = this rank's rows (lambda only), axis d-1 full
        self.op_y = backend.make_op(axes, {self.d - 2: lamy}, shift)

    # ----------------------------------------------------------------- transposes --
    def local_size(self):
        return self.R * self.shape[-2] * self.zs[self.r]

    def _z_to_y(self, x):
        """(nz_r, ny, R) z-slab -> (nz, ny_r, R) y-slab."""
        c = 2 if x.is_complex() else 1
        xr = torch.view_as_real(x).reshape(-1) if c == 2 else x
        R = self.R * c
        v = xr.view(self.zs[self.r], self.shape[-2], R)
        send = torch.cat([v[:, self.y0[q]:self.y0[q] + self.ys[q], :].reshape(-1)
                          for q in range(self.P)])
        out = torch.empty(self.shape[-1] * self.ys[self.r] * R, dtype=xr.dtype, device=xr.device)
        in_splits = [self.zs[self.r] * self.ys[q] * R for q in range(self.P)]
        out_splits = [self.zs[p] * self.ys[self.r] * R for p in range(self.P)]
        if self.P > 1:
            dist.all_to_all_single(out, send, out_splits, in_splits, group=self.group)
        else:
            out.copy_(send)
        return torch.view_as_complex(out.view(-1, 2)) if c == 2 else out

    def _y_to_z(self, x):
        """(nz, ny_r, R) y-slab -> (nz_r, ny, R) z-slab."""
        c = 2 if x.is_complex() else 1
        xr = torch.view_as_real(x).reshape(-1) if c == 2 else x
        R = self.R * c
        in_splits = [self.zs[p] * self.ys[self.r] * R for p in range(self.P)]
        out_splits = [self.zs[self.r] * self.ys[q] * R for q in range(self.P)]
        recv = torch.empty(sum(out_splits), dtype=xr.dtype, device=xr.device)
        if self.P > 1:
            dist.all_to_all_single(recv, xr.contiguous(), out_splits, in_splits, group=self.group)
        else:
            recv.copy_(xr)
        blocks = torch.split(recv, out_splits)
        out = torch.cat([b.view(self.zs[self.r], self.ys[q], R) for q, b in enumerate(blocks)],
                        dim=1).reshape(-1)
        return torch.view_as_complex(out.view(-1, 2)) if c == 2 else out

    # ------------------------------------------------------------------- operators --
    def _transform(self, x, epi, dt=0.0, diag=None, sigma=0.0):
        d, be = self.d, self.backend
        w = x
        for a in range(d - 1):  # forward, local axes
            w = be.run(self.op_z, w, a, True)
        w = self._z_to_y(w)
        w = be.run(self.op_y, w, d - 1, True, epi, dt)  # forward last axis + spectral op
        w = be.run(self.op_y, w, d - 1, False)          # backward last axis
        w = self._y_to_z(w)
        for a in range(d - 1):  # backward, local axes; the last fuses + diag u - sigma u
            last = a == d - 2
            if last and (diag is not None or sigma != 0.0):
                w = be.run(self.op_z, w, a, False, EPI_AXPY, diag=diag, sigma=sigma, u=x)
            else:
                w = be.run(self.op_z, w, a, False)
        return w

    def apply(self, u, with_diag=True, sigma: float = 0.0):
        """(A - shift) u [+ V2 u - sigma u] on this rank's slab (operators.cpp:31-40,93-105)."""
        return self._transform(u, EPI_MUL, diag=self.diag if with_diag else None, sigma=sigma)

    def solve(self, b):
        """(A - shift)^{-1} b (operators.cpp:42-61)."""
        return self._transform(b, EPI_DIV)

    def propagate(self, psi, dt: float):
        """exp(-i (A - shift) dt) psi (operators.cpp:63-75)."""
        if dt == 0.0:
            return psi.clone()
        return self._transform(psi, EPI_PHASE, dt=dt)

    # ---------------------------------------------------------------------- scalars --
    def dot(self, a, b) -> float:
        """Global dot product: local dot + all-reduce (sum) of one scalar."""
        s = self.backend.dot(a, b)
        if isinstance(s, torch.Tensor):
            s = s.item()
        vals = [s.real, s.imag] if isinstance(s, complex) else [float(s)]
        t = torch.tensor(vals, dtype=torch.float64, device=a.device)
        if self.P > 1:
            dist.all_reduce(t, group=self.group)
        return float(t[0]) if t.numel() == 1 else complex(float(t[0]), float(t[1]))


def slab_pcg(apply_a, precond, b, x, dot, rel_tol=1e-12, max_iter=500, stagnation_window=0):
    """PCG of proj/src/pcg.cpp:8-81 over slab-distributed fields: the vector updates are local,
    each scalar is one all-reduce. Returns (iterations, final_residual, converged)."""
    norm_b = math.sqrt(dot(b, b))
    if norm_b == 0.0:
        x.zero_()
        return 0, 0.0, True
    r = b.clone()
    if math.sqrt(dot(x, x)) != 0.0:
        r = r - apply_a(x)
    z = precond(r)
    p = z.clone()
    rz = dot(r, z)
    rel = math.sqrt(dot(r, r)) / norm_b
    best_rel, best_x, since, it_done = rel, x.clone(), 0, 0
    converged = False
    for it in range(max_iter):
        if rel <= rel_tol:
            converged = True
            break
        if stagnation_window > 0 and since >= stagnation_window:
            break
        q = apply_a(p)
        pq = dot(p, q)
        if pq <= 0.0:
            raise ArithmeticError("pcg: indefinite direction at iteration %d" % (it + 1))
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        z = precond(r)
        rz_next = dot(r, z)
        p = z + (rz_next / rz) * p
        rz = rz_next
        it_done += 1
        rel = math.sqrt(dot(r, r)) / norm_b
        if rel < 0.99 * best_rel:
            best_rel, best_x, since = rel, x.clone(), 0
        else:
            since += 1
    if rel <= rel_tol:
        converged = True
    elif best_rel < rel:
        x.copy_(best_x)
        rel = best_rel
    return it_done, rel, converged


# ------------------------------------------------------------ C-ABI slab operators --
def plan(n: int, parts: int):
    """kronop_slab_plan (host): the (extents, offsets) split of n planes into `parts` slabs, the
    same split the device slab operators use."""
    import ctypes as C
    from . import _lib
    e = (C.c_int * parts)()
    o = (C.c_int * parts)()
    _lib.check(_lib.lib().kronop_slab_plan(n, parts, e, o))
    return list(e), list(o)


class DeviceSlabOperator:
    """SeparableOperator / FullOperator, pcg and the a_u GPE flow on slab-decomposed fields
    through the C-ABI (kronop_slab_*, csrc/slab.cu).

    In-process: `devices` lists the CUDA device of every part (distinct GPUs exchange over
    NVLink peer copies; a repeated device gives virtual slabs on one GPU). NCCL: pass `ctx`
    (this rank's api.Context), `rank`, `nranks` and the 128-byte `unique_id` (see nccl_unique_id).
    Fields are lists of torch tensors, one per local part (this process's z-slabs)."""

    def __init__(self, axes, shift: float = 0.0, mass=None, devices=None, ctx=None, rank=0,
                 nranks=1, unique_id=None):
        import ctypes as C
        from . import _lib
        from .api import _arr_of_ptrs
        d = len(axes)
        self.axes = list(axes)
        self.shape = tuple(len(a.eigenvalues) for a in axes)
        n = (C.c_int * d)(*self.shape)
        keep = [np.asfortranarray(a.transform) for a in axes] + \
               [np.asfortranarray(a.inverse_transform) for a in axes] + \
               [np.ascontiguousarray(a.eigenvalues) for a in axes]
        T, Ti, lam = (_arr_of_ptrs(keep[:d]), _arr_of_ptrs(keep[d:2 * d]),
                      _arr_of_ptrs(keep[2 * d:]))
        self.mass = [np.ascontiguousarray(m, dtype=np.float64) for m in mass] if mass else None
        mp = _arr_of_ptrs(self.mass) if self.mass else None
        h = C.c_void_p()
        if ctx is None:
            devs = list(devices or [0])
            _lib.check(_lib.lib().kronop_slab_create(len(devs), (C.c_int * len(devs))(*devs), d, n,
                                                     T, Ti, lam, mp, shift, C.byref(h)))
        else:
            self.ctx = ctx
            _lib.check(_lib.lib().kronop_slab_create_nccl(ctx.h, bytes(unique_id), nranks, rank, d,
                                                          n, T, Ti, lam, mp, shift, C.byref(h)))
        self.h = h
        P, nl, first = C.c_int(), C.c_int(), C.c_int()
        _lib.check(_lib.lib().kronop_slab_info(h, C.byref(P), C.byref(nl), C.byref(first)))
        self.P, self.nlocal, self.first = P.value, nl.value, first.value
        self.parts = []
        for i in range(self.nlocal):
            dv, st = C.c_int(), C.c_void_p()
            z0, nz, el = C.c_longlong(), C.c_longlong(), C.c_longlong()
            _lib.check(_lib.lib().kronop_slab_part(h, i, C.byref(dv), C.byref(st), C.byref(z0),
                                                   C.byref(nz), C.byref(el)))
            self.parts.append({"device": dv.value, "stream": torch.cuda.ExternalStream(
                st.value, device="cuda:%d" % dv.value), "z0": z0.value, "nz": nz.value,
                "elems": el.value})

    def close(self):
        from . import _lib
        if getattr(self, "h", None):
            _lib.lib().kronop_slab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- field helpers --
    def plane_elems(self):
        return int(np.prod(self.shape[:-1]))

    def fused_transforms(self) -> int:
        """kronop_slab_stats: applications whose transposes ran as exchange-fused passes."""
        import ctypes as C
        from . import _lib
        v = C.c_longlong()
        _lib.check(_lib.lib().kronop_slab_stats(self.h, C.byref(v)))
        return v.value

    def scatter(self, full: torch.Tensor):
        """This process's z-slabs of a full field (host or device tensor, flat, axis 0 fastest)."""
        pe = self.plane_elems()
        out = []
        for pt in self.parts:
            sl = full[pt["z0"] * pe:(pt["z0"] + pt["nz"]) * pe]
            out.append(sl.to("cuda:%d" % pt["device"]).contiguous().clone())
        return out

    def gather(self, parts) -> torch.Tensor:
        """Concatenate local slabs (in-process: the whole field) on the first part's device."""
        return torch.cat([p.to(parts[0].device) for p in parts])

    def empty_like(self, parts):
        return [torch.empty_like(p) for p in parts]

    def _enter(self):
        for pt in self.parts:
            pt["stream"].wait_stream(torch.cuda.current_stream(pt["device"]))

    def _leave(self):
        for pt in self.parts:
            torch.cuda.current_stream(pt["device"]).wait_stream(pt["stream"])

    @staticmethod
    def _ptrs(parts):
        import ctypes as C
        if parts is None:
            return None
        return (C.c_void_p * len(parts))(*[C.c_void_p(p.data_ptr()) for p in parts])

    # -------------------------------------------------------------------- operators --
    def set_shift(self, shift: float):
        from . import _lib
        _lib.check(_lib.lib().kronop_slab_set_shift(self.h, shift))

    def apply(self, u, diag=None, sigma: float = 0.0, out=None):
        from . import _lib
        out = out or self.empty_like(u)
        self._enter()
        _lib.check(_lib.lib().kronop_slab_apply(self.h, self._ptrs(u), int(u[0].is_complex()),
                                                self._ptrs(diag), sigma, self._ptrs(out)))
        self._leave()
        return out

    def solve(self, b, out=None):
        from . import _lib
        out = out or self.empty_like(b)
        self._enter()
        _lib.check(_lib.lib().kronop_slab_solve(self.h, self._ptrs(b), int(b[0].is_complex()),
                                                self._ptrs(out)))
        self._leave()
        return out

    def propagate(self, psi, dt: float, out=None):
        from . import _lib
        out = out or self.empty_like(psi)
        self._enter()
        _lib.check(_lib.lib().kronop_slab_propagate(self.h, self._ptrs(psi), dt, self._ptrs(out)))
        self._leave()
        return out

    def dot(self, a, b, weighted: bool = False) -> float:
        import ctypes as C
        from . import _lib
        r = C.c_double()
        self._enter()
        _lib.check(_lib.lib().kronop_slab_dot(self.h, self._ptrs(a), self._ptrs(b), int(weighted),
                                              C.byref(r)))
        return r.value

    def pcg(self, b, x, config, diag=None, sigma: float = 0.0):
        """pcg(FullOperator{this, diag}.apply - sigma, this.solve, b, x&) (pcg.cpp:8-81);
        x (list of part tensors) is the warm start and receives the solution."""
        import ctypes as C
        from . import _lib
        from .api import PcgReport
        cfg = _lib.PcgConfig(config.rel_tol, config.max_iter, int(config.record_history),
                             int(config.preconditioned_norm), config.stagnation_window)
        rep = _lib.PcgReport()
        hist = np.zeros(config.max_iter + 1)
        self._enter()
        _lib.check(_lib.lib().kronop_slab_pcg(
            self.h, self._ptrs(diag), sigma, self._ptrs(b), self._ptrs(x), C.byref(cfg),
            C.byref(rep), hist.ctypes.data_as(C.POINTER(C.c_double))))
        self._leave()
        return PcgReport(rep.iterations, rep.final_residual, bool(rep.converged),
                         list(hist[:rep.history_len]))

    def gpe_au(self, beta: float, config, diag=None, initial=None):
        """a_u gradient flow (gpe.cpp:55-165) on this Hamiltonian (+ diag = V2); returns
        (state parts, api.GpeResult)."""
        import ctypes as C
        from . import _lib
        from .api import GpeResult
        gc = _lib.GpeConfig(1, config.step, config.metric_shift, config.energy_rel_tol,
                            config.max_iterations,
                            _lib.PcgConfig(config.inner.rel_tol, config.inner.max_iter,
                                           int(config.inner.record_history),
                                           int(config.inner.preconditioned_norm),
                                           config.inner.stagnation_window),
                            {"constant": 0, "eigenfunction": 1, "supplied": 2}[config.init],
                            int(config.record_history))
        res = _lib.GpeResult()
        hist = np.zeros(5 * max(config.max_iterations, 1))
        state = [torch.empty(pt["elems"], dtype=torch.float64, device="cuda:%d" % pt["device"])
                 for pt in self.parts]
        self._enter()
        _lib.check(_lib.lib().kronop_slab_gpe_au(
            self.h, self._ptrs(diag), beta, C.byref(gc), self._ptrs(initial), self._ptrs(state),
            C.byref(res), hist.ctypes.data_as(C.POINTER(C.c_double))))
        self._leave()
        rows = [tuple(hist[5 * i:5 * i + 5]) for i in range(res.history_len)]
        return state, GpeResult(state, res.energy, res.eigenvalue, res.iterations,
                                res.linear_solves, bool(res.converged), rows)


def nccl_unique_id() -> bytes:
    """kronop_nccl_unique_id: 128 bytes for kronop_slab_create_nccl (create on rank 0, broadcast)."""
    import ctypes as C
    from . import _lib
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().kronop_nccl_unique_id(buf))
    return buf.raw
