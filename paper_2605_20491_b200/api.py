"""Python mirror of the reference's operator API over the C-ABI (include/kronop_cuda.h).

Used by the tests and bench.py. Names follow proj/include/kronop/*.hpp: Grid, SeparableOperator,
FullOperator, pcg, inverse_iteration, gpe_gradient_flow, qhop_step, yoshida_step, evolve,
mode_product, kron_apply, inner, mass_field, direct_sum_grid. Fields are torch CUDA tensors
(float64 for RealField, complex128 for ComplexField, flat, axis 0 fastest). Device memory and the
stream come from torch; all arithmetic runs in libkronop.so (there is no CPU path here).
"""
from __future__ import annotations

import ctypes as C
import weakref
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib

_PD = C.POINTER(C.c_double)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_PD)


def _arr_of_ptrs(arrs):
    t = (_PD * len(arrs))()
    for i, a in enumerate(arrs):
        t[i] = _dptr(a) if a is not None else _PD()
    return t


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("kronop fields must be CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("kronop fields must be contiguous")
    return C.c_void_p(t.data_ptr())


# ------------------------------------------------------------------------------ context --
class Context:
    """kronop_ctx on one device with its own CUDA stream, ordered against torch's current
    stream at every call boundary (event waits, no host syncs)."""

    def __init__(self, device: int = 0):
        lib()
        self.device = device
        with torch.cuda.device(device):
            self.stream = torch.cuda.Stream(device=device)
        h = C.c_void_p()
        check(lib().kronop_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h
        # operators bound to this context: released before it (garbage-collected reference
        # cycles, e.g. a failed test's traceback, may finalise the context first)
        self._ops = weakref.WeakSet()

    def enter(self):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def leave(self):
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def synchronize(self):
        check(lib().kronop_ctx_synchronize(self.h))

    def trim(self):
        """Return the idle driver work buffers and the host-path staging (kronop_ctx_trim) to
        the device."""
        check(lib().kronop_ctx_trim(self.h))

    def launch_count(self) -> int:
        v = C.c_uint64()
        check(lib().kronop_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "h", None):
            for op in list(getattr(self, "_ops", ())):
                op.release()
            lib().kronop_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Call:
    def __init__(self, ctx: Context):
        self.ctx = ctx

    def __enter__(self):
        self.ctx.enter()

    def __exit__(self, *a):
        self.ctx.leave()


# ------------------------------------------------------------------ host setup (C++) --
def gll_rule(degree: int):
    n = degree + 1
    x, w, d = np.zeros(n), np.zeros(n), np.zeros(n * n)
    check(lib().kronop_host_gll_rule(degree, _dptr(x), _dptr(w), _dptr(d)))
    return x, w, d.reshape(n, n, order="F")


def gauss_legendre(points: int):
    x, w = np.zeros(points), np.zeros(points)
    check(lib().kronop_host_gauss_legendre(points, _dptr(x), _dptr(w)))
    return x, w


@dataclass
class Basis1D:
    """proj/include/kronop/basis1d.hpp:17-29 (SEM axis)."""
    half_width: float
    cell_count: int
    degree: int
    nodes: np.ndarray
    mass: np.ndarray
    stiffness: np.ndarray

    @property
    def size(self):
        return len(self.nodes)


def assemble_sem(half_width: float, cell_count: int, degree: int) -> Basis1D:
    n = cell_count * degree - 1
    if n < 1:
        raise L.ParameterError(L.KRONOP_EPARAM, "assemble_sem: no interior nodes")
    x, m, s = np.zeros(n), np.zeros(n), np.zeros(n * n)
    check(lib().kronop_host_assemble_sem(half_width, cell_count, degree, _dptr(x), _dptr(m),
                                         _dptr(s)))
    return Basis1D(half_width, cell_count, degree, x, m, s.reshape(n, n, order="F"))


def eval_weights(basis: Basis1D, x) -> np.ndarray:
    """Rows of eval_weights_row(basis, x_t) (basis1d.cpp:90-115): (len(x), n) matrix E with
    E @ u = u_h(x) for nodal values u."""
    xs = np.ascontiguousarray(np.atleast_1d(np.asarray(x, dtype=np.float64)))
    out = np.zeros((len(xs), basis.size))
    check(lib().kronop_host_eval_weights(basis.half_width, basis.cell_count, basis.degree,
                                         _dptr(xs), len(xs), _dptr(out)))
    return out


def interp_matrix(coarse: Basis1D, fine: Basis1D) -> np.ndarray:
    p = np.zeros(fine.size * coarse.size)
    check(lib().kronop_host_interp_matrix(coarse.half_width, coarse.cell_count, coarse.degree,
                                          fine.cell_count, fine.degree, _dptr(p)))
    return p.reshape(fine.size, coarse.size, order="F")


def sym_eig(a: np.ndarray):
    n = a.shape[0]
    af = np.asfortranarray(a, dtype=np.float64)
    lam, q = np.zeros(n), np.zeros(n * n)
    check(lib().kronop_host_sym_eig(n, af.ctypes.data_as(_PD), _dptr(lam), _dptr(q)))
    return lam, q.reshape(n, n, order="F")


@dataclass
class AxisEigens:
    """proj/include/kronop/axis.hpp:23-29."""
    eigenvalues: np.ndarray
    transform: np.ndarray
    inverse_transform: np.ndarray

    @property
    def size(self):
        return len(self.eigenvalues)


_AXIS_CACHE = {}


@dataclass
class HermiteBasis:
    """Hermite-function collocation axis (hermite.hpp:13-19)."""
    size: int
    nodes: np.ndarray
    psi_last: np.ndarray
    diff: np.ndarray
    mass: np.ndarray


def hermite_basis(n: int) -> HermiteBasis:
    """hermite_basis(n) (hermite.cpp:10-66) through the C++ host setup."""
    nodes, psi, mass, diff = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(max(n, 1) ** 2)
    check(lib().kronop_host_hermite_basis(n, _dptr(nodes), _dptr(psi), _dptr(mass), _dptr(diff)))
    return HermiteBasis(n, nodes, psi, diff.reshape(n, n, order="F"), mass)


def build_axis(basis, f: Optional[Callable] = None, fvals: Optional[np.ndarray] = None):
    """build_axis for an SEM basis (axis.cpp:55-74) or a Hermite basis (axis.cpp:76-84) via the
    C++ Householder+QL eigensolver."""
    n = basis.size
    if fvals is None:
        fvals = np.array([f(float(x)) for x in basis.nodes]) if f is not None else np.zeros(n)
    fvals = np.ascontiguousarray(fvals, dtype=np.float64)
    if isinstance(basis, HermiteBasis):
        key = ("hermite", n, fvals.tobytes())
        if key not in _AXIS_CACHE:
            lam, t, ti = np.zeros(n), np.zeros(n * n), np.zeros(n * n)
            check(lib().kronop_host_build_hermite_axis(n, _dptr(fvals), _dptr(lam), _dptr(t),
                                                       _dptr(ti)))
            _AXIS_CACHE[key] = AxisEigens(lam, t.reshape(n, n, order="F"),
                                          ti.reshape(n, n, order="F"))
        return _AXIS_CACHE[key]
    key = (basis.half_width, basis.cell_count, basis.degree, fvals.tobytes())
    if key in _AXIS_CACHE:
        return _AXIS_CACHE[key]
    lam, t, ti = np.zeros(n), np.zeros(n * n), np.zeros(n * n)
    check(lib().kronop_host_build_sem_axis(basis.half_width, basis.cell_count, basis.degree,
                                           _dptr(fvals), _dptr(lam), _dptr(t), _dptr(ti)))
    ax = AxisEigens(lam, t.reshape(n, n, order="F"), ti.reshape(n, n, order="F"))
    _AXIS_CACHE[key] = ax
    return ax


@dataclass
class FoldedAxis:
    """Even/odd factorisation of a mirror-symmetric axis (host_setup.hpp FoldedAxis): half-size
    forward / backward blocks on u = x_i + x_{n-1-i} (+ middle node) and v = x_i - x_{n-1-i}."""
    n: int
    eigenvalues_even: np.ndarray
    eigenvalues_odd: np.ndarray
    fe: np.ndarray
    fo: np.ndarray
    be: np.ndarray
    bo: np.ndarray
    ground: np.ndarray

    @property
    def size(self):
        return self.n

    @property
    def eigenvalues(self):
        """All eigenvalues in folded order [even | odd] (the transformed layout)."""
        return np.concatenate([self.eigenvalues_even, self.eigenvalues_odd])


def build_axis_folded(basis: Basis1D, f: Optional[Callable] = None,
                      fvals: Optional[np.ndarray] = None) -> FoldedAxis:
    """Folded build_axis for a symmetric SEM axis and an even potential (ParameterError otherwise)."""
    if not isinstance(basis, Basis1D):
        raise L.ParameterError(L.KRONOP_EPARAM, "build_axis_folded: SEM axes only")
    n = basis.size
    if fvals is None:
        fvals = np.array([f(float(x)) for x in basis.nodes]) if f is not None else np.zeros(n)
    fvals = np.ascontiguousarray(fvals, dtype=np.float64)
    key = ("folded", basis.half_width, basis.cell_count, basis.degree, fvals.tobytes())
    if key in _AXIS_CACHE:
        return _AXIS_CACHE[key]
    no = n // 2
    ne = n - no
    le, lo = np.zeros(ne), np.zeros(max(no, 1))
    fe, be = np.zeros(ne * ne), np.zeros(ne * ne)
    fo, bo = np.zeros(max(no * no, 1)), np.zeros(max(no * no, 1))
    g = np.zeros(n)
    check(lib().kronop_host_build_sem_axis_folded(basis.half_width, basis.cell_count, basis.degree,
                                                  _dptr(fvals), _dptr(le), _dptr(lo), _dptr(fe),
                                                  _dptr(fo), _dptr(be), _dptr(bo), _dptr(g)))
    ax = FoldedAxis(n, le, lo[:no].copy(), fe.reshape(ne, ne, order="F"),
                    fo[:no * no].reshape(no, no, order="F"), be.reshape(ne, ne, order="F"),
                    bo[:no * no].reshape(no, no, order="F"), g)
    _AXIS_CACHE[key] = ax
    return ax


# ---------------------------------------------------------------------------- operators --
class SeparableOperator:
    """proj/include/kronop/operators.hpp:15-53, resident on the device."""

    def __init__(self, ctx: Context, axes: Sequence[AxisEigens], shift: float = 0.0,
                 mass: Optional[Sequence[np.ndarray]] = None):
        self.ctx = ctx
        self.axes = list(axes)
        d = len(axes)
        self.shape = tuple(a.size for a in axes)
        n = (C.c_int * d)(*self.shape)
        self._keep = [np.asfortranarray(a.transform) for a in axes] + \
                     [np.asfortranarray(a.inverse_transform) for a in axes] + \
                     [np.ascontiguousarray(a.eigenvalues) for a in axes]
        T = _arr_of_ptrs(self._keep[:d])
        Ti = _arr_of_ptrs(self._keep[d:2 * d])
        lam = _arr_of_ptrs(self._keep[2 * d:])
        self.mass = [np.ascontiguousarray(m, dtype=np.float64) for m in mass] if mass else None
        mp = _arr_of_ptrs(self.mass) if self.mass else None
        h = C.c_void_p()
        check(lib().kronop_op_create(ctx.h, d, n, T, Ti, lam, mp, shift, C.byref(h)))
        self.h = h
        ctx._ops.add(self)

    @classmethod
    def folded(cls, ctx: Context, axes: Sequence[FoldedAxis], shift: float = 0.0,
               mass: Optional[Sequence[np.ndarray]] = None) -> "SeparableOperator":
        """Even/odd folded variant (kronop_op_create_folded): same operator, half-size blocks per
        axis. Per-pass entry points (transform_pass, the slab backend) are not available."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.axes = list(axes)
        d = len(axes)
        self.shape = tuple(a.n for a in axes)
        n = (C.c_int * d)(*self.shape)
        groups = [[np.asfortranarray(getattr(a, k)) if getattr(a, k).size else np.zeros(1)
                   for a in axes] for k in ("fe", "fo", "be", "bo")]
        groups += [[np.ascontiguousarray(a.eigenvalues_even) for a in axes],
                   [np.ascontiguousarray(a.eigenvalues_odd) if a.n > 1 else np.zeros(1)
                    for a in axes],
                   [np.ascontiguousarray(a.ground) for a in axes]]
        self._keep = groups
        ptrs = [_arr_of_ptrs(g) for g in groups]
        self.mass = [np.ascontiguousarray(m, dtype=np.float64) for m in mass] if mass else None
        mp = _arr_of_ptrs(self.mass) if self.mass else None
        h = C.c_void_p()
        check(lib().kronop_op_create_folded(ctx.h, d, n, *ptrs, mp, shift, C.byref(h)))
        self.h = h
        ctx._ops.add(self)
        return self

    def release(self):
        if getattr(self, "h", None):
            lib().kronop_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    @property
    def dim(self):
        return len(self.shape)

    @property
    def size(self):
        return int(np.prod(self.shape))

    def info(self):
        s, lo, hi, n = C.c_double(), C.c_double(), C.c_double(), C.c_size_t()
        check(lib().kronop_op_info(self.h, C.byref(s), C.byref(lo), C.byref(hi), C.byref(n)))
        return s.value, lo.value, hi.value

    @property
    def shift(self):
        return self.info()[0]

    def set_shift(self, shift: float):
        check(lib().kronop_op_set_shift(self.h, shift))

    def min_eigenvalue(self):
        return self.info()[1]

    def max_eigenvalue(self):
        return self.info()[2]

    def _out(self, like, out):
        return torch.empty_like(like) if out is None else out

    def apply(self, u: torch.Tensor, out=None) -> torch.Tensor:
        out = self._out(u, out)
        with _Call(self.ctx):
            check(lib().kronop_sep_apply(self.ctx.h, self.h, _ptr(u), int(u.is_complex()), _ptr(out)))
        return out

    def solve(self, b: torch.Tensor, out=None) -> torch.Tensor:
        out = self._out(b, out)
        with _Call(self.ctx):
            check(lib().kronop_sep_solve(self.ctx.h, self.h, _ptr(b), int(b.is_complex()), _ptr(out)))
        return out

    def solve_lowp(self, b: torch.Tensor, precision: str = "bf16", out=None) -> torch.Tensor:
        """Reduced-precision solve on the tcgen05 tensor cores (kronop_sep_solve_lowp, FP32
        accumulation in TMEM): "bf16" (BF16 storage, the paper's BF16 mode, ~1e-2 relative),
        "tf32" (FP32 storage, TF32 products, ~1e-3), "fp32" (3xTF32 on (hi, lo) pairs, the
        paper's FP32 mode, ~1e-6), or FP64 emulated on the INT8 tensor cores (Ozaki scheme):
        "ozaki" (7 slices of 8 bits, FP64-level), "ozaki6", "ozaki5" (fewer slices, ~1e-13 /
        ~1e-11)."""
        out = self._out(b, out)
        prec = {"bf16": 1, "tf32": 2, "fp32": 3, "ozaki": 4, "ozaki7": 4, "ozaki6": 5,
                "ozaki5": 6}[precision]
        with _Call(self.ctx):
            check(lib().kronop_sep_solve_lowp(self.ctx.h, self.h, _ptr(b), prec, _ptr(out)))
        return out

    def set_precision(self, precision: str = "fp64"):
        """kronop_op_set_precision: run every later transform of this operator (and the drivers
        built on it: PCG, inverse iteration, GPE, splitting) in "fp64" (DMMA, default) or FP64
        emulated on the INT8 tensor cores ("ozaki", "ozaki6", "ozaki5")."""
        prec = {"fp64": 0, "ozaki": 4, "ozaki7": 4, "ozaki6": 5, "ozaki5": 6}[precision]
        with _Call(self.ctx):
            check(lib().kronop_op_set_precision(self.ctx.h, self.h, prec))
        return self

    def propagate_lowp(self, psi: torch.Tensor, dt: float, precision: str = "ozaki",
                       out=None) -> torch.Tensor:
        """exp(-i dt (-Delta+V1)) psi with FP64 emulated on the INT8 tensor cores
        (kronop_sep_propagate_lowp): "ozaki" (7 slices), "ozaki6", "ozaki5"."""
        if not psi.is_complex():
            raise ValueError("propagate_lowp needs a complex128 field")
        out = self._out(psi, out)
        prec = {"ozaki": 4, "ozaki7": 4, "ozaki6": 5, "ozaki5": 6}[precision]
        with _Call(self.ctx):
            check(lib().kronop_sep_propagate_lowp(self.ctx.h, self.h, _ptr(psi), C.c_double(dt),
                                                  prec, _ptr(out)))
        return out

    def solve_bf16(self, b: torch.Tensor, out=None) -> torch.Tensor:
        return self.solve_lowp(b, "bf16", out)

    def propagate(self, psi: torch.Tensor, dt: float, out=None) -> torch.Tensor:
        if not psi.is_complex():
            raise ValueError("propagate needs a complex128 field")
        out = self._out(psi, out)
        with _Call(self.ctx):
            check(lib().kronop_sep_propagate(self.ctx.h, self.h, _ptr(psi), dt, _ptr(out)))
        return out

    def ground_state(self) -> torch.Tensor:
        out = torch.empty(self.size, dtype=torch.float64, device="cuda:%d" % self.ctx.device)
        with _Call(self.ctx):
            check(lib().kronop_op_ground_state(self.ctx.h, self.h, _ptr(out)))
        return out

    def eigenvalue_grid(self) -> torch.Tensor:
        out = torch.empty(self.size, dtype=torch.float64, device="cuda:%d" % self.ctx.device)
        with _Call(self.ctx):
            check(lib().kronop_op_eigenvalue_grid(self.ctx.h, self.h, _ptr(out)))
        return out

    def transform_pass(self, x: torch.Tensor, axis: int, forward: bool = True, out=None):
        """One mode-product pass with the resident T^{-1} (forward) or T (kronop_op_pass)."""
        out = self._out(x, out)
        with _Call(self.ctx):
            check(lib().kronop_op_pass(self.ctx.h, self.h, axis, int(forward), _ptr(x),
                                       int(x.is_complex()), _ptr(out)))
        return out

    EPI = {"store": 0, "mul": 1, "div": 2, "phase": 3, "axpy": 4}

    def transform_pass_ex(self, x: torch.Tensor, axis: int, forward: bool = True,
                          epilogue: str = "store", dt: float = 0.0, diag=None, sigma: float = 0.0,
                          u=None, out=None):
        """One pass with a fused epilogue (kronop_op_pass_ex): "store", "mul" / "div" (spectral
        x / ÷ (lambda - shift)), "phase" (x exp(-i (lambda - shift) dt)), "axpy" (+ diag u - sigma u)."""
        out = self._out(x, out)
        with _Call(self.ctx):
            check(lib().kronop_op_pass_ex(self.ctx.h, self.h, axis, int(forward), _ptr(x),
                                          int(x.is_complex()), _ptr(out), self.EPI[epilogue],
                                          C.c_double(dt), _ptr(diag), C.c_double(sigma), _ptr(u)))
        return out

    # host-buffer (end-to-end) variants
    def solve_host(self, b: np.ndarray, out: np.ndarray, is_complex=None):
        """kronop_sep_solve_host: host in / host out, copies overlapped with the passes."""
        cplx = np.iscomplexobj(b) if is_complex is None else is_complex
        check(lib().kronop_sep_solve_host(self.ctx.h, self.h, C.c_void_p(b.ctypes.data),
                                          int(cplx), C.c_void_p(out.ctypes.data)))
        return out

    def solve_host_batch(self, bs, outs, is_complex=None):
        """kronop_sep_solve_host_batch: a list of host right-hand sides -> host solutions, the
        copies of neighbouring items overlapped with each item's transform."""
        n = len(bs)
        cplx = (n > 0 and np.iscomplexobj(bs[0])) if is_complex is None else is_complex
        ins = (C.c_void_p * n)(*[b.ctypes.data for b in bs])
        ous = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
        check(lib().kronop_sep_solve_host_batch(self.ctx.h, self.h, n, ins, int(cplx), ous))
        return outs

    def propagate_host_batch(self, psis, dt: float, outs):
        n = len(psis)
        ins = (C.c_void_p * n)(*[p.ctypes.data for p in psis])
        ous = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
        check(lib().kronop_sep_propagate_host_batch(self.ctx.h, self.h, n, ins, C.c_double(dt),
                                                    ous))
        return outs

    def apply_host(self, u: np.ndarray, out: np.ndarray):
        check(lib().kronop_sep_apply_host(self.ctx.h, self.h, C.c_void_p(u.ctypes.data),
                                          int(np.iscomplexobj(u)), C.c_void_p(out.ctypes.data)))
        return out

    def propagate_host(self, psi: np.ndarray, dt: float, out: np.ndarray):
        check(lib().kronop_sep_propagate_host(self.ctx.h, self.h, C.c_void_p(psi.ctypes.data), dt,
                                              C.c_void_p(out.ctypes.data)))
        return out


@dataclass
class FullOperator:
    """sep + optional V2 diagonal (operators.hpp:56-62)."""
    sep: SeparableOperator
    diagonal: Optional[torch.Tensor] = None

    def apply(self, u: torch.Tensor, sigma: float = 0.0, out=None) -> torch.Tensor:
        out = torch.empty_like(u) if out is None else out
        with _Call(self.sep.ctx):
            check(lib().kronop_full_apply(self.sep.ctx.h, self.sep.h, _ptr(self.diagonal), sigma,
                                          _ptr(u), int(u.is_complex()), _ptr(out)))
        return out


# ------------------------------------------------------------------------------ tensor --
def _shape_arr(shape):
    return (C.c_int * len(shape))(*shape)


def mode_product(ctx: Context, x: torch.Tensor, shape, a: np.ndarray, axis: int) -> torch.Tensor:
    """tensor.hpp:79-81."""
    a = np.asfortranarray(a, dtype=np.float64)
    if not 0 <= axis < len(shape):
        raise L.ParameterError(L.KRONOP_EPARAM, "mode_product: axis out of range")
    if a.ndim != 2 or a.shape[1] != shape[axis]:
        raise L.ParameterError(L.KRONOP_EPARAM,
                               "mode_product: matrix columns do not match axis extent")
    m = a.shape[0]
    out_shape = list(shape)
    out_shape[axis] = m
    out = torch.empty(int(np.prod(out_shape)), dtype=x.dtype, device=x.device)
    with _Call(ctx):
        check(lib().kronop_mode_product(ctx.h, _ptr(x), len(shape), _shape_arr(shape),
                                        int(x.is_complex()), a.ctypes.data_as(_PD), m, axis,
                                        _ptr(out)))
    return out


def kron_apply(ctx: Context, x: torch.Tensor, shape, mats) -> torch.Tensor:
    """tensor.hpp:85-87 (None = identity)."""
    if len(mats) != len(shape):
        raise L.ParameterError(L.KRONOP_EPARAM, "kron_apply: need one matrix (or null) per axis")
    keep = [np.asfortranarray(a, dtype=np.float64) if a is not None else None for a in mats]
    for i, a in enumerate(keep):
        if a is not None and (a.ndim != 2 or a.shape[1] != shape[i]):
            raise L.ParameterError(L.KRONOP_EPARAM,
                                   "mode_product: matrix columns do not match axis extent")
    ms = [a.shape[0] if a is not None else 0 for a in keep]
    out_shape = [ms[i] if keep[i] is not None else shape[i] for i in range(len(shape))]
    out = torch.empty(int(np.prod(out_shape)), dtype=x.dtype, device=x.device)
    with _Call(ctx):
        check(lib().kronop_kron_apply(ctx.h, _ptr(x), len(shape), _shape_arr(shape),
                                      int(x.is_complex()), _arr_of_ptrs(keep),
                                      _shape_arr(ms), _ptr(out)))
    return out


def inner(ctx: Context, u: torch.Tensor, v: torch.Tensor, shape, mass=None):
    """tensor.hpp:89-98: conjugate-linear in u; mass = per-axis weights or None (plain)."""
    res = np.zeros(2)
    mk = [np.ascontiguousarray(m, dtype=np.float64) for m in mass] if mass is not None else None
    with _Call(ctx):
        check(lib().kronop_inner(ctx.h, _ptr(u), _ptr(v), len(shape), _shape_arr(shape),
                                 int(u.is_complex()), _arr_of_ptrs(mk) if mk else None,
                                 _dptr(res)))
    return complex(res[0], res[1]) if u.is_complex() else float(res[0])


def norm(ctx, u, shape, mass=None) -> float:
    s = inner(ctx, u, u, shape, mass)
    return math.sqrt(s.real if isinstance(s, complex) else s)


def mass_field(ctx: Context, shape, mass) -> torch.Tensor:
    out = torch.empty(int(np.prod(shape)), dtype=torch.float64, device="cuda:%d" % ctx.device)
    mk = [np.ascontiguousarray(m, dtype=np.float64) for m in mass]
    with _Call(ctx):
        check(lib().kronop_mass_field(ctx.h, len(shape), _shape_arr(shape), _arr_of_ptrs(mk),
                                      _ptr(out)))
    return out


def direct_sum_grid(ctx: Context, values) -> torch.Tensor:
    shape = [len(v) for v in values]
    out = torch.empty(int(np.prod(shape)), dtype=torch.float64, device="cuda:%d" % ctx.device)
    vk = [np.ascontiguousarray(v, dtype=np.float64) for v in values]
    with _Call(ctx):
        check(lib().kronop_direct_sum_grid(ctx.h, len(shape), _shape_arr(shape), _arr_of_ptrs(vk),
                                           _ptr(out)))
    return out


def splitmix_uniform(ctx: Context, seed: int, count: int, start: int = 0) -> torch.Tensor:
    """SplitMix64 uniform_pm1 stream (rng.hpp:16-35) generated on the device."""
    out = torch.empty(count, dtype=torch.float64, device="cuda:%d" % ctx.device)
    with _Call(ctx):
        check(lib().kronop_splitmix_uniform(ctx.h, seed, start, count, _ptr(out)))
    return out


# --------------------------------------------------------------------------------- grid --
class Grid:
    """Isotropic SEM tensor grid (proj/include/kronop/grid.hpp:16-39, grid.cpp:14-22)."""

    def __init__(self, axes: List[Basis1D]):
        self.axes = axes

    @staticmethod
    def sem(half_width: float, cell_count: int, degree: int, dimension: int) -> "Grid":
        if dimension < 1 or dimension > 9:
            raise L.ParameterError(L.KRONOP_EPARAM, "Grid: dimension must be in [1, 9]")
        b = assemble_sem(half_width, cell_count, degree)
        return Grid([b] * dimension)

    @staticmethod
    def hermite(n: int, dimension: int) -> "Grid":
        """Isotropic Hermite collocation grid on R^d (grid.cpp:24-32)."""
        if dimension < 1 or dimension > 9:
            raise L.ParameterError(L.KRONOP_EPARAM, "Grid: dimension must be in [1, 9]")
        return Grid([hermite_basis(n)] * dimension)

    @property
    def dim(self):
        return len(self.axes)

    @property
    def shape(self):
        return tuple(a.size for a in self.axes)

    @property
    def mass(self):
        return [a.mass for a in self.axes]

    def node_count(self):
        return int(np.prod(self.shape))

    def coords(self):
        d = self.dim
        out = []
        for a in range(d):
            shp = [1] * d
            shp[d - 1 - a] = self.axes[a].size
            out.append(self.axes[a].nodes.reshape(shp))
        return out

    def sample(self, f_vec) -> np.ndarray:
        """Nodal sampling (grid.cpp:53-69) on the host; f_vec gets per-axis coordinates."""
        v = f_vec(self.coords())
        return np.ascontiguousarray(np.broadcast_to(v, tuple(reversed(self.shape))).reshape(-1),
                                    dtype=np.float64)

    def separable_operator(self, ctx: Context, per_axis=None, shift: float = 0.0,
                           folded: bool = False):
        """grid.cpp:71-83: per_axis = list of scalar functions (or None = 0). folded=True builds
        the even/odd folded variant (symmetric axes and even per-axis potentials only)."""
        axes = []
        for a in range(self.dim):
            f = per_axis[a] if per_axis else None
            fv = np.array([f(float(x)) for x in self.axes[a].nodes]) if f else None
            build = build_axis_folded if folded else build_axis
            axes.append(build(self.axes[a], f=None, fvals=fv))
        if folded:
            return SeparableOperator.folded(ctx, axes, shift, mass=self.mass)
        return SeparableOperator(ctx, axes, shift, mass=self.mass)

    def laplacian(self, ctx: Context, shift: float = 0.0, folded: bool = False):
        return self.separable_operator(ctx, None, shift, folded=folded)


# ----------------------------------------------------------------------------- drivers --
@dataclass
class PcgConfig:
    """pcg.hpp:10-20."""
    rel_tol: float = 1e-12
    max_iter: int = 500
    record_history: bool = False
    preconditioned_norm: bool = False
    stagnation_window: int = 0

    def c(self):
        return L.PcgConfig(self.rel_tol, self.max_iter, int(self.record_history),
                           int(self.preconditioned_norm), self.stagnation_window)


@dataclass
class PcgReport:
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    history: list = field(default_factory=list)


def apply_map(op: SeparableOperator, diag=None, sigma: float = 0.0):
    """KRONOP_MAP_APPLY: v -> op.apply(v) + diag v - sigma v."""
    return (L.LinearMap(op.h, L.KRONOP_MAP_APPLY, _ptr(diag), sigma, None), (op, diag))


def solve_map(op: SeparableOperator, scale=None):
    """KRONOP_MAP_SOLVE: r -> scale .* op.solve(scale .* r)."""
    return (L.LinearMap(op.h, L.KRONOP_MAP_SOLVE, None, 0.0, _ptr(scale)), (op, scale))


def pcg(apply_a, precond, b: torch.Tensor, x: torch.Tensor, config: PcgConfig = PcgConfig()):
    """pcg.hpp:36-37; x is updated in place (warm start in, solution out)."""
    ctx = apply_a[1][0].ctx
    rep = L.PcgReport()
    hist = np.zeros(config.max_iter + 2)
    cfg = config.c()
    with _Call(ctx):
        check(lib().kronop_pcg(ctx.h, C.byref(apply_a[0]), C.byref(precond[0]), _ptr(b), _ptr(x),
                               C.byref(cfg), C.byref(rep),
                               _dptr(hist) if config.record_history else None))
    return PcgReport(rep.iterations, rep.final_residual, bool(rep.converged),
                     list(hist[:rep.history_len]) if config.record_history else [])


@dataclass
class InverseIterationConfig:
    """ground_state.hpp:24-32."""
    shift_mode: str = "fraction"
    shift_fraction: float = 0.9
    shift_offset: float = 1e-4
    eig_rel_tol: float = 1e-12
    max_outer: int = 60
    inner: PcgConfig = field(default_factory=lambda: PcgConfig(stagnation_window=100))


@dataclass
class EigenpairResult:
    eigenvalue: float
    eigenvector: torch.Tensor
    outer_iterations: int
    total_inner_iterations: int
    inner_per_outer: list
    converged: bool


def inverse_iteration(op: FullOperator, config: InverseIterationConfig, initial: torch.Tensor):
    """ground_state.hpp:47-56 (op.sep must carry mass weights)."""
    ctx = op.sep.ctx
    mode = {"fraction": 0, "offset": 1, "zero": 2}[config.shift_mode]
    cfg = L.InverseIterationConfig(mode, config.shift_fraction, config.shift_offset,
                                   config.eig_rel_tol, config.max_outer, config.inner.c())
    res = L.EigenpairResult()
    per = (C.c_int * max(1, config.max_outer))()
    vec = torch.empty_like(initial)
    with _Call(ctx):
        check(lib().kronop_inverse_iteration(ctx.h, op.sep.h, _ptr(op.diagonal), C.byref(cfg),
                                             _ptr(initial), _ptr(vec), C.byref(res), per))
    inner = list(per[:res.outer_iterations]) if op.diagonal is not None else []
    return EigenpairResult(res.eigenvalue, vec, res.outer_iterations, res.total_inner_iterations,
                           inner, bool(res.converged))


@dataclass
class GpeFlowConfig:
    """gpe.hpp:30-40."""
    kind: str = "h1"
    step: float = 0.1
    metric_shift: float = 20.0
    energy_rel_tol: float = 1e-12
    max_iterations: int = 20000
    inner: PcgConfig = field(default_factory=lambda: PcgConfig(stagnation_window=100))
    init: str = "eigenfunction"
    record_history: bool = False


@dataclass
class GpeResult:
    state: torch.Tensor
    energy: float
    eigenvalue: float
    iterations: int
    linear_solves: int
    converged: bool
    history: list


def gpe_energy(ham: FullOperator, beta: float, u: torch.Tensor) -> float:
    e = C.c_double()
    ctx = ham.sep.ctx
    with _Call(ctx):
        check(lib().kronop_gpe_energy(ctx.h, ham.sep.h, _ptr(ham.diagonal), beta, _ptr(u),
                                      C.byref(e)))
    return e.value


def gpe_gradient_flow(ham: FullOperator, laplacian: SeparableOperator, beta: float,
                      config: GpeFlowConfig, initial: Optional[torch.Tensor] = None):
    """gpe.hpp:65-66."""
    ctx = ham.sep.ctx
    cfg = L.GpeConfig({"h1": 0, "au": 1}[config.kind], config.step, config.metric_shift,
                      config.energy_rel_tol, config.max_iterations, config.inner.c(),
                      {"constant": 0, "eigenfunction": 1, "supplied": 2}[config.init],
                      int(config.record_history))
    res = L.GpeResult()
    hist = np.zeros(5 * max(1, config.max_iterations)) if config.record_history else None
    state = torch.empty(ham.sep.size, dtype=torch.float64, device="cuda:%d" % ctx.device)
    with _Call(ctx):
        check(lib().kronop_gpe_gradient_flow(ctx.h, ham.sep.h, _ptr(ham.diagonal), laplacian.h,
                                             beta, C.byref(cfg), _ptr(initial), _ptr(state),
                                             C.byref(res), _dptr(hist) if hist is not None else None))
    rows = hist[:5 * res.history_len].reshape(-1, 5).tolist() if hist is not None else []
    return GpeResult(state, res.energy, res.eigenvalue, res.iterations, res.linear_solves,
                     bool(res.converged), rows)


def yoshida_coeffs():
    g1, g2 = C.c_double(), C.c_double()
    check(lib().kronop_yoshida_coeffs(C.byref(g1), C.byref(g2)))
    return g1.value, g2.value


def qhop_step(a: SeparableOperator, b_diag: torch.Tensor, psi: torch.Tensor, h: float, m: int):
    out = torch.empty_like(psi)
    with _Call(a.ctx):
        check(lib().kronop_qhop_step(a.ctx.h, a.h, _ptr(b_diag), _ptr(psi), h, m, _ptr(out)))
    return out


def yoshida_step(a: SeparableOperator, b_diag: torch.Tensor, psi: torch.Tensor, h: float, m: int):
    out = torch.empty_like(psi)
    with _Call(a.ctx):
        check(lib().kronop_yoshida_step(a.ctx.h, a.h, _ptr(b_diag), _ptr(psi), h, m, _ptr(out)))
    return out


@dataclass
class SplitSpec:
    """splitting.hpp:26-33."""
    quad_points: int = 1
    composition: str = "single"
    dt: float = 0.0
    total_time: float = 0.0
    merge_across_steps: bool = False
    mass_weighted_error: bool = False


def evolve(spec: SplitSpec, a: SeparableOperator, b_diag: torch.Tensor, psi0: torch.Tensor,
           exact: Optional[SeparableOperator] = None, stationary_eigenvalue: float = 0.0):
    """splitting.hpp:68-69. Returns (state, error, steps)."""
    cs = L.SplitSpec(spec.quad_points, {"single": 0, "yoshida": 1}[spec.composition], spec.dt,
                     spec.total_time, int(spec.merge_across_steps), int(spec.mass_weighted_error))
    state = torch.empty_like(psi0)
    err = C.c_double()
    steps = C.c_int()
    with _Call(a.ctx):
        check(lib().kronop_evolve(a.ctx.h, C.byref(cs), a.h, _ptr(b_diag), _ptr(psi0),
                                  exact.h if exact is not None else None, stationary_eigenvalue,
                                  _ptr(state), C.byref(err), C.byref(steps)))
    return state, err.value, steps.value


@dataclass
class LevelReport:
    """ground_state.hpp:58-66."""
    n: int
    outer_iterations: int
    total_inner_iterations: int
    inner_per_outer: float
    eigenvalue: float
    setup_seconds: float = 0.0
    interp_seconds: float = 0.0


def multilevel_ground_state(ctx: Context, grids: Sequence[Grid], make_operator,
                            config: InverseIterationConfig):
    """Coarse-to-fine continuation (ground_state.cpp:101-154): solve on each SEM grid, prolong the
    eigenvector with per-axis piecewise-linear interpolation (rectangular mode products on the
    device), continue. make_operator(grid) -> FullOperator. Returns (EigenpairResult, [LevelReport])."""
    if not grids:
        raise L.ParameterError(L.KRONOP_EPARAM, "multilevel_ground_state: no levels")
    import time
    guess, prev = None, None
    levels, pair = [], None
    for grid in grids:
        t0 = time.perf_counter()
        op = make_operator(grid)
        torch.cuda.synchronize()
        setup_s, interp_s = time.perf_counter() - t0, 0.0
        if guess is None:
            initial = op.sep.ground_state()
        else:
            if not all(isinstance(b, Basis1D) for b in prev.axes + grid.axes):
                raise L.ParameterError(L.KRONOP_EPARAM,
                                       "multilevel_ground_state: levels must be SEM grids")
            t0 = time.perf_counter()
            mats = [interp_matrix(prev.axes[a], grid.axes[a]) for a in range(grid.dim)]
            initial = kron_apply(ctx, guess, prev.shape, mats)
            torch.cuda.synchronize()
            interp_s = time.perf_counter() - t0
        pair = inverse_iteration(op, config, initial)
        levels.append(LevelReport(grid.axes[0].size, pair.outer_iterations,
                                  pair.total_inner_iterations,
                                  pair.total_inner_iterations / max(1, pair.outer_iterations)
                                  if pair.outer_iterations > 0 else 0.0,
                                  pair.eigenvalue, setup_s, interp_s))
        guess, prev = pair.eigenvector, grid
    return pair, levels


# ------------------------------------------------------------------------------ field I/O --
def _shape_arr(shape):
    return (C.c_int * len(shape))(*[int(n) for n in shape])


def dump_field(path: str, field, shape: Sequence[int], ctx: Optional[Context] = None):
    """dump_field (fieldio.cpp:28-47) in the reference's binary format. `field` is a CUDA tensor
    (streamed through pinned chunks on ctx's stream) or a numpy array (host path); `shape` is the
    reference shape (axis 0 first). Complex dtype -> scalar kind 1."""
    if isinstance(field, torch.Tensor):
        if ctx is None:
            raise ValueError("dump_field: a device field needs its Context")
        with _Call(ctx):
            check(lib().kronop_field_dump(ctx.h, path.encode(), len(shape), _shape_arr(shape),
                                          int(field.is_complex()), _ptr(field)))
    else:
        a = np.ascontiguousarray(field)
        cplx = np.iscomplexobj(a)
        v = a.view(np.float64) if cplx else a.astype(np.float64, copy=False)
        check(lib().kronop_field_dump_host(path.encode(), len(shape), _shape_arr(shape),
                                           int(cplx), _dptr(v)))


def load_field_header(path: str):
    d, cplx = C.c_int(), C.c_int()
    shp = (C.c_int * 9)()
    check(lib().kronop_field_load_header(path.encode(), C.byref(d), shp, C.byref(cplx)))
    return tuple(shp[i] for i in range(d.value)), bool(cplx.value)


def load_field(path: str, ctx: Optional[Context] = None):
    """load_field (fieldio.cpp:49-73): returns (field, shape, is_complex); a CUDA tensor when ctx
    is given (uploaded through pinned chunks), else a numpy array."""
    shape, cplx = load_field_header(path)
    n = int(np.prod(shape))
    doubles = n * (2 if cplx else 1)
    if ctx is None:
        buf = np.empty(doubles, dtype=np.float64)
        check(lib().kronop_field_load_host(path.encode(), _dptr(buf), doubles))
        return (buf.view(np.complex128) if cplx else buf), shape, cplx
    t = torch.empty(n, dtype=torch.complex128 if cplx else torch.float64,
                    device="cuda:%d" % ctx.device)
    with _Call(ctx):
        check(lib().kronop_field_load(ctx.h, path.encode(), _ptr(t), doubles))
    return t, shape, cplx

