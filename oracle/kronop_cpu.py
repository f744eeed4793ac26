"""CPU ORACLE (C++ restatement), ctypes wrapper — test infrastructure and the timed CPU reference
arm only; never the product (the product path, paper_2605_20491_b200 + libkronop.so, never
imports anything under oracle/).

`oracle/cpu/kronop_cpu.cpp` restates the reference's CPU execution of the hot path
(/root/reference/proj/src/tensor.cpp:31-145, operators.cpp:7-105, pcg.cpp:8-81) with its own
structure: zero-filled std::vector fields, OpenMP static partitions of single-threaded GEMMs,
serial spectral / vector loops. The reference itself cannot be built here (Eigen3 is absent,
SURVEY.md §8c), so this is the `"kind": "port"` CPU baseline; it is checked against the numpy
oracle (`kronop_oracle.py`, pinned against the reference's golden values) in
tests/test_oracle_cpu.py.
"""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cpu", "build", "libkronop_cpu.so")
_lib = None


def blas_path() -> str:
    """numpy's bundled OpenBLAS (ILP64, `scipy_cblas_dgemm64_`)."""
    d = os.path.join(os.path.dirname(np.__file__), os.pardir, "numpy.libs")
    cands = sorted(glob.glob(os.path.join(d, "libscipy_openblas64_*.so")))
    if not cands:
        raise RuntimeError("numpy's bundled OpenBLAS (libscipy_openblas64_) not found")
    return os.path.abspath(cands[0])


def build() -> str:
    src = os.path.join(HERE, "cpu", "kronop_cpu.cpp")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["sh", os.path.join(HERE, "cpu", "build.sh")])
    return SO


def lib(threads: int = 0):
    """Load (building if needed) and initialise with `threads` OpenMP threads (0 = all)."""
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.kcpu_last_error.restype = ctypes.c_char_p
        if L.kcpu_init(blas_path().encode(), ctypes.c_int(threads)) != 0:
            raise RuntimeError(L.kcpu_last_error().decode())
        _lib = L
    return _lib


def threads() -> int:
    return int(lib().kcpu_threads())


def _check(rc):
    if rc != 0:
        msg = lib().kcpu_last_error().decode()
        if rc == 3:
            raise ArithmeticError(msg)
        raise ValueError(msg)


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class CpuOperator:
    """SeparableOperator (operators.hpp:15-53) on the C++ restatement. `axes`: objects with
    eigenvalues / transform / inverse_transform (oracle AxisEigens or the product's axes)."""

    def __init__(self, axes, shift: float = 0.0):
        L = lib()
        d = len(axes)
        self._keep = []
        n = (ctypes.c_int * d)(*[len(a.eigenvalues) for a in axes])
        T = (ctypes.POINTER(ctypes.c_double) * d)()
        Ti = (ctypes.POINTER(ctypes.c_double) * d)()
        La = (ctypes.POINTER(ctypes.c_double) * d)()
        for i, a in enumerate(axes):
            t = np.asfortranarray(a.transform, dtype=np.float64)
            ti = np.asfortranarray(a.inverse_transform, dtype=np.float64)
            la = np.ascontiguousarray(a.eigenvalues, dtype=np.float64)
            self._keep += [t, ti, la]
            T[i], Ti[i], La[i] = _dp(t), _dp(ti), _dp(la)
        self.shape = tuple(int(len(a.eigenvalues)) for a in axes)
        self.size = int(np.prod(self.shape))
        h = ctypes.c_void_p()
        _check(L.kcpu_op_create(ctypes.c_int(d), n, T, Ti, La, ctypes.c_double(shift),
                                ctypes.byref(h)))
        self._h = h
        self._keep = []

    def close(self):
        if self._h:
            lib().kcpu_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_shift(self, shift: float):
        lib().kcpu_op_set_shift(self._h, ctypes.c_double(shift))

    def solve(self, b):
        b = np.ascontiguousarray(b)
        out = np.empty_like(b)
        _check(lib().kcpu_sep_solve(self._h, _dp(b.view(np.float64)),
                                    ctypes.c_int(int(np.iscomplexobj(b))),
                                    _dp(out.view(np.float64))))
        return out

    def apply(self, u):
        u = np.ascontiguousarray(u)
        out = np.empty_like(u)
        _check(lib().kcpu_sep_apply(self._h, _dp(u.view(np.float64)),
                                    ctypes.c_int(int(np.iscomplexobj(u))),
                                    _dp(out.view(np.float64))))
        return out

    def propagate(self, psi, dt: float):
        psi = np.ascontiguousarray(psi, dtype=np.complex128)
        out = np.empty_like(psi)
        _check(lib().kcpu_sep_propagate(self._h, _dp(psi.view(np.float64)), ctypes.c_double(dt),
                                        _dp(out.view(np.float64))))
        return out

    def full_apply(self, diag, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        dg = None if diag is None else np.ascontiguousarray(diag, dtype=np.float64)
        _check(lib().kcpu_full_apply(self._h, None if dg is None else _dp(dg), _dp(u), _dp(out)))
        return out


def pcg(a_op: CpuOperator, diag, p_op: CpuOperator, b, x, rel_tol=1e-8, max_iter=1000,
        stagnation_window=0, preconditioned_norm=False):
    """pcg.cpp:8-81 with apply_a = FullOperator{a_op, diag}.apply, precond = p_op.solve.
    x is updated in place; returns (iterations, converged, final_residual, history)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert x.dtype == np.float64 and x.flags.c_contiguous
    dg = None if diag is None else np.ascontiguousarray(diag, dtype=np.float64)
    hist = np.zeros(max_iter + 1)
    its, conv, hl = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    fr = ctypes.c_double()
    _check(lib().kcpu_pcg(a_op._h, None if dg is None else _dp(dg), p_op._h, _dp(b), _dp(x),
                          ctypes.c_double(rel_tol), ctypes.c_int(max_iter),
                          ctypes.c_int(stagnation_window), ctypes.c_int(int(preconditioned_norm)),
                          ctypes.byref(its), ctypes.byref(conv), ctypes.byref(fr), _dp(hist),
                          ctypes.byref(hl)))
    return its.value, bool(conv.value), fr.value, list(hist[:hl.value])


def time_op(op: CpuOperator, kind: str, x, reps: int, dt: float = 0.0):
    """Times `reps` calls of op.<kind>(x) inside the library (the input field is built once,
    outside the timed region, as the reference's caller already holds it). Returns
    (last result, [seconds per call])."""
    x = np.ascontiguousarray(x)
    out = np.empty_like(x)
    secs = np.zeros(reps)
    k = {"solve": 0, "apply": 1, "propagate": 2}[kind]
    _check(lib().kcpu_time_op(op._h, ctypes.c_int(k), _dp(x.view(np.float64)),
                              ctypes.c_int(int(np.iscomplexobj(x))), ctypes.c_double(dt),
                              ctypes.c_int(reps), _dp(out.view(np.float64)), _dp(secs)))
    return out, list(secs)


def uniform_pm1(seed: int, count: int, start: int = 0) -> np.ndarray:
    """SplitMix64 uniform_pm1 stream (rng.hpp:16-31), OpenMP-parallel; equals
    kronop_oracle.uniform_pm1 bit for bit."""
    out = np.empty(count)
    lib().kcpu_uniform_pm1(ctypes.c_uint64(seed), ctypes.c_uint64(start), ctypes.c_int64(count),
                           _dp(out))
    return out
