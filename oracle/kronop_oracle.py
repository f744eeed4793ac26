"""CPU ORACLE — test infrastructure only, never the product.

A numpy restatement of the reference's (arxiv/paper_2605_20491, "kronop") CPU algorithm for the
tensor-product Schrodinger solver hot path. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module, and only as the
checker or as the timed CPU reference. The product path (paper_2605_20491_b200 + libkronop.so)
never imports it.

Every function cites the reference file:line it restates (paths relative to /root/reference/proj).
The reference itself cannot be compiled here (Eigen3, CLI11, doctest absent), so
this is a port ("kind": "port"); it is pinned against the reference's own golden values
(proj/tests/acceptance.cpp, see oracle/pin_golden.py and tests/golden/).

Field convention (proj/include/kronop/tensor.hpp:24-26): a field of shape (n0, ..., n_{d-1}) is a
flat array with axis 0 fastest, linear index i0 + n0*(i1 + n1*(...)). Here fields are 1-D numpy
arrays (float64 or complex128) plus the shape tuple; the numpy C-order view is reversed(shape).

Where the reference's arithmetic order is observable (GLL Newton iterations, schedule building,
stiffness assembly, lambda summation order, division rather than reciprocal multiplication), it is
followed operation for operation. Dense linear algebra (GEMM, symmetric eigensolver) goes through
numpy/LAPACK, which, like Eigen, is pinned to tolerance rather than bitwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np


class ParameterError(ValueError):
    """proj/include/kronop/errors.hpp:17-20 (exit code 2)."""


class NumericalError(ArithmeticError):
    """proj/include/kronop/errors.hpp:22-26 (exit code 3)."""


class CapabilityError(RuntimeError):
    """proj/include/kronop/errors.hpp:27-30 (exit code 4)."""


# --------------------------------------------------------------------------- rng.hpp

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs start..start+count-1 of SplitMix64(seed) (proj/include/kronop/rng.hpp:16-26)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, count: int, start: int = 0) -> np.ndarray:
    """SplitMix64::uniform_pm1 (rng.hpp:28-31): (next() >> 11) * 2^-52 - 1."""
    u = splitmix64(seed, count, start) >> np.uint64(11)
    return u.astype(np.float64) * 2.0 ** -52 - 1.0


def seeded_field(shape: Sequence[int], seed: int) -> np.ndarray:
    """random_field (proj/src/harness.cpp:184-189): f[i] = rng.uniform_pm1() in index order."""
    return uniform_pm1(seed, int(np.prod(shape)))


def seeded_complex_field(shape: Sequence[int], seed: int) -> np.ndarray:
    """{uniform, uniform} pairs in index order (proj/tests/test_operators.cpp:20-24)."""
    v = uniform_pm1(seed, 2 * int(np.prod(shape)))
    return v[0::2] + 1j * v[1::2]


# ---------------------------------------------------------------------- quadrature.cpp

def legendre_pair(k: int, x: float):
    """P_k(x), P'_k(x) (proj/src/quadrature.cpp:12-26)."""
    p0, p1 = 1.0, x
    if k == 0:
        return 1.0, 0.0
    for m in range(2, k + 1):
        p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m
        p0, p1 = p1, p2
    num, den = k * (x * p1 - p0), (x * x - 1.0)
    if den == 0.0:  # IEEE semantics of the C++ division at x = +-1 (dp unused there)
        return p1, (math.copysign(math.inf, num) if num != 0.0 else math.nan)
    return p1, num / den


def barycentric_weights(nodes):
    """proj/src/quadrature.cpp:28-39."""
    n = len(nodes)
    w = [1.0] * n
    for i in range(n):
        for j in range(n):
            if j != i:
                w[i] *= nodes[i] - nodes[j]
        w[i] = 1.0 / w[i]
    return w


def gauss_legendre(m: int, capped: bool = True):
    """Gauss-Legendre rule (proj/src/quadrature.cpp:41-87). Returns (nodes, weights) lists."""
    if capped and (m < 1 or m > 16):
        raise ParameterError("gauss_legendre: points must be in [1, 16]")
    if m == 1:
        return [0.0], [2.0]
    nodes = [0.0] * m
    weights = [0.0] * m
    for i in range(m):
        x = -math.cos(math.pi * (4.0 * i + 3.0) / (4.0 * m + 2.0))
        done = False
        for _ in range(100):
            p, dp = legendre_pair(m, x)
            dx = p / dp
            x -= dx
            if abs(dx) < 1e-15:
                done = True
                break
        if not done:
            raise NumericalError("gauss_legendre: Newton failed to converge")
        p, dp = legendre_pair(m, x)
        nodes[i] = x
        weights[i] = 2.0 / ((1.0 - x * x) * dp * dp)
    for i in range(m // 2):
        j = m - 1 - i
        xm = 0.5 * (nodes[j] - nodes[i])
        nodes[i] = -xm
        nodes[j] = xm
        wm = 0.5 * (weights[i] + weights[j])
        weights[i] = weights[j] = wm
    if m % 2 == 1:
        nodes[m // 2] = 0.0
    return nodes, weights


def lagrange_diff_matrix(nodes) -> np.ndarray:
    """proj/src/quadrature.cpp:95-110 (rows sum to zero exactly)."""
    n = len(nodes)
    b = barycentric_weights(nodes)
    d = np.zeros((n, n))
    for i in range(n):
        diag = 0.0
        for j in range(n):
            if j == i:
                continue
            d[i, j] = (b[j] / b[i]) / (nodes[i] - nodes[j])
            diag -= d[i, j]
        d[i, i] = diag
    return d


def lagrange_eval_weights(nodes, x: float):
    """proj/src/quadrature.cpp:112-122."""
    n = len(nodes)
    w = [0.0] * n
    for j in range(n):
        if x == nodes[j]:
            w[j] = 1.0
            return w
    b = barycentric_weights(nodes)
    denom = 0.0
    for j in range(n):
        w[j] = b[j] / (x - nodes[j])
        denom += w[j]
    return [wj / denom for wj in w]


@dataclass
class GllRule:
    degree: int
    nodes: list
    weights: list
    diff: np.ndarray


def gll_rule(degree: int) -> GllRule:
    """GLL rule (proj/src/quadrature.cpp:124-187): Newton from Chebyshev-Lobatto guesses with a
    bracket check and bisection fallback, then exact symmetrisation."""
    if degree < 1 or degree > 40:
        raise ParameterError("gll_rule: degree must be in [1, 40]")
    k = degree
    nodes = [0.0] * (k + 1)
    weights = [0.0] * (k + 1)
    nodes[0] = -1.0
    nodes[k] = 1.0
    for i in range(1, k):
        x = -math.cos(math.pi * i / k)
        lo = -math.cos(math.pi * (i - 0.5) / k)
        hi = -math.cos(math.pi * (i + 0.5) / k)
        done = k == 2 and i == 1
        if done:
            x = 0.0
        it = 0
        while not done and it < 100:
            p, dp = legendre_pair(k, x)
            ddp = (2.0 * x * dp - k * (k + 1.0) * p) / (1.0 - x * x)
            dx = dp / ddp
            x -= dx
            if x <= lo or x >= hi:
                break
            if abs(dx) < 1e-14:
                done = True
            it += 1
        if not done:
            _, dplo = legendre_pair(k, lo)
            plo = dplo
            for _ in range(200):
                x = 0.5 * (lo + hi)
                p, dp = legendre_pair(k, x)
                if (dp > 0) == (plo > 0):
                    lo = x
                    plo = dp
                else:
                    hi = x
                if hi - lo < 1e-15:
                    break
        nodes[i] = x
    for i in range(k // 2 + 1):
        j = k - i
        xm = 0.5 * (nodes[j] - nodes[i])
        nodes[i] = -xm
        nodes[j] = xm
    if k % 2 == 0:
        nodes[k // 2] = 0.0
    for i in range(k + 1):
        p, _ = legendre_pair(k, nodes[i])
        weights[i] = 2.0 / (k * (k + 1.0) * p * p)
    return GllRule(k, nodes, weights, lagrange_diff_matrix(nodes))


# ------------------------------------------------------------------------ basis1d.cpp

@dataclass
class Basis1D:
    half_width: float
    cell_count: int
    degree: int
    rule: GllRule
    nodes: np.ndarray
    mass: np.ndarray
    stiffness: np.ndarray

    @property
    def size(self) -> int:
        return len(self.nodes)

    def cell_width(self) -> float:
        return 2.0 * self.half_width / self.cell_count


def assemble_sem(half_width: float, cell_count: int, degree: int) -> Basis1D:
    """Q^k SEM assembly with Dirichlet trim (proj/src/basis1d.cpp:10-60)."""
    if half_width <= 0.0:
        raise ParameterError("assemble_sem: half_width must be positive")
    if cell_count < 1:
        raise ParameterError("assemble_sem: cell_count must be >= 1")
    if degree < 1:
        raise ParameterError("assemble_sem: degree must be >= 1")
    rule = gll_rule(degree)
    k = degree
    h = 2.0 * half_width / cell_count
    n_global = cell_count * k + 1
    xg = [0.0] * n_global
    for c in range(cell_count):
        left = -half_width + c * h
        for j in range(k + 1):
            xg[c * k + j] = left + (rule.nodes[j] + 1.0) * h / 2.0
    xg[0] = -half_width
    xg[-1] = half_width
    mg = [0.0] * n_global
    d = rule.diff
    w = rule.weights
    s_loc = np.zeros((k + 1, k + 1))
    for i in range(k + 1):
        for j in range(k + 1):
            acc = 0.0
            for q in range(k + 1):
                acc += w[q] * d[q, i] * d[q, j]
            s_loc[i, j] = (2.0 / h) * acc
    sg = np.zeros((n_global, n_global))
    for c in range(cell_count):
        base = c * k
        for i in range(k + 1):
            mg[base + i] += w[i] * h / 2.0
        sg[base:base + k + 1, base:base + k + 1] += s_loc
    n = n_global - 2
    return Basis1D(half_width, cell_count, degree, rule, np.array(xg[1:-1]), np.array(mg[1:-1]),
                   sg[1:n + 1, 1:n + 1].copy())


def interp_matrix(coarse: Basis1D, fine: Basis1D) -> np.ndarray:
    """Piecewise-linear prolongation (proj/src/basis1d.cpp:62-88)."""
    if coarse.half_width != fine.half_width:
        raise ParameterError("interp_matrix: bases must share the same domain")
    if fine.size < coarse.size:
        raise ParameterError("interp_matrix: fine basis must not be smaller than the coarse one")
    nc = coarse.size
    l = coarse.half_width
    xe = np.concatenate([[-l], coarse.nodes, [l]])
    p = np.zeros((fine.size, nc))
    for i in range(fine.size):
        t = fine.nodes[i]
        j = int(np.searchsorted(xe, t, side="right")) - 1
        j = min(max(j, 0), nc)
        w1 = (t - xe[j]) / (xe[j + 1] - xe[j])
        if 0 <= j - 1 < nc:
            p[i, j - 1] = 1.0 - w1
        if j < nc:
            p[i, j] = w1
    return p


# --------------------------------------------------------------------------- axis.cpp

@dataclass
class AxisEigens:
    eigenvalues: np.ndarray        # ascending
    transform: np.ndarray          # T (n x n)
    inverse_transform: np.ndarray  # T^{-1}

    @property
    def size(self) -> int:
        return len(self.eigenvalues)


def sym_eig(a: np.ndarray):
    """Deterministic symmetric eigendecomposition (proj/src/axis.cpp:29-53): symmetrise, ascending
    eigenvalues, each column's first |q_i| >= (1-1e-8) max|q| component made positive."""
    if a.shape[0] != a.shape[1]:
        raise ParameterError("sym_eig: matrix must be square")
    amax = np.abs(a).max() if a.size else 0.0
    if amax > 0.0 and np.abs(a - a.T).max() > 1e-8 * amax:
        raise ParameterError("sym_eig: input not symmetric")
    lam, q = np.linalg.eigh(0.5 * (a + a.T))
    q = q.copy()
    for j in range(q.shape[1]):
        col = q[:, j]
        max_abs = np.abs(col).max()
        i = int(np.argmax(np.abs(col) >= (1.0 - 1e-8) * max_abs))
        if col[i] < 0.0:
            q[:, j] = -col
    return lam, q


def build_axis(basis: Basis1D, f: Callable[[float], float]) -> AxisEigens:
    """SEM axis factorisation (proj/src/axis.cpp:55-74): A = M^{-1/2} S M^{-1/2} + diag(f),
    T = M^{-1/2} Q, T^{-1} = Q^T M^{1/2}."""
    n = basis.size
    sqrt_m = np.sqrt(basis.mass)
    inv_sqrt_m = 1.0 / sqrt_m
    a = (inv_sqrt_m[:, None] * basis.stiffness) * inv_sqrt_m[None, :]
    for i in range(n):
        fx = f(float(basis.nodes[i]))
        if not math.isfinite(fx):
            raise ParameterError("build_axis: f not finite at a node")
        a[i, i] += fx
    lam, q = sym_eig(a)
    return AxisEigens(lam, inv_sqrt_m[:, None] * q, q.T * sqrt_m[None, :])


# ------------------------------------------------------------------------ hermite.cpp

@dataclass
class HermiteBasis:
    size: int
    nodes: np.ndarray
    psi_last: np.ndarray
    diff: np.ndarray
    mass: np.ndarray


def hermite_basis(n: int) -> HermiteBasis:
    """Hermite-Gauss collocation (proj/src/hermite.cpp:10-66): Jacobi-matrix nodes (zero diagonal,
    off-diagonal sqrt(k/2)) symmetrised exactly, psi_{n-1} by the normalised three-term
    recurrence, D(i,j) = psi_i / (psi_j (x_i - x_j)), mass 1 / (n psi_j^2)."""
    if n < 2:
        raise ParameterError("hermite_basis: need n >= 2")
    if n > 745:
        raise CapabilityError("hermite_basis: n > 745 underflows the Hermite recurrence in FP64")
    from scipy.linalg import eigh_tridiagonal
    sub = np.sqrt(np.arange(1, n) / 2.0)
    nodes = np.sort(eigh_tridiagonal(np.zeros(n), sub, eigvals_only=True))
    for i in range(n // 2):
        j = n - 1 - i
        xm = 0.5 * (nodes[j] - nodes[i])
        nodes[i], nodes[j] = -xm, xm
    if n % 2:
        nodes[n // 2] = 0.0
    psi = np.empty(n)
    for j in range(n):
        x = float(nodes[j])
        pk, pkm1 = math.pow(math.pi, -0.25) * math.exp(-x * x / 2.0), 0.0
        for k in range(n - 1):
            pk1 = x * math.sqrt(2.0 / (k + 1)) * pk - math.sqrt(k / (k + 1.0)) * pkm1
            pkm1, pk = pk, pk1
        if pk == 0.0:
            raise CapabilityError("hermite_basis: psi_{n-1} underflowed at a node")
        psi[j] = pk
    diff = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                diff[i, j] = psi[i] / (psi[j] * (nodes[i] - nodes[j]))
    mass = 1.0 / (n * psi * psi)
    return HermiteBasis(n, nodes, psi, diff, mass)


def hermite_operator(basis: HermiteBasis, f: Callable[[float], float]):
    """Symmetrised -D^2 + diag(f) (proj/src/hermite.cpp:68-95): returns (sym, scale = psi)."""
    n = basis.size
    x = basis.nodes
    with np.errstate(divide="ignore"):
        w = 1.0 / (x[:, None] - x[None, :])
    np.fill_diagonal(w, 0.0)
    a = -(w @ w)
    for j in range(n):
        fx = f(float(x[j]))
        if not math.isfinite(fx):
            raise ParameterError("hermite_operator: f not finite at a node")
        a[j, j] += fx
    if np.abs(a - a.T).max() > 1e-8 * np.abs(a).max():
        raise NumericalError("hermite_operator: symmetrization degraded at n = %d" % n)
    return 0.5 * (a + a.T), basis.psi_last.copy()


def build_hermite_axis(basis: HermiteBasis, f: Callable[[float], float]) -> AxisEigens:
    """proj/src/axis.cpp:76-84: T = diag(psi) Q, T^{-1} = Q^T diag(1/psi)."""
    sym, scale = hermite_operator(basis, f)
    lam, q = sym_eig(sym)
    return AxisEigens(lam, scale[:, None] * q, q.T * (1.0 / scale)[None, :])


# --------------------------------------------------------------------------- grid.cpp

@dataclass
class Grid:
    axes: List[Basis1D]

    @staticmethod
    def sem(half_width: float, cell_count: int, degree: int, dimension: int) -> "Grid":
        """Isotropic SEM grid (proj/src/grid.cpp:14-22)."""
        if dimension < 1 or dimension > 9:
            raise ParameterError("Grid: dimension must be in [1, 9]")
        b = assemble_sem(half_width, cell_count, degree)
        return Grid([b] * dimension)

    @staticmethod
    def hermite(n: int, dimension: int) -> "Grid":
        """Isotropic Hermite grid on R^d (proj/src/grid.cpp:24-32)."""
        if dimension < 1 or dimension > 9:
            raise ParameterError("Grid: dimension must be in [1, 9]")
        return Grid([hermite_basis(n)] * dimension)

    @property
    def dim(self) -> int:
        return len(self.axes)

    @property
    def shape(self):
        return tuple(a.size for a in self.axes)

    @property
    def mass(self):
        return [a.mass for a in self.axes]

    def node_count(self) -> int:
        return int(np.prod(self.shape))

    def coords(self):
        """Per-axis node coordinates broadcast to the numpy (reversed) view."""
        d = self.dim
        out = []
        for a in range(d):
            shp = [1] * d
            shp[d - 1 - a] = self.axes[a].size
            out.append(self.axes[a].nodes.reshape(shp))
        return out

    def sample(self, f_vec: Callable) -> np.ndarray:
        """Nodal sampling (proj/src/grid.cpp:53-69); f_vec gets per-axis broadcast coordinates."""
        v = f_vec(self.coords())
        return np.broadcast_to(v, tuple(reversed(self.shape))).reshape(-1).astype(np.float64)

    def separable_operator(self, per_axis: Optional[Sequence[Optional[Callable]]] = None,
                           shift: float = 0.0) -> "SeparableOperator":
        """proj/src/grid.cpp:71-83."""
        if per_axis and len(per_axis) != self.dim:
            raise ParameterError("separable_operator: need one potential per axis")
        eig = []
        cache = {}
        for a in range(self.dim):
            f = per_axis[a] if per_axis and per_axis[a] is not None else (lambda t: 0.0)
            key = (id(self.axes[a]), tuple(f(float(x)) for x in self.axes[a].nodes))
            if key not in cache:
                build = build_hermite_axis if isinstance(self.axes[a], HermiteBasis) else build_axis
                cache[key] = build(self.axes[a], f)
            eig.append(cache[key])
        return SeparableOperator(eig, shift)

    def laplacian(self, shift: float = 0.0) -> "SeparableOperator":
        return self.separable_operator(None, shift)


# --------------------------------------------------------------------- potentials.cpp

@dataclass
class BuiltPotential:
    separable: list                    # per-axis scalar functions
    separable_vec: list                # same, vectorised over numpy arrays
    nonseparable: Optional[np.ndarray]  # V2 nodal field or None


def build_potential(kind: str, grid: Grid, **params) -> BuiltPotential:
    """V = V1 + V2 (proj/src/potentials.cpp:58-130); kind names as potential_kind_from_string
    (potentials.cpp:7-16)."""
    d = grid.dim
    sep, sepv, v2 = [], [], None
    if kind == "sep-osc":
        q = params.get("quad_coeffs") or [1.0] * d
        amp = params.get("osc_amplitude", 100.0)
        if len(q) != d:
            raise ParameterError("sep-osc: need one quadratic coefficient per axis")
        for a in range(d):
            qa = q[a]

            def f(t, qa=qa):
                s = math.sin(math.pi * t / 4.0)
                return qa * t * t + amp * s * s

            def fv(t, qa=qa):
                s = np.sin(np.pi * t / 4.0)
                return qa * t * t + amp * s * s
            sep.append(f)
            sepv.append(fv)
    elif kind == "harmonic":
        for _ in range(d):
            sep.append(lambda t: t * t)
            sepv.append(lambda t: t * t)
    elif kind == "quartic":
        if d != 3:
            raise ParameterError("quartic potential requires a 3D grid")
        g = params.get("gammas") or [1.0, 1.0, 3.0]
        for a in range(3):
            sep.append(lambda t, ga=g[a]: ga * t * t)
            sepv.append(lambda t, ga=g[a]: ga * t * t)
        alpha = params.get("alpha", 1.4)
        kappa = params.get("kappa", 0.3)
        lin = 2.0 * (1.0 - alpha) - 1.0
        quart = kappa / 2.0
        gx, gy = g[0], g[1]

        def v2f(c):
            x, y = c[0], c[1]
            s = gx * x * x + gy * y * y
            r2 = x * x + y * y
            return lin * s + quart * r2 * r2
        v2 = grid.sample(v2f)
    elif kind == "stirrer":
        if d != 3:
            raise ParameterError("stirrer potential requires a 3D grid")
        g = params.get("gammas") or [1.0, 1.0, 2.0]
        for a in range(3):
            g2 = g[a] * g[a]
            sep.append(lambda t, g2=g2: g2 * t * t)
            sepv.append(lambda t, g2=g2: g2 * t * t)
        w0 = params.get("stirrer_height", 4.0)
        dec = params.get("stirrer_decay", 1.0)
        r0 = params.get("stirrer_center", 1.0)

        def v2f(c):
            dx = c[0] - r0
            return 2.0 * w0 * np.exp(-dec * (dx * dx + c[1] * c[1]))
        v2 = grid.sample(v2f)
    elif kind in ("coulomb-2d2", "coulomb-3d2", "coulomb-3d3"):
        block = 2 if kind == "coulomb-2d2" else 3
        particles = 3 if kind == "coulomb-3d3" else 2
        if d != block * particles:
            raise ParameterError("soft Coulomb potential requires a %dD grid" % (block * particles))
        for _ in range(d):
            sep.append(lambda t: t * t)
            sepv.append(lambda t: t * t)
        c_s = params.get("coulomb_strength", 1.0)
        delta = params.get("coulomb_softening", 0.1)

        def v2f(c):
            v = 0.0
            for i in range(particles):
                for j in range(i + 1, particles):
                    r2 = 0.0
                    for b in range(block):
                        dd = c[i * block + b] - c[j * block + b]
                        r2 = r2 + dd * dd
                    v = v + c_s / np.sqrt(r2 + delta * delta)
            return v
        v2 = grid.sample(v2f)
    else:
        raise ParameterError("unknown potential kind: " + kind)
    return BuiltPotential(sep, sepv, v2)


def build_full_operator(grid: Grid, pot: BuiltPotential, shift: float = 0.0) -> "FullOperator":
    """proj/src/potentials.cpp:132-138."""
    return FullOperator(grid.separable_operator(pot.separable, shift), pot.nonseparable)


def separable_sum_field(grid: Grid, pot: BuiltPotential) -> np.ndarray:
    """sum_a V1_a(x_a) sampled on the grid (proj/src/harness.cpp:236-241)."""
    def f(c):
        acc = 0.0
        for a in range(grid.dim):
            acc = acc + pot.separable_vec[a](c[a])
        return acc
    return grid.sample(f)


# ------------------------------------------------------------------------- tensor.cpp

def mode_product(x: np.ndarray, shape: Sequence[int], a: np.ndarray, axis: int) -> np.ndarray:
    """(I x .. x A x .. x I) vec(X) (proj/src/tensor.cpp:105-134); complex data = A on re and im
    separately (tensor.cpp:45-53,130). Returns the flat output (axis extent replaced by a.rows)."""
    d = len(shape)
    if axis < 0 or axis >= d:
        raise ParameterError("mode_product: axis out of range")
    if a.shape[1] != shape[axis]:
        raise ParameterError("mode_product: matrix columns do not match axis extent")
    if np.iscomplexobj(x):
        return mode_product(x.real.copy(), shape, a, axis) + 1j * mode_product(
            x.imag.copy(), shape, a, axis)
    m = a.shape[0]
    nk = shape[axis]
    pre = int(np.prod(shape[:axis]))
    post = int(np.prod(shape[axis + 1:]))
    if axis == 0:
        # contract_first_axis: R = A X with X viewed as (n0 x cols) (tensor.cpp:31-55).
        y = x.reshape(post, nk) @ a.T
    elif post == 1:
        # contract_inner_axis slabs == 1: R = X A^T, X (pre x nk) (tensor.cpp:64-77).
        y = a @ x.reshape(nk, pre)
    else:
        # batched slabs (tensor.cpp:78-83).
        y = np.matmul(a, x.reshape(post, nk, pre))
    return np.ascontiguousarray(y).reshape(-1)


def kron_apply(x: np.ndarray, shape: Sequence[int], mats: Sequence[Optional[np.ndarray]]):
    """Sequential mode products, None = identity (proj/src/tensor.cpp:136-145).
    Returns (flat field, output shape)."""
    if len(mats) != len(shape):
        raise ParameterError("kron_apply: need one matrix (or null) per axis")
    out = x.copy()
    shp = list(shape)
    for axis, a in enumerate(mats):
        if a is not None:
            out = mode_product(out, shp, a, axis)
            shp[axis] = a.shape[0]
    return out, tuple(shp)


def mass_field(shape: Sequence[int], mass: Sequence[np.ndarray]) -> np.ndarray:
    """prod_a m_a[i_a] multiplied in axis order from 1.0 (proj/src/tensor.cpp:183-194)."""
    if len(mass) != len(shape):
        raise ParameterError("mass_field: dimension mismatch")
    d = len(shape)
    w = np.ones(tuple(reversed(shape)))
    for a in range(d):
        shp = [1] * d
        shp[d - 1 - a] = shape[a]
        w = w * np.asarray(mass[a]).reshape(shp)
    return w.reshape(-1)


def direct_sum_grid(values: Sequence[np.ndarray]) -> np.ndarray:
    """lambda[i..] = sum_a values[a][i_a], summed in axis order from 0.0
    (proj/src/tensor.cpp:196-209)."""
    d = len(values)
    shape = [len(v) for v in values]
    s = np.zeros(tuple(reversed(shape)))
    for a in range(d):
        shp = [1] * d
        shp[d - 1 - a] = shape[a]
        s = s + np.asarray(values[a]).reshape(shp)
    return s.reshape(-1)


def inner(u: np.ndarray, v: np.ndarray, mass_w: Optional[np.ndarray] = None):
    """Plain or mass-weighted inner product, conjugate-linear in u (proj/src/tensor.cpp:147-172).
    mass_w is the materialised mass_field (weights multiplied before u, v as in :163-167)."""
    if mass_w is None:
        return np.vdot(u, v) if np.iscomplexobj(u) else float(np.dot(u, v))
    if np.iscomplexobj(u):
        return np.sum(mass_w * np.conj(u) * v)
    return float(np.sum(mass_w * u * v))


def norm(u: np.ndarray, mass_w: Optional[np.ndarray] = None) -> float:
    """proj/src/tensor.cpp:174-181."""
    s = inner(u, u, mass_w)
    return math.sqrt(s.real if np.iscomplexobj(u) else s)


# ---------------------------------------------------------------------- operators.cpp

class SeparableOperator:
    """Kronecker-sum operator in factored form (proj/include/kronop/operators.hpp:15-53,
    proj/src/operators.cpp:7-91)."""

    def __init__(self, axes: List[AxisEigens], shift: float = 0.0):
        if not axes:
            raise ParameterError("SeparableOperator: need at least one axis")
        self.axes = axes
        self.shift = shift
        self.lam = direct_sum_grid([a.eigenvalues for a in axes])
        self.lambda_min = float(self.lam.min())
        self.lambda_max = float(self.lam.max())
        self.forward = [a.inverse_transform for a in axes]
        self.backward = [a.transform for a in axes]

    @property
    def shape(self):
        return tuple(a.size for a in self.axes)

    @property
    def dim(self):
        return len(self.axes)

    def with_shift(self, shift: float) -> "SeparableOperator":
        op = SeparableOperator.__new__(SeparableOperator)
        op.__dict__.update(self.__dict__)
        op.shift = shift
        return op

    def apply(self, u: np.ndarray) -> np.ndarray:
        """(A - shift) u = T((lambda - shift) . T^{-1}u) (operators.cpp:31-40)."""
        w, _ = kron_apply(u, self.shape, self.forward)
        w = w * (self.lam - self.shift)
        out, _ = kron_apply(w, self.shape, self.backward)
        return out

    def check_shift(self):
        """Singular-shift guard (operators.cpp:44-52)."""
        floor = 1e-14 * max(abs(self.lambda_min), abs(self.lambda_max))
        closest = min(abs(self.lambda_min - self.shift), abs(self.lambda_max - self.shift))
        if self.lambda_min < self.shift < self.lambda_max:
            closest = float(np.abs(self.lam - self.shift).min())
        if closest < floor:
            raise NumericalError("SeparableOperator::solve: shift coincides with an eigenvalue")

    def solve(self, b: np.ndarray) -> np.ndarray:
        """(A - shift)^{-1} b with a true division (operators.cpp:42-61)."""
        self.check_shift()
        w, _ = kron_apply(b, self.shape, self.forward)
        w = w / (self.lam - self.shift)
        out, _ = kron_apply(w, self.shape, self.backward)
        return out

    def propagate(self, psi: np.ndarray, dt: float) -> np.ndarray:
        """exp(-i(A - shift)dt) psi (operators.cpp:63-75): phase = -(lambda - shift) dt,
        w *= complex(cos, sin)."""
        if dt == 0.0:
            return psi.copy()
        w, _ = kron_apply(psi.astype(np.complex128), self.shape, self.forward)
        phase = -(self.lam - self.shift) * dt
        w = w * (np.cos(phase) + 1j * np.sin(phase))
        out, _ = kron_apply(w, self.shape, self.backward)
        return out

    def ground_state(self) -> np.ndarray:
        """Rank-one product of each axis's first eigenvector (operators.cpp:77-91)."""
        return mass_field(self.shape, [a.transform[:, 0] for a in self.axes])


@dataclass
class FullOperator:
    """sep + optional V2 diagonal (proj/include/kronop/operators.hpp:56-62, operators.cpp:93-105)."""
    sep: SeparableOperator
    diagonal: Optional[np.ndarray] = None

    def apply(self, u: np.ndarray) -> np.ndarray:
        out = self.sep.apply(u)
        if self.diagonal is not None:
            out = out + self.diagonal * u
        return out


# ---------------------------------------------------------------------------- pcg.cpp

@dataclass
class PcgConfig:
    """proj/include/kronop/pcg.hpp:10-20."""
    rel_tol: float = 1e-12
    max_iter: int = 500
    record_history: bool = False
    preconditioned_norm: bool = False
    stagnation_window: int = 0


@dataclass
class PcgReport:
    """proj/include/kronop/pcg.hpp:22-27."""
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    history: list = field(default_factory=list)


def pcg(apply_a, precond, b: np.ndarray, x: np.ndarray, config: PcgConfig = PcgConfig()):
    """Preconditioned CG with warm start, best iterate and stagnation window
    (proj/src/pcg.cpp:8-81). x is updated in place; returns PcgReport."""
    if config.rel_tol <= 0.0:
        raise ParameterError("pcg: rel_tol must be positive")
    if config.max_iter < 1:
        raise ParameterError("pcg: max_iter must be >= 1")
    if x.shape != b.shape:
        raise ParameterError("pcg: x0/b shape mismatch")
    rep = PcgReport()
    norm_b = float(np.linalg.norm(b))
    if norm_b == 0.0:
        x[:] = 0.0
        rep.converged = True
        return rep
    r = b.copy()
    if float(np.linalg.norm(x)) != 0.0:
        r = r - apply_a(x)
    z = precond(r)
    p = z.copy()
    rz = float(np.dot(r, z))
    pnorm0 = math.sqrt(abs(rz))

    def rel_residual(res, rz_cur):
        return math.sqrt(abs(rz_cur)) / pnorm0 if config.preconditioned_norm else \
            float(np.linalg.norm(res)) / norm_b

    rel = rel_residual(r, rz)
    if config.record_history:
        rep.history.append(rel)
    best_rel = rel
    best_x = x.copy()
    since = 0
    for it in range(config.max_iter):
        if rel <= config.rel_tol:
            rep.converged = True
            break
        if config.stagnation_window > 0 and since >= config.stagnation_window:
            break
        q = apply_a(p)
        pq = float(np.dot(p, q))
        if pq <= 0.0:
            raise NumericalError("pcg: indefinite direction at iteration %d" % (it + 1))
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        z = precond(r)
        rz_next = float(np.dot(r, z))
        p = z + (rz_next / rz) * p
        rz = rz_next
        rep.iterations += 1
        rel = rel_residual(r, rz)
        if config.record_history:
            rep.history.append(rel)
        if rel < 0.99 * best_rel:
            best_rel = rel
            best_x = x.copy()
            since = 0
        else:
            since += 1
    if rel <= config.rel_tol:
        rep.converged = True
    elif best_rel < rel:
        x[:] = best_x
        rel = best_rel
    rep.final_residual = rel
    return rep


# ------------------------------------------------------------------- ground_state.cpp

@dataclass
class InverseIterationConfig:
    """proj/include/kronop/ground_state.hpp:17-32."""
    shift_mode: str = "fraction"      # fraction | offset | zero
    shift_fraction: float = 0.9
    shift_offset: float = 1e-4
    eig_rel_tol: float = 1e-12
    max_outer: int = 60
    inner: PcgConfig = field(default_factory=lambda: PcgConfig(stagnation_window=100))


@dataclass
class EigenpairResult:
    eigenvalue: float = 0.0
    eigenvector: Optional[np.ndarray] = None
    outer_iterations: int = 0
    total_inner_iterations: int = 0
    inner_per_outer: list = field(default_factory=list)
    converged: bool = False


def shift_value(cfg: InverseIterationConfig, sep: SeparableOperator) -> float:
    """proj/src/ground_state.cpp:11-21."""
    if cfg.shift_mode == "fraction":
        return cfg.shift_fraction * sep.lambda_min
    if cfg.shift_mode == "offset":
        return sep.lambda_min - cfg.shift_offset
    return 0.0


def inverse_iteration(op: FullOperator, cfg: InverseIterationConfig, initial: np.ndarray,
                      mass: Sequence[np.ndarray]) -> EigenpairResult:
    """Shifted inverse iteration (proj/src/ground_state.cpp:35-99)."""
    if cfg.eig_rel_tol <= 0.0:
        raise ParameterError("inverse_iteration: tolerance must be positive")
    separable = op.diagonal is None
    sigma = shift_value(cfg, op.sep)
    mw = mass_field(op.sep.shape, mass)

    def wdot(a, b):
        return float(np.sum(mw * a * b))

    def rayleigh(u):
        return wdot(u, op.apply(u)) / wdot(u, u)

    res = EigenpairResult()
    u = initial / math.sqrt(wdot(initial, initial))
    lam = rayleigh(u)
    if sigma >= lam:
        raise ParameterError("inverse_iteration: shift is not below the Rayleigh estimate")
    shifted = op.sep.with_shift(sigma)
    w = np.zeros_like(u)
    for _ in range(cfg.max_outer):
        if separable:
            w = shifted.solve(u)
        else:
            rep = pcg(lambda v: op.apply(v) - sigma * v, op.sep.solve, u, w, cfg.inner)
            res.inner_per_outer.append(rep.iterations)
            res.total_inner_iterations += rep.iterations
        nxt = w / math.sqrt(wdot(w, w))
        lam_next = rayleigh(nxt)
        u = nxt
        res.outer_iterations += 1
        done = abs(lam_next - lam) < cfg.eig_rel_tol * abs(lam_next)
        lam = lam_next
        if done:
            res.converged = True
            break
    imax = int(np.argmax(np.abs(u)))   # fix_sign (ground_state.cpp:23-27)
    if u[imax] < 0.0:
        u = -u
    res.eigenvalue = lam
    res.eigenvector = u
    return res


def multilevel_ground_state(grids: Sequence[Grid], make_operator, cfg: InverseIterationConfig):
    """Coarse-to-fine continuation (proj/src/ground_state.cpp:101-154). Returns
    (finest EigenpairResult, per-level list of (n, outer, inner_total, eigenvalue))."""
    guess = None
    levels = []
    pair = None
    for li, grid in enumerate(grids):
        op = make_operator(grid)
        if guess is None:
            initial = op.sep.ground_state()
        else:
            prev = grids[li - 1]
            mats = [interp_matrix(prev.axes[a], grid.axes[a]) for a in range(grid.dim)]
            initial, _ = kron_apply(guess, prev.shape, mats)
        pair = inverse_iteration(op, cfg, initial, grid.mass)
        levels.append((grid.axes[0].size, pair.outer_iterations, pair.total_inner_iterations,
                       pair.eigenvalue))
        guess = pair.eigenvector
    return pair, levels


# ---------------------------------------------------------------------------- gpe.cpp

@dataclass
class GpeProblem:
    """proj/include/kronop/gpe.hpp:17-22."""
    hamiltonian: FullOperator
    laplacian: SeparableOperator
    beta: float
    mass: list


@dataclass
class GpeFlowConfig:
    """proj/include/kronop/gpe.hpp:30-40."""
    kind: str = "h1"             # h1 | au
    step: float = 0.1
    metric_shift: float = 20.0
    energy_rel_tol: float = 1e-12
    max_iterations: int = 20000
    inner: PcgConfig = field(default_factory=lambda: PcgConfig(stagnation_window=100))
    init: str = "eigenfunction"  # constant | eigenfunction | supplied
    record_history: bool = False


@dataclass
class GpeResult:
    state: Optional[np.ndarray] = None
    energy: float = 0.0
    eigenvalue: float = 0.0
    iterations: int = 0
    linear_solves: int = 0
    converged: bool = False
    history: list = field(default_factory=list)


def gpe_energy(problem: GpeProblem, u: np.ndarray, mw: Optional[np.ndarray] = None) -> float:
    """E(u) = 1/2 <u,Hu>_M + beta/4 sum m u^4 (proj/src/gpe.cpp:10-18)."""
    if mw is None:
        mw = mass_field(problem.laplacian.shape, problem.mass)
    hu = problem.hamiltonian.apply(u)
    quad = float(np.sum(mw * u * hu))
    quartic = float(np.sum(mw * (u * u) * (u * u)))
    return 0.5 * quad + 0.25 * problem.beta * quartic


def gpe_gradient_flow(problem: GpeProblem, cfg: GpeFlowConfig,
                      initial: Optional[np.ndarray] = None, max_iterations: Optional[int] = None):
    """Projected Riemannian gradient flow, H1 and a_u metrics (proj/src/gpe.cpp:55-165).
    max_iterations (oracle-only) truncates the run for trace-parity tests."""
    if problem.beta < 0.0:
        raise ParameterError("gpe_gradient_flow: beta must be >= 0")
    if cfg.step <= 0.0:
        raise ParameterError("gpe_gradient_flow: step must be positive")
    if cfg.metric_shift <= 0.0:
        raise ParameterError("gpe_gradient_flow: metric shift must be positive")
    if cfg.init == "supplied" and initial is None:
        raise ParameterError("gpe_gradient_flow: init = Supplied but no initial state given")
    shape = problem.laplacian.shape
    mw = mass_field(shape, problem.mass)

    def wdot(a, b):
        return float(np.sum(mw * a * b))

    if cfg.init == "supplied":
        u = initial.copy()
    elif cfg.init == "constant":
        u = np.ones(int(np.prod(shape)))
    else:
        if problem.hamiltonian.diagonal is None:
            u = problem.hamiltonian.sep.ground_state()
        else:
            g = problem.hamiltonian.sep.ground_state()
            u = inverse_iteration(problem.hamiltonian, InverseIterationConfig(), g,
                                  problem.mass).eigenvector
    u = u / math.sqrt(wdot(u, u))
    h1 = problem.laplacian.with_shift(-cfg.metric_shift)
    res = GpeResult()
    e_old = gpe_energy(problem, u, mw)
    increases = 0
    w = np.zeros_like(u)
    ham = problem.hamiltonian
    n_iter = cfg.max_iterations if max_iterations is None else min(max_iterations,
                                                                  cfg.max_iterations)
    for it in range(n_iter):
        if cfg.kind == "h1":
            r = ham.apply(u) + problem.beta * (u * u * u)
            rt = h1.solve(r)
            ut = h1.solve(u)
            res.linear_solves += 2
            proj = wdot(rt, u) / wdot(ut, u)
            grad = rt - proj * ut
        else:
            diag = problem.beta * (u * u)
            if ham.diagonal is not None:
                diag = diag + ham.diagonal
            rep = pcg(lambda v: ham.sep.apply(v) + diag * v, ham.sep.solve, u, w, cfg.inner)
            res.linear_solves += rep.iterations
            proj = wdot(u, u) / wdot(w, u)
            grad = u - proj * w
        u = u - cfg.step * grad
        u = u / math.sqrt(wdot(u, u))
        energy = gpe_energy(problem, u, mw)
        rel = abs(energy - e_old) / abs(energy)
        res.iterations = it + 1
        if cfg.record_history:
            res.history.append((it + 1, energy, rel, res.linear_solves))
        if energy - e_old > 1e-13 * abs(energy):
            increases += 1
            if increases > 10:
                raise NumericalError("gpe_gradient_flow: energy increased for more than 10 "
                                     "consecutive steps; reduce the step size")
        else:
            increases = 0
        e_old = energy
        if rel < cfg.energy_rel_tol:
            res.converged = True
            break
    hu = ham.apply(u)
    res.eigenvalue = float(np.sum(mw * u * hu)) + problem.beta * float(np.sum(mw * (u * u) * (u * u)))
    res.energy = e_old
    res.state = u
    return res


# ---------------------------------------------------------------------- splitting.cpp

def yoshida_coeffs():
    """proj/src/splitting.cpp:86-90."""
    # std::cbrt(2.0) in the reference is folded by GCC at compile time (correctly rounded); glibc's
    # runtime cbrt is 1 ulp off for 2.0, so use the correctly rounded constant.
    cbrt2 = 1.2599210498948732
    denom = 2.0 - cbrt2
    return 1.0 / denom, -cbrt2 / denom


def single_schedule(h: float, m: int):
    """(a_times[M+1], b_factors[M]) (proj/src/splitting.cpp:20-34)."""
    nodes, weights = gauss_legendre(m)
    a_times = [0.0] * (m + 1)
    b_factors = [0.0] * m
    prev = 0.0
    for k in range(m):
        sk = h * (1.0 + nodes[k]) / 2.0
        a_times[k] = sk - prev
        b_factors[k] = 0.5 * weights[k] * h
        prev = sk
    a_times[m] = h - prev
    return a_times, b_factors


def step_schedules(composition: str, quad_points: int, h: float):
    """proj/src/splitting.cpp:36-42."""
    if composition == "single":
        return [single_schedule(h, quad_points)]
    g1, g2 = yoshida_coeffs()
    return [single_schedule(g1 * h, quad_points), single_schedule(g2 * h, quad_points),
            single_schedule(g1 * h, quad_points)]


def pointwise_phase(psi: np.ndarray, b_diag: np.ndarray, factor: float) -> np.ndarray:
    """psi *= exp(-i factor B) (proj/src/splitting.cpp:44-51)."""
    phase = -factor * b_diag
    return psi * (np.cos(phase) + 1j * np.sin(phase))


def run_schedules(a: SeparableOperator, b_diag, schedules, psi, steps: int, merge: bool):
    """Alternating A-propagations / B-phases with optional cross-step merge
    (proj/src/splitting.cpp:53-82)."""
    pending = [0.0]
    state = [psi]

    def propagate_a(t):
        if merge:
            pending[0] += t
        else:
            state[0] = a.propagate(state[0], t)

    def multiply_b(factor):
        if merge and pending[0] != 0.0:
            state[0] = a.propagate(state[0], pending[0])
            pending[0] = 0.0
        state[0] = pointwise_phase(state[0], b_diag, factor)

    for _ in range(steps):
        for a_times, b_factors in schedules:
            m = len(b_factors)
            for k in range(m):
                propagate_a(a_times[k])
                multiply_b(b_factors[k])
            propagate_a(a_times[m])
    if merge and pending[0] != 0.0:
        state[0] = a.propagate(state[0], pending[0])
    return state[0]


def qhop_step(a: SeparableOperator, b_diag, psi, h: float, quad_points: int):
    """proj/src/splitting.cpp:92-96."""
    return run_schedules(a, b_diag, [single_schedule(h, quad_points)], psi, 1, False)


def yoshida_step(a: SeparableOperator, b_diag, psi, h: float, quad_points: int):
    """proj/src/splitting.cpp:98-105."""
    return run_schedules(a, b_diag, step_schedules("yoshida", quad_points, h), psi, 1, False)


@dataclass
class SplitSpec:
    """proj/include/kronop/splitting.hpp:26-33."""
    quad_points: int = 1
    composition: str = "single"   # single | yoshida
    dt: float = 0.0
    total_time: float = 0.0
    merge_across_steps: bool = False
    mass_weighted_error: bool = False


def evolve(spec: SplitSpec, a: SeparableOperator, b_diag, psi0, exact: Optional[SeparableOperator]
           = None, stationary_eigenvalue: Optional[float] = None, mass=None):
    """March and compare against the exact or stationary reference (proj/src/splitting.cpp:107-146).
    Returns (state, error, steps)."""
    if spec.dt <= 0.0 or spec.total_time <= 0.0:
        raise ParameterError("evolve: dt and total_time must be positive")
    ratio = spec.total_time / spec.dt
    steps = int(round(ratio))
    if steps < 1 or abs(ratio - steps) > 1e-9:
        raise ParameterError("evolve: total_time must be an integer multiple of dt")
    psi = psi0.astype(np.complex128)
    psi = psi / np.linalg.norm(psi)
    start = psi.copy()
    psi = run_schedules(a, b_diag, step_schedules(spec.composition, spec.quad_points, spec.dt),
                        psi, steps, spec.merge_across_steps)
    if exact is not None:
        ref = exact.propagate(start, spec.total_time)
    else:
        phase = -stationary_eigenvalue * spec.total_time
        ref = start * complex(math.cos(phase), math.sin(phase))
    diff = psi - ref
    mw = mass_field(a.shape, mass) if spec.mass_weighted_error else None
    return psi, norm(diff, mw), steps


# ---------------------------------------------------------------------- dense_ref.cpp

def dense_axis_operator(basis: Basis1D, f) -> np.ndarray:
    """M^{-1} S + diag(f) (proj/src/dense_ref.cpp:11-17)."""
    h = basis.stiffness / basis.mass[:, None]
    h = h + np.diag([f(float(x)) for x in basis.nodes])
    return h


def dense_hermite_axis_operator(basis: HermiteBasis, f) -> np.ndarray:
    """-D^2 + diag(f) from the Hermite differentiation matrix, unsymmetrised
    (proj/src/dense_ref.cpp:19-23)."""
    return -(basis.diff @ basis.diff) + np.diag([f(float(x)) for x in basis.nodes])


def clustering_report(sym_axis_ops: Sequence[np.ndarray], v2: np.ndarray, epsilon: float):
    """Spectrum of I + A^{-1/2} diag(v2) A^{-1/2} (proj/src/dense_ref.cpp:114-147): returns
    (ascending spectrum, outliers outside (1-eps, 1+eps), mu_max / mu_min)."""
    total = int(np.prod([op.shape[0] for op in sym_axis_ops]))
    if total > 5000:
        raise CapabilityError("clustering_report: N > 5000")
    a = dense_assemble(sym_axis_ops, None, 0.0)
    lam, q = np.linalg.eigh(a)
    if lam[0] <= 0.0:
        raise ParameterError("clustering_report: A is not positive definite")
    a_inv_half = (q * (1.0 / np.sqrt(lam))[None, :]) @ q.T
    b = a_inv_half @ np.diag(v2) @ a_inv_half
    mu = np.linalg.eigvalsh(0.5 * (b + b.T)) + 1.0
    outliers = int(np.sum((mu < 1.0 - epsilon) | (mu > 1.0 + epsilon)))
    return mu, outliers, float(mu[-1] / mu[0])


def dense_sym_axis_operator(basis: Basis1D, f) -> np.ndarray:
    """M^{-1/2} S M^{-1/2} + diag(f) (proj/src/dense_ref.cpp:25-34)."""
    s = 1.0 / np.sqrt(basis.mass)
    return basis.stiffness * s[:, None] * s[None, :] + np.diag([f(float(x)) for x in basis.nodes])


def dense_assemble(axis_ops: Sequence[np.ndarray], diagonal=None, shift: float = 0.0):
    """Explicit Kronecker sum, axis 0 fastest (proj/src/dense_ref.cpp:36-72)."""
    total = int(np.prod([o.shape[0] for o in axis_ops]))
    if total > 20000:
        raise CapabilityError("dense_ref::assemble: N > 20000")
    h = np.zeros((total, total))
    for a, op in enumerate(axis_ops):
        pre = int(np.prod([o.shape[0] for o in axis_ops[:a]]))
        post = int(np.prod([o.shape[0] for o in axis_ops[a + 1:]]))
        h += np.kron(np.kron(np.eye(post), op), np.eye(pre))
    if diagonal is not None:
        h += np.diag(diagonal)
    h -= shift * np.eye(total)
    return h


def expm_hermitian(h: np.ndarray, t: float) -> np.ndarray:
    """exp(-i h t) via eigendecomposition (proj/src/dense_ref.cpp:74-93)."""
    lam, v = np.linalg.eigh(h)
    p = -lam * t
    return (v * (np.cos(p) + 1j * np.sin(p))[None, :]) @ v.conj().T


# ----------------------------------------------------------------- manufactured inputs

def manufactured_rhs(grid: Grid, pot: BuiltPotential, half_width: float):
    """cmd_solve manufactured solution u* = prod sin((a+1) pi x_a / L) and
    f = (sum((a+1)pi/L)^2 + V) u* (proj/src/harness.cpp:228-249). Returns (rhs, ustar)."""
    def us(c):
        v = 1.0
        for a in range(grid.dim):
            v = v * np.sin((a + 1) * np.pi * c[a] / half_width)
        return v
    ustar = grid.sample(us)
    lap_eig = 0.0
    for a in range(grid.dim):
        lap_eig += ((a + 1) * math.pi / half_width) ** 2
    vtotal = separable_sum_field(grid, pot)
    rhs = (lap_eig + vtotal) * ustar
    if pot.nonseparable is not None:
        rhs = rhs + pot.nonseparable * ustar
    return rhs, ustar


def box_state(grid: Grid, half_width: float) -> np.ndarray:
    """prod sin(pi (x + L) / 2L) (proj/src/harness.cpp:452-462)."""
    def f(c):
        v = 1.0
        for a in range(grid.dim):
            v = v * np.sin(np.pi * (c[a] + half_width) / (2.0 * half_width))
        return v
    return grid.sample(f)


# ------------------------------------------------------------------------------ fieldio.cpp

FIELD_MAGIC = 0x4B4F5046


def dump_field(path: str, field: np.ndarray, shape: Sequence[int]):
    """Binary checkpoint (proj/src/fieldio.cpp:28-47, format fieldio.hpp:10-13)."""
    import struct
    cplx = np.iscomplexobj(field)
    with open(path, "wb") as f:
        f.write(struct.pack("<4I", FIELD_MAGIC, 1, len(shape), 1 if cplx else 0))
        f.write(struct.pack("<%dQ" % len(shape), *shape))
        f.write(np.ascontiguousarray(field, dtype=np.complex128 if cplx else np.float64).tobytes())


def load_field(path: str):
    """proj/src/fieldio.cpp:49-73: returns (field, shape)."""
    import struct
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 16:
        raise ParameterError("load_field: truncated file")
    magic, version, dim, kind = struct.unpack_from("<4I", raw, 0)
    if magic != FIELD_MAGIC:
        raise ParameterError("load_field: bad magic")
    if version != 1:
        raise ParameterError("load_field: bad version")
    if dim < 1 or dim > 9:
        raise ParameterError("load_field: bad dimension")
    if len(raw) < 16 + 8 * dim:
        raise ParameterError("load_field: truncated file")
    shape = struct.unpack_from("<%dQ" % dim, raw, 16)
    if kind not in (0, 1):
        raise ParameterError("load_field: unknown scalar kind")
    n = int(np.prod(shape)) * (2 if kind else 1)
    body = raw[16 + 8 * dim:]
    if len(body) < 8 * n:
        raise ParameterError("load_field: truncated data")
    a = np.frombuffer(body[:8 * n], dtype=np.float64).copy()
    return (a.view(np.complex128) if kind else a), tuple(shape)

