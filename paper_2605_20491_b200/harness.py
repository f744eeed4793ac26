"""Experiment harness on the B200 path: the reference's `kronop` commands (proj/src/harness.cpp)
with the same configuration grammar (proj/src/config.cpp), the same CSV columns and number format
(proj/src/csv.cpp), the same manifest and checkpoint / slice outputs, and the same exit codes
(harness.cpp:731-751: 2 configuration error, 4 capability refusal, 3 numerical failure).

Every solve, apply, PCG, inverse iteration, GPE flow and split-step run goes through the device
API (api.py -> libkronop.so); only set-up (parsing, host quadrature / eigen-factorisation, CSV
writing) runs on the host, as in the reference.

    python -m paper_2605_20491_b200.harness run.cfg [--output-dir DIR] [--allow-large]
"""
from __future__ import annotations

import math
import os
import re
import sys
import time
from typing import Dict, List, Optional

import numpy as np
import torch

from . import _lib as L
from . import api as A
from . import potentials as P

VERSION = "1.0.0"


def _perr(msg):
    return L.ParameterError(L.KRONOP_EPARAM, msg)


# ------------------------------------------------------------------------- config.cpp --
_FLOAT = re.compile(r"^[+-]?((\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|inf(inity)?|nan)$", re.I)
_INT = re.compile(r"^[+-]?\d+$")


def _g17(x: float) -> str:
    """std::ostream << double with precision 17 (default floatfield)."""
    return "%.17g" % x


class Config:
    """INI-like `[section]` / `key = value` file, '#' comments; keys are 'section.key'
    (config.cpp:37-73). Getters record the resolved value (defaults included) for the manifest;
    unknown keys are an error after the run (check_all_consumed, config.cpp:186-193)."""

    def __init__(self, origin="<string>"):
        self.origin = origin
        self.entries: Dict[str, str] = {}
        self.lines: Dict[str, int] = {}
        self.consumed = set()
        self.resolved: Dict[str, str] = {}

    @staticmethod
    def parse_file(path: str) -> "Config":
        try:
            with open(path) as f:
                text = f.read()
        except OSError:
            raise _perr("config: cannot open " + path)
        return Config.parse_string(text, path)

    @staticmethod
    def parse_string(text: str, origin: str = "<string>") -> "Config":
        cfg = Config(origin)
        section = ""
        for lineno, line in enumerate(text.split("\n"), 1):
            if "#" in line:
                line = line[:line.index("#")]
            line = line.strip(" \t\r")
            if not line:
                continue
            where = "%s:%d: " % (origin, lineno)
            if line[0] == "[":
                if line[-1] != "]":
                    raise _perr(where + "unterminated section header")
                section = line[1:-1].strip(" \t\r")
                if not section:
                    raise _perr(where + "empty section name")
                continue
            if "=" not in line:
                raise _perr(where + "expected key = value")
            key, value = line.split("=", 1)
            key, value = key.strip(" \t\r"), value.strip(" \t\r")
            if not key:
                raise _perr(where + "empty key")
            if not section:
                raise _perr(where + "key outside any [section]")
            full = section + "." + key
            if full in cfg.entries:
                raise _perr(where + "duplicate key " + full)
            cfg.entries[full] = value
            cfg.lines[full] = lineno
        return cfg

    def has(self, key):
        return key in self.entries

    def set(self, key, value):
        self.entries[key] = value
        self.lines[key] = 0

    def _raw(self, key):
        self.consumed.add(key)
        return self.entries[key]

    def _where(self, key):
        return "%s:%d: " % (self.origin, self.lines.get(key, 0))

    def get_string(self, key, fallback):
        v = self._raw(key) if self.has(key) else fallback
        self.resolved[key] = v
        return v

    def require_string(self, key):
        if not self.has(key):
            raise _perr(self.origin + ": missing required key " + key)
        v = self._raw(key)
        self.resolved[key] = v
        return v

    def require_real(self, key):
        v = self.require_string(key)
        if not _FLOAT.match(v):
            raise _perr(self._where(key) + "bad number for " + key)
        return float(v)

    def get_real(self, key, fallback):
        if not self.has(key):
            self.resolved[key] = _g17(fallback)
            return float(fallback)
        return self.require_real(key)

    def get_long(self, key, fallback):
        if not self.has(key):
            self.resolved[key] = str(int(fallback))
            return int(fallback)
        v = self.require_string(key)
        if not _INT.match(v):
            raise _perr(self._where(key) + "bad integer for " + key)
        return int(v)

    get_int = get_long

    def get_bool(self, key, fallback):
        if not self.has(key):
            self.resolved[key] = "true" if fallback else "false"
            return bool(fallback)
        v = self.require_string(key)
        if v == "true":
            return True
        if v == "false":
            return False
        raise _perr(self._where(key) + "expected true/false for " + key)

    def get_real_list(self, key, fallback):
        if not self.has(key):
            self.resolved[key] = ",".join(_g17(x) for x in fallback)
            return [float(x) for x in fallback]
        v = self.require_string(key)
        out = []
        for item in v.split(","):
            item = item.strip(" \t\r")
            if not _FLOAT.match(item):
                raise _perr(self._where(key) + "bad list entry for " + key)
            out.append(float(item))
        return out

    def get_int_list(self, key, fallback):
        return [int(x) for x in self.get_real_list(key, [float(x) for x in fallback])]

    def check_all_consumed(self):
        for key in self.entries:
            if key not in self.consumed:
                raise _perr(self._where(key) + "unknown key " + key)


# ---------------------------------------------------------------------------- csv.cpp --
class CsvWriter:
    """Header line, then rows; doubles as %.13e, integers as %d, strings verbatim
    (csv.cpp:9-44)."""

    def __init__(self, path: str, header: List[str]):
        try:
            self.f = open(path, "w")
        except OSError:
            raise _perr("CsvWriter: cannot open " + path)
        self.columns = len(header)
        self.f.write(",".join(header) + "\n")

    @staticmethod
    def fmt(v):
        if isinstance(v, bool):
            return "true" if v else "false"
        if isinstance(v, (int, np.integer)):
            return "%d" % int(v)
        if isinstance(v, (float, np.floating)):
            return "%.13e" % float(v)
        return str(v)

    def row(self, values):
        if len(values) != self.columns:
            raise _perr("CsvWriter: column count mismatch")
        self.f.write(",".join(self.fmt(v) for v in values) + "\n")
        self.f.flush()

    def close(self):
        self.f.close()


# ------------------------------------------------------------------------ harness.cpp --
class GridSpec:
    def __init__(self, cfg: Config):  # harness.cpp:56-80
        self.kind = cfg.get_string("grid.kind", "sem")
        if self.kind not in ("sem", "hermite"):
            raise _perr("grid.kind must be sem or hermite")
        self.dimension = cfg.get_int("grid.dimension", 3)
        if not 1 <= self.dimension <= 9:
            raise _perr("grid.dimension must be in [1, 9]")
        self.half_width, self.degree, self.cells, self.hermite_n = 8.0, 10, [8], 40
        if self.kind == "sem":
            self.half_width = cfg.get_real("grid.L", 8.0)
            self.degree = cfg.get_int("grid.degree", 10)
            self.cells = cfg.get_int_list("grid.cells", [8])
            if not self.cells:
                raise _perr("grid.cells must not be empty")
            if any(c < 1 for c in self.cells):
                raise _perr("grid.cells entries must be >= 1")
            if not 1 <= self.degree <= 40:
                raise _perr("grid.degree must be in [1, 40]")
        else:
            self.hermite_n = cfg.get_int("grid.n", 40)

    def levels(self):
        return len(self.cells) if self.kind == "sem" else 1

    def level_nodes(self, level):
        n = self.cells[level] * self.degree - 1 if self.kind == "sem" else self.hermite_n
        return n ** self.dimension

    def build(self, level) -> A.Grid:
        if self.kind == "sem":
            return A.Grid.sem(self.half_width, self.cells[level], self.degree, self.dimension)
        return A.Grid.hermite(self.hermite_n, self.dimension)


def check_capacity(spec: GridSpec, allow_large: bool, complex_scalars: bool):
    for level in range(spec.levels()):  # harness.cpp:89-99
        n = spec.level_nodes(level)
        if n > 200_000_000 and not allow_large:
            mib = n * (16 if complex_scalars else 8) * 6 // (1 << 20)
            raise L.CapabilityError(L.KRONOP_ECAPABILITY,
                                    "configuration needs %d scalars (~%d MiB working set); pass "
                                    "allow_large to proceed" % (n, mib))


def read_potential(cfg: Config, dim: int):  # harness.cpp:110-129
    kind = cfg.get_string("potential.kind", "harmonic")
    params = dict(
        quad_coeffs=cfg.get_real_list("potential.quad", [1.0] * dim),
        osc_amplitude=cfg.get_real("potential.amplitude", 100.0),
        alpha=cfg.get_real("potential.alpha", 1.4),
        kappa=cfg.get_real("potential.kappa", 0.3),
        gammas=cfg.get_real_list("potential.gammas", []) or None,
        stirrer_height=cfg.get_real("potential.w0", 4.0),
        stirrer_decay=cfg.get_real("potential.stirrer_delta", 1.0),
        stirrer_center=cfg.get_real("potential.r0", 1.0),
        coulomb_strength=cfg.get_real("potential.c", 1.0),
        coulomb_softening=cfg.get_real("potential.delta", 0.1))
    if kind not in P.KINDS:
        raise _perr("unknown potential kind: " + kind)
    return kind, params


def build_pot(kind, params, grid):
    try:
        return P.build_potential(kind, grid, **params)
    except ValueError as e:
        raise _perr(str(e))


def read_pcg(cfg: Config) -> A.PcgConfig:  # harness.cpp:133-141
    return A.PcgConfig(rel_tol=cfg.get_real("pcg.tol", 1e-12),
                       max_iter=cfg.get_int("pcg.max_iter", 500),
                       record_history=cfg.get_bool("pcg.history", False),
                       preconditioned_norm=cfg.get_bool("pcg.preconditioned_norm", False),
                       stagnation_window=cfg.get_int("pcg.stagnation_window", 0))


def read_eigen(cfg: Config) -> A.InverseIterationConfig:  # harness.cpp:143-160
    mode = cfg.get_string("eigen.shift", "fraction")
    if mode not in ("fraction", "offset", "zero"):
        raise _perr("eigen.shift must be fraction, offset, or zero")
    c = A.InverseIterationConfig(shift_mode=mode,
                                 shift_fraction=cfg.get_real("eigen.shift_fraction", 0.9),
                                 shift_offset=cfg.get_real("eigen.shift_offset", 1e-4),
                                 eig_rel_tol=cfg.get_real("eigen.tol", 1e-12),
                                 max_outer=cfg.get_int("eigen.max_outer", 60))
    c.inner = read_pcg(cfg)
    c.inner.stagnation_window = cfg.get_int("pcg.stagnation_window", 100)
    return c


class RunContext:
    def __init__(self, cfg: Config, ctx: A.Context):
        self.cfg = cfg
        self.ctx = ctx
        self.command = ""
        self.out_dir = "out"
        self.seed = 1
        self.allow_large = False
        self.extra: List = []

    def out_path(self, name):
        return os.path.join(self.out_dir, name)

    def note(self, key, value):
        self.extra.append((key, value if isinstance(value, str) else "%.13e" % value))


def _product(factors):
    out = 1.0
    for f in factors:  # v = 1.0; v *= f_a in axis order (harness.cpp:238-241)
        out = out * f
    return out


def _sync():
    torch.cuda.synchronize()


def _norm(t: torch.Tensor) -> float:
    return float(torch.linalg.vector_norm(t))


def full_operator(rc: RunContext, grid: A.Grid, pot) -> A.FullOperator:
    """build_full_operator (grid.cpp / potentials.cpp:132-138): separable part on the axes,
    V2 as the nodal diagonal."""
    sep = _exec_precision(rc, grid.separable_operator(rc.ctx, pot.separable))
    return A.FullOperator(sep, pot.v2_device("cuda:%d" % rc.ctx.device))


def separable_sum_field(grid: A.Grid, pot) -> np.ndarray:
    return P.separable_sum(grid, pot)


def _dev(rc: RunContext, x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda:%d" % rc.ctx.device)


def evaluate_slice(rc: RunContext, grid: A.Grid, field: torch.Tensor, axis_a: int, axis_b: int,
                   fixed: List[float], resolution: int) -> np.ndarray:
    """harness.cpp:628-668: contract the fixed axes to singletons with point-evaluation rows,
    expand the two free axes on uniform R-point grids (mode products on the device)."""
    d = grid.dim
    if axis_a == axis_b or not (0 <= axis_a < d and 0 <= axis_b < d):
        raise _perr("evaluate_slice: bad axis pair")
    if len(fixed) != d - 2:
        raise _perr("evaluate_slice: need one fixed coordinate per remaining axis")
    if resolution < 1:
        raise _perr("evaluate_slice: resolution must be >= 1")
    for a in range(d):
        if not isinstance(grid.axes[a], A.Basis1D):
            raise L.CapabilityError(L.KRONOP_ECAPABILITY, "evaluate_slice: SEM grids only")
    shape = list(grid.shape)
    work = field
    fixed_axes = [a for a in range(d) if a not in (axis_a, axis_b)]
    for i, axis in enumerate(fixed_axes):
        row = A.eval_weights(grid.axes[axis], [fixed[i]])
        work = A.mode_product(rc.ctx, work, shape, row, axis)
        shape[axis] = 1

    def targets(b):
        l = b.half_width
        return [0.0] if resolution == 1 else [-l + 2.0 * l * r / (resolution - 1.0)
                                              for r in range(resolution)]
    for axis in (axis_a, axis_b):
        e = A.eval_weights(grid.axes[axis], targets(grid.axes[axis]))
        work = A.mode_product(rc.ctx, work, shape, e, axis)
        shape[axis] = resolution
    w = work.cpu().numpy()
    stride = [1] * d
    for a in range(1, d):
        stride[a] = stride[a - 1] * shape[a - 1]
    out = np.empty((resolution, resolution))
    for i in range(resolution):
        for j in range(resolution):
            out[i, j] = w[i * stride[axis_a] + j * stride[axis_b]]
    return out


def maybe_export(rc: RunContext, grid: A.Grid, field: torch.Tensor):  # harness.cpp:190-208
    checkpoint = rc.cfg.get_string("output.checkpoint", "")
    if checkpoint:
        A.dump_field(rc.out_path(checkpoint), field, grid.shape, ctx=rc.ctx)
    slice_csv = rc.cfg.get_string("output.slice_csv", "")
    if slice_csv:
        axes = rc.cfg.get_int_list("output.slice_axes", [0, 1])
        if len(axes) != 2:
            raise _perr("output.slice_axes needs two entries")
        fixed = rc.cfg.get_real_list("output.slice_fixed", [0.0] * (grid.dim - 2))
        res = rc.cfg.get_int("output.slice_res", 300)
        values = evaluate_slice(rc, grid, field, axes[0], axes[1], fixed, res)
        ba, bb = grid.axes[axes[0]], grid.axes[axes[1]]
        csv = CsvWriter(rc.out_path(slice_csv), ["coord_a", "coord_b", "value"])
        for i in range(res):
            for j in range(res):
                xa = 0.0 if res == 1 else -ba.half_width + 2.0 * ba.half_width * i / (res - 1.0)
                xb = 0.0 if res == 1 else -bb.half_width + 2.0 * bb.half_width * j / (res - 1.0)
                csv.row([xa, xb, float(values[i, j])])
        csv.close()


def _exec_precision(rc, op):
    """Optional key `device.precision` (not in the reference grammar): "fp64" (default, DMMA) or
    "ozaki" / "ozaki6" / "ozaki5" - every transform of the operator (and the PCG / inverse
    iteration / GPE / splitting drivers on it) on the INT8 tensor cores (kronop_op_set_precision).
    """
    prec = rc.cfg.get_string("device.precision", "fp64")
    if prec != "fp64" and op is not None:
        op.set_precision(prec)
    return op


def cmd_solve(rc: RunContext, gs: GridSpec):  # harness.cpp:212-283
    kind, params = read_potential(rc.cfg, gs.dimension)
    rhs_mode = rc.cfg.get_string("solve.rhs", "manufactured")
    pcg_cfg = read_pcg(rc.cfg)
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "solve.csv")),
                    ["n", "dofs", "setup_s", "solve_s", "l2_rel_err", "residual", "pcg_iters"])
    for level in range(gs.levels()):
        t0 = time.perf_counter()
        grid = gs.build(level)
        pot = build_pot(kind, params, grid)
        op = full_operator(rc, grid, pot)
        _sync()
        setup_s = time.perf_counter() - t0
        manufactured = rhs_mode == "manufactured"
        if manufactured and gs.kind != "sem":
            raise _perr("solve.rhs = manufactured requires an SEM grid")
        ustar = None
        if manufactured:
            l = gs.half_width
            us = grid.sample(lambda c: _product(np.sin((a + 1) * np.pi * c[a] / l)
                                                for a in range(len(c))))
            lap_eig = sum(((a + 1) * math.pi / l) ** 2 for a in range(grid.dim))
            rhs_np = (lap_eig + separable_sum_field(grid, pot)) * us
            if pot.nonseparable is not None:
                rhs_np = rhs_np + pot.nonseparable * us
            ustar, rhs = _dev(rc, us), _dev(rc, rhs_np)
        elif rhs_mode == "random":
            rhs = A.splitmix_uniform(rc.ctx, rc.seed, grid.node_count())
        else:
            raise _perr("solve.rhs must be manufactured or random")
        t0 = time.perf_counter()
        iters = 0
        if op.diagonal is None:
            u = op.sep.solve(rhs)
        else:
            u = torch.zeros_like(rhs)
            rep = A.pcg(A.apply_map(op.sep, op.diagonal), A.solve_map(op.sep), rhs, u, pcg_cfg)
            iters = rep.iterations
        _sync()
        solve_s = time.perf_counter() - t0
        residual = _norm(op.apply(u) - rhs) / _norm(rhs)
        rel_err = _norm(u - ustar) / _norm(ustar) if manufactured else ""
        csv.row([grid.axes[0].size, grid.node_count(), setup_s, solve_s, rel_err, residual,
                 iters])
        maybe_export(rc, grid, u)
    csv.close()


def cmd_ground_state(rc: RunContext, gs: GridSpec):  # harness.cpp:285-315
    kind, params = read_potential(rc.cfg, gs.dimension)
    eig = read_eigen(rc.cfg)
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "ground_state.csv")),
                    ["level", "n", "dofs", "setup_s", "interp_s", "outer_iters", "pcg_per_outer",
                     "total_precond_applications", "eigenvalue"])
    grids = [gs.build(level) for level in range(gs.levels())]
    pair, levels = A.multilevel_ground_state(
        rc.ctx, grids, lambda g: full_operator(rc, g, build_pot(kind, params, g)), eig)
    for i, rep in enumerate(levels):
        csv.row([i, rep.n, grids[i].node_count(), rep.setup_seconds, rep.interp_seconds,
                 rep.outer_iterations, float(rep.inner_per_outer), rep.total_inner_iterations,
                 rep.eigenvalue])
    csv.close()
    rc.note("result.eigenvalue", pair.eigenvalue)
    rc.note("result.outer_iterations", str(pair.outer_iterations))
    rc.note("result.converged", "true" if pair.converged else "false")
    maybe_export(rc, grids[-1], pair.eigenvector)


def cmd_gpe(rc: RunContext, gs: GridSpec):  # harness.cpp:317-372
    if gs.levels() != 1:
        raise _perr("gpe expects a single grid level")
    grid = gs.build(0)
    kind, params = read_potential(rc.cfg, gs.dimension)
    ham = full_operator(rc, grid, build_pot(kind, params, grid))
    lap = _exec_precision(rc, grid.laplacian(rc.ctx))
    beta = rc.cfg.get_real("gpe.beta", 0.0)
    flow = rc.cfg.get_string("gpe.flow", "h1")
    if flow not in ("h1", "au"):
        raise _perr("gpe.flow must be h1 or au")
    cfg = A.GpeFlowConfig(kind=flow)
    cfg.step = rc.cfg.get_real("gpe.tau", 0.1 if flow == "h1" else 1.0)
    cfg.metric_shift = rc.cfg.get_real("gpe.alpha", 20.0)
    cfg.energy_rel_tol = rc.cfg.get_real("gpe.tol", 1e-12)
    cfg.max_iterations = rc.cfg.get_int("gpe.max_iter", 20000)
    cfg.inner = read_pcg(rc.cfg)
    cfg.inner.stagnation_window = rc.cfg.get_int("pcg.stagnation_window", 100)
    init = rc.cfg.get_string("gpe.init", "eigenfunction")
    if init not in ("constant", "eigenfunction"):
        raise _perr("gpe.init must be constant or eigenfunction")
    cfg.init = init
    cfg.record_history = True
    res = A.gpe_gradient_flow(ham, lap, beta, cfg)
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "gpe.csv")),
                    ["iteration", "energy", "rel_change", "linear_solves", "wall_s"])
    for row in res.history:
        csv.row([int(row[0]), row[1], row[2], int(row[3]), row[4]])
    csv.close()
    rc.note("result.energy", res.energy)
    rc.note("result.eigenvalue", res.eigenvalue)
    rc.note("result.iterations", str(res.iterations))
    rc.note("result.linear_solves", str(res.linear_solves))
    rc.note("result.converged", "true" if res.converged else "false")
    maybe_export(rc, grid, res.state)


def cmd_propagate(rc: RunContext, gs: GridSpec, table: bool):  # harness.cpp:374-493
    if gs.levels() != 1:
        raise _perr("propagate expects a single grid level")
    grid = gs.build(0)
    kind, params = read_potential(rc.cfg, gs.dimension)
    pot = build_pot(kind, params, grid)
    fully_separable = pot.nonseparable is None
    split = rc.cfg.get_string("propagate.split", "kinetic")
    v1 = separable_sum_field(grid, pot)
    if split == "kinetic":
        a = _exec_precision(rc, grid.laplacian(rc.ctx))
        b = v1 + (pot.nonseparable if pot.nonseparable is not None else 0.0)
    elif split == "kinetic+v1":
        a = _exec_precision(rc, grid.separable_operator(rc.ctx, pot.separable))
        b = pot.nonseparable if pot.nonseparable is not None else np.zeros(grid.node_count())
    else:
        raise _perr("propagate.split must be kinetic or kinetic+v1")
    b_diag = _dev(rc, np.asarray(b, dtype=np.float64))
    full = (_exec_precision(rc, grid.separable_operator(rc.ctx, pot.separable))
            if fully_separable else None)
    spec = A.SplitSpec(quad_points=rc.cfg.get_int("propagate.M", 1))
    comp = rc.cfg.get_string("propagate.composition", "qhop")
    if comp not in ("qhop", "yoshida"):
        raise _perr("propagate.composition must be qhop or yoshida")
    spec.composition = "single" if comp == "qhop" else "yoshida"
    spec.total_time = rc.cfg.get_real("propagate.T", 0.1)
    spec.merge_across_steps = rc.cfg.get_bool("propagate.merge", False)
    spec.mass_weighted_error = rc.cfg.get_bool("propagate.mass_error", False)
    ref = rc.cfg.get_string("propagate.reference", "exact" if fully_separable else "stationary")
    init = rc.cfg.get_string("propagate.initial", "box" if ref == "exact" else "ground-state")
    lam1 = 0.0
    psi0 = None
    if ref == "exact":
        if not fully_separable:
            raise _perr("propagate.reference = exact needs a separable potential")
    elif ref == "stationary":
        op = full_operator(rc, grid, pot)
        pair = A.inverse_iteration(op, read_eigen(rc.cfg), op.sep.ground_state())
        lam1 = pair.eigenvalue
        psi0 = pair.eigenvector.to(torch.complex128)
        rc.note("result.reference_eigenvalue", lam1)
    else:
        raise _perr("propagate.reference must be exact or stationary")
    if init == "box":
        if ref == "stationary":
            raise _perr("a stationary reference requires propagate.initial = ground-state")
        l = gs.half_width
        box = grid.sample(lambda c: _product(np.sin(np.pi * (c[a] + l) / (2.0 * l))
                                             for a in range(len(c))))
        psi0 = _dev(rc, box.astype(np.complex128))
    elif init != "ground-state":
        raise _perr("propagate.initial must be box or ground-state")
    if init == "ground-state" and ref == "exact":
        psi0 = full.ground_state().to(torch.complex128)
    dts = (rc.cfg.get_real_list("propagate.dt_list", [0.01, 0.005]) if table
           else [rc.cfg.get_real("propagate.dt", 0.01)])
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "propagate.csv")),
                    ["dt", "error", "rate", "steps", "wall_s", "mass_norm_drift"])
    mass = A.mass_field(rc.ctx, grid.shape, grid.mass)
    nrm = psi0 / _norm(psi0)

    def mass_norm(z):
        return math.sqrt(float(torch.sum(mass * (z.real ** 2 + z.imag ** 2))))
    prev_err = prev_dt = 0.0
    last = psi0
    for dt in dts:
        spec.dt = dt
        t0 = time.perf_counter()
        state, err, steps = A.evolve(spec, a, b_diag, psi0, exact=full if ref == "exact" else None,
                                     stationary_eigenvalue=lam1)
        _sync()
        wall = time.perf_counter() - t0
        m0 = mass_norm(nrm)
        drift = abs(mass_norm(state) - m0) / m0
        have = prev_dt > 0.0 and err > 0.0 and prev_err > 0.0
        rate = math.log(prev_err / err) / math.log(prev_dt / dt) if have else ""
        csv.row([dt, err, rate, steps, wall, drift])
        prev_err, prev_dt, last = err, dt, state
    csv.close()
    checkpoint = rc.cfg.get_string("output.checkpoint", "")
    if checkpoint:
        A.dump_field(rc.out_path(checkpoint), last, grid.shape, ctx=rc.ctx)


def cmd_pcg_bench(rc: RunContext, gs: GridSpec):  # harness.cpp:495-567
    kind, params = read_potential(rc.cfg, gs.dimension)
    pcg_cfg = read_pcg(rc.cfg)
    pre = rc.cfg.get_string("pcg.precond", "separable")
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "pcg_bench.csv")),
                    ["n", "dofs", "preconditioner", "iterations", "converged", "final_residual",
                     "setup_s", "solve_s"])
    for level in range(gs.levels()):
        t0 = time.perf_counter()
        grid = gs.build(level)
        pot = build_pot(kind, params, grid)
        op = full_operator(rc, grid, pot)
        lap = _exec_precision(rc, grid.laplacian(rc.ctx))
        _sync()
        setup_s = time.perf_counter() - t0
        if pre == "separable":
            precond = A.solve_map(op.sep)
        elif pre == "laplacian":
            precond = A.solve_map(lap)
        elif pre == "combined":  # V^{-1/2} (-Lap)^{-1} V^{-1/2}, full nodal V
            v = separable_sum_field(grid, pot)
            if pot.nonseparable is not None:
                v = v + pot.nonseparable
            if v.min() <= 0.0:
                raise _perr("combined preconditioner needs a positive potential")
            precond = A.solve_map(lap, _dev(rc, 1.0 / np.sqrt(v)))
        elif pre == "v2-scaled":
            if pot.nonseparable is None:
                raise _perr("v2-scaled preconditioner needs a non-separable part")
            if pot.nonseparable.min() <= 0.0:
                raise _perr("v2-scaled preconditioner needs positive V2")
            precond = A.solve_map(op.sep, _dev(rc, 1.0 / np.sqrt(pot.nonseparable)))
        else:
            raise _perr("pcg.precond must be separable, laplacian, combined, or v2-scaled")
        rhs = A.splitmix_uniform(rc.ctx, rc.seed, grid.node_count())
        x = torch.zeros_like(rhs)
        run = A.PcgConfig(pcg_cfg.rel_tol, pcg_cfg.max_iter, True, pcg_cfg.preconditioned_norm,
                          pcg_cfg.stagnation_window)
        t0 = time.perf_counter()
        rep = A.pcg(A.apply_map(op.sep, op.diagonal), precond, rhs, x, run)
        _sync()
        solve_s = time.perf_counter() - t0
        n = grid.axes[0].size
        csv.row([n, grid.node_count(), pre, rep.iterations, "true" if rep.converged else "false",
                 rep.final_residual, setup_s, solve_s])
        if pcg_cfg.record_history:
            hist = CsvWriter(rc.out_path("pcg_history_n%d.csv" % n),
                             ["iteration", "relative_residual"])
            for i, r in enumerate(rep.history):
                hist.row([i, r])
            hist.close()
    csv.close()


def cmd_clustering(rc: RunContext, gs: GridSpec):  # harness.cpp:569-601 (dense, host, N <= 5000)
    if gs.kind != "sem":
        raise _perr("clustering runs on SEM grids")
    kind, params = read_potential(rc.cfg, gs.dimension)
    eps = rc.cfg.get_real("clustering.epsilon", 0.1)
    csv = CsvWriter(rc.out_path(rc.cfg.get_string("output.csv", "clustering.csv")),
                    ["n", "dofs", "epsilon", "outliers", "condition"])
    spectrum_out = rc.cfg.get_bool("clustering.spectrum", False)
    for level in range(gs.levels()):
        grid = gs.build(level)
        pot = build_pot(kind, params, grid)
        if pot.nonseparable is None:
            raise _perr("clustering needs a potential with a non-separable part")
        if grid.node_count() > 5000:
            raise L.CapabilityError(L.KRONOP_ECAPABILITY, "clustering_report: N > 5000")
        ops = []
        for a in range(grid.dim):  # dense_ref.cpp:25-34 symmetric axis operators
            b = grid.axes[a]
            s = 1.0 / np.sqrt(b.mass)
            ops.append(b.stiffness * s[:, None] * s[None, :] +
                       np.diag([pot.separable[a](float(x)) for x in b.nodes]))
        a_mat = np.zeros((grid.node_count(),) * 2)
        for ax in range(grid.dim):  # Kronecker sum, axis 0 fastest (dense_ref.cpp:36-74)
            term = np.array([[1.0]])
            for bx in reversed(range(grid.dim)):
                term = np.kron(term, ops[bx] if bx == ax else np.eye(grid.shape[bx]))
            a_mat += term
        lam, q = np.linalg.eigh(a_mat)
        if lam[0] <= 0.0:
            raise _perr("clustering_report: A is not positive definite")
        ih = (q * (1.0 / np.sqrt(lam))[None, :]) @ q.T
        bm = ih @ np.diag(pot.nonseparable) @ ih
        mu = np.linalg.eigvalsh(0.5 * (bm + bm.T)) + 1.0
        outliers = int(np.sum((mu < 1.0 - eps) | (mu > 1.0 + eps)))
        n = grid.axes[0].size
        csv.row([n, grid.node_count(), eps, outliers, float(mu[-1] / mu[0])])
        if spectrum_out:
            sp = CsvWriter(rc.out_path("spectrum_n%d.csv" % n), ["index", "eigenvalue"])
            for i, m in enumerate(mu):
                sp.row([i, float(m)])
            sp.close()
    csv.close()


def write_manifest(rc: RunContext):  # harness.cpp:603-612
    try:
        with open(rc.out_path("manifest.txt"), "w") as out:
            out.write("kronop.version = %s\n" % VERSION)
            out.write("backend = libkronop.so sm_100a (FP64 DMMA)\n")
            for k in sorted(rc.cfg.resolved):
                out.write("%s = %s\n" % (k, rc.cfg.resolved[k]))
            for k, v in rc.extra:
                out.write("%s = %s\n" % (k, v))
    except OSError:
        raise _perr("cannot write manifest in " + rc.out_dir)


COMMANDS = ("solve", "ground-state", "gpe", "propagate", "convergence-table", "pcg-bench",
            "clustering")


def run(cfg: Config, ctx: Optional[A.Context] = None):  # harness.cpp:694-729
    ctx = ctx or A.Context(0)
    rc = RunContext(cfg, ctx)
    rc.command = cfg.require_string("run.command")
    rc.out_dir = cfg.get_string("run.output_dir", "out")
    rc.seed = cfg.get_long("run.seed", 1)
    rc.allow_large = cfg.get_bool("run.allow_large", False)
    cfg.get_int("run.threads", 0)  # host threads: accepted for config compatibility
    gs = GridSpec(cfg)
    check_capacity(gs, rc.allow_large, rc.command in ("propagate", "convergence-table"))
    os.makedirs(rc.out_dir, exist_ok=True)
    if rc.command == "solve":
        cmd_solve(rc, gs)
    elif rc.command == "ground-state":
        cmd_ground_state(rc, gs)
    elif rc.command == "gpe":
        cmd_gpe(rc, gs)
    elif rc.command == "propagate":
        cmd_propagate(rc, gs, False)
    elif rc.command == "convergence-table":
        cmd_propagate(rc, gs, True)
    elif rc.command == "pcg-bench":
        cmd_pcg_bench(rc, gs)
    elif rc.command == "clustering":
        cmd_clustering(rc, gs)
    else:
        raise _perr("unknown command: " + rc.command)
    cfg.check_all_consumed()
    write_manifest(rc)
    return rc


def run_to_exit_code(config_path: str, allow_large: bool = False, output_dir: str = "",
                     ctx: Optional[A.Context] = None) -> int:
    """harness.cpp:731-751."""
    try:
        cfg = Config.parse_file(config_path)
        if allow_large:
            cfg.set("run.allow_large", "true")
        if output_dir:
            cfg.set("run.output_dir", output_dir)
        run(cfg, ctx)
        return 0
    except L.ParameterError as e:
        print("configuration error: %s" % e.msg, file=sys.stderr)
        return 2
    except L.CapabilityError as e:
        print("capability refusal: %s" % e.msg, file=sys.stderr)
        return 4
    except L.NumericalError as e:
        print("numerical failure: %s" % e.msg, file=sys.stderr)
        return 3


def main(argv=None):  # tools/kronop_main.cpp
    import argparse
    ap = argparse.ArgumentParser(description="Tensor-product Schrodinger operator toolkit (B200)")
    ap.add_argument("config")
    ap.add_argument("--output-dir", default="")
    ap.add_argument("--allow-large", action="store_true")
    a = ap.parse_args(argv)
    return run_to_exit_code(a.config, a.allow_large, a.output_dir)


if __name__ == "__main__":
    sys.exit(main())
