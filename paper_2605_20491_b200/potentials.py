"""Synthetic potentials V = V1 (per-axis) + V2 (nodal field) of the experiments
(proj/src/potentials.cpp:58-130), product-side host setup: V1 as per-axis scalar functions (their
nodal values feed build_axis), V2 sampled on the host grid and uploaded once."""
import math

import numpy as np
import torch

KINDS = ("sep-osc", "harmonic", "quartic", "stirrer", "coulomb-2d2", "coulomb-3d2", "coulomb-3d3")


class BuiltPotential:
    def __init__(self, separable, separable_vec, nonseparable):
        self.separable = separable          # per-axis scalar callables
        self.separable_vec = separable_vec  # same, numpy-vectorised
        self.nonseparable = nonseparable    # host numpy field or None

    def v2_device(self, device="cuda"):
        if self.nonseparable is None:
            return None
        return torch.from_numpy(self.nonseparable).to(device)


def build_potential(kind, grid, quad_coeffs=None, osc_amplitude=100.0, alpha=1.4, kappa=0.3,
                    gammas=None, stirrer_height=4.0, stirrer_decay=1.0, stirrer_center=1.0,
                    coulomb_strength=1.0, coulomb_softening=0.1) -> BuiltPotential:
    d = grid.dim
    sep, sepv, v2 = [], [], None
    if kind == "sep-osc":
        q = quad_coeffs or [1.0] * d
        if len(q) != d:
            raise ValueError("sep-osc: need one quadratic coefficient per axis")
        for a in range(d):
            qa = q[a]
            sep.append(lambda t, qa=qa: qa * t * t + osc_amplitude * math.sin(math.pi * t / 4.0) ** 2)
            sepv.append(lambda t, qa=qa: qa * t * t + osc_amplitude * np.sin(np.pi * t / 4.0) ** 2)
    elif kind == "harmonic":
        sep = [lambda t: t * t] * d
        sepv = list(sep)
    elif kind == "quartic":
        if d != 3:
            raise ValueError("quartic potential requires a 3D grid")
        g = gammas or [1.0, 1.0, 3.0]
        sep = [lambda t, ga=g[a]: ga * t * t for a in range(3)]
        sepv = list(sep)
        lin, quart = 2.0 * (1.0 - alpha) - 1.0, kappa / 2.0
        v2 = grid.sample(lambda c: lin * (g[0] * c[0] ** 2 + g[1] * c[1] ** 2)
                         + quart * (c[0] ** 2 + c[1] ** 2) ** 2)
    elif kind == "stirrer":
        if d != 3:
            raise ValueError("stirrer potential requires a 3D grid")
        g = gammas or [1.0, 1.0, 2.0]
        sep = [lambda t, g2=g[a] * g[a]: g2 * t * t for a in range(3)]
        sepv = list(sep)
        v2 = grid.sample(lambda c: 2.0 * stirrer_height *
                         np.exp(-stirrer_decay * ((c[0] - stirrer_center) ** 2 + c[1] ** 2)))
    elif kind in ("coulomb-2d2", "coulomb-3d2", "coulomb-3d3"):
        block = 2 if kind == "coulomb-2d2" else 3
        parts = 3 if kind == "coulomb-3d3" else 2
        if d != block * parts:
            raise ValueError("soft Coulomb potential requires a %dD grid" % (block * parts))
        sep = [lambda t: t * t] * d
        sepv = list(sep)

        def f(c):
            v = 0.0
            for i in range(parts):
                for j in range(i + 1, parts):
                    r2 = 0.0
                    for b in range(block):
                        dd = c[i * block + b] - c[j * block + b]
                        r2 = r2 + dd * dd
                    v = v + coulomb_strength / np.sqrt(r2 + coulomb_softening ** 2)
            return v
        v2 = grid.sample(f)
    else:
        raise ValueError("unknown potential kind: " + kind)
    return BuiltPotential(sep, sepv, v2)


def separable_sum(grid, pot) -> np.ndarray:
    """sum_a V1_a(x_a) on the grid (harness.cpp:236-241)."""
    def f(c):
        acc = 0.0
        for a in range(grid.dim):
            acc = acc + pot.separable_vec[a](c[a])
        return acc
    return grid.sample(f)
