"""Refinement study for acceptance criterion 12 (proj/tests/acceptance.cpp:584-609) on the
ORACLE (test infrastructure): the 4D soft-Coulomb ground state (coulomb-2d2, delta = 0.1, c = 1,
L = 8, SEM Q10, sigma = lambda_min(A) - 1e-4, inner PCG tol 1e-9, multilevel from 2 cells) on
Q10 x {2, 3, 4, 5} cells = {19, 29, 39, 49}^4. The criterion compares the 29^4 value with the
paper's converged 99^4 value 5.060514417326 at 1e-4; this records how the
discretisation error closes with refinement (the 99^4 level itself runs on the GPU:
tests/test_gpu_config_parity.py::test_soft_coulomb_4d_99_matches_paper).
Writes tests/golden/oracle_c12_refinement.json.

  python -m oracle.refine_c12 [max_cells]
"""
import json
import os
import sys
import time

from oracle import kronop_oracle as K

REF_99 = 5.060514417326  # PAPER.md:1652, Q10 99^4


def main(max_cells=5):
    out = {"reference_99": REF_99, "levels": []}
    guess_grid = None
    guess = None
    for cells in range(2, max_cells + 1):
        g = K.Grid.sem(8.0, cells, 10, 4)
        op = K.build_full_operator(g, K.build_potential("coulomb-2d2", g, coulomb_softening=0.1))
        cfg = K.InverseIterationConfig(shift_mode="offset")
        cfg.inner.rel_tol = 1e-9
        t0 = time.time()
        grids = [guess_grid, g] if guess_grid is not None else [g]
        if guess_grid is None:
            pair, lv = K.multilevel_ground_state([g], lambda gg: op, cfg)
        else:
            mats = [K.interp_matrix(guess_grid.axes[a], g.axes[a]) for a in range(4)]
            init, _ = K.kron_apply(guess, guess_grid.shape, mats)
            pair = K.inverse_iteration(op, cfg, init, g.mass)
        lam = pair.eigenvalue
        out["levels"].append({"cells": cells, "n": g.shape[0], "lambda1": lam,
                              "rel_to_99": abs(lam - REF_99) / REF_99,
                              "outer": pair.outer_iterations,
                              "inner": pair.total_inner_iterations,
                              "seconds": time.time() - t0})
        print(json.dumps(out["levels"][-1]), flush=True)
        guess_grid, guess = g, pair.eigenvector
        del grids
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                        "golden", "oracle_c12_refinement.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
