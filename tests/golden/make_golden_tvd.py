"""Golden vectors for the TVD kappa-scheme line-splitting sweeps
(paqif/tvdcd.py:449-550), produced by running the REFERENCE (build
container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/make_golden_tvd.py

Cases: the manufactured quartic problem (the reference's own study and
gates: Ls0 to 1e-12 with the alternate cycle, Ls1 symmetric from the exact
solution, Ls0/Ls1/Ls2 x-cycles from zero), and seeded custom problems --
rectangular grids with odd and even line orders, the first-order "upwind"
closure, variable convection fields, omega != 1, backward order -- through
single sweep_splitting calls.  Every custom case stores f and the data ring.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from paqif.tvdcd import (ConvectionDiffusionProblem, Grid2D, KappaSchemeConfig,  # noqa: E402
                         quartic_test_problem, solve_by_sweeps, sweep_splitting)

QUARTIC = [
    # name, intervals, kappa, eps, variant, cycle, max_sweeps, tol, from_exact
    ("q16_ls0_alt", 16, 1.0 / 3.0, 1e-6, "Ls0", "alternate", 120, 1e-12, False),
    ("q16_ls1_sym", 16, 0.0, 1e-6, "Ls1", "symmetric", 5, 0.0, True),
    ("q32_ls0_x", 32, 0.0, 1e-6, "Ls0", "x", 9, 0.0, False),
    ("q32_ls1_x", 32, 0.0, 1e-6, "Ls1", "x", 9, 0.0, False),
    ("q16_ls2_alt", 16, 0.5, 1e-3, "Ls2", "alternate", 6, 0.0, False),
    ("q24_ls1_alt_k1", 24, 1.0, 1e-2, "Ls1", "alternate", 4, 0.0, False),
]

# variable fields, recreated verbatim by the test
def field_a(x, y):
    return 1.0 + 0.5 * x * x


def field_b(x, y):
    return 0.25 + y * y


CUSTOM = [
    # name, grid (x_lo, x_hi, y_lo, y_hi, nx, ny), kappa, eps, closure, variable,
    # variant, omega, order
    ("c_rect_odd_ls0", (0.0, 1.2, 0.0, 0.8, 11, 7), 1.0 / 3.0, 1e-3, "wide", False, "Ls0", 1.0, "forward"),
    ("c_rect_even_ls1", (0.0, 1.3, 0.0, 0.9, 12, 8), -0.5, 1e-2, "wide", False, "Ls1", 0.8, "backward"),
    ("c_upwind_ls0", (0.0, 1.0, 0.0, 1.0, 19, 19), 0.0, 1e-4, "upwind", False, "Ls0", 1.0, "forward"),
    ("c_upwind_ls2", (0.0, 1.0, 0.0, 1.0, 19, 19), 0.5, 1e-4, "upwind", False, "Ls2", 0.9, "backward"),
    ("c_var_ls1", (-1.0, 1.0, -1.0, 1.0, 30, 30), 1.0 / 3.0, 1e-3, "wide", True, "Ls1", 1.0, "forward"),
    ("c_var_upwind_ls0", (-1.0, 1.0, -1.0, 1.0, 25, 25), 0.0, 1e-5, "upwind", True, "Ls0", 1.1, "forward"),
]


def main():
    out = {}
    for name, iv, kappa, eps, variant, cycle, ms, tol, from_exact in QUARTIC:
        cfg = KappaSchemeConfig(kappa=kappa, eps=eps)
        prob, exact = quartic_test_problem(iv, cfg)
        u, hist = solve_by_sweeps(prob, variant, tol=tol, max_sweeps=ms, cycle=cycle,
                                  u0=exact if from_exact else None)
        out[f"{name}__u"] = u
        out[f"{name}__hist"] = np.array(hist)
    for k, (name, g, kappa, eps, closure, var, variant, omega, order) in enumerate(CUSTOM):
        rng = np.random.default_rng(100 + k)
        grid = Grid2D(*g)
        cfg = KappaSchemeConfig(kappa=kappa, eps=eps, a=field_a if var else 1.0,
                                b=field_b if var else 0.7)
        f = rng.standard_normal((grid.ny, grid.nx))
        boundary = rng.standard_normal((grid.ny + 4, grid.nx + 4))
        prob = ConvectionDiffusionProblem(grid, cfg, f, boundary, closure=closure)
        u0 = rng.standard_normal((grid.ny, grid.nx))
        u1, r1 = sweep_splitting(prob, u0, variant, omega, order)
        u2, r2 = sweep_splitting(prob, u1, variant, omega, order)
        out[f"{name}__f"], out[f"{name}__boundary"], out[f"{name}__u0"] = f, boundary, u0
        out[f"{name}__u1"], out[f"{name}__u2"] = u1, u2
        out[f"{name}__res"] = np.array([r1, r2])
    # Ls3 (line-distributive relaxation): the reference's smoke setting and
    # a variable-field custom problem, sweep by sweep, and an alternate cycle
    cfg = KappaSchemeConfig(kappa=0.0, eps=1.0)
    prob, _ = quartic_test_problem(16, cfg)
    u = np.zeros_like(prob.f)
    for k in range(3):
        u, r = sweep_splitting(prob, u, "Ls3", omega=0.7)
        out[f"ls3_q16__u{k}"], out[f"ls3_q16__r{k}"] = u, np.array(r)
    u, hist = solve_by_sweeps(prob, "Ls3", omega=0.7, tol=0.0, max_sweeps=3, cycle="alternate")
    out["ls3_q16_alt__u"], out["ls3_q16_alt__hist"] = u, np.array(hist)
    rng = np.random.default_rng(7)
    grid = Grid2D(-1.0, 1.0, -1.0, 1.0, 21, 21)
    cfg = KappaSchemeConfig(kappa=1.0 / 3.0, eps=0.5, a=field_a, b=field_b)
    f = rng.standard_normal((21, 21))
    boundary = rng.standard_normal((25, 25))
    prob = ConvectionDiffusionProblem(grid, cfg, f, boundary, closure="upwind")
    u0 = rng.standard_normal((21, 21))
    u1, r1 = sweep_splitting(prob, u0, "Ls3", omega=0.6)
    u2, r2 = sweep_splitting(prob, u1, "Ls3", omega=0.6)
    out.update({"ls3_var__f": f, "ls3_var__boundary": boundary, "ls3_var__u0": u0,
                "ls3_var__u1": u1, "ls3_var__u2": u2, "ls3_var__res": np.array([r1, r2])})
    np.savez_compressed(os.path.join(HERE, "tvd.npz"), **out)


if __name__ == "__main__":
    main()
