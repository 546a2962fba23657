"""TVD kappa-scheme line-splitting sweeps on the device (csrc/tvd_sweep.cu,
paper_2008_03276_b200/tvdcd.py) vs the reference's iterates and residual
histories (golden tvd.npz, tests/golden/make_golden_tvd.py): bit-exact, as
the sweeps are the reference's arithmetic in its order."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

T = load_golden("tvd.npz")

QUARTIC = [
    ("q16_ls0_alt", 16, 1.0 / 3.0, 1e-6, "Ls0", "alternate", 120, 1e-12, False),
    ("q16_ls1_sym", 16, 0.0, 1e-6, "Ls1", "symmetric", 5, 0.0, True),
    ("q32_ls0_x", 32, 0.0, 1e-6, "Ls0", "x", 9, 0.0, False),
    ("q32_ls1_x", 32, 0.0, 1e-6, "Ls1", "x", 9, 0.0, False),
    ("q16_ls2_alt", 16, 0.5, 1e-3, "Ls2", "alternate", 6, 0.0, False),
    ("q24_ls1_alt_k1", 24, 1.0, 1e-2, "Ls1", "alternate", 4, 0.0, False),
]


def field_a(x, y):
    return 1.0 + 0.5 * x * x


def field_b(x, y):
    return 0.25 + y * y


CUSTOM = [
    ("c_rect_odd_ls0", (0.0, 1.2, 0.0, 0.8, 11, 7), 1.0 / 3.0, 1e-3, "wide", False, "Ls0", 1.0, "forward"),
    ("c_rect_even_ls1", (0.0, 1.3, 0.0, 0.9, 12, 8), -0.5, 1e-2, "wide", False, "Ls1", 0.8, "backward"),
    ("c_upwind_ls0", (0.0, 1.0, 0.0, 1.0, 19, 19), 0.0, 1e-4, "upwind", False, "Ls0", 1.0, "forward"),
    ("c_upwind_ls2", (0.0, 1.0, 0.0, 1.0, 19, 19), 0.5, 1e-4, "upwind", False, "Ls2", 0.9, "backward"),
    ("c_var_ls1", (-1.0, 1.0, -1.0, 1.0, 30, 30), 1.0 / 3.0, 1e-3, "wide", True, "Ls1", 1.0, "forward"),
    ("c_var_upwind_ls0", (-1.0, 1.0, -1.0, 1.0, 25, 25), 0.0, 1e-5, "upwind", True, "Ls0", 1.1, "forward"),
]


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("case", QUARTIC, ids=[c[0] for c in QUARTIC])
def test_solve_by_sweeps_vs_reference(case):
    from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, solve_by_sweeps
    name, iv, kappa, eps, variant, cycle, ms, tol, from_exact = case
    prob, exact = quartic_test_problem(iv, KappaSchemeConfig(kappa=kappa, eps=eps))
    u, hist = solve_by_sweeps(prob, variant, tol=tol, max_sweeps=ms, cycle=cycle,
                              u0=exact if from_exact else None)
    assert np.array_equal(_bits(hist), _bits(T[f"{name}__hist"]))
    assert np.array_equal(_bits(u), _bits(T[f"{name}__u"]))


def _custom_problem(case):
    from paper_2008_03276_b200.tvdcd import ConvectionDiffusionProblem, Grid2D, KappaSchemeConfig
    name, g, kappa, eps, closure, var, variant, omega, order = case
    cfg = KappaSchemeConfig(kappa=kappa, eps=eps, a=field_a if var else 1.0,
                            b=field_b if var else 0.7)
    return ConvectionDiffusionProblem(Grid2D(*g), cfg, T[f"{name}__f"], T[f"{name}__boundary"],
                                      closure=closure)


@pytest.mark.parametrize("case", CUSTOM, ids=[c[0] for c in CUSTOM])
def test_sweep_splitting_vs_reference(case):
    from paper_2008_03276_b200.tvdcd import sweep_splitting
    name, _, _, _, _, _, variant, omega, order = case
    prob = _custom_problem(case)
    u1, r1 = sweep_splitting(prob, T[f"{name}__u0"], variant, omega, order)
    u2, r2 = sweep_splitting(prob, u1, variant, omega, order)
    assert np.array_equal(_bits(u1), _bits(T[f"{name}__u1"]))
    assert np.array_equal(_bits(u2), _bits(T[f"{name}__u2"]))
    assert np.array_equal(_bits([r1, r2]), _bits(T[f"{name}__res"]))


@pytest.mark.parametrize("intervals,l1_ref", [(16, 2.25826e-03), (32, 3.32640e-04)])
def test_study_l1_levels(intervals, l1_ref):
    # the reference's study gate (tests/test_tvdcd.py: published L1 levels
    # at kappa = 1/3, Ls0 to 1e-12)
    from paper_2008_03276_b200.tvdcd import (KappaSchemeConfig, error_norms,
                                             quartic_test_problem, solve_by_sweeps)
    prob, exact = quartic_test_problem(intervals, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
    u, hist = solve_by_sweeps(prob, "Ls0", tol=1e-12, max_sweeps=120)
    assert hist[-1] <= 1e-12
    _, l1, _ = error_norms(u, exact, prob.grid.h, ref_scale=2.0)
    assert l1 == pytest.approx(l1_ref, rel=0.10)


def test_residual_gate_and_errors():
    from paper_2008_03276_b200.errors import ContractViolationError
    from paper_2008_03276_b200.tvdcd import (KappaSchemeConfig, quartic_test_problem,
                                             solve_by_sweeps, sweep_splitting)
    prob, exact = quartic_test_problem(16, KappaSchemeConfig(kappa=0.0, eps=1e-6))
    f_norm = float(np.sqrt(prob.grid.h ** 2 * np.sum(prob.f ** 2)))
    _, fast = solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=5, cycle="symmetric", u0=exact)
    assert fast[4] / f_norm <= 1e-7
    with pytest.raises(ContractViolationError):
        solve_by_sweeps(prob, "Ls1", cycle="diagonal")
    with pytest.raises(ContractViolationError):
        sweep_splitting(prob, exact, "Ls9")
    with pytest.raises(NotImplementedError):
        sweep_splitting(prob, exact, "DefC")


def test_distributive_ls3_vs_reference():
    # Ls3 line-distributive relaxation (tvdcd.py:615-656), bit-exact: the
    # reference's smoke setting sweep by sweep and through an alternate
    # cycle, and a variable-field upwind-closure problem
    from paper_2008_03276_b200.tvdcd import (ConvectionDiffusionProblem, Grid2D,
                                             KappaSchemeConfig, quartic_test_problem,
                                             solve_by_sweeps, sweep_splitting)
    prob, _ = quartic_test_problem(16, KappaSchemeConfig(kappa=0.0, eps=1.0))
    u = np.zeros_like(prob.f)
    for k in range(3):
        u, r = sweep_splitting(prob, u, "Ls3", omega=0.7)
        assert np.array_equal(_bits(u), _bits(T[f"ls3_q16__u{k}"]))
        assert np.array_equal(_bits([r]), _bits([T[f"ls3_q16__r{k}"]]))
    u, hist = solve_by_sweeps(prob, "Ls3", omega=0.7, tol=0.0, max_sweeps=3, cycle="alternate")
    assert np.array_equal(_bits(u), _bits(T["ls3_q16_alt__u"]))
    assert np.array_equal(_bits(hist), _bits(T["ls3_q16_alt__hist"]))
    cfg = KappaSchemeConfig(kappa=1.0 / 3.0, eps=0.5, a=field_a, b=field_b)
    prob = ConvectionDiffusionProblem(Grid2D(-1.0, 1.0, -1.0, 1.0, 21, 21), cfg, T["ls3_var__f"],
                                      T["ls3_var__boundary"], closure="upwind")
    u1, r1 = sweep_splitting(prob, T["ls3_var__u0"], "Ls3", omega=0.6)
    u2, r2 = sweep_splitting(prob, u1, "Ls3", omega=0.6)
    assert np.array_equal(_bits(u1), _bits(T["ls3_var__u1"]))
    assert np.array_equal(_bits(u2), _bits(T["ls3_var__u2"]))
    assert np.array_equal(_bits([r1, r2]), _bits(T["ls3_var__res"]))


def test_distributive_ls3_progress():
    # the reference's smoke gate (tests/test_tvdcd.py): 30 under-relaxed
    # sweeps do not blow up and make progress
    from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, sweep_splitting
    prob, _ = quartic_test_problem(16, KappaSchemeConfig(kappa=0.0, eps=1.0))
    u = np.zeros_like(prob.f)
    first = None
    for _ in range(30):
        u, res = sweep_splitting(prob, u, "Ls3", omega=0.7)
        first = first if first is not None else res
    assert res < first


def test_large_grid_sweep_consistent():
    # size-independent property at a study-scale grid: the device residual
    # norm equals the host restatement's on the device iterate
    from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, sweep_splitting
    prob, _ = quartic_test_problem(512, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
    u, r = sweep_splitting(prob, np.zeros_like(prob.f), "Ls1")
    assert r == prob.residual_norm(u)
