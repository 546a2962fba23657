"""Time TVD line-splitting sweeps (dev tool): device solve_by_sweeps per
sweep at study grids; with --ref, the reference's numpy sweeps on this host
(build container only)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ref = "--ref" in sys.argv
if ref:
    sys.path.insert(0, "/root/reference/pkg/src")
    from paqif.tvdcd import KappaSchemeConfig, quartic_test_problem, solve_by_sweeps
else:
    import torch
    from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, solve_by_sweeps
for iv in (64, 128, 256, 512):
    prob, exact = quartic_test_problem(iv, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
    k = 2 if ref and iv >= 256 else 4
    solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=1, cycle="x")
    t = time.perf_counter()
    _, h = solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=k, cycle="x")
    dt = (time.perf_counter() - t) / k
    print(f"{'ref' if ref else 'gpu'} intervals={iv} lines={prob.grid.ny} ms/sweep={dt*1e3:.2f} "
          f"us/line={dt*1e6/prob.grid.ny:.1f} res={h[-1]:.3e}", flush=True)

if not ref and "--perline" in sys.argv:
    # per-line factorization path: the upwind closure makes the lines differ
    from paper_2008_03276_b200.tvdcd import ConvectionDiffusionProblem
    for iv in (128, 512):
        q, _ = quartic_test_problem(iv, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
        prob = ConvectionDiffusionProblem(q.grid, q.cfg, q.f, q.boundary, closure="upwind")
        solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=1, cycle="x")
        t = time.perf_counter()
        _, h = solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=3, cycle="x")
        dt = (time.perf_counter() - t) / 3
        print(f"gpu per-line (upwind) intervals={iv} ms/sweep={dt*1e3:.2f} "
              f"us/line={dt*1e6/prob.grid.ny:.1f} res={h[-1]:.3e}", flush=True)
