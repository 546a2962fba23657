"""One TVD Ls1 sweep (quartic problem, 256 intervals) for ncu (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, sweep_splitting
prob, _ = quartic_test_problem(256, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
u, r = sweep_splitting(prob, np.zeros_like(prob.f), "Ls1")
print("res", r)
