"""Line-sweep helpers (public surface of paqif/ehl/sweeps.py:38-86, 521-535).

The line-contact Newton step itself is fused into one CUDA kernel
(csrc/ehl_line.cu); these are the reference's small host-side helpers."""

from __future__ import annotations

import numpy as np

from ..errors import ContractViolationError

__all__ = ["hybrid_select", "kernel_nu", "force_balance_update", "SWITCH_THRESHOLD",
           "grid_spacing"]

SWITCH_THRESHOLD = 0.6
RATIO_GUARD = 1e-30


def grid_spacing(params, n: int) -> float:
    lo, hi = params.domain
    return (hi - lo) / n


def hybrid_select(eps_over_h, variant: str):
    eps_over_h = np.asarray(eps_over_h)
    if variant == "Lhs1":
        return np.where(eps_over_h > SWITCH_THRESHOLD, "Ls1", "Ls4")
    if variant == "Lhs2":
        return np.where(eps_over_h > SWITCH_THRESHOLD, "Ls0", "Ls5")
    raise ContractViolationError(f"unknown hybrid variant {variant!r}")


def kernel_nu(scheme: str, kappa: float) -> float:
    if scheme in ("Ls1", "Ls4", "Lhs1", "newton"):
        return (2.0 - kappa) / 2.0
    if scheme in ("Ls0", "Ls5", "Lhs2"):
        return (2.0 - kappa) / 2.0 + (1.0 - kappa) / 4.0
    raise ContractViolationError(f"unknown scheme {scheme!r}")


def force_balance_update(state, params):
    """h0 <- h0 - clip(c (target - h^d sum u), +-max_h0_step) (sweeps.py:521-535)."""
    n = state.u.shape[0] - 1
    h = grid_spacing(params, n)
    w = h if state.u.ndim == 1 else h * h
    deficit = params.load_target - w * float(np.sum(state.u))
    step = np.clip(params.relax_c * deficit, -params.max_h0_step, params.max_h0_step)
    state.h0 = state.h0 - step
    state.force_history.append(abs(deficit))
    return state.h0, deficit
