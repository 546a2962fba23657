"""Line sweeps (public surface of paqif/ehl/sweeps.py:38-86, 344-535).

The line-contact Newton step is fused into one CUDA kernel
(csrc/ehl_line.cu).  The point-contact sweeps newton_line_sweep,
weighted_change_sweep and column_sweep run on the device state of a
PointContact (csrc/ehl_point.cu) attached to the EhlState's film model:
the state is uploaded, the 2(n-1)-line sweep runs as device kernels, and
the new pressure comes back into ``state.u``."""

from __future__ import annotations

import numpy as np

from ..errors import ContractViolationError

__all__ = ["hybrid_select", "kernel_nu", "force_balance_update", "SWITCH_THRESHOLD",
           "grid_spacing", "newton_line_sweep", "weighted_change_sweep", "column_sweep"]

_NEWTON = ("Ls0", "Ls1")
_WEIGHTED = ("Ls4", "Ls5")

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


def _nu_variant(scheme: str) -> int:
    kernel_nu(scheme, 0.0)  # validates the name
    return 0 if scheme in ("Ls1", "Ls4", "Lhs1", "newton") else 1


def _device_contact(state, params, kappa, limiter):
    from .point import PointContact
    film = state.film
    if getattr(film, "contact", None) != "point" or np.ndim(state.u) != 2:
        raise ContractViolationError("x/y line sweeps need a point-contact state")
    key = (id(params), float(kappa), str(limiter))
    pc = getattr(film, "_contact", None)
    if pc is None or pc._key != key:
        pc = PointContact(params, film.n, kappa=kappa, limiter=limiter, u0=state.u,
                          h0=state.h0)
        pc._key = key
        film._contact = pc
    else:
        pc.set_state(state.u, state.h0)
    return pc


def _finish(state, pc):
    from .point import PointContact
    snap = pc.snapshot()
    PointContact.raise_for(snap["err"])
    state.u = snap["u"]
    state.film._base = None  # deformation recomputed on the next film_full
    return snap["worst"]


def newton_line_sweep(state, params, kappa: float, limiter: str, scheme: str = "Ls1",
                      omega: float | None = None, hybrid: str | None = None) -> float:
    """x-sweep with immediate line updates (sweeps.py:344-379); ``hybrid``
    picks each line's system by min(eps)/h.  Returns the worst |resid|."""
    if hybrid is not None:
        hybrid_select(1.0, hybrid)
        sel, nu = -1, 0 if hybrid == "Lhs1" else 1
    else:
        if scheme not in _NEWTON + _WEIGHTED:
            raise ContractViolationError(f"unknown scheme {scheme!r}")
        sel, nu = (1 if scheme in _WEIGHTED else 0), _nu_variant(scheme)
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(1, sel, nu, params.omega if omega is None else omega)
    return _finish(state, pc)


def weighted_change_sweep(state, params, kappa: float, limiter: str, scheme: str = "Ls4",
                          omega: float | None = None) -> float:
    """x-sweep with deferred, distributed changes (sweeps.py:382-418)."""
    if scheme not in _NEWTON + _WEIGHTED:
        raise ContractViolationError(f"unknown scheme {scheme!r}")
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(2, 1 if scheme in _WEIGHTED else 0, _nu_variant(scheme),
             params.omega if omega is None else omega)
    return _finish(state, pc)


def column_sweep(state, params, kappa: float, limiter: str, omega: float | None = None) -> float:
    """y-sweep, tridiagonal column systems, immediate updates (sweeps.py:421-518)."""
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(3, 0, 0, params.omega if omega is None else omega)
    return _finish(state, pc)
