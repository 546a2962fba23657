"""solve_ehl driver (public surface of paqif/ehl/solver.py:27-240).

The line contact runs every outer iteration as ONE fused CUDA launch
(LineContactBatch with B = 1); the host only reads back the residual and the
load deficit for the stop / divergence tests and the ``collect`` callback,
exactly as the reference loop does (solver.py:210-240).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ..errors import ContractViolationError, NonConvergenceError, PaqifError
from .film import FilmModel
from .line import LineContactBatch, line_initial_state
from .params import EhlParams

__all__ = ["EhlState", "solve_ehl"]


@dataclass
class EhlState:
    u: np.ndarray
    h0: float
    film: FilmModel
    residual_history: list = field(default_factory=list)
    force_history: list = field(default_factory=list)
    outer_iterations: int = 0

    def film_field(self) -> np.ndarray:
        return self.film.film_full(self.u, self.h0)


def _initial_state(params: EhlParams, intervals: int) -> EhlState:
    lo, hi = params.domain
    h = (hi - lo) / intervals
    film = FilmModel(params.contact, intervals, h, lo)
    if params.contact != "line":
        raise NotImplementedError("point contact: next row (DESIGN.md section 7)")
    return EhlState(u=line_initial_state(params, intervals), h0=params.h0, film=film)


def solve_ehl(params: EhlParams, intervals: int, scheme: str = "Lhs1", kappa: float = 1 / 3,
              limiter: str = "kappa", tol: float = 1e-6, tol_fb: float = 1e-4,
              max_outer: int = 10000, omega: float | None = None, state: EhlState | None = None,
              force_every: int = 5, collect=None, exact: bool = True) -> EhlState:
    """Drive the contact problem to a converged pressure/film pair."""
    if scheme not in ("Lhs1", "Lhs2"):
        raise ContractViolationError(f"unknown scheme {scheme!r}")
    if not -1.0 <= kappa <= 1.0:
        raise ContractViolationError("kappa must lie in [-1, 1]")
    if params.contact != "line":
        raise NotImplementedError("point contact: next row (DESIGN.md section 7)")
    if state is None:
        state = _initial_state(params, intervals)
    batch = LineContactBatch([params], intervals, scheme=scheme, kappa=kappa, limiter=limiter,
                             omega=omega, force_every=force_every, exact=exact,
                             u0=state.u[None], h0=[state.h0])
    grow = 0
    best = np.inf
    try:
        for outer in range(max_outer):
            batch.step()
            res = float(batch.res[0].item())
            info = int(batch.info[0].item())
            if info & (1 << 8):
                from ..errors import FactorizationBreakdownError
                raise FactorizationBreakdownError(-1, "every Ls4 rung broke down")
            if info & (1 << 3):
                raise PaqifError("non-finite change in line-contact sweep")
            if info & (1 << 2):
                deficit = float(batch.deficit[0].item())
                state.force_history.append(abs(deficit))
            else:
                deficit = state.force_history[-1] if state.force_history else np.inf
            state.residual_history.append(res)
            state.outer_iterations = outer + 1
            if collect is not None:
                state.u = batch.u[0].cpu().numpy()
                state.h0 = float(batch.h0[0].item())
                collect(state, res, deficit)
            if res <= tol and abs(deficit) <= tol_fb:
                return state
            if res < best:
                best = res
                grow = 0
            else:
                grow += 1
                if grow >= 20 and res > 1e3 * max(best, tol):
                    raise NonConvergenceError("contact iteration diverging", residual=res,
                                              iterations=outer + 1)
        raise NonConvergenceError("contact iteration exhausted its budget",
                                  residual=state.residual_history[-1], iterations=max_outer)
    finally:
        state.u = batch.u[0].cpu().numpy()
        state.h0 = float(batch.h0[0].item())
