"""solve_ehl driver (public surface of paqif/ehl/solver.py:27-240).

The line contact runs every outer iteration as ONE fused CUDA launch
(LineContactBatch with B = 1); the point contact as the native sweep driver
of csrc/ehl_point.cu (PointContact).  Without a ``collect`` callback the
whole loop runs on the device for both (drive records: the stop /
divergence tests of solver.py:219-240 after every iteration, one host
synchronisation per chunk); with ``collect`` the host steps and reads back
the residual and the load deficit each iteration, exactly as the reference
loop does (solver.py:210-240).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ..errors import ContractViolationError, NonConvergenceError, PaqifError
from .film import FilmModel
from .line import LineContactBatch, line_initial_state
from .params import EhlParams
from .point import PointContact, point_initial_state

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

    def complementarity_residual(self, params, kappa, limiter) -> float:
        """max |min(u, -r)| / h^d of the current state (solver.py:43-51)."""
        if self.film.contact == "point":
            from .sweeps import _device_contact
            return _device_contact(self, params, kappa, limiter).residual()
        b = LineContactBatch([params], self.film.n, kappa=kappa, limiter=limiter,
                             u0=np.asarray(self.u)[None], h0=[self.h0])
        return b.residual()[0]


def _initial_state(params: EhlParams, intervals: int) -> EhlState:
    lo, hi = params.domain
    h = (hi - lo) / intervals
    film = FilmModel(params.contact, intervals, h, lo, lo_y=params.lo_y)
    u = (line_initial_state(params, intervals) if params.contact == "line"
         else point_initial_state(params, intervals))
    return EhlState(u=u, h0=params.h0, film=film)


class _LineDriver:
    def __init__(self, params, intervals, state, **kw):
        self.b = LineContactBatch([params], intervals, u0=state.u[None], h0=[state.h0], **kw)

    def step(self):
        self.b.step()
        info = int(self.b.info[0].item())
        if info & (1 << 8):
            from ..errors import FactorizationBreakdownError
            raise FactorizationBreakdownError(-1, "every Ls4 rung broke down")
        if info & (1 << 3):
            raise PaqifError("non-finite change in line-contact sweep")
        deficit = float(self.b.deficit[0].item()) if info & (1 << 2) else None
        return float(self.b.res[0].item()), deficit

    def state(self):
        return self.b.u[0].cpu().numpy(), float(self.b.h0[0].item())

    def run(self, state, tol, tol_fb, max_outer, chunk=32):
        """The whole loop on the device: chunks of `chunk` launches, one
        synchronisation per chunk; the histories are replayed into `state`
        exactly as the host loop appends them."""
        from ..errors import FactorizationBreakdownError
        from .line import (DRIVE_BREAKDOWN, DRIVE_BUDGET, DRIVE_CONVERGED, DRIVE_DIVERGING,
                           DRIVE_NONFINITE, DRIVE_RUNNING)
        b = self.b
        b.drive_init(tol, tol_fb, max_outer, hist_cap=chunk)
        done_before = 0
        while True:
            b.drive_steps(chunk)
            d = b.drive_state()[0]
            k = int(d["outer"])
            hr = b.hist_res[0].cpu().numpy()
            hd = b.hist_def[0].cpu().numpy()
            last = k - 1 if d["done"] == DRIVE_NONFINITE else k  # that step raised on the host
            for it in range(done_before, last):
                if not np.isnan(hd[it % chunk]):
                    state.force_history.append(abs(float(hd[it % chunk])))
                state.residual_history.append(float(hr[it % chunk]))
            state.outer_iterations = last
            done_before = k
            b.outer = k
            if d["done"] == DRIVE_RUNNING:
                continue
            if d["done"] == DRIVE_CONVERGED:
                return state
            if d["done"] == DRIVE_BREAKDOWN:
                raise FactorizationBreakdownError(-1, "every Ls4 rung broke down")
            if d["done"] == DRIVE_NONFINITE:
                raise PaqifError("non-finite change in line-contact sweep")
            res = state.residual_history[-1]
            if d["done"] == DRIVE_DIVERGING:
                raise NonConvergenceError("contact iteration diverging", residual=res,
                                          iterations=k)
            assert d["done"] == DRIVE_BUDGET
            raise NonConvergenceError("contact iteration exhausted its budget", residual=res,
                                      iterations=max_outer)


class _PointDriver:
    def __init__(self, params, intervals, state, force_every, **kw):
        self.fe = force_every
        self.p = PointContact(params, intervals, u0=state.u, h0=state.h0,
                              force_every=force_every, **kw)

    def step(self):
        outer = self.p.outer
        self.p.step()
        _, res, deficit, err = self.p.status()
        PointContact.raise_for(err)
        return res, (deficit if (outer + 1) % self.fe == 0 else None)

    def state(self):
        snap = self.p.snapshot()
        return snap["u"], snap["h0"]

    def run(self, state, tol, tol_fb, max_outer, chunk=8):
        """The loop on the device (paqif_ehl_point_drive_steps): one
        synchronisation per chunk (the first chunk is one iteration, so the
        next chunks' deferred-run prediction has a finished x-sweep to read);
        histories replayed into `state` as the host loop appends them."""
        from ..errors import FactorizationBreakdownError
        from .line import (DRIVE_BREAKDOWN, DRIVE_CONVERGED, DRIVE_DIVERGING, DRIVE_NONFINITE,
                           DRIVE_RUNNING)
        p = self.p
        p.drive_init(tol, tol_fb, max_outer, hist_cap=chunk)
        done_before = 0
        steps = 1
        while True:
            p.drive_steps(steps)
            d = p.drive_state()
            k = int(d["outer"])
            hr = p.hist_res.cpu().numpy()
            hd = p.hist_def.cpu().numpy()
            for it in range(done_before, k):
                if not np.isnan(hd[it % chunk]):
                    state.force_history.append(abs(float(hd[it % chunk])))
                state.residual_history.append(float(hr[it % chunk]))
            state.outer_iterations = k
            done_before = k
            steps = chunk
            if d["done"] == DRIVE_RUNNING:
                continue
            if d["done"] == DRIVE_CONVERGED:
                return state
            if d["done"] == DRIVE_BREAKDOWN:
                raise FactorizationBreakdownError(-1, "every rung of a point line solve broke down")
            if d["done"] == DRIVE_NONFINITE:
                raise PaqifError("non-finite change in point-contact sweep")
            res = state.residual_history[-1]
            if d["done"] == DRIVE_DIVERGING:
                raise NonConvergenceError("contact iteration diverging", residual=res,
                                          iterations=k)
            raise NonConvergenceError("contact iteration exhausted its budget", residual=res,
                                      iterations=max_outer)


def solve_ehl(params: EhlParams, intervals: int, scheme: str = "Lhs1", kappa: float = 1 / 3,
              limiter: str = "kappa", tol: float = 1e-6, tol_fb: float = 1e-4,
              max_outer: int = 10000, omega: float | None = None, state: EhlState | None = None,
              force_every: int = 5, collect=None, exact: bool = True) -> EhlState:
    """Drive the contact problem to a converged pressure/film pair."""
    if scheme not in ("Lhs1", "Lhs2"):
        raise ContractViolationError(f"unknown scheme {scheme!r}")
    if not -1.0 <= kappa <= 1.0:
        raise ContractViolationError("kappa must lie in [-1, 1]")
    if state is None:
        state = _initial_state(params, intervals)
    kw = dict(scheme=scheme, kappa=kappa, limiter=limiter, omega=omega,
              force_every=force_every, exact=exact)
    drv = (_LineDriver(params, intervals, state, **kw) if params.contact == "line"
           else _PointDriver(params, intervals, state, **kw))
    grow = 0
    best = np.inf
    try:
        if collect is None and max_outer > 0:
            return drv.run(state, tol, tol_fb, max_outer)
        for outer in range(max_outer):
            res, fb = drv.step()
            if fb is not None:
                deficit = fb
                state.force_history.append(abs(deficit))
            else:
                deficit = state.force_history[-1] if state.force_history else np.inf
            state.residual_history.append(res)
            state.outer_iterations = outer + 1
            if collect is not None:
                state.u, state.h0 = drv.state()
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
        state.u, state.h0 = drv.state()
