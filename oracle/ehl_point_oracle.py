"""Point-contact EHL oracle -- TEST INFRASTRUCTURE ONLY.

numpy/scipy restatement of one reference outer iteration for the circular
point contact (configs 4/5), pinned against reference-generated goldens
(tests/golden/make_golden_point.py, tests/test_ehl_point_oracle.py).

Reference functions restated (paths under /root/reference/pkg/src/paqif):
  kernel_point                         ehl/kernels.py:78-100
  FilmModel (point): FFT deformation,  ehl/film.py:43-56, 67-78,
    pending line corrections, folds     83-146 (_FOLD_LIMIT = 8)
  _line_quantities                     ehl/sweeps.py:318-341
  assemble_line_system (point terms)   ehl/sweeps.py:157-267
  robust_line_solve / _solve_line      ehl/sweeps.py:270-295
  _hybrid_x_sweep                      ehl/solver.py:76-128
  newton_line_sweep                    ehl/sweeps.py:344-379
  weighted_change_sweep                ehl/sweeps.py:382-418
  column_sweep                         ehl/sweeps.py:421-518
  force_balance_update (h^2 weight)    ehl/sweeps.py:521-535
  reynolds_residual_field (2-D),
  complementarity_residual             ehl/sweeps.py:124-140, ehl/solver.py:43-51
The y-domain adapter of SURVEY.md 8(c) (x in [lo, lo+6], y in [lo_y, lo_y+6])
is built in: geometry 0.5(x^2 + y^2) on the two axes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.fft

from .ehl_oracle import (Breakdown, faces, guarded_ratio, limiter_weight_plus, kernel_nu,
                         padded_bands, rheology, solve_bands, SWITCH)

FOLD_LIMIT = 8


@dataclass
class PointCase:
    p_hertz: float
    lam: float
    alpha: float = 1.7e-8
    z: float = 0.68
    p0: float = 1.98e8
    compressible: bool = True
    lo: float = -4.5
    hi: float = 1.5
    lo_y: float = -3.0
    relax_c: float = 0.05
    omega: float = 0.5
    load_target: float = 3.0 * math.pi / 2.0
    max_change: float = 0.1
    max_h0_step: float = 0.02
    h0: float = -0.5


def point_case(m, l, alpha=1.7e-8, **kw) -> PointCase:
    p_h = l * (3.0 * m) ** (1.0 / 3.0) / (2.0 * math.pi * alpha)
    lam = 4.0 * math.pi * 3.0 ** (-1.0 / 3.0) * m ** (-4.0 / 3.0)
    return PointCase(p_hertz=p_h, lam=lam, alpha=alpha, **kw)


def kernel_point(n, h):
    dx = np.arange(n + 1, dtype=np.float64)[:, None] * h
    dy = np.arange(n + 1, dtype=np.float64)[None, :] * h
    xp, xm, yp, ym = dx + h / 2.0, dx - h / 2.0, dy + h / 2.0, dy - h / 2.0

    def term(a, b):
        return np.abs(a) * np.arcsinh(b / a)
    t = (term(xp, yp) + term(yp, xp) - term(xm, yp) - term(yp, xm)
         - term(xp, ym) - term(ym, xp) + term(xm, ym) + term(ym, xm))
    return t * (2.0 / np.pi ** 2)


class PointFilm:
    """FilmModel('point') with the reference's pending-line bookkeeping."""

    def __init__(self, n, c: PointCase):
        self.n = n
        self.h = (c.hi - c.lo) / n
        self.x = c.lo + self.h * np.arange(n + 1)
        # the SURVEY 8(c) adapter builds y as (x - x[0]) + lo_y; same rounding
        self.y = (self.x - self.x[0]) + c.lo_y
        self.table = kernel_point(n, self.h)
        gx, gy = np.meshgrid(self.x, self.y)
        self.geometry = 0.5 * (gx ** 2 + gy ** 2)
        t = self.table
        full = np.zeros((2 * n + 1, 2 * n + 1))
        full[n:, n:] = t
        full[n:, :n + 1] = t[:, ::-1]
        full[:n + 1, n:] = t[::-1, :]
        full[:n + 1, :n + 1] = t[::-1, ::-1]
        self.shape = [scipy.fft.next_fast_len(3 * n + 1)] * 2
        self.kfft = scipy.fft.rfftn(full, self.shape)
        self.base = None
        self.pending = []
        self.folds = 0

    def deformation_full(self, u):
        uf = scipy.fft.rfftn(u, self.shape)
        conv = scipy.fft.irfftn(uf * self.kfft, self.shape)
        self.base = conv[self.n:2 * self.n + 1, self.n:2 * self.n + 1].copy()
        self.pending = []
        self.folds += 1
        return self.base

    def film_full(self, u, h0):
        return h0 + self.geometry + self.deformation_full(u)

    def note(self, axis, index, delta, u):
        if not np.any(delta):
            return
        self.pending.append((axis, index, delta.copy()))
        if len(self.pending) > FOLD_LIMIT:
            self.deformation_full(u)

    def _row_corr(self, r):
        n = self.n
        corr = np.zeros(n + 1)
        for axis, ell, delta in self.pending:
            if axis == "row":
                kc = self.table[:, abs(r - ell)]
                corr += np.convolve(delta, np.concatenate([kc[::-1], kc[1:]]))[n:2 * n + 1]
            else:
                d1 = np.abs(np.arange(n + 1) - ell)
                d2 = np.abs(r - np.arange(n + 1))
                corr += self.table[np.ix_(d1, d2)] @ delta
        return corr

    def _col_corr(self, cidx):
        n = self.n
        corr = np.zeros(n + 1)
        for axis, ell, delta in self.pending:
            if axis == "col":
                kc = self.table[:, abs(cidx - ell)]
                corr += np.convolve(delta, np.concatenate([kc[::-1], kc[1:]]))[n:2 * n + 1]
            else:
                d_k = np.abs(np.arange(n + 1) - cidx)
                d_m = np.abs(ell - np.arange(n + 1))
                corr += delta @ self.table[np.ix_(d_k, d_m)]
        return corr

    def rows(self, rows, h0):
        out = np.empty((len(rows), self.n + 1))
        for k, r in enumerate(rows):
            out[k] = h0 + self.geometry[r] + self.base[r]
            if self.pending:
                out[k] += self._row_corr(r)
        return out

    def cols(self, cols, h0):
        out = np.empty((len(cols), self.n + 1))
        for k, cc in enumerate(cols):
            out[k] = h0 + self.geometry[:, cc] + self.base[:, cc]
            if self.pending:
                out[k] += self._col_corr(cc)
        return out

    def sens(self, d, off=0):
        return float(self.table[abs(d), abs(off)])


def assemble_point(q, rho, ex_p, ex_m, ey_p, ey_m, resid, film: PointFilm, h, kappa, limiter,
                   scheme, jacobian="scheme"):
    """assemble_line_system for an x-line of the point contact (hy = h, cross
    kernel terms in the weighted schemes)."""
    n = q.size - 1
    _, phi_p, phi_m = faces(q, limiter, kappa)
    if jacobian in ("first-order", "diagonal"):
        phi_p = np.zeros_like(phi_p)
        phi_m = np.zeros_like(phi_m)
    weighted = scheme in ("Ls4", "Ls5")
    s = film.sens
    if weighted:
        nu = kernel_nu(scheme, kappa)
        cross = 2.0 * s(0, 1)
        cross1 = 2.0 * s(1, 1)
        ks0 = nu * (s(0) - 0.25 * (2.0 * s(1) + cross))
        ks1 = nu * (s(1) - 0.25 * (s(0) + s(2) + cross1))
    else:
        ks0, ks1 = s(0), s(1)
    i = np.arange(1, n)
    rw, rc, re = rho[i - 1], rho[i], rho[i + 1]
    a_p, b_p = 1.0 - 0.5 * phi_p, 0.5 * phi_p
    a_m, b_m = 1.0 - 0.5 * phi_m, 0.5 * phi_m
    hy = h
    if jacobian == "diagonal":
        z = np.zeros(n - 1)
        c_m2, c_m1, c_p1, c_p2 = z, z, z, z
        c_0 = -hy * rc * abs(ks0)
    else:
        c_m2 = hy * (a_m * rw * ks1)
        c_m1 = -hy * (a_p * rc * ks1 - a_m * rw * ks0 - b_m * rc * ks1)
        c_0 = -hy * (a_p * rc * ks0 + b_p * re * ks1 - a_m * rw * ks1 - b_m * rc * ks0)
        c_p1 = -hy * (a_p * rc * ks1 + b_p * re * ks0 - b_m * rc * ks1)
        c_p2 = -hy * (b_p * re * ks1)
    ey_sum = ey_p + ey_m
    if weighted:
        p_m2 = -0.25 * ex_m / h
        p_m1 = (1.25 * ex_m + 0.25 * ex_p) / h + 0.25 * ey_sum / h
        p_0 = -1.25 * (ex_p + ex_m + ey_sum) / h
        p_p1 = (1.25 * ex_p + 0.25 * ex_m) / h + 0.25 * ey_sum / h
        p_p2 = -0.25 * ex_p / h
    else:
        zz = np.zeros(n - 1)
        p_m2, p_p2 = zz, zz
        p_m1 = ex_m / h
        p_0 = -(ex_p + ex_m + ey_sum) / h
        p_p1 = ex_p / h
    ent = {-2: -(c_m2 + p_m2), -1: -(c_m1 + p_m1), 0: -(c_0 + p_0), 1: -(c_p1 + p_p1),
           2: -(c_p2 + p_p2)}
    off_mag = np.abs(ent[-2]) + np.abs(ent[-1]) + np.abs(ent[1]) + np.abs(ent[2])
    floor = 0.05 * hy * np.abs(rc) * abs(ks0)
    bad = np.abs(ent[0]) < np.maximum(0.2 * off_mag, floor)
    if np.any(bad):
        fo_m2 = hy * rw * ks1
        fo_m1 = -hy * (rc * ks1 - rw * ks0)
        fo_0 = -hy * (rc * ks0 - rw * ks1)
        fo_p1 = -hy * rc * ks1
        ent[-2] = np.where(bad, -(fo_m2 + p_m2), ent[-2])
        ent[-1] = np.where(bad, -(fo_m1 + p_m1), ent[-1])
        ent[0] = np.where(bad, -(fo_0 + p_0), ent[0])
        ent[1] = np.where(bad, -(fo_p1 + p_p1), ent[1])
        ent[2] = np.where(bad, -p_p2, ent[2])
    bands = padded_bands(ent, n - 1)
    rhs = np.zeros(bands.shape[1])
    rhs[:n - 1] = resid
    return bands, rhs


def robust_solve(args, film, h, kappa, limiter, scheme):
    n_int = args[0].size - 2
    for jac in ("scheme", "first-order", "diagonal"):
        bands, rhs = assemble_point(*args[1:], film, h, kappa, limiter, scheme, jacobian=jac)
        try:
            return solve_bands(bands, rhs, n_int), jac
        except Breakdown:
            continue
    raise Breakdown(-1)


def line_quantities(u, film: PointFilm, c: PointCase, j, h0, kappa, limiter):
    n = u.shape[0] - 1
    h = film.h
    films = film.rows([j - 1, j, j + 1], h0)
    rho3, _, eps3 = rheology(u[j - 1:j + 2], c, film=films)
    i = np.arange(1, n)
    e = eps3[1]
    ex_p = 0.5 * (e[i] + e[i + 1]) * h
    ex_m = 0.5 * (e[i] + e[i - 1]) * h
    ey_p = 0.5 * (e[i] + eps3[2, i]) * h
    ey_m = 0.5 * (e[i] + eps3[0, i]) * h
    q = rho3[1] * films[1]
    fd, _, _ = faces(q, limiter, kappa)
    resid = (ex_p * (u[j, i + 1] - u[j, i]) + ex_m * (u[j, i - 1] - u[j, i])) / h \
        + (ey_p * (u[j + 1, i] - u[j, i]) + ey_m * (u[j - 1, i] - u[j, i])) / h - h * fd
    return (u[j], q, rho3[1], ex_p, ex_m, ey_p, ey_m, resid), eps3[1]


def hybrid_x_sweep(u, h0, film: PointFilm, c: PointCase, kappa=1 / 3, limiter="kappa",
                   variant="Lhs1"):
    """Returns (u, tags, rungs); u updated in place for Newton lines."""
    n = u.shape[0] - 1
    h = film.h
    omega = c.omega
    sigma = np.zeros_like(u)
    any_w = False
    ns, ws = ("Ls1", "Ls4") if variant == "Lhs1" else ("Ls0", "Ls5")
    tags, rungs = [], []
    for j in range(1, n):
        args, eps_line = line_quantities(u, film, c, j, h0, kappa, limiter)
        ratio = float(np.min(eps_line)) / h
        if ratio > SWITCH:
            sig, rung = robust_solve(args, film, h, kappa, limiter, ns)
            tags.append(1)
            sig = np.clip(sig, -c.max_change, c.max_change)
            new = np.maximum(0.0, u[j, 1:n] + omega * sig)
            delta = np.zeros(n + 1)
            delta[1:n] = new - u[j, 1:n]
            u[j, 1:n] = new
            film.note("row", j, delta, u)
        else:
            any_w = True
            tags.append(0)
            sig, rung = robust_solve(args, film, h, kappa, limiter, ws)
            sigma[j, 1:n] = np.clip(sig, -c.max_change, c.max_change)
        rungs.append(rung)
    if any_w:
        spread = np.zeros_like(sigma)
        spread[:, 1:] += sigma[:, :-1]
        spread[:, :-1] += sigma[:, 1:]
        spread[1:, :] += sigma[:-1, :]
        spread[:-1, :] += sigma[1:, :]
        u = np.maximum(0.0, u + omega * (sigma - 0.25 * spread))
        u[0, :] = u[-1, :] = 0.0
        u[:, 0] = u[:, -1] = 0.0
        film.deformation_full(u)
    return u, tags, rungs


def x_sweep_lines(u, h0, c: PointCase, film: PointFilm, budget_s, kappa=1 / 3,
                  limiter="kappa", variant="Lhs1"):
    """A bounded sample of hybrid_x_sweep for CPU-baseline timing (bench.py
    config 5): the sweep's lines in order, Newton lines updating u and the
    pending list (folds included) as in hybrid_x_sweep, until budget_s
    seconds have passed.  Returns the number of lines done."""
    import time
    n = u.shape[0] - 1
    h = film.h
    ns, ws = ("Ls1", "Ls4") if variant == "Lhs1" else ("Ls0", "Ls5")
    t0 = time.perf_counter()
    done = 0
    for j in range(1, n):
        args, eps_line = line_quantities(u, film, c, j, h0, kappa, limiter)
        newton = float(np.min(eps_line)) / h > SWITCH
        sig, _ = robust_solve(args, film, h, kappa, limiter, ns if newton else ws)
        if newton:
            sig = np.clip(sig, -c.max_change, c.max_change)
            new = np.maximum(0.0, u[j, 1:n] + c.omega * sig)
            delta = np.zeros(n + 1)
            delta[1:n] = new - u[j, 1:n]
            u[j, 1:n] = new
            film.note("row", j, delta, u)
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return done


def newton_line_sweep(u, h0, film: PointFilm, c: PointCase, kappa=1 / 3, limiter="kappa",
                      scheme="Ls1", omega=None, hybrid=None):
    """sweeps.newton_line_sweep (sweeps.py:344-379): immediate updates, the
    line system fixed or picked per line by hybrid_select.  Returns
    (u, worst |resid|)."""
    n = u.shape[0] - 1
    h = film.h
    omega = c.omega if omega is None else omega
    worst = 0.0
    for j in range(1, n):
        args, eps_line = line_quantities(u, film, c, j, h0, kappa, limiter)
        sch = scheme
        if hybrid is not None:
            pair = ("Ls1", "Ls4") if hybrid == "Lhs1" else ("Ls0", "Ls5")
            sch = pair[0] if float(np.min(eps_line)) / h > SWITCH else pair[1]
        sig, _ = robust_solve(args, film, h, kappa, limiter, sch)
        sig = np.clip(sig, -c.max_change, c.max_change)
        new = np.maximum(0.0, u[j, 1:n] + omega * sig)
        delta = np.zeros(n + 1)
        delta[1:n] = new - u[j, 1:n]
        u[j, 1:n] = new
        film.note("row", j, delta, u)
        worst = max(worst, float(np.max(np.abs(args[-1]))))
    return u, worst


def weighted_change_sweep(u, h0, film: PointFilm, c: PointCase, kappa=1 / 3, limiter="kappa",
                          scheme="Ls4", omega=None):
    """sweeps.weighted_change_sweep (sweeps.py:382-418): every line against
    the sweep-start state, changes spread to the 4 neighbours at the end.
    Returns (u, worst |resid|)."""
    n = u.shape[0] - 1
    h = film.h
    omega = c.omega if omega is None else omega
    sigma = np.zeros_like(u)
    worst = 0.0
    for j in range(1, n):
        args, _ = line_quantities(u, film, c, j, h0, kappa, limiter)
        sig, _ = robust_solve(args, film, h, kappa, limiter, scheme)
        sigma[j, 1:n] = np.clip(sig, -c.max_change, c.max_change)
        worst = max(worst, float(np.max(np.abs(args[-1]))))
    spread = np.zeros_like(sigma)
    spread[:, 1:] += sigma[:, :-1]
    spread[:, :-1] += sigma[:, 1:]
    spread[1:, :] += sigma[:-1, :]
    spread[:-1, :] += sigma[1:, :]
    u = np.maximum(0.0, u + omega * (sigma - 0.25 * spread))
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    film.deformation_full(u)
    return u, worst


def column_sweep(u, h0, film: PointFilm, c: PointCase, kappa=1 / 3, limiter="kappa",
                 omega=None, stats=None):
    """sweeps.column_sweep (sweeps.py:421-518).  Returns (u, rungs); the
    worst |resid| goes to stats['worst'] when a dict is passed."""
    n = u.shape[0] - 1
    h = film.h
    omega = c.omega if omega is None else omega
    s = film.sens
    rungs = []
    worst = 0.0
    for i in range(1, n):
        lo = max(0, i - 2)
        films = film.cols(list(range(lo, i + 2)), h0)
        cols = np.ascontiguousarray(u[:, lo:i + 2].T)
        rho_c, _, eps_c = rheology(cols, c, film=films)
        pos = i - lo
        j = np.arange(1, n)
        e = eps_c[pos]
        ey_p = 0.5 * (e[j] + e[j + 1]) * h
        ey_m = 0.5 * (e[j] + e[j - 1]) * h
        ex_p = 0.5 * (e[j] + eps_c[pos + 1, j]) * h
        ex_m = 0.5 * (e[j] + eps_c[pos - 1, j]) * h
        q = rho_c * films
        dq_p = q[pos + 1, j] - q[pos, j]
        dq_m = q[pos, j] - q[pos - 1, j]
        qs = float(np.max(np.abs(q)))
        phi_p = limiter_weight_plus(guarded_ratio(dq_p, dq_m, qs), limiter, kappa)
        if pos >= 2:
            dq_mm = q[pos - 1, j] - q[pos - 2, j]
            phi_m = limiter_weight_plus(guarded_ratio(dq_m, dq_mm, qs), limiter, kappa)
        else:
            phi_m = np.zeros(n - 1)
        flux_p = q[pos, j] + 0.5 * phi_p * dq_p
        flux_m = q[pos - 1, j] + 0.5 * phi_m * dq_m
        resid = (ex_p * (u[j, i + 1] - u[j, i]) + ex_m * (u[j, i - 1] - u[j, i])) / h \
            + (ey_p * (u[j + 1, i] - u[j, i]) + ey_m * (u[j - 1, i] - u[j, i])) / h \
            - h * (flux_p - flux_m)
        a_p, b_p = 1.0 - 0.5 * phi_p, 0.5 * phi_p
        a_m, b_m = 1.0 - 0.5 * phi_m, 0.5 * phi_m
        rho_i, rho_w, rho_e = rho_c[pos, j], rho_c[pos - 1, j], rho_c[pos + 1, j]
        c_diag = -h * ((a_p - b_m) * rho_i * s(0, 0) + (b_p * rho_e - a_m * rho_w) * s(1, 0))
        c_off = -h * ((a_p - b_m) * rho_i * s(0, 1) + (b_p * rho_e - a_m * rho_w) * s(1, 1))
        diag_full = -(ey_p + ey_m + ex_p + ex_m) / h + c_diag
        floor = 0.05 * h * np.abs(rho_i) * s(0, 0)
        bad = np.abs(diag_full) < floor
        if np.any(bad):
            fo_diag = -h * (rho_i * s(0, 0) - rho_w * s(1, 0))
            fo_off = -h * (rho_i * s(0, 1) - rho_w * s(1, 1))
            c_diag = np.where(bad, fo_diag, c_diag)
            c_off = np.where(bad, fo_off, c_off)
            diag_full = -(ey_p + ey_m + ex_p + ex_m) / h + c_diag
        ent = {-1: -(ey_m / h + c_off), 0: -diag_full, 1: -(ey_p / h + c_off)}
        bands = padded_bands(ent, n - 1)
        rhs = np.zeros(bands.shape[1])
        rhs[:n - 1] = resid
        try:
            sigma = solve_bands(bands, rhs, n - 1)
            rungs.append("scheme")
        except Breakdown:
            diag = (ey_p + ey_m + ex_p + ex_m) / h + h * np.abs(rho_i) * s(0, 0)
            bands = padded_bands({0: diag}, n - 1)
            sigma = solve_bands(bands, rhs, n - 1)
            rungs.append("diagonal")
        sigma = np.clip(sigma, -c.max_change, c.max_change)
        new = np.maximum(0.0, u[1:n, i] + omega * sigma)
        delta = np.zeros(n + 1)
        delta[1:n] = new - u[1:n, i]
        u[1:n, i] = new
        film.note("col", i, delta, u)
        worst = max(worst, float(np.max(np.abs(resid))))
    if stats is not None:
        stats["worst"] = worst
    return u, rungs


def residual_field(u, fv, c: PointCase, film: PointFilm, kappa, limiter):
    rho, _, eps = rheology(u, c, film=fv)
    q = rho * fv
    n = u.shape[0] - 1
    h = film.h
    r = np.zeros_like(u)
    i = np.arange(1, n)
    for j in range(1, n):
        e = eps[j]
        exp_ = 0.5 * (e[i] + e[i + 1]) * h
        exm = 0.5 * (e[i] + e[i - 1]) * h
        eyp = 0.5 * (e[i] + eps[j + 1, i]) * h
        eym = 0.5 * (e[i] + eps[j - 1, i]) * h
        fd, _, _ = faces(q[j], limiter, kappa)
        r[j, i] = (exp_ * (u[j, i + 1] - u[j, i]) + exm * (u[j, i - 1] - u[j, i])) / h \
            + (eyp * (u[j + 1, i] - u[j, i]) + eym * (u[j - 1, i] - u[j, i])) / h - h * fd
    return r


def complementarity_residual(u, h0, c: PointCase, film: PointFilm, kappa=1 / 3,
                             limiter="kappa"):
    """EhlState.complementarity_residual (solver.py:43-51), point contact."""
    fv = film.film_full(u, h0)
    r = residual_field(u, fv, c, film, kappa, limiter)
    return float(np.max(np.abs(np.minimum(u, -r)))) / (film.h * film.h)


def point_step(u, h0, outer, c: PointCase, film: PointFilm, kappa=1 / 3, limiter="kappa",
               force_every=5):
    """One solve_ehl outer iteration (point).  Returns (u, h0, film, res, info)."""
    u = u.copy()
    film.deformation_full(u)
    u, tags, xr = hybrid_x_sweep(u, h0, film, c, kappa, limiter)
    u_x = u.copy()
    u, yr = column_sweep(u, h0, film, c, kappa, limiter)
    applied = False
    if (outer + 1) % force_every == 0:
        h = film.h
        deficit = c.load_target - h * h * float(np.sum(u))
        step = np.clip(c.relax_c * deficit, -c.max_h0_step, c.max_h0_step)
        h0 = h0 - step
        applied = True
    fv = film.film_full(u, h0)
    r = residual_field(u, fv, c, film, kappa, limiter)
    res = float(np.max(np.abs(np.minimum(u, -r)))) / (film.h * film.h)
    return u, h0, fv, res, dict(tags=np.array(tags), x_rungs=xr, y_rungs=yr, u_x=u_x,
                                fb_applied=applied)


def hertz_start(c: PointCase, film: PointFilm):
    gx, gy = np.meshgrid(film.x, film.y)
    u = np.sqrt(np.maximum(0.0, 1.0 - gx * gx - gy * gy))
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    return u * (c.load_target / (2.0 * np.pi / 3.0))
