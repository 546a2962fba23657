"""EHL Newton-step oracle -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's line-contact outer iteration, used as
the checker for the CUDA step (tests/, smoke, bench cpu_baseline).  Banded
solves go through the bit-exact C AQIF oracle (oracle/paqif_oracle.c).
Pinned against goldens produced by the reference itself
(tests/golden/make_golden_ehl.py, tests/test_ehl_oracle.py).

Reference functions restated (paths under /root/reference/pkg/src/paqif):
  moes_convert / line_dimensionless / moes_from_line   ehl/params.py:108-146
  rheology                                             ehl/params.py:149-175
  hertzian_init                                        ehl/params.py:178-186
  kernel_line / _log_antiderivative                    ehl/kernels.py:55-75
  FilmModel line deformation (np.convolve)             ehl/film.py:57-61, 67-71
  limiter_psi / limiter_weight_plus                    tvdcd.py:207-235
  _guarded_ratio / _faces                              ehl/sweeps.py:47-56, 89-103
  _padded_matrix / assemble_line_system                ehl/sweeps.py:143-267
  _solve_line / robust_line_solve                      ehl/sweeps.py:270-295
  _line_contact_sweep                                  ehl/solver.py:131-183
  force_balance_update                                 ehl/sweeps.py:521-535
  reynolds_residual_field (line) / complementarity    ehl/sweeps.py:106-123,
                                                       ehl/solver.py:43-51
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import factor_batch, solve_w_batch, solve_z_batch

P0 = 1.98e8
ZEXP = 0.68
DENS_A = 0.59e9
DENS_B = 1.34
RATIO_GUARD = 1e-30
SWITCH = 0.6


@dataclass
class LineCase:
    """Dimensionless line-contact problem (the fields of EhlParams the line
    step reads)."""
    p_hertz: float
    lam: float
    alpha: float = 1.7e-8
    z: float = ZEXP
    p0: float = P0
    compressible: bool = True
    lo: float = -4.5
    hi: float = 1.5
    relax_c: float = 0.05
    omega: float = 0.5
    load_target: float = math.pi / 2.0
    max_change: float = 0.1
    max_h0_step: float = 0.02
    h0: float = -0.5


def line_dimensionless(g, u, w, alpha):
    e_prime = g / alpha
    p_h = e_prime * math.sqrt(w / (2.0 * math.pi))
    lam = 12.0 * u / ((8.0 * w / math.pi) ** 1.5 * math.sqrt(w / (2.0 * math.pi)))
    return p_h, lam


def line_case(m, l, g=5000.0, alpha=1.7e-8, **kw) -> LineCase:
    two_u = (l / g) ** 4.0
    u, w = two_u / 2.0, m * two_u ** 0.5
    p_h, lam = line_dimensionless(g, u, w, alpha)
    return LineCase(p_hertz=p_h, lam=lam, alpha=alpha, **kw)


def rheology(u, c: LineCase, film=None):
    u = np.asarray(u, dtype=np.float64)
    if c.compressible:
        p = u * c.p_hertz
        rho = (DENS_A + DENS_B * p) / (DENS_A + p)
        arg = (c.alpha * c.p0 / c.z) * (-1.0 + (1.0 + p / c.p0) ** c.z)
        eta = np.exp(np.minimum(arg, 200.0))
    else:
        rho = np.ones_like(u)
        eta = np.ones_like(u)
    coeff = rho / (eta * c.lam)
    if film is not None:
        gap = np.maximum(np.asarray(film), 1e-8)
        return rho, eta, coeff * gap ** 3
    return rho, eta, coeff


def kernel_line(n, h):
    d = np.arange(n + 1, dtype=np.float64)
    xp, xm = d * h + h / 2.0, d * h - h / 2.0

    def anti(t):
        out = np.zeros_like(t)
        nz = t != 0.0
        out[nz] = t[nz] * (np.log(np.abs(t[nz])) - 1.0)
        return out
    return anti(xp) - anti(xm)


class LineFilm:
    def __init__(self, n, c: LineCase):
        self.n = n
        self.h = (c.hi - c.lo) / n
        self.x = c.lo + self.h * np.arange(n + 1)
        self.table = kernel_line(n, self.h)
        self.ext = np.concatenate([self.table[::-1], self.table[1:]])
        self.geometry = 0.5 * self.x ** 2
        self.sign = -1.0 / np.pi

    def deformation(self, u):
        return self.sign * np.convolve(u, self.ext)[self.n:2 * self.n + 1]

    def sensitivity(self, d):
        return self.sign * float(self.table[abs(d)])


def limiter_psi(r, name, kappa):
    if name == "none":
        return ((1.0 + kappa) * r + (1.0 - kappa)) / 2.0
    if name == "van-albada":
        return np.where(r > 0.0, (r * r + r) / (1.0 + r * r), 0.0)
    if name == "minmod":
        return np.maximum(0.0, np.minimum(r, 1.0))
    if name == "koren":
        return np.maximum(0.0, np.minimum(np.minimum(2.0 * r, (1.0 + 2.0 * r) / 3.0), 2.0))
    if name == "kappa":
        lin = ((1.0 + kappa) * r + (1.0 - kappa)) / 2.0
        return np.maximum(0.0, np.minimum(np.minimum(2.0 * r, lin), 2.0))
    raise ValueError(name)


def limiter_weight_plus(r, name, kappa):
    psi = limiter_psi(r, name, kappa)
    safe = np.where(np.abs(r) > RATIO_GUARD, r, np.where(r >= 0.0, RATIO_GUARD, -RATIO_GUARD))
    return np.where(r > 0.0, psi / safe, 0.0)


def guarded_ratio(num, den, scale):
    floor = 1e-12 * max(float(scale), RATIO_GUARD)
    den_safe = np.where(np.abs(den) > floor, den, 1.0)
    return np.where(np.abs(den) > floor, num / den_safe, 0.0)


def faces(q, limiter, kappa):
    n = q.size - 1
    i = np.arange(1, n)
    dq = np.diff(q)
    scale = float(np.max(np.abs(q)))
    phi_p = limiter_weight_plus(guarded_ratio(dq[i], dq[i - 1], scale), limiter, kappa)
    phi_m = np.zeros(n - 1)
    phi_m[1:] = limiter_weight_plus(guarded_ratio(dq[i[1:] - 1], dq[i[1:] - 2], scale),
                                    limiter, kappa)
    flux_p = q[i] + 0.5 * phi_p * dq[i]
    flux_m = q[i - 1] + 0.5 * phi_m * dq[i - 1]
    return flux_p - flux_m, phi_p, phi_m


def kernel_nu(scheme, kappa):
    if scheme in ("Ls1", "Ls4"):
        return (2.0 - kappa) / 2.0
    return (2.0 - kappa) / 2.0 + (1.0 - kappa) / 4.0


def padded_bands(entries, n_int, beta=2):
    n_sys = n_int + 1 if (n_int + 1) % 2 == 0 else n_int + 2
    bands = np.zeros((2 * beta + 1, n_sys))
    bands[beta, :] = 1.0
    for off, vals in entries.items():
        lo = max(0, -off)
        bands[beta + off, lo:n_int] = vals[lo:n_int]
    bands[beta, n_int:] = 1.0
    for o in range(1, beta + 1):
        bands[beta + o, n_sys - o:] = 0.0
        bands[beta - o, :o] = 0.0
    return bands


def assemble(u, q, rho, ex_p, ex_m, resid, film: LineFilm, h, kappa, limiter, scheme,
             jacobian="scheme"):
    """Pentadiagonal change system of the line (sweeps.py:157-267), line
    contact (hy = 1, no transverse mobility)."""
    n = u.size - 1
    i = np.arange(1, n)
    _, phi_p, phi_m = faces(q, limiter, kappa)
    if jacobian in ("first-order", "diagonal"):
        phi_p = np.zeros_like(phi_p)
        phi_m = np.zeros_like(phi_m)
    weighted = scheme in ("Ls4", "Ls5")
    sens = film.sensitivity
    if weighted:
        nu = kernel_nu(scheme, kappa)
        ks0 = nu * (sens(0) - 0.25 * (2.0 * sens(1) + 0.0))
        ks1 = nu * (sens(1) - 0.25 * (sens(0) + sens(2) + 0.0))
    else:
        ks0, ks1 = sens(0), sens(1)
    rw, rc, re = rho[i - 1], rho[i], rho[i + 1]
    a_p = 1.0 - 0.5 * phi_p
    b_p = 0.5 * phi_p
    a_m = 1.0 - 0.5 * phi_m
    b_m = 0.5 * phi_m
    hy = 1.0
    if jacobian == "diagonal":
        zero = np.zeros(n - 1)
        c_m2, c_m1, c_p1, c_p2 = zero, zero, zero, zero
        c_0 = -hy * rc * abs(ks0)
    else:
        c_m2 = hy * (a_m * rw * ks1)
        c_m1 = -hy * (a_p * rc * ks1 - a_m * rw * ks0 - b_m * rc * ks1)
        c_0 = -hy * (a_p * rc * ks0 + b_p * re * ks1 - a_m * rw * ks1 - b_m * rc * ks0)
        c_p1 = -hy * (a_p * rc * ks1 + b_p * re * ks0 - b_m * rc * ks1)
        c_p2 = -hy * (b_p * re * ks1)
    zeros = np.zeros(n - 1)
    ey_sum = zeros + zeros
    if weighted:
        p_m2 = -0.25 * ex_m / h
        p_m1 = (1.25 * ex_m + 0.25 * ex_p) / h + 0.25 * ey_sum / h
        p_0 = -1.25 * (ex_p + ex_m + ey_sum) / h
        p_p1 = (1.25 * ex_p + 0.25 * ex_m) / h + 0.25 * ey_sum / h
        p_p2 = -0.25 * ex_p / h
    else:
        p_m2 = zeros
        p_m1 = ex_m / h
        p_0 = -(ex_p + ex_m + ey_sum) / h
        p_p1 = ex_p / h
        p_p2 = zeros
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
    return bands, rhs, bad


class Breakdown(Exception):
    pass


def solve_bands(bands, rhs, n_int):
    """factorize_wz -> solve_w -> solve_z through the bit-exact C kernels;
    raises Breakdown like FactorizationBreakdownError."""
    n = bands.shape[1]
    beta = (bands.shape[0] - 1) // 2
    s = n // 2
    band = np.ascontiguousarray(bands[None]).copy()
    anti = np.zeros_like(band)
    z2 = np.zeros((1, s + 1, 2, 2))
    zl = np.zeros((1, s + 1, 2, beta + 1))
    zr = np.zeros_like(zl)
    ww = np.zeros((1, s + 1, 2 * beta, 2))
    st = np.zeros(1, np.int64)
    factor_batch(band, anti, z2, zl, zr, ww, 1e-14, st)
    if st[0]:
        raise Breakdown(int(st[0]))
    y = rhs[None].copy()
    solve_w_batch(ww, y)
    x = np.zeros((1, n))
    zs = np.zeros(1, np.int64)
    tr = np.full((1, n), -1, np.int64)
    solve_z_batch(z2, zl, zr, y, x, 1, 1e-14, zs, tr)
    if zs[0]:
        raise Breakdown(int(zs[0]))
    return x[0, :n_int]


def residual(u, film_vals, c: LineCase, film: LineFilm, kappa, limiter):
    rho, eta, eps = rheology(u, c, film=film_vals)
    q = rho * film_vals
    n = u.size - 1
    h = film.h
    r = np.zeros_like(u)
    i = np.arange(1, n)
    e_p = 0.5 * (eps[i] + eps[i + 1])
    e_m = 0.5 * (eps[i] + eps[i - 1])
    fd, _, _ = faces(q, limiter, kappa)
    r[i] = (e_p * (u[i + 1] - u[i]) + e_m * (u[i - 1] - u[i])) / h - fd
    return r


def line_step(u, h0, outer, c: LineCase, film: LineFilm, kappa=1.0 / 3.0, limiter="kappa",
              variant="Lhs1", force_every=5):
    """One outer iteration of solve_ehl for the line contact.  Returns
    (u_new, h0_new, film_new, res, info)."""
    n = u.size - 1
    h = film.h
    omega = c.omega
    fv = h0 + film.geometry + film.deformation(u)
    rho, eta, eps = rheology(u, c, film=fv)
    i = np.arange(1, n)
    e_p = 0.5 * (eps[i] + eps[i + 1])
    e_m = 0.5 * (eps[i] + eps[i - 1])
    q = rho * fv
    fd, _, _ = faces(q, limiter, kappa)
    resid = (e_p * (u[i + 1] - u[i]) + e_m * (u[i - 1] - u[i])) / h - fd
    ns, ws = ("Ls1", "Ls4") if variant == "Lhs1" else ("Ls0", "Ls5")
    mat_n, rhs_n, _ = assemble(u, q, rho, e_p, e_m, resid, film, h, kappa, limiter, ns)
    mat_w, _, _ = assemble(u, q, rho, e_p, e_m, resid, film, h, kappa, limiter, ws)
    wmask = (eps[i] / h) <= SWITCH
    mat = mat_n.copy()
    cols = np.where(wmask)[0]
    mat[:, cols] = mat_w[:, cols]
    rung = "combined"
    try:
        sigma = solve_bands(mat, rhs_n, n - 1)
    except Breakdown:
        sigma = None
        for jac in ("scheme", "first-order", "diagonal"):
            b2, r2, _ = assemble(u, q, rho, e_p, e_m, resid, film, h, kappa, limiter, ws,
                                 jacobian=jac)
            try:
                sigma = solve_bands(b2, r2, n - 1)
                rung = jac
                break
            except Breakdown:
                continue
        if sigma is None:
            raise Breakdown(-1)
    sigma = np.clip(sigma, -c.max_change, c.max_change)
    full = np.zeros(n + 1)
    full[1:n] = sigma
    spread = np.zeros(n + 1)
    wsig = np.zeros(n + 1)
    wsig[1:n][wmask] = sigma[wmask]
    spread[1:] += wsig[:-1]
    spread[:-1] += wsig[1:]
    u_new = np.maximum(0.0, u + omega * (full - 0.25 * spread))
    u_new[0] = u_new[-1] = 0.0
    h0_new = h0
    applied = False
    if (outer + 1) % force_every == 0:
        deficit = c.load_target - h * float(np.sum(u_new))
        step = np.clip(c.relax_c * deficit, -c.max_h0_step, c.max_h0_step)
        h0_new = h0 - step
        applied = True
    film_new = h0_new + film.geometry + film.deformation(u_new)
    r = residual(u_new, film_new, c, film, kappa, limiter)
    res = float(np.max(np.abs(np.minimum(u_new, -r)))) / h
    return u_new, h0_new, film_new, res, dict(rung=rung, weighted=wmask, fb_applied=applied)


def hertz_start(c: LineCase, film: LineFilm):
    u = np.sqrt(np.maximum(0.0, 1.0 - film.x * film.x))
    u[0] = u[-1] = 0.0
    return u * (c.load_target / (np.pi / 2.0))
