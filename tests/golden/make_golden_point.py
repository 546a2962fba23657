"""Golden vectors for the point-contact outer iteration, produced by running
the REFERENCE (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_point.py

Configs 4/5 put x in [-4.5, 1.5] and y in [-3, 3]; the reference takes one
(lo, hi) for both axes (ehl/film.py:38,44-45, ehl/solver.py:59), so the
adapter of SURVEY.md 8(c) is applied: after _initial_state the geometry is
0.5*(gx^2+gy^2) with gy on [-3, 3] and u the Hertzian hemisphere there,
scaled by (3 pi/2)/(2 pi/3), boundary ring zeroed, deformation recomputed.
Kernel and h are unchanged (both axes have length 6).

Teacher forcing: from recorded states (u, h0) one
reference outer iteration (_hybrid_x_sweep, column_sweep, force balance
every 5th, complementarity residual) is run and stored, together with the
per-line Newton/weighted tags of the x-sweep.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from paqif.ehl import params as ref_params  # noqa: E402
from paqif.ehl import solver as ref_solver  # noqa: E402
from paqif.ehl import sweeps as ref_sweeps  # noqa: E402

KAPPA = 1.0 / 3.0
LO_Y = -3.0


def adapted_state(p, intervals):
    st = ref_solver._initial_state(p, intervals)
    film = st.film
    gx, gy0 = np.meshgrid(film.x, film.x)
    gy = gy0 - film.x[0] + LO_Y
    film.geometry = 0.5 * (gx ** 2 + gy ** 2)
    u = ref_params.hertzian_init(gx, gy)
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    u *= p.load_target / (2.0 * np.pi / 3.0)
    st.u = u
    film.deformation_full(u)
    return st


def one_step(p, intervals, u, h0, outer):
    st = adapted_state(p, intervals)
    st.u = u.copy()
    st.h0 = float(h0)
    st.film.deformation_full(st.u)
    tags = []
    orig = ref_solver.robust_line_solve

    def wrapped(*a, **k):
        tags.append(a[11])  # the scheme argument
        return orig(*a, **k)

    ref_solver.robust_line_solve = wrapped
    try:
        ref_solver._hybrid_x_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
    finally:
        ref_solver.robust_line_solve = orig
    u_x = st.u.copy()
    ref_sweeps.column_sweep(st, p, KAPPA, "kappa", p.omega)
    applied = 0
    if (outer + 1) % 5 == 0:
        ref_sweeps.force_balance_update(st, p)
        applied = 1
    res = st.complementarity_residual(p, KAPPA, "kappa")
    film = st.film.film_full(st.u, st.h0)
    newton = np.array([1 if t == "Ls1" else 0 for t in tags], dtype=np.int64)
    return dict(u_x=u_x, u_out=st.u.copy(), h0_out=np.float64(st.h0), film_out=film,
                res_out=np.float64(res), newton=newton, fb_applied=np.int64(applied))


def main():
    out = {}
    idx = 0
    for tag, m, intervals, ks, max_k in [("p32", 100.0, 32, [0, 1, 4, 10], 11),
                                         ("q64", 100.0, 64, [0, 2, 4], 5),
                                         ("h32", 1000.0, 32, [0, 3], 4)]:
        p = ref_params.EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5))
        st = adapted_state(p, intervals)
        states = {}
        hist = []
        for outer in range(max_k):
            if outer in ks:
                states[outer] = (st.u.copy(), st.h0)
            ref_solver._hybrid_x_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
            ref_sweeps.column_sweep(st, p, KAPPA, "kappa", p.omega)
            if (outer + 1) % 5 == 0:
                ref_sweeps.force_balance_update(st, p)
            hist.append(st.complementarity_residual(p, KAPPA, "kappa"))
        for k in ks:
            u, h0 = states[k]
            r = one_step(p, intervals, u, h0, k)
            key = f"e{idx}"
            out[f"{key}__tag"] = np.array(tag)
            out[f"{key}__meta"] = np.array([m, 10.0, intervals, k])
            out[f"{key}__p_hertz"] = np.float64(p.p_hertz)
            out[f"{key}__lam"] = np.float64(p.lam)
            out[f"{key}__u_in"] = u
            out[f"{key}__h0_in"] = np.float64(h0)
            for kk, v in r.items():
                out[f"{key}__{kk}"] = v
            print(tag, k, "newton lines", int(r["newton"].sum()), "/", r["newton"].size,
                  "res", float(r["res_out"]))
            idx += 1
        out[f"hist_{tag}"] = np.array(hist)
        if tag == "p32":
            out["init__u"] = adapted_state(p, intervals).u
    np.savez_compressed(os.path.join(HERE, "ehl_point.npz"), **out)
    print("size", os.path.getsize(os.path.join(HERE, "ehl_point.npz")))


if __name__ == "__main__":
    main()
