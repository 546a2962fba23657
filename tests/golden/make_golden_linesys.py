"""Golden vectors for the per-line building blocks of paqif/ehl/sweeps.py --
assemble_line_system (all schemes and Jacobians), robust_line_solve and
reynolds_residual_field -- produced by running the REFERENCE (build
container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/make_golden_linesys.py

Point-contact lines come from recorded states of ehl_point.npz through the
reference's own _line_quantities (x-line j: films with pending corrections,
rheology, face mobilities, residual); line-contact lines from states of
ehl_line.npz with the same quantities the reference's _line_contact_sweep
forms (ey = 0); FilmModel pending-update sequences (note_line_update,
film_rows / film_cols, the fold past 8 pending).  Every case stores its
inputs, so the GPU test needs no reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden_point import KAPPA, adapted_state, ref_params, ref_solver, ref_sweeps  # noqa: E402

POINT_CASES = [
    # (name, point golden key, row j, limiter, scheme, jacobian)
    ("p_ls1_scheme", "e1", 16, "kappa", "Ls1", "scheme"),
    ("p_ls4_scheme", "e1", 16, "kappa", "Ls4", "scheme"),
    ("p_ls5_first", "e2", 12, "van-albada", "Ls5", "first-order"),
    ("p_ls0_diag", "e5", 20, "minmod", "Ls0", "diagonal"),
    ("p_ls1_koren", "e7", 9, "koren", "Ls1", "scheme"),
    ("p_ls4_none", "e8", 25, "none", "Ls4", "scheme"),
]
LINE_CASES = [
    # (name, line golden key, limiter, scheme, jacobian)
    ("l_ls1_scheme", "e0", "kappa", "Ls1", "scheme"),
    ("l_ls4_first", "e3", "kappa", "Ls4", "first-order"),
    ("l_ls5_diag", "e5", "minmod", "Ls5", "diagonal"),
]


def store(out, name, vals):
    for k, v in vals.items():
        out[f"{name}__{k}"] = np.asarray(v)


def main():
    GP = np.load(os.path.join(HERE, "ehl_point.npz"))
    GL = np.load(os.path.join(HERE, "ehl_line.npz"))
    out = {}
    for name, key, j, lim, scheme, jac in POINT_CASES:
        m, l, n, _ = GP[f"{key}__meta"]
        p = ref_params.EhlParams.point_from_moes(float(m), float(l), domain=(-4.5, 1.5))
        st = adapted_state(p, int(n))
        st.u = GP[f"{key}__u_in"].copy()
        st.h0 = float(GP[f"{key}__h0_in"])
        st.film.deformation_full(st.u)
        q = ref_sweeps._line_quantities(st, p, j, KAPPA, lim)
        u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, _, h = q
        mat, rhs = ref_sweeps.assemble_line_system(u_line, q_line, rho_line, ex_p, ex_m, ey_p,
                                                   ey_m, resid, p, KAPPA, lim, scheme, st.film,
                                                   h, jacobian=jac)
        sigma = ref_sweeps.robust_line_solve(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m,
                                             resid, p, KAPPA, lim, scheme, st.film, h)
        film = st.film.film_full(st.u, st.h0)
        field = ref_sweeps.reynolds_residual_field(st.u, film, p, KAPPA, lim)
        store(out, name, dict(contact="point", src=key, limiter=lim, scheme=scheme, jac=jac,
                              h=h, u_line=u_line, q_line=q_line, rho_line=rho_line, ex_p=ex_p,
                              ex_m=ex_m, ey_p=ey_p, ey_m=ey_m, resid=resid, bands=mat.bands,
                              rhs=rhs, sigma=sigma, u=st.u, film=film, field=field))
    for name, key, lim, scheme, jac in LINE_CASES:
        m, l, n = GL[f"{key}__meta"][:3]
        U, W = ref_params.moes_convert(m=float(m), l=float(l), g=5000.0)
        p = ref_params.EhlParams.line_from_loads(5000.0, U, W, domain=(-4.5, 1.5))
        st = ref_solver._initial_state(p, int(n))
        st.u = GL[f"{key}__u_in"].copy()
        st.h0 = float(GL[f"{key}__h0_in"])
        film = st.film.film_full(st.u, st.h0)
        rho, _, eps = ref_params.rheology(st.u, p, film=film)
        nn = st.u.size - 1
        h = ref_sweeps.grid_spacing(p, nn)
        i = np.arange(1, nn)
        ex_p = 0.5 * (eps[i] + eps[i + 1])
        ex_m = 0.5 * (eps[i] + eps[i - 1])
        zeros = np.zeros(nn - 1)
        field = ref_sweeps.reynolds_residual_field(st.u, film, p, KAPPA, lim)
        resid = field[1:nn]
        q_line = rho * film
        mat, rhs = ref_sweeps.assemble_line_system(st.u, q_line, rho, ex_p, ex_m, zeros, zeros,
                                                   resid, p, KAPPA, lim, scheme, st.film, h,
                                                   jacobian=jac)
        sigma = ref_sweeps.robust_line_solve(st.u, q_line, rho, ex_p, ex_m, zeros, zeros, resid,
                                             p, KAPPA, lim, scheme, st.film, h)
        store(out, name, dict(contact="line", src=key, limiter=lim, scheme=scheme, jac=jac, h=h,
                              u_line=st.u, q_line=q_line, rho_line=rho, ex_p=ex_p, ex_m=ex_m,
                              ey_p=zeros, ey_m=zeros, resid=resid, bands=mat.bands, rhs=rhs,
                              sigma=sigma, u=st.u, film=film, field=field))
    # FilmModel pending line updates: note rows / columns, read films of
    # rows and columns with the exact corrections, then past the fold limit
    rng = np.random.default_rng(5)
    for name, key in (("f_e1", "e1"), ("f_e5", "e5")):
        m, l, n, _ = GP[f"{key}__meta"]
        n = int(n)
        p = ref_params.EhlParams.point_from_moes(float(m), float(l), domain=(-4.5, 1.5))
        st = adapted_state(p, n)
        u = GP[f"{key}__u_in"].copy()
        h0 = float(GP[f"{key}__h0_in"])
        fm = st.film
        fm.deformation_full(u)
        notes, reads = [], []
        plan = [("row", n // 2), ("row", n // 2 + 1), ("col", n // 3), ("row", 3),
                ("col", n - 2)]
        for axis, idx in plan:
            delta = np.zeros(n + 1)
            delta[1:n] = 1e-2 * rng.standard_normal(n - 1)
            fm.note_line_update(axis, idx, delta, u)
            notes.append((0 if axis == "row" else 1, idx, delta))
        rows = [n // 2 - 1, n // 2, n // 2 + 1, 7]
        cols = [n // 3 - 1, n // 3, n - 2]
        reads.append((0, rows, fm.film_rows(rows, h0)))
        reads.append((1, cols, fm.film_cols(cols, h0)))
        zero = np.zeros(n + 1)
        fm.note_line_update("row", 5, zero, u)  # ignored
        for k in range(5):  # past the fold limit (9 > 8 folds)
            delta = np.zeros(n + 1)
            delta[1:n] = 1e-2 * rng.standard_normal(n - 1)
            fm.note_line_update("row", 10 + k, delta, u)
            notes.append((0, 10 + k, delta))
        reads.append((0, rows, fm.film_rows(rows, h0)))
        out[f"{name}__src"] = np.array(key)
        out[f"{name}__u"] = u
        out[f"{name}__h0"] = np.array(h0)
        out[f"{name}__note_axis"] = np.array([a for a, _, _ in notes])
        out[f"{name}__note_idx"] = np.array([i for _, i, _ in notes])
        out[f"{name}__note_delta"] = np.stack([d for _, _, d in notes])
        for q, (mode, idx, val) in enumerate(reads):
            out[f"{name}__read{q}_mode"] = np.array(mode)
            out[f"{name}__read{q}_idx"] = np.array(idx)
            out[f"{name}__read{q}_val"] = val
    np.savez_compressed(os.path.join(HERE, "ehl_linesys.npz"), **out)
    print("wrote", len(POINT_CASES) + len(LINE_CASES), "cases")


if __name__ == "__main__":
    main()
