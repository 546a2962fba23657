"""Reference goldens for the point contact AT THE CONFIGURED GRIDS
(configs 4 and 5), produced by running the REFERENCE (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_point_big.py [c4] [c5]

c4 -> tests/golden/ehl_point_c4.npz: 513^2 (512 intervals), M=100, L=10.
      Teacher-forced single outer iterations from the adapted Hertz start
      (k=0) and from the reference's own state after 2 iterations (k=2).
      Full fields: u_in, u_x (after the x-sweep), u_out, film_out; the
      x-sweep's Newton tags and ladder rungs, the y-sweep's rungs, h0, the
      residual.  ~11 s per reference iteration here.
c5 -> tests/golden/ehl_point_c5.npz: 2049^2 (2048 intervals), M=1000, L=10,
      one outer iteration from the adapted Hertz start (~11-15 min here).
      A digest, not the 34 MB fields: the packed cavitated bitmap of u_out,
      tags and rungs, h0, residual, per-row max and L1 of u_out / film_out /
      u_x, 8 full rows and 8 full columns of u_out and film_out, and a digest
      of the start state (per-row L1 + the same rows) so the GPU test can
      confirm it starts from the same bits.

Same adapter as make_golden_point.py (y in [-3, 3]).
Rungs are recorded by wrapping the reference's own functions (no source
edits): the x-lines' jacobian rung is the last ``assemble_line_system``
jacobian that ``robust_line_solve`` tried; a column's rung is 1 when its
first ``_solve_line`` raised (the diagonal fallback, sweeps.py:501-508).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden_point import KAPPA, adapted_state, ref_params, ref_solver, ref_sweeps  # noqa: E402

RUNG = {"scheme": 0, "first-order": 1, "diagonal": 2}
DIGEST_ROWS = None  # set per grid


def one_step_traced(p, intervals, u, h0, outer):
    st = adapted_state(p, intervals)
    st.u = u.copy()
    st.h0 = float(h0)
    st.film.deformation_full(st.u)
    tags, x_rungs, y_rungs, jacs = [], [], [], []
    o_rls, o_asm, o_sl = ref_solver.robust_line_solve, ref_sweeps.assemble_line_system, \
        ref_sweeps._solve_line

    def asm(*a, **k):
        jacs.append(k.get("jacobian", "scheme"))
        return o_asm(*a, **k)

    def rls(*a, **k):
        jacs.clear()
        tags.append(a[11])
        r = o_rls(*a, **k)
        x_rungs.append(RUNG[jacs[-1]])
        return r

    col_calls = []

    def sl(*a, **k):
        try:
            r = o_sl(*a, **k)
        except Exception:
            col_calls.append(0)
            raise
        col_calls.append(1)
        return r

    ref_solver.robust_line_solve = rls
    ref_sweeps.assemble_line_system = asm
    try:
        ref_solver._hybrid_x_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
    finally:
        ref_solver.robust_line_solve = o_rls
        ref_sweeps.assemble_line_system = o_asm
    u_x = st.u.copy()
    ref_sweeps._solve_line = sl
    try:
        ref_sweeps.column_sweep(st, p, KAPPA, "kappa", p.omega)
    finally:
        ref_sweeps._solve_line = o_sl
    # each column: [ok] -> rung 0, [fail, ok] -> rung 1
    i = 0
    while i < len(col_calls):
        if col_calls[i] == 1:
            y_rungs.append(0)
            i += 1
        else:
            y_rungs.append(1)
            i += 2
    applied = 0
    if (outer + 1) % 5 == 0:
        ref_sweeps.force_balance_update(st, p)
        applied = 1
    res = st.complementarity_residual(p, KAPPA, "kappa")
    film = st.film.film_full(st.u, st.h0)
    newton = np.array([1 if t == "Ls1" else 0 for t in tags], dtype=np.int64)
    return dict(u_x=u_x, u_out=st.u.copy(), h0_out=np.float64(st.h0), film_out=film,
                res_out=np.float64(res), newton=newton, x_rungs=np.array(x_rungs, np.int64),
                y_rungs=np.array(y_rungs, np.int64), fb_applied=np.int64(applied))


def config4():
    intervals, m = 512, 100.0
    p = ref_params.EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5))
    st = adapted_state(p, intervals)
    out = {}
    states = {0: (st.u.copy(), st.h0)}
    for outer in range(2):
        ref_solver._hybrid_x_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
        ref_sweeps.column_sweep(st, p, KAPPA, "kappa", p.omega)
        if (outer + 1) % 5 == 0:
            ref_sweeps.force_balance_update(st, p)
    states[2] = (st.u.copy(), st.h0)
    for idx, k in enumerate((0, 2)):
        u, h0 = states[k]
        t0 = time.time()
        r = one_step_traced(p, intervals, u, h0, k)
        key = f"e{idx}"
        out[f"{key}__meta"] = np.array([m, 10.0, intervals, k])
        out[f"{key}__p_hertz"] = np.float64(p.p_hertz)
        out[f"{key}__lam"] = np.float64(p.lam)
        out[f"{key}__u_in"] = u
        out[f"{key}__h0_in"] = np.float64(h0)
        for kk, v in r.items():
            out[f"{key}__{kk}"] = v
        print("c4 k", k, "newton", int(r["newton"].sum()), "/", r["newton"].size,
              "x rungs", np.bincount(r["x_rungs"]).tolist(), "y rungs",
              np.bincount(r["y_rungs"]).tolist(), "res", float(r["res_out"]),
              f"{time.time() - t0:.1f}s", flush=True)
    path = os.path.join(HERE, "ehl_point_c4.npz")
    np.savez_compressed(path, **out)
    print("c4 size", os.path.getsize(path))


def digest_rows(n1):
    return np.array(sorted({1, n1 // 8, n1 // 3, (2 * n1) // 5, n1 // 2, (3 * n1) // 5,
                            (3 * n1) // 4, n1 - 2}), dtype=np.int64)


def config5():
    intervals, m = 2048, 1000.0
    p = ref_params.EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5))
    st = adapted_state(p, intervals)
    u_in, h0 = st.u.copy(), st.h0
    rows = digest_rows(intervals + 1)
    t0 = time.time()
    r = one_step_traced(p, intervals, u_in, h0, 0)
    print("c5 newton", int(r["newton"].sum()), "/", r["newton"].size, "x rungs",
          np.bincount(r["x_rungs"]).tolist(), "y rungs", np.bincount(r["y_rungs"]).tolist(),
          "res", float(r["res_out"]), f"{time.time() - t0:.1f}s", flush=True)
    u, film, ux = r["u_out"], r["film_out"], r["u_x"]
    out = {
        "meta": np.array([m, 10.0, intervals, 0]), "p_hertz": np.float64(p.p_hertz),
        "lam": np.float64(p.lam), "h0_in": np.float64(h0), "digest_rows": rows,
        "in_row_l1": np.abs(u_in).sum(axis=1), "in_rows": u_in[rows], "in_cols": u_in[:, rows].T,
        "cav_bits": np.packbits((u == 0.0).ravel()), "shape": np.array(u.shape),
        "newton": r["newton"], "x_rungs": r["x_rungs"], "y_rungs": r["y_rungs"],
        "h0_out": r["h0_out"], "res_out": r["res_out"], "fb_applied": r["fb_applied"],
        "u_row_max": np.abs(u).max(axis=1), "u_row_l1": np.abs(u).sum(axis=1),
        "film_row_max": np.abs(film).max(axis=1), "film_row_l1": np.abs(film).sum(axis=1),
        "ux_row_max": np.abs(ux).max(axis=1), "ux_row_l1": np.abs(ux).sum(axis=1),
        "u_rows": u[rows], "u_cols": u[:, rows].T, "film_rows": film[rows],
        "film_cols": film[:, rows].T,
    }
    path = os.path.join(HERE, "ehl_point_c5.npz")
    np.savez_compressed(path, **out)
    print("c5 size", os.path.getsize(path))


def films513():
    """FilmModel pending line updates at 513^2 (the multi-segment films
    path): from the c4 golden's k=2 state, note 8 row / column deltas, read
    the films of rows and columns (8 exact corrections each), note a 9th
    (past the fold limit: full deformation), read again."""
    g = np.load(os.path.join(HERE, "ehl_point_c4.npz"))
    n = 512
    p = ref_params.EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5))
    st = adapted_state(p, n)
    u = g["e1__u_in"].copy()
    h0 = float(g["e1__h0_in"])
    fm = st.film
    fm.deformation_full(u)
    rng = np.random.default_rng(513)
    plan = [("row", 256), ("col", 200), ("row", 257), ("row", 100), ("col", 201), ("col", 450),
            ("row", 400), ("col", 3)]
    notes, reads = [], []
    for axis, idx in plan:
        delta = np.zeros(n + 1)
        delta[1:n] = 1e-2 * rng.standard_normal(n - 1)
        fm.note_line_update(axis, idx, delta, u)
        notes.append((0 if axis == "row" else 1, idx, delta))
    rows = [255, 256, 257, 99, 100, 401, 1]
    cols = [199, 200, 201, 202, 449, 2]
    reads.append((0, rows, fm.film_rows(rows, h0)))
    reads.append((1, cols, fm.film_cols(cols, h0)))
    delta = np.zeros(n + 1)
    delta[1:n] = 1e-2 * rng.standard_normal(n - 1)
    fm.note_line_update("row", 300, delta, u)  # 9 pending > 8: folded
    notes.append((0, 300, delta))
    reads.append((0, rows, fm.film_rows(rows, h0)))
    reads.append((1, cols, fm.film_cols(cols, h0)))
    out = {"h0": np.float64(h0), "note_axis": np.array([a for a, _, _ in notes]),
           "note_idx": np.array([i for _, i, _ in notes]),
           "note_delta": np.stack([d for _, _, d in notes])}
    for q, (mode, idx, val) in enumerate(reads):
        out[f"read{q}_mode"] = np.array(mode)
        out[f"read{q}_idx"] = np.array(idx)
        out[f"read{q}_val"] = val
    path = os.path.join(HERE, "ehl_point_films513.npz")
    np.savez_compressed(path, **out)
    print("films513 size", os.path.getsize(path))


if __name__ == "__main__":
    which = sys.argv[1:] or ["c4", "c5", "films"]
    if "films" in which:
        films513()
    if "c4" in which:
        config4()
    if "c5" in which:
        config5()
