"""Golden vectors for the EHL Newton step, produced by running the REFERENCE
(build container only; /root/reference is absent on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_ehl.py

Teacher-forced single outer iterations (protocol P2): the
reference trajectory is recorded at several outer indices k; from each
recorded state (u, h0) exactly one reference outer iteration is run with the
reference's own functions (_line_contact_sweep, force_balance_update every
force_every-th iteration, EhlState.complementarity_residual) and its outputs
stored.  A short reference trajectory (protocol P3) is stored too.

Line parameters follow SURVEY.md 8(c): U, W = moes_convert(m=M, l=L,
g=5000); EhlParams.line_from_loads(5000, U, W, domain=(-4.5, 1.5)).
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
from paqif.errors import FactorizationBreakdownError  # noqa: E402

G_FIXED = 5000.0
KAPPA = 1.0 / 3.0


def line_params(m, l):
    u, w = ref_params.moes_convert(m=m, l=l, g=G_FIXED)
    return ref_params.EhlParams.line_from_loads(G_FIXED, u, w, domain=(-4.5, 1.5))


class Counter:
    """Counts breakdowns of the combined system inside _line_contact_sweep
    (wraps the name the solver module resolves)."""

    def __init__(self):
        self.breaks = 0
        self.orig = ref_solver._solve_line

    def __enter__(self):
        def wrapped(mat, rhs, n_int):
            try:
                return self.orig(mat, rhs, n_int)
            except FactorizationBreakdownError:
                self.breaks += 1
                raise
        ref_solver._solve_line = wrapped
        return self

    def __exit__(self, *a):
        ref_solver._solve_line = self.orig


def one_step(p, intervals, u, h0, outer, force_every=5):
    st = ref_solver._initial_state(p, intervals)
    st.u = u.copy()
    st.h0 = float(h0)
    st.film.deformation_full(st.u)
    with Counter() as c:
        ref_solver._line_contact_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
    applied = 0
    deficit = np.nan
    if (outer + 1) % force_every == 0:
        _, deficit = ref_sweeps.force_balance_update(st, p)
        applied = 1
    res = st.complementarity_residual(p, KAPPA, "kappa")
    film = st.film.film_full(st.u, st.h0)
    return dict(u_out=st.u.copy(), h0_out=np.float64(st.h0), film_out=film,
                res_out=np.float64(res), breaks=np.int64(c.breaks),
                fb_applied=np.int64(applied), deficit=np.float64(deficit))


def trajectory(p, intervals, ks, max_k):
    """Reference trajectory states (u, h0) at outer indices ks (state BEFORE
    iteration k), plus per-iteration residual history."""
    st = ref_solver._initial_state(p, intervals)
    states = {}
    hist = []
    for outer in range(max_k):
        if outer in ks:
            states[outer] = (st.u.copy(), st.h0)
        try:
            ref_solver._line_contact_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
        except Exception:
            break
        if (outer + 1) % 5 == 0:
            ref_sweeps.force_balance_update(st, p)
        hist.append(st.complementarity_residual(p, KAPPA, "kappa"))
    return states, np.array(hist)


def main():
    out = {}
    cases = []
    # config 1: M=20, L=10, N=513
    cases.append(("c1", 20.0, 10.0, 512, [0, 1, 4, 9, 30, 120, 400], 401))
    # config-3 style: N=1025, a spread of loads including breakdown-prone M
    for tag, m, l in [("m5", 5.0, 5.0), ("m20", 20.0, 10.0), ("m60", 60.0, 8.0),
                      ("m90", 90.0, 12.0), ("m150", 150.0, 15.0)]:
        cases.append((tag, m, l, 1024, [0, 2, 7, 25], 26))
    # small grid for fast CPU tests
    cases.append(("s1", 20.0, 10.0, 128, [0, 3, 9, 50], 51))
    idx = 0
    for tag, m, l, intervals, ks, max_k in cases:
        p = line_params(m, l)
        states, hist = trajectory(p, intervals, set(ks), max_k)
        for k in ks:
            if k not in states:
                continue
            u, h0 = states[k]
            r = one_step(p, intervals, u, h0, k)
            key = f"e{idx}"
            out[f"{key}__tag"] = np.array(tag)
            out[f"{key}__meta"] = np.array([m, l, intervals, k, G_FIXED])
            out[f"{key}__p_hertz"] = np.float64(p.p_hertz)
            out[f"{key}__lam"] = np.float64(p.lam)
            out[f"{key}__u_in"] = u
            out[f"{key}__h0_in"] = np.float64(h0)
            for kk, v in r.items():
                out[f"{key}__{kk}"] = v
            print(tag, k, "breaks", int(r["breaks"]), "res", float(r["res_out"]))
            idx += 1
        out[f"hist_{tag}"] = hist
    # short trajectory (protocol P3) on the small grid from the Hertzian start
    p = line_params(20.0, 10.0)
    st = ref_solver._initial_state(p, 128)
    traj_u, traj_h0, traj_res = [], [], []
    for outer in range(8):
        ref_solver._line_contact_sweep(st, p, KAPPA, "kappa", "Lhs1", p.omega)
        if (outer + 1) % 5 == 0:
            ref_sweeps.force_balance_update(st, p)
        traj_res.append(st.complementarity_residual(p, KAPPA, "kappa"))
        traj_u.append(st.u.copy())
        traj_h0.append(st.h0)
    out["traj__u"] = np.array(traj_u)
    out["traj__h0"] = np.array(traj_h0)
    out["traj__res"] = np.array(traj_res)
    np.savez_compressed(os.path.join(HERE, "ehl_line.npz"), **out)
    print("size", os.path.getsize(os.path.join(HERE, "ehl_line.npz")))


if __name__ == "__main__":
    main()
