"""Golden vectors for the public point-contact sweep functions, produced by
running the REFERENCE (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_point_sweeps.py

From recorded states of ehl_point.npz (same adapter as make_golden_point.py)
each case runs ONE reference call -- newton_line_sweep (fixed scheme or
hybrid), weighted_change_sweep, column_sweep, EhlState.complementarity_residual
-- and stores the new pressure and the returned value.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden_point import KAPPA, adapted_state, ref_params, ref_sweeps  # noqa: E402

CASES = [
    # (name, source golden key, call, kwargs)
    ("newton_ls1", "e1", "newton", dict(limiter="kappa", scheme="Ls1")),
    ("newton_lhs2", "e1", "newton", dict(limiter="kappa", hybrid="Lhs2")),
    ("newton_ls4_va", "e2", "newton", dict(limiter="van-albada", scheme="Ls4")),
    ("weighted_ls5", "e1", "weighted", dict(limiter="kappa", scheme="Ls5")),
    ("weighted_ls4_minmod", "e5", "weighted", dict(limiter="minmod", scheme="Ls4")),
    ("column_kappa", "e1", "column", dict(limiter="kappa")),
    ("column_koren", "e7", "column", dict(limiter="koren")),
    ("residual_none", "e2", "residual", dict(limiter="none")),
    ("residual_koren", "e8", "residual", dict(limiter="koren")),
]


def main():
    G = np.load(os.path.join(HERE, "ehl_point.npz"))
    out = {}
    for name, key, call, kw in CASES:
        m, l, n, _ = G[f"{key}__meta"]
        p = ref_params.EhlParams.point_from_moes(float(m), float(l), domain=(-4.5, 1.5))
        st = adapted_state(p, int(n))
        st.u = G[f"{key}__u_in"].copy()
        st.h0 = float(G[f"{key}__h0_in"])
        st.film.deformation_full(st.u)
        lim = kw.pop("limiter")
        if call == "newton":
            val = ref_sweeps.newton_line_sweep(st, p, KAPPA, lim, **kw)
        elif call == "weighted":
            val = ref_sweeps.weighted_change_sweep(st, p, KAPPA, lim, **kw)
        elif call == "column":
            val = ref_sweeps.column_sweep(st, p, KAPPA, lim)
        else:
            val = st.complementarity_residual(p, KAPPA, lim)
        out[f"{name}__src"] = np.array(key)
        out[f"{name}__call"] = np.array(call)
        out[f"{name}__limiter"] = np.array(lim)
        out[f"{name}__scheme"] = np.array(kw.get("scheme", ""))
        out[f"{name}__hybrid"] = np.array(kw.get("hybrid", ""))
        out[f"{name}__u_out"] = st.u.copy()
        out[f"{name}__value"] = np.float64(val)
        print(name, call, float(val))
    np.savez_compressed(os.path.join(HERE, "ehl_point_sweeps.npz"), **out)
    print("size", os.path.getsize(os.path.join(HERE, "ehl_point_sweeps.npz")))


if __name__ == "__main__":
    main()
