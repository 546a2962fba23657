"""Line contacts finer than one CTA's shared memory holds (N > 2049; the
reference has no size limit, ehl/solver.py:131-183), produced by running the
REFERENCE (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_line_big.py

-> tests/golden/ehl_line_big.npz: teacher-forced single outer iterations
(same protocol and fields as make_golden_ehl.py) at n = 4096 and 8192
intervals, from the Hertzian start and from the reference's own state a
few iterations later, with a load that breaks the combined system.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden_ehl import G_FIXED, line_params, one_step, trajectory  # noqa: E402


def main():
    out = {}
    idx = 0
    for tag, m, l, intervals, ks, max_k in [("b4k", 20.0, 10.0, 4096, [0, 3], 4),
                                            ("b4h", 90.0, 12.0, 4096, [0, 2, 6], 7),
                                            ("b8k", 60.0, 8.0, 8192, [0, 2], 3)]:
        p = line_params(m, l)
        states, _ = trajectory(p, intervals, set(ks), max_k)
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
            print(tag, k, "breaks", int(r["breaks"]), "res", float(r["res_out"]), flush=True)
            idx += 1
    path = os.path.join(HERE, "ehl_line_big.npz")
    np.savez_compressed(path, **out)
    print("size", os.path.getsize(path))


if __name__ == "__main__":
    main()
