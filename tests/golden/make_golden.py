"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Outputs (committed, small):
  tests/golden/aqif_kernels.npz   _kernels.factor_batch / solve_w_batch /
                                  solve_z_batch / band_matvec_batch outputs
  tests/golden/lcp.npz            paqif_solve_lcp(r=1) on seeded systems
  tests/golden/paqif_r.npz        paqif_solve(L, f, r) for r in {1,2,4,8}
  tests/golden/paqif_proj.npz     paqif_solve(L, f, r, project=True)
The EHL goldens are produced by make_golden_ehl.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from paqif import _kernels  # noqa: E402  (the reference)
from paqif.bandcore import BandedMatrix  # noqa: E402
from paqif.lcp import LcpProblem, psor_oracle  # noqa: E402
from paqif.parallel import paqif_solve, paqif_solve_lcp  # noqa: E402
import paqif.parallel as ref_parallel  # noqa: E402

from paper_2008_03276_b200.workloads import lcp_system, random_banded  # noqa: E402


def run_kernels(bands, rhs, start, tol=1e-14):
    """Run the reference kernels on a batch of one and return every output."""
    n = bands.shape[1]
    beta = (bands.shape[0] - 1) // 2
    s = n // 2
    band = bands[None].copy()
    anti = np.zeros_like(band)
    z2x2 = np.zeros((1, s + 1, 2, 2))
    zl = np.zeros((1, s + 1, 2, beta + 1))
    zr = np.zeros((1, s + 1, 2, beta + 1))
    ww = np.zeros((1, s + 1, 2 * beta, 2))
    status = np.zeros(1, dtype=np.int64)
    _kernels.factor_batch(band, anti, z2x2, zl, zr, ww, tol, status)
    y = rhs[None].copy()
    _kernels.solve_w_batch(ww, y)
    x = np.zeros((1, n))
    if start > 1:
        p = start - 1
        x[0, :p] = 0.25 * rhs[:p]
        x[0, n - p:] = 0.25 * rhs[n - p:]
    x_in = x.copy()
    zstatus = np.zeros(1, dtype=np.int64)
    trace = np.full((1, n), -1, dtype=np.int64)
    _kernels.solve_z_batch(z2x2, zl, zr, y, x, start, tol, zstatus, trace)
    mv = np.zeros((1, n))
    _kernels.band_matvec_batch(bands[None], rhs[None], mv)
    return dict(bands=bands, rhs=rhs, start=np.int64(start), band_out=band[0],
                anti_out=anti[0], z2x2=z2x2[0], zl=zl[0], zr=zr[0], ww=ww[0],
                status=status[0], y=y[0], x_in=x_in[0], x=x[0], zstatus=zstatus[0],
                trace=trace[0], matvec=mv[0])


def aqif_cases():
    rng = np.random.default_rng(20240817)
    cases = {}
    k = 0
    for n, beta in [(8, 1), (16, 2), (32, 3), (64, 2), (40, 4), (64, 8), (130, 8),
                    (34, 5), (36, 6), (46, 7), (512, 2), (66, 16)]:
        bands = random_banded(n, beta, rng)
        rhs = rng.standard_normal(n)
        cases[f"c{k}"] = run_kernels(bands, rhs, 1)
        k += 1
    # middle solve (start > 1), M-matrix, non-dominant (may break down)
    for n, beta, start in [(24, 2, 3), (64, 8, 9), (130, 8, 9)]:
        bands = random_banded(n, beta, rng)
        rhs = rng.standard_normal(n)
        cases[f"c{k}"] = run_kernels(bands, rhs, start)
        k += 1
    bands = random_banded(64, 3, rng, m_matrix=True)
    cases[f"c{k}"] = run_kernels(bands, rng.standard_normal(64), 1); k += 1
    for _ in range(6):
        bands = random_banded(32, 2, rng, dominant=False)
        cases[f"c{k}"] = run_kernels(bands, rng.standard_normal(32), 1); k += 1
    # exact breakdowns: zero matrix, identity, tiny order 2, pinned rows
    cases[f"c{k}"] = run_kernels(np.zeros((3, 8)), rng.standard_normal(8), 1); k += 1
    eye = np.zeros((5, 12)); eye[2] = 1.0
    cases[f"c{k}"] = run_kernels(eye, rng.standard_normal(12), 1); k += 1
    two = np.zeros((3, 2)); two[1] = [3.0, 4.0]; two[2, 0] = 1.0; two[0, 1] = 2.0
    cases[f"c{k}"] = run_kernels(two, np.array([1.0, 2.0]), 1); k += 1
    # singular middle 2x2 at level 3: rows built so det vanishes mid-way
    sing = random_banded(16, 1, rng)
    sing[1, 5] = 1.0; sing[2, 5] = 1.0; sing[0, 6] = 1.0; sing[1, 10] = 1.0
    sing[1, 6] = 1.0; sing[2, 6] = 1.0; sing[1, 9] = 1.0; sing[0, 10] = 1.0
    cases[f"c{k}"] = run_kernels(sing, rng.standard_normal(16), 1); k += 1
    # pinned rows (LCP style): rows zeroed except the diagonal
    pin = random_banded(130, 8, rng)
    mask = rng.random(130) < 0.5
    d = pin[8, mask].copy()
    pin[:, mask] = 0.0
    pin[8, mask] = d
    f = rng.standard_normal(130); f[mask] = 0.0
    cases[f"c{k}"] = run_kernels(pin, f, 1); k += 1
    # near-threshold determinant: scale a 2x2 pivot to sit near 1e-14
    near = np.zeros((3, 4)); near[1] = [1.0, 1.0, 1.0, 1.0]
    near[2, 1] = 1.0; near[0, 2] = 1.0 - 2e-14
    cases[f"c{k}"] = run_kernels(near, np.ones(4), 1); k += 1
    near2 = near.copy(); near2[0, 2] = 1.0 - 5e-15
    cases[f"c{k}"] = run_kernels(near2, np.ones(4), 1); k += 1
    return cases


def flatten(cases):
    out = {}
    for name, d in cases.items():
        for key, val in d.items():
            out[f"{name}__{key}"] = np.asarray(val)
    return out


def lcp_cases():
    """paqif_solve_lcp(r=1) on config-2-style systems (small n and full n)
    plus the reference tests' obstacle problems; records passes via a
    module-attribute wrapper around paqif_solve."""
    out = {}
    calls = [0]
    orig = ref_parallel.paqif_solve

    def counted(*a, **k):
        calls[0] += 1
        return orig(*a, **k)

    ref_parallel.paqif_solve = counted
    try:
        specs = [(7, b, 65, 8) for b in range(12)] + [(7, b, 129, 4) for b in range(4)] \
            + [(11, b, 1025, 8) for b in range(3)] + [(13, b, 33, 2) for b in range(4)]
        for k, (seed, b, n, beta) in enumerate(specs):
            bands, f = lcp_system(seed, b, n, beta)
            calls[0] = 0
            u = paqif_solve_lcp(LcpProblem(BandedMatrix(bands.shape[1], beta, bands), f), 1,
                                tol=1e-10)
            psor = psor_oracle(LcpProblem(BandedMatrix(bands.shape[1], beta, bands), f),
                               omega=1.0, tol=1e-14)
            out[f"l{k}__bands"] = bands
            out[f"l{k}__f"] = f
            out[f"l{k}__u"] = u
            out[f"l{k}__passes"] = np.int64(calls[0])
            out[f"l{k}__psor"] = psor
            out[f"l{k}__meta"] = np.array([seed, b, n, beta], dtype=np.int64)
        # obstacle_1d(64), the reference test problem (tests/test_parallel.py:16-21)
        n = 64
        h = 1.0 / (n + 1)
        bands = np.zeros((3, n)); bands[0, 1:] = -1.0 / h**2; bands[1] = 2.0 / h**2
        bands[2, :-1] = -1.0 / h**2
        x = np.linspace(h, 1 - h, n)
        f = 50.0 * np.sin(2 * np.pi * x)
        calls[0] = 0
        u = paqif_solve_lcp(LcpProblem(BandedMatrix(n, 1, bands), f), 1, tol=1e-10)
        k = len(specs)
        out[f"l{k}__bands"] = bands; out[f"l{k}__f"] = f; out[f"l{k}__u"] = u
        out[f"l{k}__passes"] = np.int64(calls[0])
        out[f"l{k}__psor"] = psor_oracle(LcpProblem(BandedMatrix(n, 1, bands), f), omega=1.7,
                                         tol=1e-13)
        out[f"l{k}__meta"] = np.array([-1, -1, n, 1], dtype=np.int64)
    finally:
        ref_parallel.paqif_solve = orig
    return out


def paqif_r_cases():
    rng = np.random.default_rng(99)
    out = {}
    k = 0
    for n, beta in [(64, 2), (128, 3), (512, 2), (256, 8)]:
        bands = random_banded(n, beta, rng)
        f = rng.standard_normal(n)
        for r in (1, 2, 4, 8):
            t = n // r
            if n % r or t % 2 or t <= 2 * beta:
                continue
            u = paqif_solve(BandedMatrix(n, beta, bands), f, r)
            out[f"p{k}__bands"] = bands; out[f"p{k}__f"] = f; out[f"p{k}__u"] = u
            out[f"p{k}__r"] = np.int64(r)
            k += 1
    return out


def paqif_project_cases():
    """paqif_solve(L, f, r, project=True): corners projected before the
    middles' Z solve, middles projected (parallel.py:278-289)."""
    rng = np.random.default_rng(7)
    out = {}
    k = 0
    for n, beta, r in [(128, 2, 4), (96, 3, 4), (256, 8, 8), (64, 1, 8), (160, 5, 2)]:
        for _ in range(2):
            bands = random_banded(n, beta, rng)
            f = rng.standard_normal(n)
            u = paqif_solve(BandedMatrix(n, beta, bands), f, r, project=True)
            out[f"p{k}__bands"] = bands; out[f"p{k}__f"] = f; out[f"p{k}__u"] = u
            out[f"p{k}__r"] = np.int64(r)
            k += 1
    return out


def main():
    if "--project-only" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "paqif_proj.npz"), **paqif_project_cases())
        return
    np.savez_compressed(os.path.join(HERE, "paqif_proj.npz"), **paqif_project_cases())
    np.savez_compressed(os.path.join(HERE, "aqif_kernels.npz"), **flatten(aqif_cases()))
    np.savez_compressed(os.path.join(HERE, "lcp.npz"), **lcp_cases())
    np.savez_compressed(os.path.join(HERE, "paqif_r.npz"), **paqif_r_cases())
    for f in ("aqif_kernels.npz", "lcp.npz", "paqif_r.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
