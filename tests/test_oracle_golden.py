"""The CPU oracle (oracle/) pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

import oracle as O
from conftest import cavitated, golden_cases


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def run_oracle_kernels(G):
    bands = G["bands"]
    n = bands.shape[1]
    beta = (bands.shape[0] - 1) // 2
    s = n // 2
    band = bands[None].copy()
    anti = np.zeros_like(band)
    z2 = np.zeros((1, s + 1, 2, 2))
    zl = np.zeros((1, s + 1, 2, beta + 1))
    zr = np.zeros_like(zl)
    ww = np.zeros((1, s + 1, 2 * beta, 2))
    st = np.zeros(1, np.int64)
    O.factor_batch(band, anti, z2, zl, zr, ww, 1e-14, st)
    y = G["rhs"][None].copy()
    O.solve_w_batch(ww, y)
    x = G["x_in"][None].copy()
    zs = np.zeros(1, np.int64)
    tr = np.full((1, n), -1, np.int64)
    O.solve_z_batch(z2, zl, zr, y, x, int(G["start"]), 1e-14, zs, tr)
    mv = np.zeros((1, n))
    O.band_matvec_batch(bands[None].copy(), G["rhs"][None].copy(), mv)
    return dict(band_out=band[0], anti_out=anti[0], z2x2=z2[0], zl=zl[0], zr=zr[0], ww=ww[0],
                status=st[0], y=y[0], x=x[0], zstatus=zs[0], trace=tr[0], matvec=mv[0])


@pytest.mark.parametrize("case", range(len(golden_cases("aqif_kernels.npz"))))
def test_aqif_kernels_bit_exact(case):
    G = golden_cases("aqif_kernels.npz")[case]
    out = run_oracle_kernels(G)
    for k, v in out.items():
        assert np.array_equal(_bits(v), _bits(G[k])), k


def test_golden_covers_breakdowns():
    st = [int(G["status"]) for G in golden_cases("aqif_kernels.npz")]
    assert any(s > 0 for s in st) and any(s == 0 for s in st)


@pytest.mark.parametrize("case", range(len(golden_cases("lcp.npz"))))
def test_lcp_matches_reference(case):
    G = golden_cases("lcp.npz")[case]
    u, act, passes, res, st = O.lcp_batch(G["bands"][None], G["f"][None])
    assert st[0] == 0
    assert passes[0] == int(G["passes"])
    ref = G["u"]
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(u[0] - ref)) <= 1e-13 * scale
    assert np.array_equal(cavitated(u[0]), cavitated(ref))
    # final pinned set agrees with the cavitated set of the reference answer
    assert np.array_equal(act[0] | (u[0] == 0), cavitated(ref))
    assert np.max(np.abs(u[0] - G["psor"])) <= 1e-8 * scale


def test_lcp_threads_deterministic():
    from paper_2008_03276_b200.workloads import lcp_batch
    bands, f = lcp_batch(3, 6, n=129, beta=8)
    a = O.lcp_batch(bands, f, threads=1)
    b = O.lcp_batch(bands, f, threads=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_psor_oracle_matches_golden():
    G = golden_cases("lcp.npz")[0]
    u, sweeps, ch = O.psor(G["bands"], G["f"], omega=1.0, tol=1e-14)
    assert np.array_equal(_bits(u), _bits(G["psor"]))
