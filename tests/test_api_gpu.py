"""The reference's own test families (tests/test_aqif.py, test_parallel.py,
test_lcp.py PSOR parts) run against this package's API on the GPU, plus the
r-block PAQIF goldens produced by the reference."""

import numpy as np
import pytest

from conftest import cavitated, golden_cases

pytestmark = pytest.mark.gpu


def rb(n, beta, rng, **kw):
    from paper_2008_03276_b200.bandcore import BandedMatrix
    from paper_2008_03276_b200.workloads import random_banded
    return BandedMatrix(n, beta, random_banded(n, beta, rng, **kw))


def w_pattern_ok(w):
    n = w.shape[0]
    half = n // 2
    for j1 in range(1, half + 1):
        for i1 in range(j1 + 1, n - j1 + 2):
            if i1 != j1 and w[i1 - 1, j1 - 1] != 0.0:
                return False
    for j1 in range(n + 1 - half, n + 1):
        for i1 in range(n - j1 + 1, j1):
            if i1 != j1 and w[i1 - 1, j1 - 1] != 0.0:
                return False
    return np.allclose(np.diag(w), 1.0)


def z_pattern_ok(z):
    n = z.shape[0]
    half = n // 2
    for i1 in range(1, (n - 1) // 2 + 1):
        for j1 in range(i1 + 1, n - i1 + 1):
            if z[i1 - 1, j1 - 1] != 0.0:
                return False
    for i1 in range(n + 1 - half, n + 1):
        for j1 in range(n - i1 + 2, i1):
            if z[i1 - 1, j1 - 1] != 0.0:
                return False
    return True


class TestAqif:
    def test_identity_and_order_two(self):
        from paper_2008_03276_b200 import BandedMatrix, factorize_wz
        f = factorize_wz(BandedMatrix.identity(4))
        assert np.array_equal(f.w_dense(), np.eye(4)) and np.array_equal(f.z_dense(), np.eye(4))
        l = BandedMatrix.from_dense(np.array([[3.0, 1.0], [2.0, 4.0]]), 1)
        f = factorize_wz(l)
        assert np.array_equal(f.w_dense(), np.eye(2)) and np.array_equal(f.z_dense(), l.to_dense())

    def test_errors(self):
        from paper_2008_03276_b200 import (BandedMatrix, FactorizationBreakdownError,
                                           UnsupportedOrderError, factorize_wz)
        with pytest.raises(UnsupportedOrderError):
            factorize_wz(BandedMatrix.from_diagonals(7, {-1: -1.0, 0: 4.0, 1: -1.0}))
        with pytest.raises(FactorizationBreakdownError):
            factorize_wz(BandedMatrix(8, 1))

    def test_pattern_and_reconstruction_family(self, rng):
        from paper_2008_03276_b200 import factorize_wz
        for n in (8, 16, 32, 64):
            for beta in (1, 2, 3):
                l = rb(n, beta, rng)
                f = factorize_wz(l)
                w, z = f.w_dense(), f.z_dense()
                assert w_pattern_ok(w) and z_pattern_ok(z)
                d = l.to_dense()
                assert np.max(np.abs(w @ z - d)) / np.max(np.abs(d)) <= 1e-10

    def test_dense_oracle_family(self, rng):
        from paper_2008_03276_b200 import aqif_solve
        for n in (8, 16, 32, 64, 128):
            for beta in (1, 2, 3, 8):
                if n <= beta:
                    continue
                l = rb(n, beta, rng)
                rhs = rng.standard_normal(n)
                u = aqif_solve(l, rhs)
                ud = np.linalg.solve(l.to_dense(), rhs)
                assert np.max(np.abs(u - ud)) / np.max(np.abs(ud)) <= 1e-9

    def test_outside_in_trace_and_middle_solve(self, rng):
        from paper_2008_03276_b200 import factorize_wz, solve_z
        l = rb(16, 2, rng)
        f = factorize_wz(l)
        trace = []
        solve_z(f, rng.standard_normal(16), trace=trace)
        assert trace == [v for lev in range(8) for v in (lev, 15 - lev)]
        l = rb(24, 2, rng)
        f = factorize_wz(l)
        y = rng.standard_normal(24)
        xf = solve_z(f, y)
        xm = solve_z(f, y, start_level=3, boundary=xf)
        np.testing.assert_allclose(xm[2:-2], xf[2:-2], atol=1e-12)

    def test_poisson_manufactured(self):
        from paper_2008_03276_b200 import BandedMatrix, aqif_solve, band_matvec
        n = 64
        h = 1.0 / (n + 1)
        l = BandedMatrix.from_diagonals(n, {-1: -1.0 / h**2, 0: 2.0 / h**2, 1: -1.0 / h**2})
        x = np.linspace(h, 1 - h, n)
        exact = np.sin(np.pi * x)
        u = aqif_solve(l, band_matvec(l, exact))
        assert np.max(np.abs(u - exact)) <= 1e-10


class TestPaqif:
    @pytest.mark.parametrize("case", range(len(golden_cases("paqif_r.npz", "__"))))
    def test_r_blocks_vs_reference(self, case):
        from paper_2008_03276_b200.bandcore import BandedMatrix
        from paper_2008_03276_b200.parallel import paqif_solve
        G = golden_cases("paqif_r.npz")[case]
        bands = G["bands"]
        l = BandedMatrix(bands.shape[1], (bands.shape[0] - 1) // 2, bands)
        u = paqif_solve(l, G["f"], int(G["r"]))
        ref = G["u"]
        assert np.max(np.abs(u - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))

    def test_r_independence_and_identity(self, rng):
        from paper_2008_03276_b200 import BandedMatrix
        from paper_2008_03276_b200.parallel import paqif_solve
        l = BandedMatrix.identity(32)
        f = rng.standard_normal(32)
        for r in (1, 2, 4, 8):
            np.testing.assert_allclose(paqif_solve(l, f, r), f, atol=1e-14)
        n = 64
        h = 1.0 / (n + 1)
        l = BandedMatrix.from_diagonals(n, {-1: -1.0 / h**2, 0: 2.0 / h**2, 1: -1.0 / h**2})
        f = rng.standard_normal(n)
        sols = [paqif_solve(l, f, r) for r in (1, 2, 4)]
        for s in sols[1:]:
            assert np.max(np.abs(s - sols[0])) <= 1e-12 * np.max(np.abs(sols[0]))

    def test_large_vs_dense(self, rng):
        from paper_2008_03276_b200.parallel import paqif_solve
        l = rb(512, 2, rng)
        f = rng.standard_normal(512)
        u = paqif_solve(l, f, 8)
        ud = np.linalg.solve(l.to_dense(), f)
        assert np.max(np.abs(u - ud)) / np.max(np.abs(ud)) <= 1e-9


def obstacle_1d(n, amplitude=50.0):
    from paper_2008_03276_b200 import BandedMatrix
    from paper_2008_03276_b200.lcp import LcpProblem
    h = 1.0 / (n + 1)
    l = BandedMatrix.from_diagonals(n, {-1: -1.0 / h**2, 0: 2.0 / h**2, 1: -1.0 / h**2})
    x = np.linspace(h, 1 - h, n)
    return LcpProblem(l, amplitude * np.sin(2 * np.pi * x))


class TestLcpApi:
    def test_trivially_complementary(self):
        from paper_2008_03276_b200 import BandedMatrix
        from paper_2008_03276_b200.lcp import LcpProblem
        from paper_2008_03276_b200.parallel import paqif_solve_lcp
        n = 32
        l = BandedMatrix.from_diagonals(n, {-1: -1.0, 0: 4.0, 1: -1.0})
        u = paqif_solve_lcp(LcpProblem(l, -np.abs(np.linspace(0.5, 2.0, n))), 1)
        assert np.array_equal(u, np.zeros(n))

    def test_obstacle_vs_psor_and_cross_r(self):
        from paper_2008_03276_b200.lcp import psor_oracle
        from paper_2008_03276_b200.parallel import paqif_solve_lcp
        prob = obstacle_1d(64)
        u_ref = psor_oracle(prob, omega=1.7, tol=1e-13)
        u1 = paqif_solve_lcp(prob, 1, tol=1e-10)
        assert np.max(np.abs(u1 - u_ref)) <= 1e-8
        for r in (2, 4):
            assert np.max(np.abs(paqif_solve_lcp(prob, r, tol=1e-10) - u1)) <= 1e-8

    def test_golden_lcp_through_api(self):
        from paper_2008_03276_b200 import BandedMatrix
        from paper_2008_03276_b200.lcp import LcpProblem
        from paper_2008_03276_b200.parallel import paqif_solve_lcp
        for G in golden_cases("lcp.npz")[:6]:
            b = G["bands"]
            l = BandedMatrix(b.shape[1], (b.shape[0] - 1) // 2, b)
            u = paqif_solve_lcp(LcpProblem(l, G["f"]), 1, tol=1e-10)
            ref = G["u"]
            assert np.max(np.abs(u - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
            assert np.array_equal(cavitated(u), cavitated(ref))

    def test_psor_positive_diagonal_required(self):
        from paper_2008_03276_b200 import BandedMatrix, ContractViolationError
        from paper_2008_03276_b200.lcp import LcpProblem, psor_oracle
        l = BandedMatrix.from_diagonals(4, {0: -1.0, 1: 0.0, -1: 0.0})
        with pytest.raises(ContractViolationError):
            psor_oracle(LcpProblem(l, np.ones(4)))


class TestRblockDevice:
    """paqif_solve(r > 1) runs all seven steps on the device (csrc/rblock.cu)."""

    @pytest.mark.parametrize("n,beta,r", [(96, 2, 4), (256, 3, 8), (1026, 8, 27), (512, 8, 8),
                                          (640, 12, 10), (64, 1, 16)])
    def test_batch_vs_dense(self, n, beta, r):
        from paper_2008_03276_b200.batch import solve_rblock_batch
        from paper_2008_03276_b200.workloads import lcp_batch as gen
        bands, f = gen(7 + n, 12, n=n, beta=beta)
        x, st = solve_rblock_batch(bands, f, r)
        assert np.all(st == 0)
        from paper_2008_03276_b200 import BandedMatrix
        for b in range(bands.shape[0]):
            l = BandedMatrix(n, beta, bands[b])
            ud = np.linalg.solve(l.to_dense(), f[b])
            assert np.max(np.abs(x[b] - ud)) <= 1e-12 * max(1.0, np.max(np.abs(ud)))

    @pytest.mark.parametrize("case", range(len(golden_cases("paqif_proj.npz", "__"))))
    def test_project_flag_vs_reference(self, case):
        """project=True against the reference's paqif_solve(..., project=True)
        (tests/golden/paqif_proj.npz, make_golden.py)."""
        from paper_2008_03276_b200 import BandedMatrix
        from paper_2008_03276_b200.parallel import paqif_solve
        G = golden_cases("paqif_proj.npz")[case]
        bands = G["bands"]
        l = BandedMatrix(bands.shape[1], (bands.shape[0] - 1) // 2, bands)
        u = paqif_solve(l, G["f"], int(G["r"]), project=True)
        ref = G["u"]
        assert np.max(np.abs(u - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        assert np.array_equal(u[ref == 0.0] == 0.0, np.ones(int((ref == 0.0).sum()), bool))

    def test_statuses(self):
        from paper_2008_03276_b200.batch import solve_rblock_batch
        from paper_2008_03276_b200._native import LCP_FACTOR_BREAKDOWN
        n, beta = 64, 2
        bands = np.zeros((1, 5, n))
        bands[0, 2] = 1.0
        bands[0, 2, 8:24] = 0.0  # singular middle of block 0 of 4 (t = 16)
        x, st = solve_rblock_batch(bands, np.ones((1, n)), 4)
        assert int(st[0]) == LCP_FACTOR_BREAKDOWN

    def test_no_host_reduced_system(self, monkeypatch):
        """The public paqif_solve(r>1) runs on the device: no host linear
        algebra is reachable from it (numpy.linalg / scipy patched to fail)."""
        import scipy.linalg
        from paper_2008_03276_b200 import BandedMatrix, parallel
        def boom(*a, **k):
            raise AssertionError("host path used")
        for mod, name in ((np.linalg, "inv"), (np.linalg, "solve"), (scipy.linalg, "cho_factor"),
                          (scipy.linalg, "cho_solve")):
            monkeypatch.setattr(mod, name, boom)
        rng = np.random.default_rng(5)
        n = 128
        l = BandedMatrix.from_diagonals(n, {-1: -1.0, 0: 4.0, 1: -1.0})
        f = rng.standard_normal(n)
        from paper_2008_03276_b200.lcp import LcpProblem
        u = parallel.paqif_solve(l, f, 4)
        u2 = parallel.paqif_solve_lcp(LcpProblem(l, f), 4, tol=1e-10)
        u1 = parallel.paqif_solve_lcp(LcpProblem(l, f), 1, tol=1e-10)
        monkeypatch.undo()
        assert np.max(np.abs(u - np.linalg.solve(l.to_dense(), f))) <= 1e-12
        assert np.max(np.abs(u2 - u1)) <= 1e-10
