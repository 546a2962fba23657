"""Fused batched LCP kernel (config 2 hot path) against the CPU oracle and the
reference's golden answers.

Tolerances: EXACT mode is bit-identical to the oracle (same operation order
everywhere, including the corner normal equations); FMA mode must give the
same pass count and pinned set and pressures within 1e-9 relative (the
north_star tolerance); both match the reference goldens to 1e-12 relative."""

import numpy as np
import pytest

import oracle as O
from conftest import cavitated, golden_cases

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.asarray(a).view(np.uint64)


def test_lcp_matches_reference_goldens():
    from paper_2008_03276_b200.batch import lcp_batch
    for G in golden_cases("lcp.npz"):
        if (G["bands"].shape[0] - 1) // 2 > 8:
            continue
        r = lcp_batch(G["bands"][None], G["f"][None], exact=True)
        ref = G["u"]
        assert r.status[0] == 0
        assert r.passes[0] == int(G["passes"])
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(r.u[0] - ref)) <= 1e-12 * scale
        assert np.array_equal(cavitated(r.u[0]), cavitated(ref))


@pytest.mark.parametrize("n,beta,B", [(1025, 8, 48), (129, 8, 64), (65, 4, 64), (33, 2, 64),
                                      (257, 1, 16), (101, 3, 16), (91, 5, 16), (99, 6, 8),
                                      (131, 7, 8)])
def test_lcp_exact_bitwise_vs_oracle(n, beta, B):
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(1234, B, n=n, beta=beta)
    u, act, passes, res, st = O.lcp_batch(bands, f, threads=8)
    r = lcp_batch(bands, f, exact=True)
    assert np.array_equal(r.status, st)
    assert np.array_equal(r.passes, passes)
    assert np.array_equal(r.active, act)
    assert np.array_equal(_bits(r.u), _bits(u))
    assert np.array_equal(_bits(r.res), _bits(res))


@pytest.mark.parametrize("n,beta,B", [(1025, 8, 64), (129, 8, 64), (33, 2, 64), (257, 1, 16),
                                      (101, 3, 16), (91, 5, 16), (99, 6, 8), (131, 7, 8)])
def test_lcp_fma_within_tolerance(n, beta, B):
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(99, B, n=n, beta=beta)
    u, act, passes, res, st = O.lcp_batch(bands, f, threads=8)
    r = lcp_batch(bands, f, exact=False)
    assert np.array_equal(r.status, st)
    assert np.array_equal(r.passes, passes)
    assert np.array_equal(r.active, act)
    scale = np.maximum(1.0, np.max(np.abs(u), axis=1, keepdims=True))
    assert np.max(np.abs(r.u - u) / scale) <= 1e-9


def test_lcp_full_config2_properties():
    """All 4096 config-2 systems: KKT conditions hold for every system and a
    sampled subset matches the oracle exactly (size-independent properties)."""
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(2024, 4096)
    r = lcp_batch(bands, f, exact=True)
    assert np.all(r.status == 0)
    assert np.all((r.passes >= 2) & (r.passes <= 4))
    B, d, n = bands.shape
    beta = (d - 1) // 2
    lam = np.zeros_like(r.u)
    for o in range(-beta, beta + 1):
        lo, hi = max(0, -o), n - max(0, o)
        lam[:, lo:hi] += bands[:, beta + o, lo:hi] * r.u[:, lo + o:hi + o]
    lam -= f
    assert np.all(r.u >= 0.0)
    assert np.min(lam) >= -1e-10
    assert np.max(np.abs(np.minimum(r.u, lam))) <= 1e-10
    assert np.all(r.res <= 1e-10)
    pick = np.arange(0, 4096, 128)
    u, act, passes, res, st = O.lcp_batch(bands[pick], f[pick], threads=8)
    assert np.array_equal(_bits(r.u[pick]), _bits(u))
    assert np.array_equal(r.passes[pick], passes)


def test_lcp_host_entry_matches_device_entry():
    from paper_2008_03276_b200.batch import lcp_batch, lcp_batch_host
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(5, 40, n=257, beta=8)
    a = lcp_batch(bands, f)
    b = lcp_batch_host(bands, f)
    assert np.array_equal(_bits(a.u), _bits(b.u))
    assert np.array_equal(a.passes, b.passes)


def test_lcp_edge_cases():
    from paper_2008_03276_b200.batch import lcp_batch
    n = 32
    # f <= 0 everywhere: trivially complementary, zero solution in one pass
    bands = np.zeros((1, 3, n)); bands[0, 1] = 4.0; bands[0, 0, 1:] = -1.0; bands[0, 2, :-1] = -1.0
    f = -np.abs(np.linspace(0.5, 2.0, n))[None]
    r = lcp_batch(bands, f)
    assert r.status[0] == 0 and r.passes[0] == 1 and np.all(r.u == 0.0)
    # max_outer = 0 -> NonConvergence status, zero answer
    r = lcp_batch(bands, f, max_outer=0)
    assert r.status[0] == 4
    # zero diagonal -> factor breakdown reported per system, others unaffected
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bb, ff = gen(8, 3, n=65, beta=8)
    bb[1] = 0.0
    ff[1] = 1.0
    r = lcp_batch(bb, ff)
    assert r.status[1] == 1 and r.status[0] == 0 and r.status[2] == 0
    assert r.res[1] == -1.0  # a breakdown reports -(1-based level) in res
    # ... which the API raises as FactorizationBreakdownError.level
    from paper_2008_03276_b200 import BandedMatrix, FactorizationBreakdownError
    from paper_2008_03276_b200.lcp import LcpProblem
    from paper_2008_03276_b200.parallel import paqif_solve, paqif_solve_lcp
    d = np.ones(64)
    d[5] = 0.0  # the level-27 corner (rows 5, 58) is singular: the reference
    l = BandedMatrix.from_diagonals(64, {0: d, 1: np.zeros(63)})  # raises level=27
    with pytest.raises(FactorizationBreakdownError) as ei:
        paqif_solve_lcp(LcpProblem(l, np.ones(64)), 1)
    assert ei.value.level == 27
    with pytest.raises(FactorizationBreakdownError) as ei:
        paqif_solve(l, np.ones(64), 1)
    assert ei.value.level == 27


def test_solve_r1_matches_oracle():
    from paper_2008_03276_b200.batch import solve_r1_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(77, 32, n=257, beta=8)
    x, st = solve_r1_batch(bands, f)
    xo, sto = O.paqif_solve_r1_batch(bands, f, threads=8)
    assert np.array_equal(st, sto)
    assert np.array_equal(_bits(x), _bits(xo))


def test_lcp_full_config2_fma_matches_exact():
    """The bench headline runs FMA arithmetic: on all 4096 config-2 systems it
    takes the same passes and ends in the same active sets as the exact
    (bit-exact vs the oracle) arithmetic, values within 1e-9 relative."""
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    bands, f = gen(2024, 4096)
    re_ = lcp_batch(bands, f, exact=True)
    rf = lcp_batch(bands, f, exact=False)
    assert np.array_equal(re_.passes, rf.passes)
    assert np.array_equal(re_.active, rf.active)
    assert np.all(rf.status == 0)
    scale = np.maximum(1.0, np.max(np.abs(re_.u), axis=1, keepdims=True))
    assert np.max(np.abs(rf.u - re_.u) / scale) <= 1e-9


@pytest.mark.parametrize("beta", [2, 8])
def test_lcp_wild_systems_status_vs_oracle(beta):
    """Non-dominant systems (random diagonals): factor breakdowns at inner
    levels, non-convergence and ordinary solves mixed in one batch -- status,
    passes and answers equal to the oracle bit for bit (exact arithmetic;
    the breakdown test runs after the factorization, lazily)."""
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    rng = np.random.default_rng(77 + beta)
    B, n = 48, 129
    bands, f = gen(5, B, n=n, beta=beta)
    diag = bands[:, beta, :]
    wild = rng.random(B) < 0.5
    diag[wild, :n] = rng.uniform(-1.0, 1.0, (int(wild.sum()), n))  # pad row stays identity
    u, act, passes, res, st = O.lcp_batch(bands, f, threads=8)
    r = lcp_batch(bands, f, exact=True)
    assert np.array_equal(r.status, st)
    assert np.array_equal(r.passes, passes)
    ok = st == 0
    assert np.array_equal(r.active[ok], act[ok])
    assert np.array_equal(_bits(r.u[ok]), _bits(u[ok]))
    assert len(set(st.tolist())) >= 2, "the batch should mix outcomes"


@pytest.mark.parametrize("beta", [2, 8])
def test_lcp_wild_systems_fma_status(beta):
    """FMA arithmetic (the pipelined factorization, which defers the level
    test to the records the Z solve and the corner system read) on the same
    non-dominant systems: the same outcome per system as the oracle -- the
    same breakdown level, the same passes -- and values within 1e-9 where
    the solve succeeds."""
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    rng = np.random.default_rng(77 + beta)
    B, n = 48, 129
    bands, f = gen(5, B, n=n, beta=beta)
    diag = bands[:, beta, :]
    wild = rng.random(B) < 0.5
    diag[wild, :n] = rng.uniform(-1.0, 1.0, (int(wild.sum()), n))
    u, act, passes, res, st = O.lcp_batch(bands, f, threads=8)
    r = lcp_batch(bands, f, exact=False)
    assert np.array_equal(r.status, st)
    assert np.array_equal(r.passes, passes)
    brk = st == 1
    assert np.array_equal(r.res[brk], res[brk]), "breakdown levels"
    ok = st == 0
    assert np.array_equal(r.active[ok], act[ok])
    scale = np.maximum(1.0, np.max(np.abs(u[ok]), axis=1, keepdims=True))
    assert np.max(np.abs(r.u[ok] - u[ok]) / scale) <= 1e-9


@pytest.mark.parametrize("exact", [True, False])
def test_lcp_breakdown_levels_both_arithmetics(exact):
    """Breakdown levels in every range the level test covers: an inner level
    (found by the Z solve's scan in FMA arithmetic), an outer corner level
    (found by the corner system), and level 1 -- the same level in both
    arithmetics, reported as -(level) in res."""
    from paper_2008_03276_b200.batch import lcp_batch
    n, beta = 64, 4
    s = n // 2
    bands = np.zeros((3, 2 * beta + 1, n))
    bands[:, beta, :] = 2.0
    f = np.ones((3, n))
    # system 0: row 2 singular -> the level-30 pivot (rows 2, 61): a corner level
    bands[0, beta, 2] = 0.0
    # system 1: row 20 singular -> level 12 (rows 20, 43): an inner level
    bands[1, beta, 20] = 0.0
    # system 2: the middle rows singular -> level 1
    bands[2, beta, s - 1] = 0.0
    r = lcp_batch(bands, f, exact=exact)
    assert list(r.status) == [1, 1, 1]
    assert list(r.res) == [-float(s - 2), -float(s - 20), -1.0]


@pytest.mark.parametrize("beta", [1, 2, 5, 8])
@pytest.mark.parametrize("exact", [True, False])
def test_lcp_minimum_order_and_odd_batches(beta, exact):
    """The smallest order the block method allows (n = 2*beta + 2: every
    hook past the matrix, one middles level) and batches that leave a
    system group of the last warp empty, both arithmetics, against the
    oracle (bit-exact / within 1e-9)."""
    from paper_2008_03276_b200.batch import lcp_batch
    from paper_2008_03276_b200.workloads import lcp_batch as gen
    for n, B in ((2 * beta + 2, 3), (2 * beta + 4, 1), (4 * beta + 2, 5)):
        bands, f = gen(31 + n, B, n=n, beta=beta)
        u, act, passes, res, st = O.lcp_batch(bands, f, threads=4)
        r = lcp_batch(bands, f, exact=exact)
        assert np.array_equal(r.status, st)
        assert np.array_equal(r.passes, passes)
        assert np.array_equal(r.active, act)
        if exact:
            assert np.array_equal(_bits(r.u), _bits(u))
        else:
            scale = np.maximum(1.0, np.max(np.abs(u), axis=1, keepdims=True))
            assert np.max(np.abs(r.u - u) / scale) <= 1e-9


def test_lcp_fma_matches_reference_goldens():
    """The headline arithmetic against the reference's own answers: same
    pass count and cavitated set, values within 1e-9 relative."""
    from paper_2008_03276_b200.batch import lcp_batch
    for G in golden_cases("lcp.npz"):
        if (G["bands"].shape[0] - 1) // 2 > 8:
            continue
        r = lcp_batch(G["bands"][None], G["f"][None], exact=False)
        ref = G["u"]
        assert r.status[0] == 0
        assert r.passes[0] == int(G["passes"])
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(r.u[0] - ref)) <= 1e-9 * scale
        assert np.array_equal(cavitated(r.u[0]), cavitated(ref))
