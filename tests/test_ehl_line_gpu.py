"""Fused line-contact Newton step on the GPU vs teacher-forced reference
steps (golden) and the numpy oracle.  Protocol SURVEY.md 8(c): single-step
parity from identical states -- pressure and film within 1e-9 relative,
identical cavitated set, identical solve rung (combined system vs the Ls4
breakdown ladder) and force-balance application; plus a short horizon."""

import math

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

G = load_golden("ehl_line.npz")
KEYS = sorted({k.split("__")[0] for k in G.files if k.startswith("e")}, key=lambda s: int(s[1:]))
TOL = 1e-9


def gcase(key):
    return {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(key + "__")}


def params_for(d):
    from paper_2008_03276_b200.ehl import EhlParams, moes_convert
    m, l = float(d["meta"][0]), float(d["meta"][1])
    u, w = moes_convert(m=m, l=l, g=5000.0)
    p = EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))
    assert p.p_hertz == float(d["p_hertz"]) and p.lam == float(d["lam"])
    return p


def run_step(params_list, intervals, u_in, h0_in, k, exact=True, path="auto"):
    from paper_2008_03276_b200.ehl import LineContactBatch
    b = LineContactBatch(params_list, intervals, u0=u_in, h0=h0_in, exact=exact, path=path)
    b.outer = k
    b.step()
    return b.snapshot()


def check_against(d, u, h0, film, res, info):
    ref = d["u_out"]
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(u - ref)) <= TOL * scale
    assert np.array_equal(u == 0.0, ref == 0.0), "cavitated set differs"
    assert math.isclose(h0, float(d["h0_out"]), rel_tol=1e-13, abs_tol=1e-15)
    fref = d["film_out"]
    assert np.max(np.abs(film - fref)) <= TOL * max(1.0, float(np.max(np.abs(fref))))
    assert math.isclose(res, float(d["res_out"]), rel_tol=TOL)
    assert ((info & 3) != 0) == (int(d["breaks"]) > 0), "solve rung differs"
    assert bool(info & 4) == bool(d["fb_applied"])


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("path", ["fused", "split"])
def test_single_step_vs_reference(key, exact, path):
    d = gcase(key)
    p = params_for(d)
    n, k = int(d["meta"][2]), int(d["meta"][3])
    u, h0, film, res, _, info = run_step([p], n, d["u_in"][None], [float(d["h0_in"])], k, exact,
                                         path)
    check_against(d, u[0], h0[0], film[0], res[0], int(info[0]))


@pytest.mark.parametrize("path", ["fused", "split"])
def test_batched_config3_cases_match_individually(path):
    """All N=1025 golden states of one outer index in ONE launch."""
    by_k = {}
    for key in KEYS:
        d = gcase(key)
        if int(d["meta"][2]) == 1024:
            by_k.setdefault(int(d["meta"][3]), []).append(d)
    assert by_k
    for k, ds in by_k.items():
        ps = [params_for(d) for d in ds]
        u0 = np.stack([d["u_in"] for d in ds])
        h0 = [float(d["h0_in"]) for d in ds]
        u, h0o, film, res, _, info = run_step(ps, 1024, u0, h0, k, path=path)
        for j, d in enumerate(ds):
            check_against(d, u[j], h0o[j], film[j], res[j], int(info[j]))


def test_short_horizon_vs_oracle():
    import oracle.ehl_oracle as E
    from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert
    u_, w_ = moes_convert(m=20.0, l=10.0, g=5000.0)
    p = EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))
    c = E.LineCase(p_hertz=p.p_hertz, lam=p.lam)
    film = E.LineFilm(128, c)
    ur, h0r = E.hertz_start(c, film), c.h0
    b = LineContactBatch([p], 128)
    for k in range(8):
        ur, h0r, fr, rr, _ = E.line_step(ur, h0r, k, c, film)
        b.step()
        u, h0, f, res, _, _ = b.snapshot()
        assert np.max(np.abs(u[0] - ur)) <= 1e-9 * max(1.0, np.max(np.abs(ur)))
        assert math.isclose(res[0], rr, rel_tol=1e-8)
        np.testing.assert_allclose(u[0], G["traj__u"][k], rtol=0, atol=1e-9)


def test_line_deformation_matches_convolve(rng):
    from paper_2008_03276_b200.ehl import kernel_line, line_deformation
    n = 300
    t = kernel_line(n, 0.02).table
    u = np.abs(rng.standard_normal((3, n + 1)))
    ext = np.concatenate([t[::-1], t[1:]])
    ref = np.stack([-(1.0 / np.pi) * np.convolve(x, ext)[n:2 * n + 1] for x in u])
    got = line_deformation(t, u)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_solve_ehl_line_api():
    """solve_ehl runs the fused step; the reference never converges on config 1
    (SURVEY.md 0.3), so a short budget raises NonConvergenceError with the
    same residual history as the oracle's first iterations."""
    import oracle.ehl_oracle as E
    from paper_2008_03276_b200.errors import NonConvergenceError
    from paper_2008_03276_b200.ehl import EhlParams, moes_convert, solve_ehl
    u_, w_ = moes_convert(m=20.0, l=10.0, g=5000.0)
    p = EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))
    seen = []
    with pytest.raises(NonConvergenceError):
        solve_ehl(p, 512, max_outer=6, collect=lambda st, r, d: seen.append(r))
    c = E.LineCase(p_hertz=p.p_hertz, lam=p.lam)
    film = E.LineFilm(512, c)
    ur, h0r = E.hertz_start(c, film), c.h0
    for k in range(3):
        ur, h0r, _, rr, _ = E.line_step(ur, h0r, k, c, film)
        assert math.isclose(seen[k], rr, rel_tol=1e-8)


@pytest.mark.parametrize("key", KEYS[:3])
def test_line_complementarity_residual(key):
    """EhlState.complementarity_residual for a line state equals the residual
    the reference reports after its step (residual-only kernel)."""
    from paper_2008_03276_b200.ehl import solver
    d = gcase(key)
    p = params_for(d)
    n = int(d["meta"][2])
    st = solver._initial_state(p, n)
    st.u = d["u_out"].copy()
    st.h0 = float(d["h0_out"])
    assert math.isclose(st.complementarity_residual(p, 1.0 / 3.0, "kappa"), float(d["res_out"]),
                        rel_tol=TOL)


def _line_params():
    from paper_2008_03276_b200.ehl import EhlParams, moes_convert
    u_, w_ = moes_convert(m=20.0, l=10.0, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))


@pytest.mark.parametrize("tol,tol_fb,max_outer", [(1e-6, 1e-4, 70), (1e30, 1e30, 40),
                                                  (1e30, 1e-300, 12)])
def test_device_driver_matches_host_loop(tol, tol_fb, max_outer):
    """solve_ehl without `collect` runs the stop / divergence tests on the
    device (paqif_ehl_line_drive_steps, chunks of 32 launches); with
    `collect` it steps from the host.  Same histories, state and outcome."""
    from paper_2008_03276_b200.ehl import solve_ehl
    from paper_2008_03276_b200.errors import NonConvergenceError
    p = _line_params()
    out = []
    for collect in (None, lambda st, r, d: None):
        err = None
        try:
            st = solve_ehl(p, 512, tol=tol, tol_fb=tol_fb, max_outer=max_outer, collect=collect)
        except NonConvergenceError as e:
            err, st = (e.iterations, e.residual), None
        out.append((err, st))
    (e_dev, s_dev), (e_host, s_host) = out
    assert e_dev == e_host
    if s_dev is not None:
        assert s_dev.residual_history == s_host.residual_history
        assert s_dev.force_history == s_host.force_history
        assert s_dev.outer_iterations == s_host.outer_iterations
        assert np.array_equal(s_dev.u, s_host.u) and s_dev.h0 == s_host.h0


def test_device_driver_batch_stops_per_case():
    """Per-case drive records: a case that converged skips later launches
    while the others keep iterating."""
    import torch
    from paper_2008_03276_b200.ehl.line import DRIVE_BUDGET, DRIVE_CONVERGED, LineContactBatch
    p = _line_params()
    b = LineContactBatch([p, p], 512)
    b.drive_init(1e30, 1e30, 9, hist_cap=16)
    rec = b.drive_state()
    rec["tol_fb"][1] = 1e-300  # case 1 can never pass the force test
    b.drive.copy_(torch.from_numpy(rec.view(np.uint8)))
    b.drive_steps(16)
    d = b.drive_state()
    assert d["done"][0] == DRIVE_CONVERGED and d["outer"][0] == 5
    assert d["done"][1] == DRIVE_BUDGET and d["outer"][1] == 9
    ref = LineContactBatch([p], 512)
    res = []
    for k in range(9):
        ref.step()
        res.append(float(ref.res[0].item()))
        if k == 4:
            assert np.array_equal(b.u[0].cpu().numpy(), ref.u[0].cpu().numpy())
    assert np.array_equal(b.u[1].cpu().numpy(), ref.u[0].cpu().numpy())
    assert list(b.hist_res[0, :5].cpu().numpy()) == res[:5]
    assert list(b.hist_res[1, :9].cpu().numpy()) == res


def test_queued_batch_matches_one_case_launches():
    """B > SM count: one CTA per SM pulls the cases from a queue ordered by
    the previous step's ladder use; every case's state equals a B = 1 run of
    the same case (bit for bit, over several steps so the order is live)."""
    from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert
    rng = np.random.default_rng(11)
    cases = list(zip(np.exp(rng.uniform(np.log(5), np.log(200), 300)), rng.uniform(5, 15, 300)))

    def params(m, l):
        u_, w_ = moes_convert(m=float(m), l=float(l), g=5000.0)
        return EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))

    ps = [params(m, l) for m, l in cases]
    b = LineContactBatch(ps, 128, path="fused")
    for _ in range(4):
        b.step()
    u, h0, film, res, _, info = b.snapshot()
    for j in (0, 17, 149, 150, 299):
        one = LineContactBatch([ps[j]], 128)
        for _ in range(4):
            one.step()
        u1, h01, film1, res1, _, info1 = one.snapshot()
        assert np.array_equal(u[j], u1[0]) and h0[j] == h01[0]
        assert np.array_equal(film[j], film1[0]) and res[j] == res1[0] and info[j] == info1[0]


def _config3_params(count, seed=2024):
    import bench
    from paper_2008_03276_b200.ehl import EhlParams, moes_convert
    out = []
    for m, l in bench.config3_cases(0, count=count, seed=seed):
        u_, w_ = moes_convert(m=float(m), l=float(l), g=5000.0)
        out.append(EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5)))
    return out


@pytest.mark.parametrize("exact", [True, False])
def test_split_path_matches_fused_config3(exact):
    """Config 3 (N = 1025, load-sweep cases): the split path (phase A, every
    ladder rung of every case solved side by side by the throughput
    engine, phase C) against the fused one-CTA-per-case kernel from the
    same states: identical rungs / force balance / weighted-row counts and
    pressures within 1e-12 after one step, then 1e-9 (exact) / 1e-6 (FMA:
    the two engines contract differently) -- the iteration is chaotic,
    SURVEY.md 0.4, so later steps amplify last-bit differences."""
    from paper_2008_03276_b200.ehl import LineContactBatch
    ps = _config3_params(320)
    a = LineContactBatch(ps, 1024, exact=exact, path="fused")
    b = LineContactBatch(ps, 1024, exact=exact, path="split")
    for k in range(4 if exact else 1):
        a.step()
        b.step()
        ua, h0a, fa, ra, _, ia = a.snapshot()
        ub, h0b, fb, rb, _, ib = b.snapshot()
        tol = 1e-12 if k == 0 else (1e-9 if exact else 1e-6)
        scale = np.maximum(1.0, np.max(np.abs(ua), axis=1, keepdims=True))
        assert np.max(np.abs(ub - ua) / scale) <= tol, k
        assert np.max(np.abs(fb - fa) / np.maximum(1.0, np.abs(fa))) <= tol, k
        if k == 0:
            assert np.array_equal(ia, ib), "rungs / force balance / weighted rows"
            assert np.array_equal(ua == 0.0, ub == 0.0)
    assert int(np.sum((ia & 3) > 0)) >= 1, "no ladder case in the batch"


def test_split_path_device_driver():
    """The device-driven loop (per-case stop / divergence records) on the
    split path: same outcome as the fused path's records."""
    from paper_2008_03276_b200.ehl import LineContactBatch
    ps = _config3_params(300)
    recs = []
    for path in ("fused", "split"):
        b = LineContactBatch(ps, 256, path=path)
        b.drive_init(1e-6, 1e-4, 12, hist_cap=16)
        b.drive_steps(16)
        recs.append((b.drive_state(), b.hist_res.cpu().numpy()))
    (d0, h0), (d1, h1) = recs
    assert np.array_equal(d0["done"], d1["done"]) and np.array_equal(d0["outer"], d1["outer"])
    np.testing.assert_allclose(h1[:, :12], h0[:, :12], rtol=1e-7)


GB = load_golden("ehl_line_big.npz")
BIG = sorted({k.split("__")[0] for k in GB.files}, key=lambda s: int(s[1:]))


@pytest.mark.parametrize("key", BIG)
@pytest.mark.parametrize("exact", [True, False])
def test_fine_grid_single_step_vs_reference(key, exact):
    """Line contacts finer than one CTA's shared memory (n = 4096 / 8192
    intervals; the reference has no size limit): the split path with its
    phase arrays in HBM, teacher-forced against the reference
    (tests/golden/make_golden_line_big.py), incl. a ladder state."""
    d = {k.split("__", 1)[1]: GB[k] for k in GB.files if k.startswith(key + "__")}
    p = params_for(d)
    n, k = int(d["meta"][2]), int(d["meta"][3])
    u, h0, film, res, _, info = run_step([p], n, d["u_in"][None], [float(d["h0_in"])], k, exact)
    check_against(d, u[0], h0[0], film[0], res[0], int(info[0]))


def test_fine_grid_residual_and_deformation(rng):
    """complementarity_residual and the line deformation past the shared-
    memory size (arrays in HBM)."""
    from paper_2008_03276_b200.ehl import kernel_line, line_deformation, solver
    d = {k.split("__", 1)[1]: GB[k] for k in GB.files if k.startswith(BIG[-1] + "__")}
    p = params_for(d)
    n = int(d["meta"][2])
    st = solver._initial_state(p, n)
    st.u = d["u_out"].copy()
    st.h0 = float(d["h0_out"])
    assert math.isclose(st.complementarity_residual(p, 1.0 / 3.0, "kappa"), float(d["res_out"]),
                        rel_tol=TOL)
    m = 9000
    t = kernel_line(m, 6.0 / m).table
    u = np.abs(rng.standard_normal((2, m + 1)))
    ext = np.concatenate([t[::-1], t[1:]])
    ref = np.stack([-(1.0 / np.pi) * np.convolve(x, ext)[m:2 * m + 1] for x in u])
    got = line_deformation(t, u)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_fine_grid_solve_ehl_device_loop():
    """solve_ehl at n = 4096 runs on the device loop like the coarse grids:
    same histories with and without the host loop."""
    from paper_2008_03276_b200.ehl import solve_ehl
    from paper_2008_03276_b200.errors import NonConvergenceError
    p = _line_params()
    hists = []
    for collect in (None, lambda st, r, dd: None):
        try:
            solve_ehl(p, 4096, max_outer=6, collect=collect)
        except NonConvergenceError as e:
            hists.append((e.iterations, e.residual))
    assert len(hists) == 2 and hists[0] == hists[1]
