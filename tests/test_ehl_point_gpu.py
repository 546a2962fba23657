"""Point-contact outer iteration on the GPU (csrc/ehl_point.cu through the
C ABI paqif_ehl_point_*) vs teacher-forced reference iterations (golden,
tests/golden/make_golden_point.py) and the numpy oracle.

Protocol SURVEY.md 8(c) P2: from identical states (u, h0) one outer
iteration -- identical per-line Newton/weighted decisions in the x-sweep,
pressure and film within 1e-9 relative, identical cavitated set, force
balance on the same iterations, residual within 1e-9 relative; plus the
FFT deformation against scipy's and a short free-running horizon."""

import math

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

G = load_golden("ehl_point.npz")
KEYS = sorted({k.split("__")[0] for k in G.files if k.startswith("e")}, key=lambda s: int(s[1:]))
TOL = 1e-9


def gcase(key):
    return {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(key + "__")}


def params_for(m, l=10.0):
    from paper_2008_03276_b200.ehl import EhlParams
    return EhlParams.point_from_moes(m, l, domain=(-4.5, 1.5), lo_y=-3.0)


def close_field(got, ref, tol=TOL):
    return np.max(np.abs(got - ref)) <= tol * max(1.0, float(np.max(np.abs(ref))))


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("exact", [True, False])
def test_single_step_vs_reference(key, exact):
    from paper_2008_03276_b200.ehl import PointContact
    d = gcase(key)
    m, l, n, k = d["meta"]
    p = params_for(float(m), float(l))
    assert p.p_hertz == float(d["p_hertz"]) and p.lam == float(d["lam"])
    pc = PointContact(p, int(n), u0=d["u_in"], h0=float(d["h0_in"]), exact=exact)
    pc.outer = int(k)
    pc.step()
    s = pc.snapshot()
    pc.close()
    assert s["err"] == 0
    assert np.array_equal(s["newton"], d["newton"]), "x-sweep Newton/weighted decisions"
    assert close_field(s["u"], d["u_out"])
    assert np.array_equal(s["u"] == 0.0, d["u_out"] == 0.0), "cavitated set differs"
    assert math.isclose(s["h0"], float(d["h0_out"]), rel_tol=1e-13, abs_tol=1e-15)
    assert close_field(s["film"], d["film_out"])
    assert math.isclose(s["res"], float(d["res_out"]), rel_tol=TOL)


def test_rungs_match_oracle():
    """Fallback-ladder rungs of every x line and y column equal the oracle's."""
    from oracle import ehl_point_oracle as P
    from paper_2008_03276_b200.ehl import PointContact
    d = gcase(KEYS[-1])
    m, l, n, k = d["meta"]
    pc = PointContact(params_for(float(m)), int(n), u0=d["u_in"], h0=float(d["h0_in"]))
    pc.outer = int(k)
    pc.step()
    s = pc.snapshot()
    c = P.PointCase(p_hertz=float(d["p_hertz"]), lam=float(d["lam"]))
    _, _, _, _, info = P.point_step(d["u_in"], float(d["h0_in"]), int(k), c, P.PointFilm(int(n), c))
    names = {"scheme": 0, "first-order": 1, "diagonal": 2}
    assert list(s["x_rungs"]) == [names[r] for r in info["x_rungs"]]
    assert list(s["y_rungs"]) == [0 if r == "scheme" else 1 for r in info["y_rungs"]]


@pytest.mark.parametrize("n", [32, 64, 100, 256])
def test_fft_deformation_vs_scipy(n):
    from oracle import ehl_point_oracle as P
    from paper_2008_03276_b200.ehl import FilmModel
    c = P.point_case(100.0, 10.0)
    f = P.PointFilm(n, c)
    rng = np.random.default_rng(n)
    u = np.maximum(0.0, rng.standard_normal((n + 1, n + 1)))
    ref = f.deformation_full(u)
    fm = FilmModel("point", n, f.h, c.lo, lo_y=c.lo_y)
    got = fm.deformation_full(u)
    assert np.max(np.abs(got - ref)) <= 1e-12 * float(np.max(np.abs(ref)))
    assert np.array_equal(fm.geometry, f.geometry)


def test_horizon_matches_reference_history():
    """11 free-running outer iterations from the adapted Hertz start; the
    residual history follows the reference's (golden hist_p32)."""
    from paper_2008_03276_b200.ehl import PointContact
    pc = PointContact(params_for(100.0), 32)
    assert np.array_equal(pc.snapshot()["u"], G["init__u"])
    hist = []
    for _ in range(11):
        pc.step()
        hist.append(pc.status()[1])
    np.testing.assert_allclose(hist, G["hist_p32"], rtol=1e-7)


def test_solve_ehl_point_runs():
    from paper_2008_03276_b200.ehl import solve_ehl
    from paper_2008_03276_b200.errors import NonConvergenceError
    seen = []
    try:
        solve_ehl(params_for(100.0), 32, max_outer=6, collect=lambda st, r, dfc: seen.append(r))
    except NonConvergenceError as e:
        assert e.iterations == 6
    np.testing.assert_allclose(seen, G["hist_p32"][:6], rtol=1e-7)


def test_no_host_fallback(monkeypatch):
    """The point path must not route through the oracle."""
    import sys
    from paper_2008_03276_b200.ehl import PointContact
    monkeypatch.setitem(sys.modules, "oracle.ehl_point_oracle", None)
    pc = PointContact(params_for(100.0), 32)
    pc.step()
    assert math.isfinite(pc.status()[1])


S = load_golden("ehl_point_sweeps.npz")
SWEEPS = sorted({k.split("__")[0] for k in S.files})


@pytest.mark.parametrize("name", SWEEPS)
def test_public_sweeps_vs_reference(name):
    """newton_line_sweep / weighted_change_sweep / column_sweep /
    complementarity_residual on an EhlState (reference signatures)."""
    from paper_2008_03276_b200.ehl import sweeps
    from paper_2008_03276_b200.ehl.solver import _initial_state
    d = {k.split("__", 1)[1]: S[k] for k in S.files if k.startswith(name + "__")}
    src = gcase(str(d["src"]))
    m, l, n, _ = src["meta"]
    p = params_for(float(m), float(l))
    st = _initial_state(p, int(n))
    st.u = src["u_in"].copy()
    st.h0 = float(src["h0_in"])
    call, lim, kappa = str(d["call"]), str(d["limiter"]), 1.0 / 3.0
    if call == "newton":
        hyb = str(d["hybrid"]) or None
        val = sweeps.newton_line_sweep(st, p, kappa, lim, scheme=str(d["scheme"]) or "Ls1",
                                       hybrid=hyb)
    elif call == "weighted":
        val = sweeps.weighted_change_sweep(st, p, kappa, lim, scheme=str(d["scheme"]))
    elif call == "column":
        val = sweeps.column_sweep(st, p, kappa, lim)
    else:
        val = st.complementarity_residual(p, kappa, lim)
    ref = d["u_out"]
    assert close_field(st.u, ref)
    assert np.array_equal(st.u == 0.0, ref == 0.0)
    assert math.isclose(val, float(d["value"]), rel_tol=TOL)


@pytest.mark.parametrize("n,steps", [(64, 4), (128, 3)])
def test_batched_deferred_runs_match_line_by_line(monkeypatch, n, steps):
    """Runs of deferred x-lines solved side by side (pt_xrun_kernel, runs
    predicted from the previous sweep) give bit-identical states, tags and
    residuals to solving every line on its own in Gauss-Seidel order."""
    from paper_2008_03276_b200.ehl import PointContact
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("PAQIF_PT_RUNS", flag)
        pc = PointContact(params_for(100.0), n)
        hist = []
        for _ in range(steps):
            pc.step()
            hist.append(pc.status()[1])
        s = pc.snapshot()
        pc.close()
        out.append((hist, s))
    (h1, s1), (h0, s0) = out
    assert h1 == h0
    assert np.array_equal(s1["u"], s0["u"]) and s1["h0"] == s0["h0"]
    assert np.array_equal(s1["newton"], s0["newton"])
    assert np.array_equal(s1["x_rungs"], s0["x_rungs"])
    assert int(np.sum(np.asarray(s1["newton"]) == 0)) >= 4, "no deferred run to batch"


@pytest.mark.parametrize("tol,tol_fb,max_outer", [(1e30, 1e30, 12), (0.0, 0.0, 11),
                                                  (1e30, 1e-300, 10)])
def test_point_device_driver_matches_host_loop(tol, tol_fb, max_outer):
    """solve_ehl for a point contact without `collect` runs the loop on the
    device (paqif_ehl_point_drive_steps: stop / divergence tests after every
    iteration, force balance on the record's schedule, later iterations of
    a stopped chunk no-ops); with `collect` the host steps.  Same residual
    and force histories, state and outcome."""
    from paper_2008_03276_b200.ehl import solve_ehl
    from paper_2008_03276_b200.errors import NonConvergenceError
    p = params_for(100.0)
    out = []
    for collect in (None, lambda st, r, d: None):
        err, st = None, None
        try:
            st = solve_ehl(p, 32, tol=tol, tol_fb=tol_fb, max_outer=max_outer, collect=collect)
        except NonConvergenceError as e:
            err = (e.iterations, e.residual)
        out.append((err, st))
    (e_dev, s_dev), (e_host, s_host) = out
    assert e_dev == e_host
    if s_dev is not None:
        assert s_dev.residual_history == s_host.residual_history
        assert s_dev.force_history == s_host.force_history
        assert s_dev.outer_iterations == s_host.outer_iterations
        assert np.array_equal(s_dev.u, s_host.u) and s_dev.h0 == s_host.h0


def test_point_drive_stopped_chunk_is_noop():
    """A record that is already done turns a whole enqueued chunk into
    no-ops: the state does not move."""
    from paper_2008_03276_b200.ehl import PointContact
    pc = PointContact(params_for(100.0), 32)
    pc.drive_init(1e30, 1e30, 3, hist_cap=8)
    pc.drive_steps(6)
    d = pc.drive_state()
    assert d["done"] == 3 and d["outer"] == 3
    s1 = pc.snapshot()
    pc.drive_steps(4)
    d2 = pc.drive_state()
    s2 = pc.snapshot()
    assert d2["outer"] == 3 and np.array_equal(s1["u"], s2["u"]) and s1["h0"] == s2["h0"]
    pc.step()  # an explicit step runs again
    assert not np.array_equal(pc.snapshot()["u"], s2["u"])
    pc.close()
