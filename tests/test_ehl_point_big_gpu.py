"""Point contact at the CONFIGURED grids (configs 4 and 5) vs the reference.

Goldens (tests/golden/make_golden_point_big.py, produced by running the
reference in the build container):
  ehl_point_c4.npz       513^2, M=100: teacher-forced outer iterations from
                         the adapted Hertz start (k=0) and the reference's
                         state after 2 iterations (k=2), full fields
  ehl_point_c5.npz       2049^2, M=1000: one outer iteration from the adapted
                         Hertz start, as a digest (cavitated bitmap, per-row
                         max / L1, 8 full rows and columns, tags, rungs)
  ehl_point_films513.npz FilmModel with 8 pending line updates (the
                         multi-segment register-tiled films path) and the
                         fold on the 9th, at 513^2

Protocol SURVEY.md 8(c) P2: identical x-sweep Newton/weighted decisions and
ladder rungs, identical cavitated set, pressure and film within 1e-9
relative (exact and FMA arithmetic), same h0 and residual.
"""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
TOL = 1e-9


def params_for(m, l=10.0):
    from paper_2008_03276_b200.ehl import EhlParams
    return EhlParams.point_from_moes(m, l, domain=(-4.5, 1.5), lo_y=-3.0)


def rel_max(got, ref):
    return float(np.max(np.abs(got - ref))) / max(1.0, float(np.max(np.abs(ref))))


def _g(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path)


@pytest.mark.parametrize("key", ["e0", "e1"])
@pytest.mark.parametrize("exact", [True, False])
def test_config4_single_step_vs_reference(key, exact):
    from paper_2008_03276_b200.ehl import PointContact
    G = _g("ehl_point_c4.npz")
    d = {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(key + "__")}
    m, l, n, k = d["meta"]
    p = params_for(float(m), float(l))
    assert p.p_hertz == float(d["p_hertz"]) and p.lam == float(d["lam"])
    if int(k) == 0:
        from paper_2008_03276_b200.ehl import point_initial_state
        assert np.array_equal(point_initial_state(p, int(n)), d["u_in"]), "adapted Hertz start"
    # the x half-step alone (hybrid x-sweep, kind 0)
    px = PointContact(p, int(n), u0=d["u_in"], h0=float(d["h0_in"]), exact=exact)
    px.sweep(0)
    sx = px.snapshot()
    px.close()
    assert rel_max(sx["u"], d["u_x"]) <= TOL
    assert np.array_equal(sx["u"] == 0.0, d["u_x"] == 0.0)
    # the whole outer iteration
    pc = PointContact(p, int(n), u0=d["u_in"], h0=float(d["h0_in"]), exact=exact)
    pc.outer = int(k)
    pc.step()
    s = pc.snapshot()
    pc.close()
    assert s["err"] == 0
    assert np.array_equal(s["newton"], d["newton"]), "x-sweep Newton/weighted decisions"
    assert np.array_equal(np.asarray(s["x_rungs"]), d["x_rungs"]), "x-line ladder rungs"
    assert np.array_equal(np.asarray(s["y_rungs"]), d["y_rungs"]), "column ladder rungs"
    assert rel_max(s["u"], d["u_out"]) <= TOL
    assert np.array_equal(s["u"] == 0.0, d["u_out"] == 0.0), "cavitated set differs"
    assert math.isclose(s["h0"], float(d["h0_out"]), rel_tol=1e-13, abs_tol=1e-15)
    assert rel_max(s["film"], d["film_out"]) <= TOL
    assert math.isclose(s["res"], float(d["res_out"]), rel_tol=TOL)


@pytest.mark.parametrize("exact", [True, False])
def test_config5_single_step_vs_reference(exact):
    from paper_2008_03276_b200.ehl import PointContact, point_initial_state
    D = _g("ehl_point_c5.npz")
    m, l, n, k = D["meta"]
    p = params_for(float(m), float(l))
    assert p.p_hertz == float(D["p_hertz"]) and p.lam == float(D["lam"])
    rows = D["digest_rows"]
    u0 = point_initial_state(p, int(n))
    assert np.array_equal(u0[rows], D["in_rows"]) and np.array_equal(u0[:, rows].T, D["in_cols"])
    assert np.array_equal(np.abs(u0).sum(axis=1), D["in_row_l1"]), "adapted Hertz start"
    pc = PointContact(p, int(n), u0=u0, h0=float(D["h0_in"]), exact=exact)
    pc.outer = int(k)
    pc.step()
    s = pc.snapshot()
    pc.close()
    assert s["err"] == 0
    assert np.array_equal(s["newton"], D["newton"]), "x-sweep Newton/weighted decisions"
    assert np.array_equal(np.asarray(s["x_rungs"]), D["x_rungs"]), "x-line ladder rungs"
    assert np.array_equal(np.asarray(s["y_rungs"]), D["y_rungs"]), "column ladder rungs"
    u, film = s["u"], s["film"]
    cav = np.unpackbits(D["cav_bits"])[:u.size].reshape(u.shape).astype(bool)
    assert np.array_equal(u == 0.0, cav), f"cavitated set differs at {int(np.sum((u == 0.0) != cav))} nodes"
    umax = float(np.max(np.abs(u)))
    for name, got, ref in (("u_row_max", np.abs(u).max(axis=1), D["u_row_max"]),
                           ("film_row_max", np.abs(film).max(axis=1), D["film_row_max"])):
        assert np.max(np.abs(got - ref)) <= TOL * max(1.0, float(np.max(ref))), name
    for name, got, ref in (("u_row_l1", np.abs(u).sum(axis=1), D["u_row_l1"]),
                           ("film_row_l1", np.abs(film).sum(axis=1), D["film_row_l1"])):
        assert np.max(np.abs(got - ref) / np.maximum(ref, 1.0)) <= TOL, name
    assert np.max(np.abs(u[rows] - D["u_rows"])) <= TOL * max(1.0, umax)
    assert np.max(np.abs(u[:, rows].T - D["u_cols"])) <= TOL * max(1.0, umax)
    fmax = max(1.0, float(np.max(np.abs(D["film_rows"]))))
    assert np.max(np.abs(film[rows] - D["film_rows"])) <= TOL * fmax
    assert np.max(np.abs(film[:, rows].T - D["film_cols"])) <= TOL * fmax
    assert math.isclose(s["h0"], float(D["h0_out"]), rel_tol=1e-13, abs_tol=1e-15)
    assert math.isclose(s["res"], float(D["res_out"]), rel_tol=TOL)


def test_films_513_pending_vs_reference():
    """8 pending row/column updates (the multi-segment register-tiled
    corrections at n >= 256), then the fold on the 9th, vs the reference's
    FilmModel."""
    from paper_2008_03276_b200.ehl import FilmModel
    G4 = _g("ehl_point_c4.npz")
    F = _g("ehl_point_films513.npz")
    n = 512
    p = params_for(100.0)
    h = (p.domain[1] - p.domain[0]) / n
    fm = FilmModel("point", n, h, p.domain[0], lo_y=-3.0)
    u = G4["e1__u_in"]
    h0 = float(F["h0"])
    fm.deformation_full(u)
    axes, idxs, deltas = F["note_axis"], F["note_idx"], F["note_delta"]

    def check(q):
        mode, idx, val = int(F[f"read{q}_mode"]), list(F[f"read{q}_idx"]), F[f"read{q}_val"]
        got = fm.film_rows(idx, h0) if mode == 0 else fm.film_cols(idx, h0)
        assert np.max(np.abs(got - val)) <= 1e-12 * float(np.max(np.abs(val))), q

    for k in range(8):
        fm.note_line_update("row" if axes[k] == 0 else "col", int(idxs[k]), deltas[k], u)
    check(0)
    check(1)
    fm.note_line_update("row" if axes[8] == 0 else "col", int(idxs[8]), deltas[8], u)
    check(2)
    check(3)


@pytest.mark.parametrize("n", [512, 2048])
def test_fft_deformation_vs_scipy_configured(n):
    """The device fold (power-of-two period P = 1024 / 4096) against the
    reference's scipy rfftn on next_fast_len(3n+1) at the configured grids."""
    from oracle import ehl_point_oracle as P
    from paper_2008_03276_b200.ehl import FilmModel
    c = P.point_case(100.0, 10.0)
    f = P.PointFilm(n, c)
    rng = np.random.default_rng(n)
    u = np.maximum(0.0, rng.standard_normal((n + 1, n + 1)))
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    ref = f.deformation_full(u)
    fm = FilmModel("point", n, f.h, c.lo, lo_y=c.lo_y)
    got = fm.deformation_full(u)
    assert np.max(np.abs(got - ref)) <= 1e-12 * float(np.max(np.abs(ref)))
