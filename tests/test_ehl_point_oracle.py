"""Point-contact oracle (oracle/ehl_point_oracle.py) pinned against
teacher-forced reference outer iterations (tests/golden/make_golden_point.py)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import ehl_point_oracle as P

G = load_golden("ehl_point.npz")
KEYS = sorted({k.split("__")[0] for k in G.files if k.startswith("e")}, key=lambda s: int(s[1:]))


def gcase(key):
    return {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(key + "__")}


def test_initial_state_matches_adapter():
    d = gcase(KEYS[0])
    c = P.PointCase(p_hertz=float(d["p_hertz"]), lam=float(d["lam"]))
    film = P.PointFilm(32, c)
    assert np.array_equal(P.hertz_start(c, film), G["init__u"])


@pytest.mark.parametrize("key", KEYS)
def test_point_step_matches_reference(key):
    d = gcase(key)
    m, l, n, k = d["meta"]
    c = P.PointCase(p_hertz=float(d["p_hertz"]), lam=float(d["lam"]))
    assert P.point_case(float(m), float(l)).p_hertz == c.p_hertz
    film = P.PointFilm(int(n), c)
    u, h0, fv, res, info = P.point_step(d["u_in"], float(d["h0_in"]), int(k), c, film)
    assert np.array_equal(info["tags"], d["newton"])
    for got, ref in ((info["u_x"], d["u_x"]), (u, d["u_out"]), (fv, d["film_out"])):
        assert np.max(np.abs(got - ref)) <= 1e-11 * max(1.0, float(np.max(np.abs(ref))))
    assert np.array_equal(u == 0.0, d["u_out"] == 0.0)
    assert h0 == pytest.approx(float(d["h0_out"]), rel=1e-13)
    assert res == pytest.approx(float(d["res_out"]), rel=1e-9)


S = load_golden("ehl_point_sweeps.npz")
SWEEPS = sorted({k.split("__")[0] for k in S.files})


def sweep_case(name):
    d = {k.split("__", 1)[1]: S[k] for k in S.files if k.startswith(name + "__")}
    src = gcase(str(d["src"]))
    return d, src


def run_oracle_sweep(d, src):
    m, l, n, k = src["meta"]
    c = P.PointCase(p_hertz=float(src["p_hertz"]), lam=float(src["lam"]))
    film = P.PointFilm(int(n), c)
    u = src["u_in"].copy()
    h0 = float(src["h0_in"])
    film.deformation_full(u)
    call, lim = str(d["call"]), str(d["limiter"])
    kappa = 1.0 / 3.0
    if call == "newton":
        hyb = str(d["hybrid"]) or None
        return P.newton_line_sweep(u, h0, film, c, kappa, lim, scheme=str(d["scheme"]) or "Ls1",
                                   hybrid=hyb)
    if call == "weighted":
        return P.weighted_change_sweep(u, h0, film, c, kappa, lim, scheme=str(d["scheme"]))
    if call == "column":
        st = {}
        u, _ = P.column_sweep(u, h0, film, c, kappa, lim, stats=st)
        return u, st["worst"]
    return u, P.complementarity_residual(u, h0, c, film, kappa, lim)


@pytest.mark.parametrize("name", SWEEPS)
def test_sweep_functions_match_reference(name):
    d, src = sweep_case(name)
    u, val = run_oracle_sweep(d, src)
    ref = d["u_out"]
    assert np.max(np.abs(u - ref)) <= 1e-11 * max(1.0, float(np.max(np.abs(ref))))
    assert np.array_equal(u == 0.0, ref == 0.0)
    assert val == pytest.approx(float(d["value"]), rel=1e-10)
