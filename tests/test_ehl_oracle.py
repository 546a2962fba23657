"""The EHL line-step oracle (oracle/ehl_oracle.py) pinned against
teacher-forced reference steps (tests/golden/make_golden_ehl.py)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import ehl_oracle as E

G = load_golden("ehl_line.npz")
KEYS = sorted({k.split("__")[0] for k in G.files if k.startswith("e")}, key=lambda s: int(s[1:]))


def case(key):
    d = {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(key + "__")}
    m, l, intervals, k, g = d["meta"]
    c = E.LineCase(p_hertz=float(d["p_hertz"]), lam=float(d["lam"]))
    return d, c, int(intervals), int(k)


def test_case_parameters_rederive():
    d, c, n, _ = case(KEYS[0])
    m, l = float(d["meta"][0]), float(d["meta"][1])
    c2 = E.line_case(m, l)
    assert c2.p_hertz == c.p_hertz and c2.lam == c.lam


@pytest.mark.parametrize("key", KEYS)
def test_line_step_matches_reference(key):
    d, c, n, k = case(key)
    film = E.LineFilm(n, c)
    u, h0, fv, res, info = E.line_step(d["u_in"], float(d["h0_in"]), k, c, film)
    scale = max(1.0, float(np.max(np.abs(d["u_out"]))))
    assert np.max(np.abs(u - d["u_out"])) <= 1e-12 * scale
    assert np.array_equal(u == 0.0, d["u_out"] == 0.0)
    assert h0 == pytest.approx(float(d["h0_out"]), rel=1e-14, abs=1e-15)
    assert np.max(np.abs(fv - d["film_out"])) <= 1e-12 * max(1.0, np.max(np.abs(fv)))
    assert res == pytest.approx(float(d["res_out"]), rel=1e-9)
    assert (info["rung"] != "combined") == (int(d["breaks"]) > 0)
    assert info["fb_applied"] == bool(d["fb_applied"])


def test_goldens_exercise_the_breakdown_ladder():
    assert sum(int(G[k + "__breaks"]) for k in KEYS) >= 3


def test_short_trajectory():
    c = E.line_case(20.0, 10.0)
    film = E.LineFilm(128, c)
    u = E.hertz_start(c, film)
    h0 = c.h0
    for k in range(8):
        u, h0, _, res, _ = E.line_step(u, h0, k, c, film)
        ref = G["traj__u"][k]
        assert np.max(np.abs(u - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))
        assert res == pytest.approx(float(G["traj__res"][k]), rel=1e-8)
