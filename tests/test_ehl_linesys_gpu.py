"""Per-line building blocks of paqif/ehl/sweeps.py on the GPU
(csrc/ehl_linesys.cu: assemble_line_system, splitting_ls4/ls5,
robust_line_solve, reynolds_residual_field) vs the reference's outputs on
the same inputs (golden ehl_linesys.npz, tests/golden/make_golden_linesys.py:
point-contact x-lines from recorded states through the reference's own
_line_quantities, line-contact lines with ey = 0)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

S = load_golden("ehl_linesys.npz")
GP = load_golden("ehl_point.npz")
GL = load_golden("ehl_line.npz")
NAMES = sorted({k.split("__")[0] for k in S.files if not k.startswith("f_")})
FILMS = sorted({k.split("__")[0] for k in S.files if k.startswith("f_")})


def case(name):
    return {k.split("__", 1)[1]: S[k] for k in S.files if k.startswith(name + "__")}


def model_for(d):
    from paper_2008_03276_b200.ehl import EhlParams, FilmModel, moes_convert
    src = str(d["src"])
    if str(d["contact"]) == "point":
        m, l, n, _ = GP[f"{src}__meta"]
        p = EhlParams.point_from_moes(float(m), float(l), domain=(-4.5, 1.5), lo_y=-3.0)
        n = int(n)
        h = (p.domain[1] - p.domain[0]) / n
        return p, FilmModel("point", n, h, p.domain[0], lo_y=-3.0)
    m, l, n = GL[f"{src}__meta"][:3]
    u_, w_ = moes_convert(m=float(m), l=float(l), g=5000.0)
    p = EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))
    n = int(n)
    h = (p.domain[1] - p.domain[0]) / n
    return p, FilmModel("line", n, h, p.domain[0])


def args(d):
    return (d["u_line"], d["q_line"], d["rho_line"], d["ex_p"], d["ex_m"], d["ey_p"], d["ey_m"],
            d["resid"])


def rel(got, ref):
    return float(np.max(np.abs(got - ref)) / max(1e-300, float(np.max(np.abs(ref)))))


@pytest.mark.parametrize("name", NAMES)
def test_assemble_line_system(name):
    from paper_2008_03276_b200.ehl import sweeps
    d = case(name)
    p, fm = model_for(d)
    mat, rhs = sweeps.assemble_line_system(*args(d), p, 1.0 / 3.0, str(d["limiter"]),
                                           str(d["scheme"]), fm, float(d["h"]),
                                           jacobian=str(d["jac"]))
    assert mat.bands.shape == d["bands"].shape
    assert rel(mat.bands, d["bands"]) <= 1e-12
    assert np.array_equal(mat.bands == 0.0, d["bands"] == 0.0), "band sparsity differs"
    assert np.array_equal(rhs, d["rhs"])


@pytest.mark.parametrize("name", NAMES)
def test_robust_line_solve(name):
    from paper_2008_03276_b200.ehl import sweeps
    d = case(name)
    p, fm = model_for(d)
    sigma = sweeps.robust_line_solve(*args(d), p, 1.0 / 3.0, str(d["limiter"]), str(d["scheme"]),
                                     fm, float(d["h"]))
    assert rel(sigma, d["sigma"]) <= 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_reynolds_residual_field(name):
    from paper_2008_03276_b200.ehl import sweeps
    d = case(name)
    p, _ = model_for(d)
    r = sweeps.reynolds_residual_field(d["u"], d["film"], p, 1.0 / 3.0, str(d["limiter"]))
    assert r.shape == d["field"].shape
    assert rel(r, d["field"]) <= 1e-12


def test_splitting_aliases():
    from paper_2008_03276_b200.ehl import sweeps
    d = case(NAMES[0])
    p, fm = model_for(d)
    a4 = sweeps.splitting_ls4(*args(d), p, 1.0 / 3.0, str(d["limiter"]), fm, float(d["h"]))
    b4 = sweeps.assemble_line_system(*args(d), p, 1.0 / 3.0, str(d["limiter"]), "Ls4", fm,
                                     float(d["h"]))
    assert np.array_equal(a4[0].bands, b4[0].bands)
    a5 = sweeps.splitting_ls5(*args(d), p, 1.0 / 3.0, str(d["limiter"]), fm, float(d["h"]))
    assert not np.array_equal(a5[0].bands, a4[0].bands)


def test_contract_errors():
    from paper_2008_03276_b200.errors import ContractViolationError
    from paper_2008_03276_b200.ehl import sweeps
    d = case(NAMES[0])
    p, fm = model_for(d)
    with pytest.raises(ContractViolationError):
        sweeps.assemble_line_system(*args(d), p, 1.0 / 3.0, "kappa", "Ls1", fm, float(d["h"]),
                                    jacobian="bogus")
    with pytest.raises(ContractViolationError):
        sweeps.assemble_line_system(*args(d), p, 1.0 / 3.0, "kappa", "Ls9", fm, float(d["h"]))


@pytest.mark.parametrize("name", FILMS)
def test_film_pending_updates(name):
    """FilmModel.note_line_update / film_rows / film_cols on the device list
    of pending line updates (exact corrections, fold past 8 pending) vs the
    reference's sequence."""
    from paper_2008_03276_b200.ehl import EhlParams, FilmModel
    d = case(name)
    m, l, n, _ = GP[f"{str(d['src'])}__meta"]
    n = int(n)
    p = EhlParams.point_from_moes(float(m), float(l), domain=(-4.5, 1.5), lo_y=-3.0)
    h = (p.domain[1] - p.domain[0]) / n
    fm = FilmModel("point", n, h, p.domain[0], lo_y=-3.0)
    u, h0 = d["u"], float(d["h0"])
    with pytest.raises(Exception):
        fm.film_rows([1], h0)  # before deformation_full
    fm.deformation_full(u)

    def check(q):
        mode, idx, val = int(d[f"read{q}_mode"]), list(d[f"read{q}_idx"]), d[f"read{q}_val"]
        got = fm.film_rows(idx, h0) if mode == 0 else fm.film_cols(idx, h0)
        assert rel(got, val) <= 1e-12

    axes, idxs, deltas = d["note_axis"], d["note_idx"], d["note_delta"]
    for k in range(len(axes)):
        fm.note_line_update("row" if axes[k] == 0 else "col", int(idxs[k]), deltas[k], u)
        if k == 4:
            check(0)
            check(1)
            fm.note_line_update("row", 5, np.zeros(n + 1), u)  # ignored
    check(2)
