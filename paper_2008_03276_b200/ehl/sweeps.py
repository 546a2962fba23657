"""Line sweeps (public surface of paqif/ehl/sweeps.py:38-86, 344-535).

The line-contact Newton step is fused into one CUDA kernel
(csrc/ehl_line.cu).  The point-contact sweeps newton_line_sweep,
weighted_change_sweep and column_sweep run on the device state of a
PointContact (csrc/ehl_point.cu) attached to the EhlState's film model:
the state is uploaded, the 2(n-1)-line sweep runs as device kernels, and
the new pressure comes back into ``state.u``."""

from __future__ import annotations

import numpy as np

from ..errors import ContractViolationError

__all__ = ["hybrid_select", "kernel_nu", "force_balance_update", "SWITCH_THRESHOLD",
           "grid_spacing", "newton_line_sweep", "weighted_change_sweep", "column_sweep"]

_NEWTON = ("Ls0", "Ls1")
_WEIGHTED = ("Ls4", "Ls5")

SWITCH_THRESHOLD = 0.6
RATIO_GUARD = 1e-30


def grid_spacing(params, n: int) -> float:
    lo, hi = params.domain
    return (hi - lo) / n


def hybrid_select(eps_over_h, variant: str):
    eps_over_h = np.asarray(eps_over_h)
    if variant == "Lhs1":
        return np.where(eps_over_h > SWITCH_THRESHOLD, "Ls1", "Ls4")
    if variant == "Lhs2":
        return np.where(eps_over_h > SWITCH_THRESHOLD, "Ls0", "Ls5")
    raise ContractViolationError(f"unknown hybrid variant {variant!r}")


def kernel_nu(scheme: str, kappa: float) -> float:
    if scheme in ("Ls1", "Ls4", "Lhs1", "newton"):
        return (2.0 - kappa) / 2.0
    if scheme in ("Ls0", "Ls5", "Lhs2"):
        return (2.0 - kappa) / 2.0 + (1.0 - kappa) / 4.0
    raise ContractViolationError(f"unknown scheme {scheme!r}")


def force_balance_update(state, params):
    """h0 <- h0 - clip(c (target - h^d sum u), +-max_h0_step) (sweeps.py:521-535)."""
    n = state.u.shape[0] - 1
    h = grid_spacing(params, n)
    w = h if state.u.ndim == 1 else h * h
    deficit = params.load_target - w * float(np.sum(state.u))
    step = np.clip(params.relax_c * deficit, -params.max_h0_step, params.max_h0_step)
    state.h0 = state.h0 - step
    state.force_history.append(abs(deficit))
    return state.h0, deficit


def _nu_variant(scheme: str) -> int:
    kernel_nu(scheme, 0.0)  # validates the name
    return 0 if scheme in ("Ls1", "Ls4", "Lhs1", "newton") else 1


def _device_contact(state, params, kappa, limiter):
    from .point import PointContact
    film = state.film
    if getattr(film, "contact", None) != "point" or np.ndim(state.u) != 2:
        raise ContractViolationError("x/y line sweeps need a point-contact state")
    key = (id(params), float(kappa), str(limiter))
    pc = getattr(film, "_contact", None)
    if pc is None or pc._key != key:
        pc = PointContact(params, film.n, kappa=kappa, limiter=limiter, u0=state.u,
                          h0=state.h0)
        pc._key = key
        film._contact = pc
    else:
        pc.set_state(state.u, state.h0)
    return pc


def _finish(state, pc):
    from .point import PointContact
    snap = pc.snapshot()
    PointContact.raise_for(snap["err"])
    state.u = snap["u"]
    state.film._base = None  # deformation recomputed on the next film_full
    return snap["worst"]


def newton_line_sweep(state, params, kappa: float, limiter: str, scheme: str = "Ls1",
                      omega: float | None = None, hybrid: str | None = None) -> float:
    """x-sweep with immediate line updates (sweeps.py:344-379); ``hybrid``
    picks each line's system by min(eps)/h.  Returns the worst |resid|."""
    if hybrid is not None:
        hybrid_select(1.0, hybrid)
        sel, nu = -1, 0 if hybrid == "Lhs1" else 1
    else:
        if scheme not in _NEWTON + _WEIGHTED:
            raise ContractViolationError(f"unknown scheme {scheme!r}")
        sel, nu = (1 if scheme in _WEIGHTED else 0), _nu_variant(scheme)
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(1, sel, nu, params.omega if omega is None else omega)
    return _finish(state, pc)


def weighted_change_sweep(state, params, kappa: float, limiter: str, scheme: str = "Ls4",
                          omega: float | None = None) -> float:
    """x-sweep with deferred, distributed changes (sweeps.py:382-418)."""
    if scheme not in _NEWTON + _WEIGHTED:
        raise ContractViolationError(f"unknown scheme {scheme!r}")
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(2, 1 if scheme in _WEIGHTED else 0, _nu_variant(scheme),
             params.omega if omega is None else omega)
    return _finish(state, pc)


def column_sweep(state, params, kappa: float, limiter: str, omega: float | None = None) -> float:
    """y-sweep, tridiagonal column systems, immediate updates (sweeps.py:421-518)."""
    pc = _device_contact(state, params, kappa, limiter)
    pc.sweep(3, 0, 0, params.omega if omega is None else omega)
    return _finish(state, pc)


# ---------------------------------------------------------------------------
# Per-line building blocks on the GPU (csrc/ehl_linesys.cu, C ABI
# paqif_ehl_assemble_line / paqif_ehl_robust_line_solve /
# paqif_ehl_residual_field): the reference's arrays in, the same arrays out.
# ---------------------------------------------------------------------------

import ctypes as _ct

__all__ += ["reynolds_residual_field", "assemble_line_system", "robust_line_solve",
            "splitting_ls4", "splitting_ls5"]

_LIMITERS = {"kappa": 0, "none": 1, "van-albada": 2, "minmod": 3, "koren": 4}
_JACOBIANS = {"scheme": 0, "first-order": 1, "diagonal": 2}


class _LineSys(_ct.Structure):
    """Mirror of paqif_ehl_linesys (include/paqif_ehl.h)."""
    _fields_ = [("n", _ct.c_int32), ("limiter", _ct.c_int32), ("weighted", _ct.c_int32),
                ("reserved", _ct.c_int32), ("kappa", _ct.c_double), ("ks0", _ct.c_double),
                ("ks1", _ct.c_double), ("h", _ct.c_double), ("hy", _ct.c_double),
                ("q", _ct.c_void_p), ("rho", _ct.c_void_p), ("ex_p", _ct.c_void_p),
                ("ex_m", _ct.c_void_p), ("ey_p", _ct.c_void_p), ("ey_m", _ct.c_void_p),
                ("resid", _ct.c_void_p)]


class _Rheo(_ct.Structure):
    """Mirror of paqif_ehl_rheo."""
    _fields_ = [("compressible", _ct.c_int32), ("reserved", _ct.c_int32),
                ("alpha", _ct.c_double), ("z", _ct.c_double), ("p0", _ct.c_double),
                ("p_hertz", _ct.c_double), ("lam", _ct.c_double)]


def _lib():
    from .. import _native
    L = _native.lib()
    if not getattr(L, "_linesys_bound", False):
        vp = _ct.c_void_p
        L.paqif_ehl_assemble_line.argtypes = [_ct.POINTER(_LineSys), _ct.c_int32, vp, vp, vp]
        L.paqif_ehl_assemble_line.restype = _ct.c_int
        L.paqif_ehl_robust_line_solve.argtypes = [_ct.POINTER(_LineSys), vp, vp, vp]
        L.paqif_ehl_robust_line_solve.restype = _ct.c_int
        L.paqif_ehl_residual_field.argtypes = [vp, vp, _ct.c_int64, _ct.c_int32,
                                               _ct.POINTER(_Rheo), _ct.c_double, _ct.c_int32,
                                               _ct.c_double, vp, vp]
        L.paqif_ehl_residual_field.restype = _ct.c_int
        L._linesys_bound = True
    return L


def _kernel_strengths(scheme, kappa, film_model):
    """(weighted, ks0, ks1, hy) as assemble_line_system derives them
    (sweeps.py:186-199)."""
    if scheme not in _NEWTON + _WEIGHTED:
        raise ContractViolationError(f"unknown scheme {scheme!r}")
    weighted = scheme in _WEIGHTED
    sens = film_model.sensitivity
    point = film_model.contact == "point"
    if weighted:
        nu = kernel_nu(scheme, kappa)
        cross = 2.0 * sens(0, 1) if point else 0.0
        cross1 = 2.0 * sens(1, 1) if point else 0.0
        ks0 = nu * (sens(0) - 0.25 * (2.0 * sens(1) + cross))
        ks1 = nu * (sens(1) - 0.25 * (sens(0) + sens(2) + cross1))
    else:
        ks0, ks1 = sens(0), sens(1)
    return weighted, ks0, ks1, point


def _line_args(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, kappa, limiter,
               scheme, film_model, h):
    from .. import _native
    torch = _native.torch_cuda()
    if limiter not in _LIMITERS:
        raise ContractViolationError(f"unknown limiter {limiter!r}")
    n = int(np.asarray(u_line).size) - 1
    if n < 4:
        raise ContractViolationError("line too short")
    weighted, ks0, ks1, point = _kernel_strengths(scheme, kappa, film_model)

    def dev(a, size):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
        if a.size != size:
            raise ContractViolationError(f"expected {size} entries, got {a.size}")
        return torch.from_numpy(a).cuda()

    keep = [dev(q_line, n + 1), dev(rho_line, n + 1), dev(ex_p, n - 1), dev(ex_m, n - 1),
            dev(ey_p, n - 1), dev(ey_m, n - 1), dev(resid, n - 1)]
    a = _LineSys(n=n, limiter=_LIMITERS[limiter], weighted=1 if weighted else 0, reserved=0,
                 kappa=float(kappa), ks0=float(ks0), ks1=float(ks1), h=float(h),
                 hy=float(h) if point else 1.0, q=keep[0].data_ptr(), rho=keep[1].data_ptr(),
                 ex_p=keep[2].data_ptr(), ex_m=keep[3].data_ptr(), ey_p=keep[4].data_ptr(),
                 ey_m=keep[5].data_ptr(), resid=keep[6].data_ptr())
    return a, keep, n


def assemble_line_system(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params,
                         kappa: float, limiter: str, scheme: str, film_model, h: float,
                         jacobian: str = "scheme"):
    """Change system of one x-line: (BandedMatrix, rhs) (sweeps.py:157-267),
    assembled on the GPU."""
    from .. import _native
    from ..bandcore import BandedMatrix
    if jacobian not in _JACOBIANS:
        raise ContractViolationError(f"unknown jacobian {jacobian!r}")
    torch = _native.torch_cuda()
    a, keep, n = _line_args(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, kappa,
                            limiter, scheme, film_model, h)
    n_int = n - 1
    n_sys = n_int + 1 if (n_int + 1) % 2 == 0 else n_int + 2
    bands = torch.empty((5, n_sys), dtype=torch.float64, device="cuda")
    rhs = torch.empty(n_sys, dtype=torch.float64, device="cuda")
    L = _lib()
    _native.check(L.paqif_ehl_assemble_line(_ct.byref(a), _JACOBIANS[jacobian], bands.data_ptr(),
                                            rhs.data_ptr(), _native.stream_ptr()),
                  "paqif_ehl_assemble_line")
    return BandedMatrix(n_sys, 2, bands.cpu().numpy()), rhs.cpu().numpy()


def splitting_ls4(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params, kappa,
                  limiter, film_model, h):
    """Distributive line system with the plain kernel strength."""
    return assemble_line_system(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params,
                                kappa, limiter, "Ls4", film_model, h)


def splitting_ls5(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params, kappa,
                  limiter, film_model, h):
    """Distributive line system with the reinforced kernel strength."""
    return assemble_line_system(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params,
                                kappa, limiter, "Ls5", film_model, h)


def robust_line_solve(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, params, kappa,
                      limiter, scheme, film_model, h):
    """Solve the line system, degrading the linearization until the
    factorization succeeds (sweeps.py:270-295); one kernel: assembly and
    the AQIF solve per rung on the GPU."""
    from .. import _native
    from ..errors import FactorizationBreakdownError
    torch = _native.torch_cuda()
    a, keep, n = _line_args(u_line, q_line, rho_line, ex_p, ex_m, ey_p, ey_m, resid, kappa,
                            limiter, scheme, film_model, h)
    sigma = torch.empty(n - 1, dtype=torch.float64, device="cuda")
    rung = torch.empty(1, dtype=torch.int32, device="cuda")
    L = _lib()
    _native.check(L.paqif_ehl_robust_line_solve(_ct.byref(a), sigma.data_ptr(), rung.data_ptr(),
                                                _native.stream_ptr()),
                  "paqif_ehl_robust_line_solve")
    if int(rung.item()) < 0:
        raise FactorizationBreakdownError(-1, "every line-system rung broke down")
    return sigma.cpu().numpy()


def reynolds_residual_field(u, film, params, kappa: float, limiter: str) -> np.ndarray:
    """Residual of the discrete balance on all interior nodes, boundary
    entries zero (sweeps.py:106-138); 1-d arrays for the line contact,
    u[j, i] for the point contact."""
    from .. import _native
    if limiter not in _LIMITERS:
        raise ContractViolationError(f"unknown limiter {limiter!r}")
    torch = _native.torch_cuda()
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    film = np.array(np.broadcast_to(np.asarray(film, dtype=np.float64), u.shape))
    point = u.ndim == 2
    n = u.shape[0] - 1
    h = grid_spacing(params, n)
    tu, tf = torch.from_numpy(u).cuda(), torch.from_numpy(film).cuda()
    out = torch.empty_like(tu)
    rp = _Rheo(compressible=1 if params.compressible else 0, reserved=0, alpha=params.alpha,
               z=params.z, p0=params.p0, p_hertz=params.p_hertz, lam=params.lam)
    L = _lib()
    _native.check(L.paqif_ehl_residual_field(tu.data_ptr(), tf.data_ptr(), n, 1 if point else 0,
                                             _ct.byref(rp), h, _LIMITERS[limiter], float(kappa),
                                             out.data_ptr(), _native.stream_ptr()),
                  "paqif_ehl_residual_field")
    return out.cpu().numpy()
