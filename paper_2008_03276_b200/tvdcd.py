"""TVD kappa-scheme linear study (the reference's paqif/tvdcd.py; the
paper's Sec. 6): ``(a u)_x + (b u)_y - eps Lap(u) = f`` on a uniform grid,
relaxed by x-line splittings whose line systems are solved with the AQIF
factorization.

The problem set-up (grid, scheme coefficients, stencil operator, line-band
arrays, manufactured quartic problem, transposed twin) is host numpy, as in
the reference, and runs once per problem.  The sweeps -- the part that
repeats -- run on the device: one CTA per sweep walks the x-lines in order
(residual line, padded AQIF line solve, relaxed update) and ends with the
residual norm in numpy's summation order (csrc/tvd_sweep.cu,
include/paqif_tvd.h), bit for bit the reference's iterates.  Lines with
varying coefficients are factored one by one on the beta = 2 latency
engine; constant-coefficient lines share one factorization, as in the
reference, and each line is then only W and Z solves.

Variants on the device: Ls0, Ls1, Ls2 (Gauss-Seidel line sweeps) and Ls3
(the line-distributive relaxation, tvdcd.py:615-656: all lines' changes
from the current iterate, one CTA per line).  DefC (a sparse direct
first-order solve, tvdcd.py:553-570) is not on the device path and raises
NotImplementedError.
"""

from __future__ import annotations

import ctypes as _ct
from dataclasses import dataclass, field

import numpy as np

from .errors import ContractViolationError, FactorizationBreakdownError

__all__ = [
    "Grid2D", "KappaSchemeConfig", "StencilOperator", "ConvectionDiffusionProblem",
    "quartic_test_problem", "assemble_kappa_operator", "sweep_splitting", "solve_by_sweeps",
    "transposed_problem", "error_norms", "convergence_order", "limiter_psi",
    "limiter_weight_plus", "inject_fine_to_coarse",
]

RATIO_GUARD = 1e-30
_LINE_OFFSETS = (-2, -1, 0, 1)


@dataclass
class Grid2D:
    """Uniform interior grid with Dirichlet boundary (tvdcd.py:40-75)."""
    x_lo: float
    x_hi: float
    y_lo: float
    y_hi: float
    nx: int
    ny: int

    def __post_init__(self):
        hx = (self.x_hi - self.x_lo) / (self.nx + 1)
        hy = (self.y_hi - self.y_lo) / (self.ny + 1)
        if abs(hx - hy) > 1e-12 * abs(hx):
            raise ContractViolationError("grid spacing must be uniform")

    @classmethod
    def square(cls, intervals: int, lo: float = -1.0, hi: float = 1.0):
        return cls(lo, hi, lo, hi, intervals - 1, intervals - 1)

    @property
    def h(self) -> float:
        return (self.x_hi - self.x_lo) / (self.nx + 1)

    def x_nodes(self) -> np.ndarray:
        return self.x_lo + self.h * np.arange(self.nx + 2)

    def y_nodes(self) -> np.ndarray:
        return self.y_lo + self.h * np.arange(self.ny + 2)

    def interior_mesh(self):
        return np.meshgrid(self.x_nodes()[1:-1], self.y_nodes()[1:-1])


@dataclass
class KappaSchemeConfig:
    """kappa in [-1, 1], limiter name, convection a, b (constants or
    callables of (x, y)), diffusion eps > 0 (tvdcd.py:78-98)."""
    kappa: float = 0.0
    limiter: str = "van-albada"
    a: float = 1.0
    b: float = 1.0
    eps: float = 1e-6

    def __post_init__(self):
        if not -1.0 <= self.kappa <= 1.0:
            raise ContractViolationError("kappa must lie in [-1, 1]")
        if self.eps <= 0.0:
            raise ContractViolationError("eps must be positive")

    def a_field(self, x, y):
        return self.a(x, y) if callable(self.a) else np.full_like(x, self.a)

    def b_field(self, x, y):
        return self.b(x, y) if callable(self.b) else np.full_like(x, self.b)


@dataclass
class StencilOperator:
    """Per-node coefficients at x offsets (cx), y offsets (cy) and the
    centre (tvdcd.py:101-134); fields carry a two-wide border."""
    cx: dict
    cy: dict
    c0: np.ndarray

    def _gather(self, u_full, rows):
        ny, nx = self.c0.shape
        out = self.c0[rows] * u_full[2:ny + 2][rows, 2:nx + 2]
        for o, c in self.cx.items():
            out += c[rows] * u_full[2:ny + 2][rows, 2 + o:nx + 2 + o]
        for o, c in self.cy.items():
            out += c[rows] * u_full[2 + o:ny + 2 + o][rows, 2:nx + 2]
        return out

    def apply(self, u_full: np.ndarray) -> np.ndarray:
        return self._gather(u_full, slice(None))

    def apply_line(self, u_full: np.ndarray, j: int) -> np.ndarray:
        return self._gather(u_full, j)

    def row_sums(self) -> np.ndarray:
        total = self.c0.copy()
        for c in list(self.cx.values()) + list(self.cy.values()):
            total += c
        return total


def _kappa_coeffs(kappa):
    """Upwind-biased weights for a > 0 at offsets -2..+1 (tvdcd.py:137-145)."""
    return ((1.0 - kappa) / 4.0, -1.0 + (3.0 * kappa - 1.0) / 4.0,
            1.0 - (1.0 + 3.0 * kappa) / 4.0, (1.0 + kappa) / 4.0)


def assemble_kappa_operator(cfg: KappaSchemeConfig, grid: Grid2D,
                            closure: str = "wide") -> StencilOperator:
    """Unlimited kappa-scheme convection + 5-point diffusion, "wide" or
    first-order "upwind" closure (tvdcd.py:148-204)."""
    h = grid.h
    gx, gy = grid.interior_mesh()
    a, b = cfg.a_field(gx, gy), cfg.b_field(gx, gy)
    if np.any(a < 0.0) or np.any(b < 0.0):
        raise ContractViolationError("upwind orientation assumes a, b >= 0 per cell")
    if closure not in ("wide", "upwind"):
        raise ContractViolationError(f"unknown closure {closure!r}")
    eps_h2 = cfg.eps / h ** 2
    w = _kappa_coeffs(cfg.kappa)
    ny, nx = a.shape
    cx = {o: np.zeros((ny, nx)) for o in (-2, -1, 1, 2)}
    cy = {o: np.zeros((ny, nx)) for o in (-2, -1, 1, 2)}
    diag = np.zeros((ny, nx))
    for vel, c, first in ((a, cx, (slice(None), 0)), (b, cy, (0, slice(None)))):
        c[-2] += (vel / h) * w[0]
        c[-1] += (vel / h) * w[1]
        diag += (vel / h) * w[2]
        c[1] += (vel / h) * w[3]
        if closure == "upwind":
            c[-2][first] = 0.0
            c[-1][first] = -vel[first] / h
            diag[first] += (vel[first] / h) * (1.0 - w[2])
            c[1][first] = 0.0
    for c in (cx, cy):
        c[-1] -= eps_h2
        c[1] -= eps_h2
    diag += 4.0 * eps_h2
    return StencilOperator(cx=cx, cy=cy, c0=diag)


@dataclass
class ConvectionDiffusionProblem:
    """Operator, right side f (ny, nx) and the two-wide Dirichlet data ring
    boundary (ny+4, nx+4) (tvdcd.py:312-343)."""
    grid: Grid2D
    cfg: KappaSchemeConfig
    f: np.ndarray
    boundary: np.ndarray
    closure: str = "wide"
    operator: StencilOperator = field(init=False)

    def __post_init__(self):
        self.operator = assemble_kappa_operator(self.cfg, self.grid, self.closure)

    def embed(self, u: np.ndarray) -> np.ndarray:
        full = self.boundary.copy()
        full[2:-2, 2:-2] = u
        return full

    def residual_field(self, u: np.ndarray) -> np.ndarray:
        return self.f - self.operator.apply(self.embed(u))

    def residual_norm(self, u: np.ndarray) -> float:
        r = self.residual_field(u)
        return float(np.sqrt(self.grid.h ** 2 * np.sum(r * r)))


def quartic_test_problem(intervals: int, cfg: KappaSchemeConfig):
    """Manufactured problem, exact solution x^4 + y^4 on [-1, 1]^2 with a
    two-deep data ring (tvdcd.py:345-371).  Returns (problem, exact on the
    solved nodes)."""
    if callable(cfg.a) or callable(cfg.b):
        raise ContractViolationError("the quartic case derives f for constant convection")
    if intervals < 8:
        raise ContractViolationError("study grids start at 8 intervals")
    h = 2.0 / intervals
    core = intervals - 3
    grid = Grid2D(-1.0 + h, 1.0 - h, -1.0 + h, 1.0 - h, core, core)
    xs = -1.0 + h * np.arange(intervals + 1)
    gxa, gya = np.meshgrid(xs, xs)
    exact = gxa ** 4 + gya ** 4
    gx, gy = grid.interior_mesh()
    f = (4.0 * cfg.a * gx ** 3 + 4.0 * cfg.b * gy ** 3
         - cfg.eps * (12.0 * gx ** 2 + 12.0 * gy ** 2))
    return ConvectionDiffusionProblem(grid, cfg, f, exact, closure="wide"), exact[2:-2, 2:-2]


def _line_system_coeffs(problem: ConvectionDiffusionProblem, variant: str) -> dict:
    """Band arrays (offset -> (ny, nx)) of the x-line operator of a
    splitting (tvdcd.py:374-416)."""
    cfg, grid = problem.cfg, problem.grid
    h = grid.h
    gx, gy = grid.interior_mesh()
    a, b = cfg.a_field(gx, gy), cfg.b_field(gx, gy)
    eps_h2 = cfg.eps / h ** 2
    k = cfg.kappa
    cm2, _, c0, cp1 = _kappa_coeffs(k)
    nu = {"Ls0": (5.0 - 3.0 * k) / 4.0, "Ls1": (2.0 - k) / 2.0, "Ls2": 1.0}.get(variant)
    if nu is None:
        raise ContractViolationError(f"unknown line variant {variant!r}")
    bands = {-1: -(a / h) * nu - eps_h2,
             0: (a / h) * nu + (b / h) * c0 + 4.0 * eps_h2,
             1: np.full_like(a, -eps_h2) + (0.0 if variant == "Ls2" else (a / h) * cp1)}
    if variant != "Ls2":
        bands[-2] = (a / h) * cm2
    if problem.closure == "upwind":
        bands[-1][:, 0] = -a[:, 0] / h - eps_h2
        bands[0][:, 0] = a[:, 0] / h + (b[:, 0] / h) * c0 + 4.0 * eps_h2
        bands[1][:, 0] = -eps_h2
        if -2 in bands:
            bands[-2][:, 0] = 0.0
        bands[0][0, :] += (b[0, :] / h) * (1.0 - c0)
    return bands


def _padded_even_order(nx: int) -> int:
    return nx + 1 if (nx + 1) % 2 == 0 else nx + 2


def _line_matrix(band_rows: dict, nx: int, beta: int):
    """Line matrix padded with pinned trailing unknowns to an even order
    (tvdcd.py:424-436)."""
    from .bandcore import BandedMatrix
    mat = BandedMatrix(_padded_even_order(nx), beta)
    mat.bands[beta, :] = 1.0
    for off, vals in band_rows.items():
        lo = max(0, -off)
        mat.bands[beta + off][lo:nx] = vals[lo:nx]
    mat.bands[beta, nx:] = 1.0
    mat._zero_out_of_range()
    return mat


def transposed_problem(problem: ConvectionDiffusionProblem) -> ConvectionDiffusionProblem:
    """x and y exchanged, so a y-sweep is an x-sweep of the twin
    (tvdcd.py:492-511)."""
    cfg = problem.cfg
    if callable(cfg.a) or callable(cfg.b):
        a_t = (lambda x, y: cfg.b(y, x)) if callable(cfg.b) else cfg.b
        b_t = (lambda x, y: cfg.a(y, x)) if callable(cfg.a) else cfg.a
    else:
        a_t, b_t = cfg.b, cfg.a
    cfg_t = KappaSchemeConfig(kappa=cfg.kappa, limiter=cfg.limiter, a=a_t, b=b_t, eps=cfg.eps)
    g = problem.grid
    grid_t = Grid2D(g.y_lo, g.y_hi, g.x_lo, g.x_hi, g.ny, g.nx)
    return ConvectionDiffusionProblem(grid_t, cfg_t, np.ascontiguousarray(problem.f.T),
                                      np.ascontiguousarray(problem.boundary.T),
                                      closure=problem.closure)


# ---------------------------------------------------------------- device path

class _TvdProblem(_ct.Structure):
    """Mirror of paqif_tvd_problem (include/paqif_tvd.h)."""
    _fields_ = [("nx", _ct.c_int32), ("ny", _ct.c_int32), ("kx", _ct.c_int32),
                ("ky", _ct.c_int32), ("ox", _ct.c_int32 * 4), ("oy", _ct.c_int32 * 4),
                ("line_mask", _ct.c_int32), ("reserved", _ct.c_int32),
                ("omega", _ct.c_double), ("h2", _ct.c_double), ("f", _ct.c_void_p),
                ("c0", _ct.c_void_p), ("cx", _ct.c_void_p), ("cy", _ct.c_void_p),
                ("lb", _ct.c_void_p), ("z2x2", _ct.c_void_p), ("zl", _ct.c_void_p),
                ("zr", _ct.c_void_p), ("ww", _ct.c_void_p), ("zf_beta", _ct.c_int32),
                ("reserved2", _ct.c_int32)]


def _lib():
    from . import _native
    L = _native.lib()
    if not getattr(L, "_tvd_bound", False):
        vp = _ct.c_void_p
        L.paqif_tvd_sweep.argtypes = [_ct.POINTER(_TvdProblem), vp, _ct.c_int32, _ct.c_int32,
                                      vp, vp, vp, vp]
        L.paqif_tvd_sweep.restype = _ct.c_int
        L.paqif_tvd_transpose.argtypes = [vp, _ct.c_int32, _ct.c_int32, vp, vp]
        L.paqif_tvd_transpose.restype = _ct.c_int
        L.paqif_tvd_distributive.argtypes = [_ct.POINTER(_TvdProblem), vp, vp, vp, _ct.c_double,
                                             _ct.c_double, vp, vp, vp, vp, vp, vp]
        L.paqif_tvd_distributive.restype = _ct.c_int
        L._tvd_bound = True
    return L


class _DeviceSplitting:
    """One problem's operator, line bands and buffers resident on the
    device for one line variant and omega."""

    def __init__(self, problem: ConvectionDiffusionProblem, variant: str, omega: float):
        from . import _native
        torch = _native.torch_cuda()
        self.variant = variant
        bands = _line_system_coeffs(problem, "Ls1" if variant == "Ls3" else variant)
        op = problem.operator
        ny, nx = problem.f.shape
        if len(op.cx) > 4 or len(op.cy) > 4 or any(abs(o) > 2 for o in list(op.cx) + list(op.cy)):
            raise ContractViolationError("stencil offsets must lie in -2..2")

        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

        zero = np.zeros((ny, nx))
        self.f = dev(problem.f)
        self.c0 = dev(op.c0)
        self.cx = dev(np.stack(list(op.cx.values())) if op.cx else zero[None])
        self.cy = dev(np.stack(list(op.cy.values())) if op.cy else zero[None])
        self.lb = dev(np.stack([bands.get(o, zero) for o in _LINE_OFFSETS]))
        self.resid = torch.empty((ny, nx), dtype=torch.float64, device="cuda")
        self.scal = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        s = _TvdProblem(nx=nx, ny=ny, kx=len(op.cx), ky=len(op.cy), line_mask=0, reserved=0,
                        omega=float(omega), h2=problem.grid.h ** 2)
        for t, o in enumerate(op.cx):
            s.ox[t] = o
        for t, o in enumerate(op.cy):
            s.oy[t] = o
        for t, o in enumerate(_LINE_OFFSETS):
            if o in bands:
                s.line_mask |= 1 << t
        s.f, s.c0, s.cx, s.cy, s.lb = (self.f.data_ptr(), self.c0.data_ptr(),
                                       self.cx.data_ptr(), self.cy.data_ptr(),
                                       self.lb.data_ptr())
        if variant == "Ls3":
            self._distributive_setup(problem, dev)
        # constant-coefficient problems share one line factorization, as
        # the reference caches it (tvdcd.py:466-477): factored once
        # (paqif_factor_batch), each line then only solve_w + solve_z
        cfg = problem.cfg
        if variant != "Ls3" and not (callable(cfg.a) or callable(cfg.b)) and all(
                np.ptp(c, axis=0).max() == 0.0 for c in bands.values()):
            from .aqif import factorize_wz
            beta = 2 if -2 in bands else 1
            fac = factorize_wz(_line_matrix({o: c[0] for o, c in bands.items()}, nx, beta))
            self.fac = [dev(a) for a in (fac.z2x2, fac.zl, fac.zr, fac.ww)]
            s.z2x2, s.zl, s.zr, s.ww = (t.data_ptr() for t in self.fac)
            s.zf_beta = beta
        self.struct = s
        self.shape = (ny, nx)
        self._bands = bands
        self._f_src = None

    def refresh_f(self, f: np.ndarray) -> None:
        """Re-upload the right side (the reference re-reads problem.f on
        every line, so edits between calls must be seen)."""
        from . import _native
        torch = _native.torch_cuda()
        self.f.copy_(torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)))

    def _distributive_setup(self, problem, dev):
        """Ls3's line operator and explicit-term weights
        (tvdcd.py:615-645), per node; they do not depend on the iterate."""
        from . import _native
        torch = _native.torch_cuda()
        grid, cfg = problem.grid, problem.cfg
        h, k, eps = grid.h, cfg.kappa, cfg.eps
        gx, gy = grid.interior_mesh()
        a = cfg.a_field(gx, gy)
        ny, nx = a.shape
        a_pad = np.pad(a, ((0, 0), (1, 1)), mode="edge")
        a_p = 0.5 * (a_pad[:, 1:-1] + a_pad[:, 2:])
        a_m = 0.5 * (a_pad[:, 1:-1] + a_pad[:, :-2])
        cm2 = eps / (4 * h ** 2) + a_m * (2 + k) / (8 * h)
        cm1 = -(7 * eps / (4 * h ** 2) + a_p * (2 + k) / (2 * h) + a_m * (2 + k) / (8 * h))
        c0 = 20 * eps / (4 * h ** 2) + a_p * (2 + k) / (2 * h) + a_m * (2 + k) / (8 * h)
        cp1 = -(8 * eps / (4 * h ** 2) + a_p * (2 + k) / (2 * h))
        cp2 = np.full((ny, nx), eps / (4 * h ** 2))
        self.db = dev(np.stack([cm2, cm1, c0, cp1, cp2]))
        self.ah = dev(a / h)
        self.k12 = ((1 + k) / 4.0, (1 - k) / 4.0)
        self.sigma = torch.empty((ny, nx), dtype=torch.float64, device="cuda")
        self.lst = torch.zeros(ny, dtype=torch.int32, device="cuda")

    def sweep(self, u_full, backward: bool, want_norm: bool) -> None:
        from . import _native
        L = _lib()
        if self.variant == "Ls3":
            _native.check(L.paqif_tvd_distributive(
                _ct.byref(self.struct), u_full.data_ptr(), self.ah.data_ptr(), self.db.data_ptr(),
                self.k12[0], self.k12[1], self.sigma.data_ptr(), self.lst.data_ptr(),
                self.resid.data_ptr(), self.scal.data_ptr(), self.status.data_ptr(),
                _native.stream_ptr()), "paqif_tvd_distributive")
            return
        _native.check(L.paqif_tvd_sweep(_ct.byref(self.struct), u_full.data_ptr(),
                                        1 if backward else 0, 1 if want_norm else 0,
                                        self.resid.data_ptr(), self.scal.data_ptr(),
                                        self.status.data_ptr(), _native.stream_ptr()),
                      "paqif_tvd_sweep")

    def check_status(self) -> None:
        st = int(self.status.item())
        if st:
            j = st - 1
            raise FactorizationBreakdownError(self._breakdown_level(j),
                                              f"x-line {j}: AQIF breakdown")

    def _breakdown_level(self, j: int) -> int:
        """1-based level at which line j's factorization breaks down (the
        reference's FactorizationBreakdownError.level), from the device
        engine on that line's matrix; error path only."""
        from .aqif import factorize_wz
        nx = self.shape[1]
        if self.variant == "Ls3":
            db = self.db.cpu().numpy()
            rows = {o: db[o + 2, j] for o in range(-2, 3)}
            beta = 2
        else:
            rows = {o: c[j] for o, c in self._bands.items()}
            beta = 2 if -2 in rows else 1
        try:
            factorize_wz(_line_matrix(rows, nx, beta))
        except FactorizationBreakdownError as exc:
            return exc.level
        return -1  # the Z solve broke down, not the factorization


def _device_splitting(problem, variant, omega) -> _DeviceSplitting:
    if variant == "DefC":
        raise NotImplementedError(
            "DefC (the sparse direct first-order baseline) is not on the device path "
            "-- see DESIGN.md")
    # keyed on the operator object too: a problem whose operator / grid was
    # replaced gets fresh device planes; f is re-uploaded on every call
    cache = problem.__dict__.setdefault("_device", {})
    key = (variant, float(omega), id(problem.operator), problem.closure, problem.f.shape)
    d = cache.get(key)
    if d is None:
        d = cache[key] = _DeviceSplitting(problem, variant, omega)
    d.refresh_f(problem.f)
    return d


def _transpose(src_full, ny, nx, dst_full):
    from . import _native
    _native.check(_lib().paqif_tvd_transpose(src_full.data_ptr(), ny, nx, dst_full.data_ptr(),
                                             _native.stream_ptr()), "paqif_tvd_transpose")


def sweep_splitting(problem: ConvectionDiffusionProblem, u: np.ndarray, variant: str,
                    omega: float = 1.0, order: str = "forward"):
    """One full x-line sweep of a splitting on the device (tvdcd.py:449-489).
    Returns (u_next, residual_norm)."""
    from . import _native
    torch = _native.torch_cuda()
    d = _device_splitting(problem, variant, omega)
    uf = torch.from_numpy(problem.embed(np.asarray(u, dtype=np.float64))).cuda()
    d.sweep(uf, order == "backward", True)
    d.check_status()
    return uf[2:-2, 2:-2].cpu().numpy(), float(d.scal[0].item())


def solve_by_sweeps(problem: ConvectionDiffusionProblem, variant: str, omega: float = 1.0,
                    tol: float = 1e-12, max_sweeps: int = 400, cycle: str = "alternate",
                    u0: np.ndarray | None = None):
    """Sweeps to the discrete solution (tvdcd.py:514-550), the iterate
    resident on the device: "x" = forward x-sweeps, "alternate" adds a
    y-sweep (x-sweep of the transposed twin), "symmetric" the reverse-order
    pair.  One host synchronisation per cycle (the stop test).  Returns
    (u, residual_history)."""
    from . import _native
    torch = _native.torch_cuda()
    passes = {"x": ("f",), "alternate": ("f", "tf"), "symmetric": ("f", "tf", "b", "tb")}
    if variant == "DefC":
        passes = {k: ("f",) for k in passes}
    if cycle not in passes:
        raise ContractViolationError(f"unknown cycle {cycle!r}")
    seq = passes[cycle]
    u = np.zeros_like(problem.f) if u0 is None else np.array(u0, dtype=np.float64)
    ny, nx = problem.f.shape
    d = _device_splitting(problem, variant, omega)
    uf = torch.from_numpy(problem.embed(u)).cuda()
    twin = dt = uft = None
    if any(p.startswith("t") for p in seq):
        twin = transposed_problem(problem)  # per call, as the reference builds it
        dt = _device_splitting(twin, variant, omega)
        uft = torch.from_numpy(np.ascontiguousarray(twin.boundary)).cuda()
    history = []
    for _ in range(max_sweeps):
        last = None
        for k, p in enumerate(seq):
            final = k == len(seq) - 1
            if p.startswith("t"):
                _transpose(uf, ny, nx, uft)
                dt.sweep(uft, p.endswith("b"), final)
                _transpose(uft, nx, ny, uf)
                last = dt
            else:
                d.sweep(uf, p.endswith("b"), final)
                last = d
        d.check_status()
        if dt is not None:
            dt.check_status()
        res = float(last.scal[0].item())
        history.append(res)
        if res <= tol:
            break
    return uf[2:-2, 2:-2].cpu().numpy(), history


# ---------------------------------------------------------------- host helpers

def limiter_psi(r, name, kappa=0.0):
    """Limited slope weight, backward-difference convention (tvdcd.py:207-225)."""
    r = np.asarray(r, dtype=np.float64)
    lin = ((1.0 + kappa) * r + (1.0 - kappa)) / 2.0
    if name == "none":
        return lin
    if name == "van-albada":
        return np.where(r > 0.0, (r * r + r) / (1.0 + r * r), 0.0)
    if name == "minmod":
        return np.maximum(0.0, np.minimum(r, 1.0))
    if name == "koren":
        return np.maximum(0.0, np.minimum(np.minimum(2.0 * r, (1.0 + 2.0 * r) / 3.0), 2.0))
    if name == "kappa":
        return np.maximum(0.0, np.minimum(np.minimum(2.0 * r, lin), 2.0))
    raise ContractViolationError(f"unknown limiter {name!r}")


def limiter_weight_plus(r, name, kappa=0.0):
    """psi(r) / r, the forward-difference convention (tvdcd.py:228-235)."""
    r = np.asarray(r, dtype=np.float64)
    psi = limiter_psi(r, name, kappa)
    safe = np.where(np.abs(r) > RATIO_GUARD, r, np.where(r >= 0.0, RATIO_GUARD, -RATIO_GUARD))
    return np.where(r > 0.0, psi / safe, 0.0)


def error_norms(u, reference, h: float, dim: int = 2, normalization: str = "max",
                ref_scale: float | None = None):
    """(L_inf, L_1, L_2) error norms (tvdcd.py:719-752)."""
    u, reference = np.asarray(u), np.asarray(reference)
    diff = u - reference
    if normalization == "max":
        scale = ref_scale if ref_scale is not None else np.max(np.abs(reference))
        s = diff / scale
        return (float(np.max(np.abs(s))), float(np.mean(np.abs(s))),
                float(np.sqrt(np.mean(s * s))))
    w = h ** dim
    linf = float(np.max(np.abs(diff)))
    l1 = float(w * np.sum(np.abs(diff)))
    l2 = float(np.sqrt(w * np.sum(diff * diff)))
    if normalization == "reference":
        linf /= np.max(np.abs(reference))
        l1 /= w * np.sum(np.abs(reference))
        l2 /= np.sqrt(w * np.sum(reference * reference))
    elif normalization != "absolute":
        raise ContractViolationError(f"unknown normalization {normalization!r}")
    return linf, l1, l2


def inject_fine_to_coarse(u_fine: np.ndarray) -> np.ndarray:
    return u_fine[1::2, 1::2]


def convergence_order(errors) -> list:
    """p = (log E(k-1) - log E(k)) / log 2 (tvdcd.py:761-766)."""
    e = list(errors)
    return [float((np.log(e[k - 1]) - np.log(e[k])) / np.log(2.0)) for k in range(1, len(e))]
