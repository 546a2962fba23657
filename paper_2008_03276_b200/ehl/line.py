"""Batched line-contact Newton steps on the device (configs 1 and 3).

``LineContactBatch`` keeps B independent line contacts (same grid, per-case
load numbers) resident in HBM and advances all of them by one outer
iteration of solve_ehl per ``step()`` (csrc/ehl_line.cu, C ABI
include/paqif_ehl.h): one fused kernel launch (one CTA per case) for small
batches, or, from 2 x SM-count cases on (config 3), the split path -- phase
A per case, every case's ladder-rung systems solved side by side by the
throughput AQIF engine, phase C per case.  ``path`` forces either.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _native
from ..errors import ContractViolationError
from .kernels import kernel_line
from .params import EhlParams, hertzian_init

LIMITERS = {"kappa": 0, "none": 1, "van-albada": 2, "minmod": 3, "koren": 4}
SCHEMES = {"Lhs1": 0, "Lhs2": 1}


class LineCfg(ctypes.Structure):
    """Mirror of paqif_ehl_line_cfg (include/paqif_ehl.h)."""
    _fields_ = [("n", ctypes.c_int32), ("limiter", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("compressible", ctypes.c_int32),
                ("force_every", ctypes.c_int32), ("outer", ctypes.c_int32),
                ("h", ctypes.c_double), ("lo", ctypes.c_double), ("kappa", ctypes.c_double),
                ("omega", ctypes.c_double), ("max_change", ctypes.c_double),
                ("relax_c", ctypes.c_double), ("max_h0_step", ctypes.c_double),
                ("load_target", ctypes.c_double), ("alpha", ctypes.c_double),
                ("z", ctypes.c_double), ("p0", ctypes.c_double)]


def _bind(L):
    if getattr(L, "_ehl_bound", False):
        return L
    vp, i64, sz, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_uint32
    L.paqif_ehl_line_workspace_bytes.argtypes = [i64, i64]
    L.paqif_ehl_line_workspace_bytes.restype = sz
    L.paqif_ehl_line_step.argtypes = [ctypes.POINTER(LineCfg), i64, vp, vp, vp, vp, vp, vp, vp,
                                      vp, vp, u32, vp, sz, vp]
    L.paqif_ehl_line_step.restype = ctypes.c_int
    L.paqif_ehl_line_drive_steps.argtypes = [ctypes.POINTER(LineCfg), i64, ctypes.c_int32, vp,
                                             vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             ctypes.c_int32, u32, vp, sz, vp]
    L.paqif_ehl_line_drive_steps.restype = ctypes.c_int
    L.paqif_ehl_line_residual.argtypes = [ctypes.POINTER(LineCfg), i64, vp, vp, vp, vp, vp, vp,
                                          vp, vp]
    L.paqif_ehl_line_residual.restype = ctypes.c_int
    L.paqif_line_deformation.argtypes = [i64, i64, vp, vp, vp, vp]
    L.paqif_line_deformation.restype = ctypes.c_int
    L._ehl_bound = True
    return L


# mirror of paqif_ehl_line_drive (include/paqif_ehl.h)
DRIVE_DTYPE = np.dtype([("tol", "<f8"), ("tol_fb", "<f8"), ("best", "<f8"), ("deficit", "<f8"),
                        ("max_outer", "<i4"), ("outer", "<i4"), ("grow", "<i4"),
                        ("done", "<i4")])
DRIVE_RUNNING, DRIVE_CONVERGED, DRIVE_DIVERGING, DRIVE_BUDGET, DRIVE_BREAKDOWN, DRIVE_NONFINITE = \
    range(6)


def line_initial_state(params: EhlParams, intervals: int):
    """Hertzian start scaled to the load target (solver.py:54-73)."""
    lo, hi = params.domain
    h = (hi - lo) / intervals
    x = lo + h * np.arange(intervals + 1)
    u = hertzian_init(x)
    u[0] = u[-1] = 0.0
    u *= params.load_target / (np.pi / 2.0)
    return u


class LineContactBatch:
    """B line contacts on one grid, advanced together on the GPU."""

    def __init__(self, params_list, intervals: int, scheme: str = "Lhs1",
                 kappa: float = 1 / 3, limiter: str = "kappa", omega: float | None = None,
                 force_every: int = 5, exact: bool = True, u0=None, h0=None,
                 path: str = "auto"):
        torch = _native.torch_cuda()
        self.L = _bind(_native.lib())
        params_list = list(params_list)
        if path not in ("auto", "split", "fused"):
            raise ContractViolationError(f"unknown path {path!r}")
        if not params_list:
            raise ContractViolationError("empty batch")
        p = params_list[0]
        if any(q.contact != "line" for q in params_list):
            raise ContractViolationError("LineContactBatch needs line contacts")
        common = ("domain", "compressible", "alpha", "z", "p0", "relax_c", "max_change",
                  "max_h0_step", "load_target", "omega")
        for q in params_list[1:]:
            for f in common:
                if getattr(q, f) != getattr(p, f):
                    raise ContractViolationError(f"batched cases must share {f}")
        if scheme not in SCHEMES:
            raise ContractViolationError(f"unknown scheme {scheme!r}")
        if limiter not in LIMITERS:
            raise ContractViolationError(f"unknown limiter {limiter!r}")
        if not -1.0 <= kappa <= 1.0:
            raise ContractViolationError("kappa must lie in [-1, 1]")
        self.B = len(params_list)
        self.n = int(intervals)
        lo, hi = p.domain
        self.h = (hi - lo) / intervals
        self.cfg = LineCfg(n=self.n, limiter=LIMITERS[limiter], variant=SCHEMES[scheme],
                           compressible=1 if p.compressible else 0, force_every=force_every,
                           outer=0, h=self.h, lo=lo, kappa=kappa,
                           omega=p.omega if omega is None else omega, max_change=p.max_change,
                           relax_c=p.relax_c, max_h0_step=p.max_h0_step,
                           load_target=p.load_target, alpha=p.alpha, z=p.z, p0=p.p0)
        self.flags = (_native.FLAG_EXACT if exact else 0) | {
            "auto": 0, "split": _native.FLAG_LINE_SPLIT, "fused": _native.FLAG_LINE_FUSED}[path]
        dev = "cuda"
        N = self.n + 1
        self.table = torch.from_numpy(kernel_line(self.n, self.h).table).to(dev)
        self.p_hertz = torch.tensor([q.p_hertz for q in params_list], dtype=torch.float64,
                                    device=dev)
        self.lam = torch.tensor([q.lam for q in params_list], dtype=torch.float64, device=dev)
        if u0 is None:
            u0 = np.stack([line_initial_state(q, intervals) for q in params_list])
        self.u = torch.from_numpy(np.ascontiguousarray(u0, dtype=np.float64).reshape(self.B, N)
                                  ).to(dev)
        if h0 is None:
            h0 = [q.h0 for q in params_list]
        self.h0 = torch.tensor(np.broadcast_to(np.asarray(h0, dtype=np.float64), (self.B,)).copy(),
                               device=dev)
        self.film = torch.empty((self.B, N), dtype=torch.float64, device=dev)
        self.res = torch.empty(self.B, dtype=torch.float64, device=dev)
        self.deficit = torch.empty(self.B, dtype=torch.float64, device=dev)
        self.info = torch.empty(self.B, dtype=torch.int32, device=dev)
        nbytes = self.L.paqif_ehl_line_workspace_bytes(self.B, self.n)
        self.ws = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev)
        self.ws_bytes = nbytes
        self.outer = 0

    def step(self, stream=None) -> None:
        """One outer iteration for every case (asynchronous)."""
        self.cfg.outer = self.outer
        rc = self.L.paqif_ehl_line_step(ctypes.byref(self.cfg), self.B, self.table.data_ptr(),
                                        self.p_hertz.data_ptr(), self.lam.data_ptr(),
                                        self.u.data_ptr(), self.h0.data_ptr(),
                                        self.film.data_ptr(), self.res.data_ptr(),
                                        self.deficit.data_ptr(), self.info.data_ptr(),
                                        self.flags, self.ws.data_ptr(), self.ws_bytes,
                                        _native.stream_ptr(stream))
        _native.check(rc, "paqif_ehl_line_step")
        self.outer += 1

    def drive_init(self, tol: float, tol_fb: float, max_outer: int, hist_cap: int = 64):
        """Device solve_ehl state for every case (ehl/solver.py:210-240):
        the stop / divergence tests run on the GPU after each iteration."""
        torch = _native.torch_cuda()
        rec = np.zeros(self.B, dtype=DRIVE_DTYPE)
        rec["tol"], rec["tol_fb"] = tol, tol_fb
        rec["best"] = rec["deficit"] = np.inf
        rec["max_outer"], rec["outer"] = max_outer, self.outer
        self.drive = torch.from_numpy(rec.view(np.uint8)).cuda()
        self.hist_cap = int(hist_cap)
        self.hist_res = torch.empty((self.B, self.hist_cap), dtype=torch.float64, device="cuda")
        self.hist_def = torch.empty_like(self.hist_res)

    def drive_steps(self, steps: int, stream=None) -> None:
        """Enqueue `steps` device-driven iterations (stopped cases skip)."""
        rc = self.L.paqif_ehl_line_drive_steps(
            ctypes.byref(self.cfg), self.B, int(steps), self.table.data_ptr(),
            self.p_hertz.data_ptr(), self.lam.data_ptr(), self.u.data_ptr(), self.h0.data_ptr(),
            self.film.data_ptr(), self.res.data_ptr(), self.deficit.data_ptr(),
            self.info.data_ptr(), self.drive.data_ptr(), self.hist_res.data_ptr(),
            self.hist_def.data_ptr(), self.hist_cap, self.flags, self.ws.data_ptr(),
            self.ws_bytes, _native.stream_ptr(stream))
        _native.check(rc, "paqif_ehl_line_drive_steps")

    def drive_state(self):
        """Host copy of the drive records (numpy structured array)."""
        return self.drive.cpu().numpy().view(DRIVE_DTYPE).copy()

    def residual(self, stream=None) -> np.ndarray:
        """Complementarity residual of every case's current state (host array)."""
        torch = _native.torch_cuda()
        out = torch.empty(self.B, dtype=torch.float64, device="cuda")
        rc = self.L.paqif_ehl_line_residual(ctypes.byref(self.cfg), self.B, self.table.data_ptr(),
                                            self.p_hertz.data_ptr(), self.lam.data_ptr(),
                                            self.u.data_ptr(), self.h0.data_ptr(),
                                            self.film.data_ptr(), out.data_ptr(),
                                            _native.stream_ptr(stream))
        _native.check(rc, "paqif_ehl_line_residual")
        return out.cpu().numpy()

    def snapshot(self):
        """Host copies: (u, h0, film, res, deficit, info)."""
        return (self.u.cpu().numpy(), self.h0.cpu().numpy(), self.film.cpu().numpy(),
                self.res.cpu().numpy(), self.deficit.cpu().numpy(), self.info.cpu().numpy())


def line_deformation(table, u):
    """-(1/pi) sum_j table[|i-j|] u_j on the GPU for a (B, n+1) or (n+1,) array."""
    torch = _native.torch_cuda()
    L = _bind(_native.lib())
    u = np.asarray(u, dtype=np.float64)
    one = u.ndim == 1
    uu = np.ascontiguousarray(u[None] if one else u)
    B, N = uu.shape
    tt = torch.from_numpy(np.ascontiguousarray(table, dtype=np.float64)).cuda()
    tu = torch.from_numpy(uu).cuda()
    to = torch.empty_like(tu)
    rc = L.paqif_line_deformation(B, N - 1, tt.data_ptr(), tu.data_ptr(), to.data_ptr(),
                                  _native.stream_ptr())
    _native.check(rc, "paqif_line_deformation")
    out = to.cpu().numpy()
    return out[0] if one else out
