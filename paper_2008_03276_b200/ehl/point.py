"""Point-contact Newton steps on the device (configs 4 and 5).

``PointContact`` owns one circular point contact on an (n+1)^2 grid in HBM
(handle ``paqif_ehl_point``, csrc/ehl_point.cu, C ABI include/paqif_ehl.h)
and advances it by one outer iteration of solve_ehl per ``step()``:
the hybrid x-sweep (ehl/solver.py:76-128), the column sweep
(ehl/sweeps.py:421-518), the force balance every ``force_every`` iterations
and the complementarity residual.  The 2(n-1) line solves, the exact
pending-line film corrections and the FFT folds are all device kernels
enqueued by a native host loop on the handle's stream.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _native
from ..errors import ContractViolationError, FactorizationBreakdownError, PaqifError
from .kernels import kernel_point
from .params import EhlParams, hertzian_init

LIMITERS = {"kappa": 0, "none": 1, "van-albada": 2, "minmod": 3, "koren": 4}
SCHEMES = {"Lhs1": 0, "Lhs2": 1}


class PointCfg(ctypes.Structure):
    """Mirror of paqif_ehl_point_cfg (include/paqif_ehl.h)."""
    _fields_ = [("n", ctypes.c_int32), ("limiter", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("compressible", ctypes.c_int32),
                ("force_every", ctypes.c_int32), ("outer", ctypes.c_int32),
                ("h", ctypes.c_double), ("kappa", ctypes.c_double),
                ("omega", ctypes.c_double), ("max_change", ctypes.c_double),
                ("relax_c", ctypes.c_double), ("max_h0_step", ctypes.c_double),
                ("load_target", ctypes.c_double), ("alpha", ctypes.c_double),
                ("z", ctypes.c_double), ("p0", ctypes.c_double),
                ("p_hertz", ctypes.c_double), ("lam", ctypes.c_double)]


def _bind(L):
    if getattr(L, "_ehl_point_bound", False):
        return L
    vp, i32, u32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
    L.paqif_ehl_point_create.argtypes = [ctypes.POINTER(PointCfg), vp, vp]
    L.paqif_ehl_point_create.restype = vp
    L.paqif_ehl_point_destroy.argtypes = [vp]
    L.paqif_ehl_point_destroy.restype = None
    L.paqif_ehl_point_set_state.argtypes = [vp, vp, f64]
    L.paqif_ehl_point_set_state.restype = ctypes.c_int
    L.paqif_ehl_point_step.argtypes = [vp, i32, u32]
    L.paqif_ehl_point_step.restype = ctypes.c_int
    L.paqif_ehl_point_drive_steps.argtypes = [vp, i32, vp, vp, vp, i32, u32]
    L.paqif_ehl_point_drive_steps.restype = ctypes.c_int
    L.paqif_ehl_point_get.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.paqif_ehl_point_get.restype = ctypes.c_int
    L.paqif_ehl_point_stream.argtypes = [vp]
    L.paqif_ehl_point_stream.restype = vp
    L.paqif_ehl_point_sync.argtypes = [vp]
    L.paqif_ehl_point_sync.restype = ctypes.c_int
    L.paqif_ehl_point_sweep.argtypes = [vp, i32, i32, i32, f64, u32]
    L.paqif_ehl_point_sweep.restype = ctypes.c_int
    L.paqif_ehl_point_force_balance.argtypes = [vp]
    L.paqif_ehl_point_force_balance.restype = ctypes.c_int
    L.paqif_ehl_point_residual.argtypes = [vp]
    L.paqif_ehl_point_residual.restype = ctypes.c_int
    L.paqif_ehl_point_deformation.argtypes = [vp, vp, vp]
    L.paqif_ehl_point_deformation.restype = ctypes.c_int
    L.paqif_ehl_point_note_update.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp]
    L.paqif_ehl_point_note_update.restype = ctypes.c_int
    L.paqif_ehl_point_film_lines.argtypes = [vp, ctypes.c_int32, vp, ctypes.c_int32,
                                             ctypes.c_double, vp]
    L.paqif_ehl_point_film_lines.restype = ctypes.c_int
    L.paqif_ehl_point_ipc_handles.argtypes = [vp, vp]
    L.paqif_ehl_point_ipc_handles.restype = ctypes.c_int
    L.paqif_ehl_point_attach_peers.argtypes = [vp, i32, i32, vp]
    L.paqif_ehl_point_attach_peers.restype = ctypes.c_int
    L.paqif_ehl_point_fold_emulated.argtypes = [vp, i32, vp, vp]
    L.paqif_ehl_point_fold_emulated.restype = ctypes.c_int
    L.paqif_ehl_point_fold_bench.argtypes = [vp, i32]
    L.paqif_ehl_point_fold_bench.restype = ctypes.c_int
    L._ehl_point_bound = True
    return L


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def point_grid(params: EhlParams, intervals: int):
    """x, y, h of the point grid (film.py:38-45; y through the lo_y adapter)."""
    lo, hi = params.domain
    h = (hi - lo) / intervals
    x = lo + h * np.arange(intervals + 1)
    y = x if params.lo_y is None else (x - x[0]) + params.lo_y
    return x, y, h


def point_initial_state(params: EhlParams, intervals: int) -> np.ndarray:
    """Hertzian hemisphere scaled to the load target, boundary ring zero
    (solver.py:54-73)."""
    x, y, _ = point_grid(params, intervals)
    gx, gy = np.meshgrid(x, y)
    u = hertzian_init(gx, gy)
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    return u * (params.load_target / (2.0 * np.pi / 3.0))


class _Handle:
    def __init__(self, L, cfg: PointCfg, table: np.ndarray, geometry: np.ndarray):
        self.L = L
        t = np.ascontiguousarray(table, dtype=np.float64)
        g = np.ascontiguousarray(geometry, dtype=np.float64)
        N = cfg.n + 1
        if t.shape != (N, N) or g.shape != (N, N):
            raise ContractViolationError("table and geometry must be (n+1, n+1)")
        self.ptr = L.paqif_ehl_point_create(ctypes.byref(cfg), _ptr(t), _ptr(g))
        if not self.ptr:
            _native.check(-1, "paqif_ehl_point_create")

    def close(self):
        if self.ptr:
            self.L.paqif_ehl_point_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PointDevice:
    """Deformation-only use of the handle (FilmModel('point').deformation_full)."""

    def __init__(self, table: np.ndarray, geometry: np.ndarray):
        L = _bind(_native.lib())
        n = table.shape[0] - 1
        cfg = PointCfg(n=n, force_every=1, h=1.0, p_hertz=1.0, lam=1.0, z=1.0, p0=1.0,
                       alpha=1.0)
        self.n = n
        self.h = _Handle(L, cfg, table, geometry)

    def deformation(self, u) -> np.ndarray:
        uu = np.ascontiguousarray(u, dtype=np.float64)
        if uu.shape != (self.n + 1, self.n + 1):
            raise ContractViolationError("u must be (n+1, n+1)")
        out = np.empty_like(uu)
        rc = self.h.L.paqif_ehl_point_deformation(self.h.ptr, _ptr(uu), _ptr(out))
        _native.check(rc, "paqif_ehl_point_deformation")
        return out

    def fold_emulated(self, world: int, u) -> np.ndarray:
        """The sharded fold's decomposition over `world` ranks emulated in
        order on this GPU (test of the slab arithmetic; fft_shard.cuh)."""
        uu = np.ascontiguousarray(u, dtype=np.float64)
        if uu.shape != (self.n + 1, self.n + 1):
            raise ContractViolationError("u must be (n+1, n+1)")
        out = np.empty_like(uu)
        rc = self.h.L.paqif_ehl_point_fold_emulated(self.h.ptr, int(world), _ptr(uu), _ptr(out))
        _native.check(rc, "paqif_ehl_point_fold_emulated")
        return out

    def note_update(self, axis: int, index: int, delta) -> None:
        """Append a pending line update (device list; see FilmModel)."""
        dd = np.ascontiguousarray(delta, dtype=np.float64)
        if dd.shape != (self.n + 1,):
            raise ContractViolationError("delta must have n+1 entries")
        rc = self.h.L.paqif_ehl_point_note_update(self.h.ptr, int(axis), int(index), _ptr(dd))
        _native.check(rc, "paqif_ehl_point_note_update")

    def film_lines(self, mode: int, idx, h0: float) -> np.ndarray:
        """Films of rows (mode 0) / columns (mode 1) idx with the pending
        corrections."""
        ii = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1)
        out = np.empty((ii.size, self.n + 1))
        rc = self.h.L.paqif_ehl_point_film_lines(self.h.ptr, int(mode), ii.ctypes.data,
                                                 int(ii.size), float(h0), _ptr(out))
        _native.check(rc, "paqif_ehl_point_film_lines")
        return out


class PointContact:
    """One point contact resident on the GPU, advanced by ``step()``."""

    def __init__(self, params: EhlParams, intervals: int, scheme: str = "Lhs1",
                 kappa: float = 1 / 3, limiter: str = "kappa", omega: float | None = None,
                 force_every: int = 5, exact: bool = True, u0=None, h0=None):
        if params.contact != "point":
            raise ContractViolationError("PointContact needs a point contact")
        if scheme not in SCHEMES:
            raise ContractViolationError(f"unknown scheme {scheme!r}")
        if limiter not in LIMITERS:
            raise ContractViolationError(f"unknown limiter {limiter!r}")
        if not -1.0 <= kappa <= 1.0:
            raise ContractViolationError("kappa must lie in [-1, 1]")
        if intervals < 8:
            raise ContractViolationError("point grid needs at least 8 intervals")
        self.L = _bind(_native.lib())
        self.n = int(intervals)
        x, y, h = point_grid(params, intervals)
        self.h = h
        self.x, self.y = x, y
        gx, gy = np.meshgrid(x, y)
        self.geometry = 0.5 * (gx ** 2 + gy ** 2)
        self.table = kernel_point(self.n, self.n, h).table
        self.cfg = PointCfg(n=self.n, limiter=LIMITERS[limiter], variant=SCHEMES[scheme],
                            compressible=1 if params.compressible else 0,
                            force_every=force_every, outer=0, h=h, kappa=kappa,
                            omega=params.omega if omega is None else omega,
                            max_change=params.max_change, relax_c=params.relax_c,
                            max_h0_step=params.max_h0_step, load_target=params.load_target,
                            alpha=params.alpha, z=params.z, p0=params.p0,
                            p_hertz=params.p_hertz, lam=params.lam)
        self.flags = _native.FLAG_EXACT if exact else 0
        self._h = _Handle(self.L, self.cfg, self.table, self.geometry)
        if u0 is None:
            u0 = point_initial_state(params, intervals)
        self.set_state(u0, params.h0 if h0 is None else h0)
        self.outer = 0

    def set_state(self, u, h0: float) -> None:
        uu = np.ascontiguousarray(u, dtype=np.float64)
        if uu.shape != (self.n + 1, self.n + 1):
            raise ContractViolationError("u must be (n+1, n+1)")
        rc = self.L.paqif_ehl_point_set_state(self._h.ptr, _ptr(uu), float(h0))
        _native.check(rc, "paqif_ehl_point_set_state")

    def step(self) -> None:
        """One outer iteration (asynchronous on the handle's stream)."""
        rc = self.L.paqif_ehl_point_step(self._h.ptr, self.outer, self.flags)
        _native.check(rc, "paqif_ehl_point_step")
        self.outer += 1

    def shard_folds(self, group=None) -> int:
        """Config 5 on several GPUs: split every later full deformation of
        this contact over the ranks of `group` (torch.distributed, one rank
        per GPU, every rank running the same contact): the handles' CUDA IPC
        handles are exchanged with all_gather_object and each rank's fold
        phases write straight into the peers' buffers (fft_shard.cuh).
        Returns the world size (1: nothing to do)."""
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized():
            return 1
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world == 1:
            return 1
        if world > 8:
            raise ContractViolationError("sharded folds: at most 8 ranks")
        self.sync()
        mine = ctypes.create_string_buffer(192)
        _native.check(self.L.paqif_ehl_point_ipc_handles(self._h.ptr, mine),
                      "paqif_ehl_point_ipc_handles")
        got = [None] * world
        dist.all_gather_object(got, bytes(mine.raw), group=group)
        blob = ctypes.create_string_buffer(b"".join(got), 192 * world)
        _native.check(self.L.paqif_ehl_point_attach_peers(self._h.ptr, rank, world, blob),
                      "paqif_ehl_point_attach_peers")
        dist.barrier(group=group)  # every rank attached before anyone folds
        return world

    def fold_bench(self, reps: int) -> None:
        """Enqueue `reps` forced full deformations (sharded when attached)."""
        _native.check(self.L.paqif_ehl_point_fold_bench(self._h.ptr, int(reps)),
                      "paqif_ehl_point_fold_bench")

    def drive_init(self, tol: float, tol_fb: float, max_outer: int, hist_cap: int = 16):
        """Device solve_ehl record (the line contact's layout, DRIVE_DTYPE):
        the stop / divergence tests run on the GPU after every iteration."""
        from .line import DRIVE_DTYPE
        torch = _native.torch_cuda()
        rec = np.zeros(1, dtype=DRIVE_DTYPE)
        rec["tol"], rec["tol_fb"] = tol, tol_fb
        rec["best"] = rec["deficit"] = np.inf
        rec["max_outer"], rec["outer"] = max_outer, self.outer
        self.drive = torch.from_numpy(rec.view(np.uint8)).cuda()
        self.hist_cap = int(hist_cap)
        self.hist_res = torch.empty(self.hist_cap, dtype=torch.float64, device="cuda")
        self.hist_def = torch.empty_like(self.hist_res)

    def drive_steps(self, steps: int) -> None:
        """Enqueue `steps` device-driven outer iterations (asynchronous on
        the handle's stream; a stopped record turns the rest into no-ops)."""
        torch = _native.torch_cuda()
        torch.cuda.current_stream().synchronize()  # drive buffers written on torch's stream
        rc = self.L.paqif_ehl_point_drive_steps(self._h.ptr, int(steps), self.drive.data_ptr(),
                                                self.hist_res.data_ptr(),
                                                self.hist_def.data_ptr(), self.hist_cap,
                                                self.flags)
        _native.check(rc, "paqif_ehl_point_drive_steps")

    def drive_state(self):
        """Host copy of the drive record (synchronises the handle's stream)."""
        from .line import DRIVE_DTYPE
        self.sync()
        d = self.drive.cpu().numpy().view(DRIVE_DTYPE).copy()[0]
        self.outer = int(d["outer"])
        return d

    def sweep(self, kind: int, sel: int = -1, nu_variant: int | None = None,
              omega: float | None = None) -> None:
        """One public sweep on the resident state (kinds: 0 hybrid x, 1 Newton
        x, 2 weighted x, 3 column; see include/paqif_ehl.h)."""
        nu = self.cfg.variant if nu_variant is None else nu_variant
        om = self.cfg.omega if omega is None else omega
        rc = self.L.paqif_ehl_point_sweep(self._h.ptr, kind, sel, nu, float(om), self.flags)
        _native.check(rc, "paqif_ehl_point_sweep")

    def force_balance(self) -> None:
        _native.check(self.L.paqif_ehl_point_force_balance(self._h.ptr),
                      "paqif_ehl_point_force_balance")

    def residual(self) -> float:
        """complementarity_residual of the resident state (synchronises)."""
        _native.check(self.L.paqif_ehl_point_residual(self._h.ptr), "paqif_ehl_point_residual")
        return self.status()[1]

    def stream_handle(self) -> int:
        """The handle's cudaStream_t (e.g. for torch.cuda.ExternalStream)."""
        return int(self.L.paqif_ehl_point_stream(self._h.ptr) or 0)

    def sync(self) -> None:
        _native.check(self.L.paqif_ehl_point_sync(self._h.ptr), "paqif_ehl_point_sync")

    def status(self):
        """(h0, residual, deficit, err) after the last step (synchronises)."""
        scal = np.zeros(4)
        err = np.zeros(1, dtype=np.int32)
        rc = self.L.paqif_ehl_point_get(self._h.ptr, None, None, _ptr(scal), None, None,
                                        _ptr(err))
        _native.check(rc, "paqif_ehl_point_get")
        return float(scal[0]), float(scal[1]), float(scal[2]), int(err[0])

    def snapshot(self):
        """Host copies: dict(u, film, h0, res, deficit, worst, newton, deferred,
        x_rungs, y_rungs, err)."""
        N = self.n + 1
        u = np.empty((N, N))
        film = np.empty((N, N))
        scal = np.zeros(4)
        xi = np.zeros(self.n - 1, dtype=np.int32)
        yi = np.zeros(self.n - 1, dtype=np.int32)
        err = np.zeros(1, dtype=np.int32)
        rc = self.L.paqif_ehl_point_get(self._h.ptr, _ptr(u), _ptr(film), _ptr(scal), _ptr(xi),
                                        _ptr(yi), _ptr(err))
        _native.check(rc, "paqif_ehl_point_get")
        return dict(u=u, film=film, h0=float(scal[0]), res=float(scal[1]),
                    deficit=float(scal[2]), worst=float(scal[3]),
                    newton=(xi & 1).astype(np.int64), deferred=((xi >> 1) & 1).astype(np.int64),
                    x_rungs=(xi >> 4) & 3, y_rungs=yi, err=int(err[0]))

    @staticmethod
    def raise_for(err: int) -> None:
        if err & 5:
            raise FactorizationBreakdownError(-1, "every rung of a point line solve broke down")
        if err & 10:
            raise PaqifError("non-finite change in point-contact sweep")
        if err & 64:
            raise PaqifError("sharded fold: a peer rank did not reach the barrier")

    def close(self) -> None:
        self._h.close()
