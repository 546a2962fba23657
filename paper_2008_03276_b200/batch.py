"""Batched device API: many independent banded LCPs / linear systems in one
kernel launch (the config-2 hot path).

Inputs may be torch CUDA tensors (zero-copy; the stream is torch's current
stream) or host numpy arrays (copied in and out).  Layout is the reference's
batched layout: ``bands (B, 2*beta+1, n)`` diagonal-major, ``f (B, n)``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ContractViolationError


@dataclass
class LcpBatchResult:
    u: object          # (B, n) float64 solution (projected)
    active: object     # (B, n) bool, pinned (cavitated) set of the returned pass
    passes: object     # (B,) int64 active-set passes (paqif_solve calls)
    res: object        # (B,) float64 complementarity residual of u
    status: object     # (B,) int64 PAQIF_LCP_* codes


def _shape(bands, f):
    if bands.ndim != 3 or f.ndim != 2:
        raise ContractViolationError("bands must be (B, 2beta+1, n) and f (B, n)")
    B, d, n = bands.shape
    if d % 2 != 1 or f.shape != (B, n):
        raise ContractViolationError("inconsistent batch shapes")
    return B, (d - 1) // 2, n


class LcpSolver:
    """Preallocated device workspace for repeated batches of one shape."""

    def __init__(self, B: int, n: int, beta: int, exact: bool = True):
        torch = _native.torch_cuda()
        self.L = _native.lib()
        self.B, self.n, self.beta = B, n, beta
        self.flags = _native.FLAG_EXACT if exact else 0
        nbytes = self.L.paqif_lcp_workspace_bytes(B, n, beta)
        if nbytes == 0 and B > 0:
            raise ContractViolationError(
                f"unsupported LCP shape B={B} n={n} beta={beta} (n even, n > 2beta+1, beta<=8)")
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        self.ws_bytes = nbytes
        dev = "cuda"
        self.u = torch.empty((B, n), dtype=torch.float64, device=dev)
        self.active = torch.empty((B, n), dtype=torch.uint8, device=dev)
        self.passes = torch.empty(B, dtype=torch.int64, device=dev)
        self.res = torch.empty(B, dtype=torch.float64, device=dev)
        self.status = torch.empty(B, dtype=torch.int64, device=dev)

    def launch(self, bands, f, tol: float = 1e-10, max_outer: int = 100, stream=None) -> None:
        """Asynchronous launch on device tensors (results in self.u etc.)."""
        rc = self.L.paqif_lcp_batch(self.B, self.n, self.beta, bands.data_ptr(), f.data_ptr(),
                                    float(tol), int(max_outer), self.flags, self.u.data_ptr(),
                                    self.active.data_ptr(), self.passes.data_ptr(),
                                    self.res.data_ptr(), self.status.data_ptr(),
                                    self.ws.data_ptr(), self.ws_bytes,
                                    _native.stream_ptr(stream))
        _native.check(rc, "paqif_lcp_batch")

    def solve_r1(self, bands, f, stream=None):
        """paqif_solve(L_b, f_b, r=1) for every b; returns (x, status) tensors."""
        rc = self.L.paqif_solve_r1_batch(self.B, self.n, self.beta, bands.data_ptr(),
                                         f.data_ptr(), self.u.data_ptr(), self.status.data_ptr(),
                                         self.flags, self.ws.data_ptr(), self.ws_bytes,
                                         _native.stream_ptr(stream))
        _native.check(rc, "paqif_solve_r1_batch")
        return self.u, self.status


def lcp_batch(bands, f, tol: float = 1e-10, max_outer: int = 100, exact: bool = True,
              solver: LcpSolver | None = None) -> LcpBatchResult:
    """Solve every ``u >= 0, L_b u >= f_b, u.(L_b u - f_b) = 0`` with the
    reference's projected-pass policy (paqif_solve_lcp, parallel.py:298-347)."""
    torch = _native.torch_cuda()
    host = isinstance(bands, np.ndarray)
    if host:
        tb = torch.from_numpy(np.ascontiguousarray(bands, dtype=np.float64)).cuda()
        tf = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda()
    else:
        tb, tf = bands.contiguous(), f.contiguous()
    B, beta, n = _shape(tb, tf)
    s = solver or LcpSolver(B, n, beta, exact)
    s.launch(tb, tf, tol, max_outer)
    if host:
        torch.cuda.current_stream().synchronize()
        return LcpBatchResult(s.u.cpu().numpy(), s.active.cpu().numpy().astype(bool),
                              s.passes.cpu().numpy(), s.res.cpu().numpy(),
                              s.status.cpu().numpy())
    return LcpBatchResult(s.u, s.active.bool(), s.passes, s.res, s.status)


def lcp_batch_host(bands: np.ndarray, f: np.ndarray, tol: float = 1e-10, max_outer: int = 100,
                   exact: bool = True) -> LcpBatchResult:
    """The host-buffer C-ABI entry (paqif_lcp_batch_host): H2D, kernel, D2H."""
    L = _native.lib()
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    B, d, n = bands.shape
    u = np.empty((B, n))
    act = np.empty((B, n), dtype=np.uint8)
    passes = np.empty(B, dtype=np.int64)
    res = np.empty(B)
    st = np.empty(B, dtype=np.int64)
    rc = L.paqif_lcp_batch_host(B, n, (d - 1) // 2, bands.ctypes.data, f.ctypes.data, float(tol),
                                int(max_outer), _native.FLAG_EXACT if exact else 0,
                                u.ctypes.data, act.ctypes.data, passes.ctypes.data,
                                res.ctypes.data, st.ctypes.data)
    _native.check(rc, "paqif_lcp_batch_host")
    return LcpBatchResult(u, act.astype(bool), passes, res, st)


def solve_r1_batch(bands, f, exact: bool = True):
    """Batched paqif_solve(L_b, f_b, r=1): returns (x, status) like the inputs."""
    torch = _native.torch_cuda()
    host = isinstance(bands, np.ndarray)
    tb = torch.from_numpy(np.ascontiguousarray(bands, dtype=np.float64)).cuda() if host else bands
    tf = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda() if host else f
    B, beta, n = _shape(tb, tf)
    s = LcpSolver(B, n, beta, exact)
    x, st = s.solve_r1(tb, tf)
    if host:
        torch.cuda.current_stream().synchronize()
        return x.cpu().numpy(), st.cpu().numpy()
    return x, st


def _dev(a, dtype=None):
    torch = _native.torch_cuda()
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype or np.float64)).cuda(), True
    return a.contiguous(), False


def solve_rblock_batch(bands, f, r: int, project: bool = False, exact: bool = True,
                       stream=None):
    """Batched paqif_solve(L_b, f_b, r) with all seven steps on the device
    (csrc/rblock.cu).  Returns (x, status) like the inputs (numpy or torch)."""
    torch = _native.torch_cuda()
    L = _native.lib()
    tb, host = _dev(bands)
    tf, _ = _dev(f)
    B, beta, n = _shape(tb, tf)
    nbytes = L.paqif_solve_rblock_workspace_bytes(B, n, beta, r)
    if nbytes == 0:
        raise ContractViolationError(f"r-block solve: unsupported sizes n={n} beta={beta} r={r}")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    x = torch.zeros((B, n), dtype=torch.float64, device="cuda")
    st = torch.zeros(B, dtype=torch.int64, device="cuda")
    rc = L.paqif_solve_rblock_batch(B, n, beta, int(r), tb.data_ptr(), tf.data_ptr(),
                                    x.data_ptr(), 1 if project else 0, st.data_ptr(),
                                    _native.FLAG_EXACT if exact else 0, ws.data_ptr(), nbytes,
                                    _native.stream_ptr(stream))
    _native.check(rc, "paqif_solve_rblock_batch")
    if host:
        torch.cuda.current_stream().synchronize()
        return x.cpu().numpy(), st.cpu().numpy()
    return x, st


def lcp_rblock(bands, f, r: int, tol: float = 1e-10, max_outer: int = 100, exact: bool = True):
    """paqif_solve_lcp(LcpProblem(L, f), r) for r > 1 on the device for one
    system (parallel.py:298-347): every pass pins the active rows, runs the
    r-block solve and the multiplier / projection / residual / next-set
    kernels; the host only reads (res, changed) per pass.  Returns
    (u, status, passes, res) with status a PAQIF_LCP_* code."""
    torch = _native.torch_cuda()
    L = _native.lib()
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    nd, n = bands.shape
    beta = (nd - 1) // 2
    tb = torch.from_numpy(bands[None]).cuda()
    tf = torch.from_numpy(f[None]).cuda()
    scale = float(np.abs(bands).sum(axis=0).max() + np.abs(f).max())
    floor = 1e3 * np.finfo(float).eps * scale
    act = (tf <= 0.0).to(torch.uint8)
    nact = torch.empty_like(act)
    lmod = torch.empty_like(tb)
    fmod = torch.empty_like(tf)
    u = torch.empty_like(tf)
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    chg = torch.empty(1, dtype=torch.int32, device="cuda")
    nbytes = L.paqif_solve_rblock_workspace_bytes(1, n, beta, r)
    if nbytes == 0:
        raise ContractViolationError(f"r-block solve: unsupported sizes n={n} beta={beta} r={r}")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ue = torch.zeros_like(tf)
    st = torch.zeros(1, dtype=torch.int64, device="cuda")
    sp = _native.stream_ptr()
    best_res, best_u = np.inf, np.zeros(n)
    last = np.inf
    for k in range(max_outer):
        _native.check(L.paqif_lcp_pin_batch(1, n, beta, tb.data_ptr(), tf.data_ptr(),
                                             act.data_ptr(), lmod.data_ptr(), fmod.data_ptr(), sp),
                      "paqif_lcp_pin_batch")
        _native.check(L.paqif_solve_rblock_batch(1, n, beta, int(r), lmod.data_ptr(),
                                                 fmod.data_ptr(), ue.data_ptr(), 0, st.data_ptr(),
                                                 _native.FLAG_EXACT if exact else 0,
                                                 ws.data_ptr(), nbytes, sp),
                      "paqif_solve_rblock_batch")
        _native.check(L.paqif_lcp_pass_batch(1, n, beta, tb.data_ptr(), tf.data_ptr(),
                                              ue.data_ptr(), act.data_ptr(), u.data_ptr(),
                                              nact.data_ptr(), res.data_ptr(), chg.data_ptr(), sp),
                      "paqif_lcp_pass_batch")
        code = int(st.item())
        if code:
            return u[0].cpu().numpy(), code, k + 1, float("nan")
        last = float(res.item())
        if last <= tol:
            return u[0].cpu().numpy(), 0, k + 1, last
        if last < best_res:
            best_res, best_u = last, u[0].cpu().numpy()
        if not int(chg.item()):
            if best_res <= max(tol, floor):
                return best_u, 0, k + 1, best_res
            break
        act, nact = nact, act
    if best_res <= max(tol, floor):
        return best_u, 0, max_outer, best_res
    return best_u, _native.LCP_NONCONVERGED, max_outer, last
